timeout 900 python profiles/kexp.py time prev,base --cfg c3,c3_32k,c3b4 --reps 7 --rounds 2
timeout 1200 python -m pytest tests -m gpu -x -q -k "decode or decoder or paged or composition or dist_gpu or concurrent" 2>&1 | tail -5
