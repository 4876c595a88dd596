timeout 1200 python -m pytest tests -m gpu -x -q -k "decode or decoder or paged or composition or dist_gpu or concurrent or replay" 2>&1 | tail -5
timeout 600 python profiles/kexp.py time base --cfg c3b1,c3b4,c3 --reps 9
