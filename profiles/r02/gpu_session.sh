python -m pytest tests -m gpu -x -q -k "decode or decoder or single_row or smoke" 2>&1 | tail -4 > gpurun_out/pytest8.log
python profiles/kexp.py time base --cfg c3,c3_32k,c3b1,c3b4 --reps 9 > gpurun_out/kexp8.jsonl 2>&1
cat gpurun_out/pytest8.log gpurun_out/kexp8.jsonl
