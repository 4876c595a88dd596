python profiles/kexp.py time prev,base --cfg c2,c4 --reps 7 --rounds 2 > gpurun_out/kexp_fastmax.jsonl 2>&1
python -m pytest tests -m gpu -x -q -k "attention or layer or exact_case or sinkwin or full_size or wide or gqa or multi_query or host" 2>&1 | tail -3
cat gpurun_out/kexp_fastmax.jsonl
