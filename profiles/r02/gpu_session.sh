python profiles/kexp.py time tma4s,base --cfg c2,c4 --reps 7 > gpurun_out/kexp_tma4s2.jsonl 2>&1
cat gpurun_out/kexp_tma4s2.jsonl
