# round-2 GPU session script (profiling aid): variant timings through profiles/kexp.py
python profiles/kexp.py time base --cfg c4,c2,c3 --reps 7 --rounds 3 > gpurun_out/kexp3.jsonl 2>&1
for S in 1 2 4 8; do HIPATTN_SPLITS=$S python profiles/kexp.py time tune --cfg c3b1,c3b4 --reps 9 | sed "s/^/S=$S /"; done > gpurun_out/splits2.log 2>&1
cat gpurun_out/kexp3.jsonl gpurun_out/splits2.log
