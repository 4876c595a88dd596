# round-2 GPU session script (profiling aid)
python -m pytest tests -m gpu -x -q -k "decode or single_row or sinkwin or split or concurrent or decoder" 2>&1 | tail -5 > gpurun_out/pytest5.log
python profiles/kexp.py time base --cfg c3,c3_32k,c3b1,c3b4 --reps 9 --rounds 2 > gpurun_out/kexp5.jsonl 2>&1
LIB=paper_2406_09827_b200/libhipattn.so
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_row1_kernel" -s 1 -c 1 \
  -o gpurun_out/ncu_c3_r02b python profiles/kexp.py _time $LIB c3 1 > gpurun_out/ncu_c3b.log 2>&1
cat gpurun_out/pytest5.log gpurun_out/kexp5.jsonl
