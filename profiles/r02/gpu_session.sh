CS=/usr/local/cuda/bin/compute-sanitizer
rm -f gpurun_out/sanitizer_rc3.log
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1200 $CS --tool $tool --print-limit 50 python profiles/sanitize.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_rc3.log
done
cat gpurun_out/sanitizer_rc3.log; grep -h "SUMMARY" gpurun_out/sanitizer_*.log; grep -c "done" gpurun_out/sanitizer_memcheck.log
