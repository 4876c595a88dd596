python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_final2.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1
python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err
cat gpurun_out/pytest_final2.log gpurun_out/smoke_final2.log
