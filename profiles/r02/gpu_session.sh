# round-2 final validation: full GPU suite, smoke, default bench
python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
cat gpurun_out/pytest_final.log gpurun_out/smoke_final.log
