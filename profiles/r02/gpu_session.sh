# round-2 GPU session: full GPU suite (incl. slow full-size parity), default bench, C5 1M-token bench
python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/pytest_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1
python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err
python bench.py --config c5 --no-e2e --no-cpu --steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
cat gpurun_out/pytest_full.log gpurun_out/smoke2.log; tail -2 gpurun_out/bench4.err gpurun_out/bench_c5.err
