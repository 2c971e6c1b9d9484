# round-2 re-entry baseline: full GPU suite, smoke, default bench, 7T bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/pytest_r2f.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2f.log; tail -8 gpurun_out/pytest_r2f.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2f.log 2>&1; tail -2 gpurun_out/smoke_r2f.log
timeout 900 python bench.py > gpurun_out/bench_r2f.json 2> gpurun_out/bench_r2f.err
tail -c 4000 gpurun_out/bench_r2f.json
timeout 600 python bench.py --config C3_hcp7t --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_r2f.json 2> gpurun_out/bench7_r2f.err
tail -c 2500 gpurun_out/bench7_r2f.json
