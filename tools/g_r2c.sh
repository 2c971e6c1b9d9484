mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -k "batch or resident or correct_pipeline or host_stream" > gpurun_out/pytest_r2c.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2c.log; tail -3 gpurun_out/pytest_r2c.log
for B in 8; do timeout 600 python bench.py --steps 10 --warmup 3 --batch $B --no-cpu-baseline > gpurun_out/bench_r2c_b$B.json 2> gpurun_out/bench_r2c_b$B.err; tail -1 gpurun_out/bench_r2c_b$B.json | cut -c1-300; done
