# cp.async march + tile choice: flat tests, 7T and C5 bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -m gpu -q --timeout 900 -x -rf -k "flat or solve_fixed or pipeline or slab or production" > gpurun_out/pytest_r2r.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2r.log; tail -3 gpurun_out/pytest_r2r.log
timeout 600 python bench.py --config C3_hcp7t --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_r2r.json 2> gpurun_out/bench7_r2r.err
tail -1 gpurun_out/bench7_r2r.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('7T', d['value'], d['ms_per_step'], r['kernel_share_of_step'], r['hbm_kernels'])"
timeout 900 python bench.py --config C5_512 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench5_r2r.json 2> gpurun_out/bench5_r2r.err
tail -1 gpurun_out/bench5_r2r.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C5', d['value'], d['ms_per_step'], r['kernel_share_of_step'], r['hbm_kernels'])"
