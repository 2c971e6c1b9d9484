# march eval: full GPU suite + 3T / 7T bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -x -rf > gpurun_out/pytest_r2m.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2m.log; tail -6 gpurun_out/pytest_r2m.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench3_r2m.json 2> gpurun_out/bench3_r2m.err
tail -1 gpurun_out/bench3_r2m.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('3T', d['value'], d['ms_per_step'], d['solver'], r['kernel_share_of_step'], r['hbm_kernels'].get('eval'))"
timeout 600 python bench.py --config C3_hcp7t --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_r2m.json 2> gpurun_out/bench7_r2m.err
tail -1 gpurun_out/bench7_r2m.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('7T', d['value'], d['ms_per_step'], d['solver'], r['kernel_share_of_step'], r['hbm_kernels'])"
tail -3 gpurun_out/bench7_r2m.err
