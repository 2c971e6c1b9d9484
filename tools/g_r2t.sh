# XU-light eval: parity tests touching eval + 3T / 7T bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shipped.py -m gpu -q --timeout 900 -x -rf > gpurun_out/pytest_r2t.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2t.log; tail -3 gpurun_out/pytest_r2t.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench3_r2t.json 2> gpurun_out/bench3_r2t.err
tail -1 gpurun_out/bench3_r2t.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('3T', d['value'], d['ms_per_step'], r['kernel_share_of_step'], r['hbm_kernels'].get('eval'))"
timeout 600 python bench.py --config C3_hcp7t --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_r2t.json 2> gpurun_out/bench7_r2t.err
tail -1 gpurun_out/bench7_r2t.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('7T', d['value'], d['ms_per_step'], r['kernel_share_of_step'], r['hbm_kernels'].get('eval'))"
