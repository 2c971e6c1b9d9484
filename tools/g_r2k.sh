# full GPU suite + smoke + 7T and 3T bench with the flat/march PCG
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/pytest_r2k.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2k.log; tail -12 gpurun_out/pytest_r2k.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2k.log 2>&1; tail -2 gpurun_out/smoke_r2k.log
timeout 600 python bench.py --config C3_hcp7t --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_r2k.json 2> gpurun_out/bench7_r2k.err
tail -1 gpurun_out/bench7_r2k.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], d['solver'], r['kernel'], r['frac'], r['kernel_share_of_step'])"
HYSCO_NO_RESIDENT=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench3s_r2k.json 2> gpurun_out/bench3s_r2k.err
tail -1 gpurun_out/bench3s_r2k.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('3T streaming', d['value'], d['ms_per_step'], r['kernel_share_of_step'], r['hbm_kernels'])"
