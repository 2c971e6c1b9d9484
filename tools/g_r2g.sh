# flat two-launch streaming PCG: parity (new + affected tests), 7T bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -x -k "flat or solve_fixed or pipeline or production or halving or graph_and_host or l2_persistent or resident_pcg_matches" > gpurun_out/pytest_r2g.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2g.log; tail -5 gpurun_out/pytest_r2g.log
timeout 600 python bench.py --config C3_hcp7t --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_r2g.json 2> gpurun_out/bench7_r2g.err
tail -1 gpurun_out/bench7_r2g.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['ms_per_step'], r['kernel'], r['frac'], r['kernel_share_of_step'], r['hbm_kernels'])"
tail -3 gpurun_out/bench7_r2g.err
