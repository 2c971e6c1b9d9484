# ticket all-reduce in the resident PCG: resident / shipped / L2 tests + 3T bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_shipped.py tests/test_gpu_parity.py -m gpu -q --timeout 900 -x -rf -k "resident or shipped or hcp3t or l2_persistent or C1 or pipeline or solve_fixed" > gpurun_out/pytest_r2v.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2v.log; tail -3 gpurun_out/pytest_r2v.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench3_r2v.json 2> gpurun_out/bench3_r2v.err
tail -1 gpurun_out/bench3_r2v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('3T', d['value'], d['ms_per_step'], r['kernel_share_of_step'], r['achieved'], r['peak'], r['frac'])"
tail -2 gpurun_out/bench3_r2v.err
