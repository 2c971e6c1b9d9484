# pcg_upd with 4 groups in flight per thread: flat / slab parity subset, bench 7T and C5
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_shipped.py -m gpu -q -x -k "flat or hcp7t or slab" > gpurun_out/pytest_g.log 2>&1; tail -2 gpurun_out/pytest_g.log
for cfg in C3_hcp7t C5_512; do
timeout 900 python bench.py --no-cpu-baseline --config $cfg --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/bench_g_$cfg.json 2> gpurun_out/bench_g_$cfg.err
tail -1 gpurun_out/bench_g_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg value',round(d['value'],2),'ms',round(d['ms_per_step'],3),'hbm',{k:round(v['frac_cold'],3) for k,v in r.get('hbm_kernels',{}).items()}, 'avg_ms', {k: round(v,4) for k,v in r.get('kernel_share_of_step',{}).items()})"
done
