# fp32 eval column body: eval parity subset + shipped, bench C2 / C3
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shipped.py -m gpu -q -x -k "objective or ot_init or solve_fixed or pipeline or shipped or resident or hcp3t or hcp7t or noise or guard" > gpurun_out/pytest_w.log 2>&1; tail -3 gpurun_out/pytest_w.log
for cfg in C2_hcp3t C3_hcp7t; do
timeout 600 python bench.py --no-cpu-baseline --config $cfg > gpurun_out/bench_w_$cfg.json 2> gpurun_out/bench_w_$cfg.err
tail -1 gpurun_out/bench_w_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value',round(d['value'],2),'ms',round(d['ms_per_step'],3),'e2e',round(d['e2e']['value'],2),'share',{k:round(v,3) for k,v in r['kernel_share_of_step'].items()},'hbm',{k:round(v['frac_cold'],3) for k,v in r.get('hbm_kernels',{}).items()})"
done
