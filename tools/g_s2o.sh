# A/B: fp32 eval with a segment of consecutive cells per lane (EVAL_SEG=1) vs chunked (0)
mkdir -p gpurun_out
for v in seg0 seg1; do
cp ab/libhysco_$v.so paper_2403_10706_b200/libhysco.so
touch -d '+1 hour' paper_2403_10706_b200/libhysco.so
for cfg in C2_hcp3t C3_hcp7t; do
timeout 600 python bench.py --no-cpu-baseline --config $cfg --e2e-steps 2 > gpurun_out/bench_o_${v}_$cfg.json 2> gpurun_out/bench_o_${v}_$cfg.err
tail -1 gpurun_out/bench_o_${v}_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v $cfg value',round(d['value'],2),'ms',round(d['ms_per_step'],4),'eval share',round(r['kernel_share_of_step'].get('eval',0),4),'eval hbm',round(r['hbm_kernels'].get('eval',{}).get('frac_cold',0),3))"
done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shipped.py -m gpu -q -x -k "objective or ot_init or solve_fixed or pipeline or shipped or resident or hcp3t or hcp7t or noise or guard or history or graph" 2>&1 | tail -2
