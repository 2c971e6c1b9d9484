# A/B: eval tiles of 4 columns (128 threads, 6 CTAs/SM) vs 8 (256 threads, 3 CTAs/SM)
mkdir -p gpurun_out
for rep in 1 2; do
for v in ev8 ev4; do
cp ab/libhysco_$v.so paper_2403_10706_b200/libhysco.so
touch -d '+1 hour' paper_2403_10706_b200/libhysco.so
for cfg in C2_hcp3t C3_hcp7t; do
timeout 600 python bench.py --no-cpu-baseline --config $cfg --e2e-steps 2 > gpurun_out/bench_u_${v}_$cfg.json 2> gpurun_out/bench_u_${v}_$cfg.err
tail -1 gpurun_out/bench_u_${v}_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v $cfg', round(d['value'],2), 'median ms', round(d['step_ms']['median'],4), 'eval hbm', round(r['hbm_kernels'].get('eval',{}).get('frac_cold',0),3))"
done
done
done
cp ab/libhysco_ev4.so paper_2403_10706_b200/libhysco.so; touch -d '+1 hour' paper_2403_10706_b200/libhysco.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shipped.py -m gpu -q -x --timeout 240 -k "objective or pipeline or shipped or hcp3t or graph or apply" 2>&1 | tail -2
