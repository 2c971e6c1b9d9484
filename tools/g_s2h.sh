# A/B: march with 1 vs 2 CTAs per SM (HYSCO_MARCH_CPS), 7T and C5 bench
mkdir -p gpurun_out
for v in cps1 cps2; do
cp ab/libhysco_$v.so paper_2403_10706_b200/libhysco.so
touch -d '+1 hour' paper_2403_10706_b200/libhysco.so
for cfg in C3_hcp7t C5_512; do
timeout 900 python bench.py --no-cpu-baseline --config $cfg --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/bench_h_${v}_$cfg.json 2> gpurun_out/bench_h_${v}_$cfg.err
tail -1 gpurun_out/bench_h_${v}_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v $cfg value',round(d['value'],2),'ms',round(d['ms_per_step'],3),'hbm',{k:round(v['frac_cold'],3) for k,v in r.get('hbm_kernels',{}).items()})"
done
done
if [ -f gpurun_out/bench_h_cps2_C3_hcp7t.json ]; then timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "flat" 2>&1 | tail -2; fi
