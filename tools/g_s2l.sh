# A/B: resident prologue by cp.async into shared memory (RES_PRO_ASYNC=1) vs per-slot loads (0), 3T bench x2
mkdir -p gpurun_out
timeout 60 ./tools/res_trace tiled 4 37 42 3 | grep -E "err=|init|period|tiled"
for rep in 1 2; do
for v in pro0 pro1; do
cp ab/libhysco_$v.so paper_2403_10706_b200/libhysco.so
touch -d '+1 hour' paper_2403_10706_b200/libhysco.so
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_l_$v.json 2> gpurun_out/bench_l_$v.err
tail -1 gpurun_out/bench_l_$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v value',round(d['value'],2),'ms',round(d['ms_per_step'],4),'res us/it',round(r['achieved'],3))"
done
done
timeout 600 python -m pytest tests/test_gpu_shipped.py tests/test_gpu_parity.py -m gpu -q -x -k "resident or tiled or hcp3t" 2>&1 | tail -2
