# resident limb reductions: resident / shipped parity subset, bench C2, ncu of the eval kernel (3T) with source
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shipped.py tests/test_gpu_parity.py -m gpu -q -x -k "resident or shipped or hcp3t or graph or repeat or history or batch" > gpurun_out/pytest_v.log 2>&1; tail -3 gpurun_out/pytest_v.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err
tail -1 gpurun_out/bench_v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value'],2),'ms',round(d['ms_per_step'],3),'e2e',round(d['e2e']['value'],2),'roof',d['roofline']['achieved'],d['roofline']['peak'])"
export HYSCO_NO_GRAPH=1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:eval_kernel" -s 3 -c 1 -o gpurun_out/prof_eval3t python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 1 > gpurun_out/ncu_eval.log 2>&1
ls -la gpurun_out | grep prof_
