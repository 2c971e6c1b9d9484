# unrolled Armijo retries on the streaming graph, early exit of empty retry evaluations: full suite + benches
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 240 > gpurun_out/pytest_r.log 2>&1; tail -3 gpurun_out/pytest_r.log
for v in 0 2; do
HYSCO_LS_UNROLL=$v timeout 900 python bench.py --no-cpu-baseline --config C3_hcp7t --e2e-steps 2 > gpurun_out/bench_r_$v.json 2> gpurun_out/bench_r_$v.err
tail -1 gpurun_out/bench_r_$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('unroll=$v 7T', round(d['value'],2), round(d['ms_per_step'],3), d['solver']['f_evals'])"
done
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('3T', round(d['value'],2))"
