# streaming graph: two unrolled Armijo retry evaluations per GN step before the WHILE node
mkdir -p gpurun_out
for v in 0 2; do
HYSCO_LS_UNROLL=$v timeout 900 python bench.py --no-cpu-baseline --config C3_hcp7t --e2e-steps 2 > gpurun_out/bench_q_$v.json 2> gpurun_out/bench_q_$v.err
tail -1 gpurun_out/bench_q_$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('unroll=$v 7T', round(d['value'],2), round(d['ms_per_step'],3), d['solver']['f_evals'])"
done
timeout 900 python bench.py --no-cpu-baseline --config C5_512 --steps 5 --warmup 3 --e2e-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', round(d['value'],3), d['solver']['f_evals'])"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_q.log 2>&1; tail -2 gpurun_out/pytest_q.log
