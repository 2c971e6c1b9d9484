# host-stream entry without a per-item synchronisation: its tests, bench 3T e2e
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "host or stream or cli or infeasible or repeat" > gpurun_out/pytest_i.log 2>&1; tail -2 gpurun_out/pytest_i.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err
tail -1 gpurun_out/bench_i.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value'],2),'ms',round(d['ms_per_step'],3),'e2e',d['e2e'])"
