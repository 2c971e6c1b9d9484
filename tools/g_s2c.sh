# cooperative Armijo search: full GPU suite, bench C2 / C3, smoke
mkdir -p gpurun_out
for cfg in C2_hcp3t C3_hcp7t; do
timeout 600 python bench.py --no-cpu-baseline --config $cfg > gpurun_out/bench_x_$cfg.json 2> gpurun_out/bench_x_$cfg.err
tail -1 gpurun_out/bench_x_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value',round(d['value'],2),'ms',round(d['ms_per_step'],3),'e2e',round(d['e2e']['value'],2),'solver',d['solver'],'share',{k:round(v,3) for k,v in r['kernel_share_of_step'].items()})"
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_x.log 2>&1; tail -3 gpurun_out/pytest_x.log
