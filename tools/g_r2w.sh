# A/B: max shared carve-out for eval (no SM reconfiguration at eval <-> resident boundaries)
mkdir -p gpurun_out
for v in 0 1 0 1; do
HYSCO_CARVEOUT_MAX=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2> /dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('carveout_max=$v', round(d['value'],1), round(d['step_ms']['median'],4), r['kernel_share_of_step'])"
done
