#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench, and (optionally) ncu captures.
# usage: tools/gpu_round.sh [tag] [ncu]   (run under gpurun from the repo root)
TAG=${1:-dev}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -4 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -1 gpurun_out/bench_$TAG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value'],2),'ms',round(d['ms_per_step'],3),'e2e',round(d['e2e']['value'],2),'roof',d['roofline']['kernel'],d['roofline']['bound'],round(d['roofline']['frac'],4),'share',{k:round(v,3) for k,v in d['roofline']['kernel_share_of_step'].items()},'hbm',{k:round(v['frac_cold'],3) for k,v in d['roofline']['hbm_kernels'].items()},'clk',d['clocks'],'launches',d['gpu_launches'])"
if [ "$2" == "ncu" ]; then
  export HYSCO_NO_GRAPH=1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 1 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${NCU_KERNELS:-pcg_resident|eval_kernel|trial_init|ot_column|apply_kernel}" -s ${NCU_SKIP:-3} -c ${NCU_COUNT:-5} -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 1 > gpurun_out/ncu_$TAG.log 2>&1
  ls -la gpurun_out | grep $TAG
fi
