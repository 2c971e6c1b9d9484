#!/bin/bash
# A/B timing of library variants on one box: tools/ab_bench.sh tag lib1.so lib2.so ...
# (each variant copied over the in-tree libhysco.so; bench runs alternate A B A B)
TAG=$1; shift
mkdir -p gpurun_out
cp paper_2403_10706_b200/libhysco.so /tmp/libhysco_keep.so
for rep in 1 2; do
  for L in "$@"; do
    cp "$L" paper_2403_10706_b200/libhysco.so
    timeout 300 python bench.py --steps ${STEPS:-30} --warmup 5 --no-cpu-baseline --e2e-steps 2 $BENCH_EXTRA > gpurun_out/ab_${TAG}.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/ab_${TAG}.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$L', round(d['value'],1), round(d['ms_per_step'],4), {k: round(v*d['ms_per_step']*1e3/r['launches_per_step'][k],1) for k,v in r['kernel_share_of_step'].items()})"
  done
done
cp /tmp/libhysco_keep.so paper_2403_10706_b200/libhysco.so
