#!/bin/bash
# ncu --set full captures of the NEXT-row kernels (run under gpurun)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:admm_b_kernel|admm_u_kernel|admm_rhs|admm_zscale" -s 4 -c 4 -o gpurun_out/prof_admm python bench.py --solver admm --steps 1 --warmup 0 > gpurun_out/ncu_admm.log 2>&1; echo "admm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:lsq_kernel|push_forward_kernel" -s 2 -c 2 -o gpurun_out/prof_lsq python bench.py --stage lsq --steps 1 --warmup 1 > gpurun_out/ncu_lsq.log 2>&1; echo "lsq rc=$?"
timeout 900 ncu --set full --clock-control none -k "regex:permute_kernel|fieldmap_cells" -c 3 -o gpurun_out/prof_cli python bench.py --stage cli --steps 1 --warmup 0 > gpurun_out/ncu_cli.log 2>&1; echo "cli rc=$?"
ls -la gpurun_out | grep prof_
for t in admm lsq cli; do python profiles/summarize_ncu.py full gpurun_out/prof_$t.ncu-rep gpurun_out/ncu_next_$t.json > gpurun_out/ncu_next_$t.txt 2>&1; rm -f gpurun_out/prof_$t.ncu-rep; done
cat gpurun_out/ncu_next_*.txt
