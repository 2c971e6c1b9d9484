# ncu of eval_kernel at 3T: raw + SASS-level stalls
mkdir -p gpurun_out
export HYSCO_NO_GRAPH=1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:eval_kernel" -s 3 -c 1 -o /tmp/prof_e python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 1 > gpurun_out/ncu_r2s.log 2>&1
ncu -i /tmp/prof_e.ncu-rep --page raw --csv > gpurun_out/prof_r2s_3t.csv
ncu -i /tmp/prof_e.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_r2s_3t_sass.csv 2>&1
