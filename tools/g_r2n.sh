# ncu of pcg_march (slot version) at 7T: raw + source stalls
mkdir -p gpurun_out
export HYSCO_NO_GRAPH=1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:pcg_march" -s 3 -c 1 -o /tmp/prof_e python bench.py --config C3_hcp7t --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 1 > gpurun_out/ncu_r2o.log 2>&1
ncu -i /tmp/prof_e.ncu-rep --page raw --csv > gpurun_out/prof_r2o_7t.csv
ncu -i /tmp/prof_e.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_r2o_7t_sass.csv 2>&1
