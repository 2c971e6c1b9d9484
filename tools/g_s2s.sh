# ncu --set full of the final build at 7T (flat PCG kernels, eval, trial, init)
mkdir -p gpurun_out
export HYSCO_NO_GRAPH=1
timeout 900 ncu --set full --clock-control none -k "regex:pcg_march|pcg_upd|eval_kernel|trial_flat|pcg_init_flat" -s 4 -c 10 -o gpurun_out/prof_r2f_7t python bench.py --config C3_hcp7t --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 1 > gpurun_out/ncu_r2f_7t.log 2>&1
python profiles/summarize_ncu.py full gpurun_out/prof_r2f_7t.ncu-rep gpurun_out/ncu_r2f_7t.json > /dev/null
ls -la gpurun_out/ncu_r2f_7t.json
