set -x
mkdir -p gpurun_out
export HYSCO_NO_GRAPH=1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:eval_kernel|matvec_kernel|pcg_update|pcg_dir|trial_init" -s 30 -c 5 -o gpurun_out/prof_r2base_7t python bench.py --config C3_hcp7t --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 2 > gpurun_out/ncu_r2base_7t.log 2>&1
unset HYSCO_NO_GRAPH
timeout 300 python bench.py --config C3_hcp7t --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_r2base.json 2>gpurun_out/bench7_r2base.err
tail -c 600 gpurun_out/bench7_r2base.json
ls -la gpurun_out | grep r2base
