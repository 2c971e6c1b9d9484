# C5 (512x512x384) single GPU with the flat PCG + ncu of its kernels; 3T streaming ncu
mkdir -p gpurun_out
timeout 900 python bench.py --config C5_512 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench5_r2q.json 2> gpurun_out/bench5_r2q.err
tail -1 gpurun_out/bench5_r2q.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C5', d['value'], d['ms_per_step'], d['solver'], r['kernel'], r['frac'], r['kernel_share_of_step'], r['hbm_kernels'])"
tail -2 gpurun_out/bench5_r2q.err
export HYSCO_NO_GRAPH=1
timeout 900 ncu --set full --clock-control none -k "regex:pcg_march|pcg_upd|eval_kernel|trial_flat" -s 8 -c 4 -o /tmp/prof_c5 python bench.py --config C5_512 --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 1 > gpurun_out/ncu_r2q_c5.log 2>&1
ncu -i /tmp/prof_c5.ncu-rep --page raw --csv > gpurun_out/prof_r2q_c5.csv
timeout 900 ncu --set full --clock-control none -k "regex:pcg_march|pcg_upd|eval_kernel|trial_flat" -s 8 -c 4 -o /tmp/prof_c3 python bench.py --config C3_hcp7t --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 1 > gpurun_out/ncu_r2q_c3.log 2>&1
ncu -i /tmp/prof_c3.ncu-rep --page raw --csv > gpurun_out/prof_r2q_c3.csv
ls -la gpurun_out | grep r2q
