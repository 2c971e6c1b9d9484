# ncu evidence for the tiled resident build: --set full of the 3T kernels, launch list of the bench command
mkdir -p gpurun_out
export HYSCO_NO_GRAPH=1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pcg_resident|eval_kernel|pcg_sync_floor" -s 2 -c 6 -o gpurun_out/prof_r2t_3t python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 1 > gpurun_out/ncu_r2t_3t.log 2>&1
python profiles/summarize_ncu.py full gpurun_out/prof_r2t_3t.ncu-rep gpurun_out/ncu_r2t_3t.json > /dev/null
unset HYSCO_NO_GRAPH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2t.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 1 > gpurun_out/ncu_launches_r2t.log 2>&1
python profiles/summarize_ncu.py launches gpurun_out/launches_r2t.csv gpurun_out/launches_r2t.json > /dev/null
ls -la gpurun_out | grep r2t
