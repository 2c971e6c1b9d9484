# round-2 evidence pass: ncu --set full summaries at C2 / C3 / C5 of the current build,
# the smoke launch list, and compute-sanitizer memcheck of the flat / march / slab kernels
mkdir -p gpurun_out
export HYSCO_NO_GRAPH=1
timeout 900 ncu --set full --clock-control none -k "regex:pcg_resident|eval_kernel|pcg_sync_floor" -s 2 -c 6 -o /tmp/p2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 1 > gpurun_out/ncu_r2u_c2.log 2>&1
python profiles/summarize_ncu.py full /tmp/p2.ncu-rep gpurun_out/ncu_r2u_c2.json > /dev/null
timeout 900 ncu --set full --clock-control none -k "regex:pcg_march|pcg_upd|eval_kernel|trial_flat|pcg_init_flat" -s 4 -c 10 -o /tmp/p3 python bench.py --config C3_hcp7t --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 1 > gpurun_out/ncu_r2u_c3.log 2>&1
python profiles/summarize_ncu.py full /tmp/p3.ncu-rep gpurun_out/ncu_r2u_c3.json > /dev/null
timeout 1200 ncu --set full --clock-control none -k "regex:pcg_march|pcg_upd|eval_kernel|trial_flat|pcg_init_flat" -s 4 -c 10 -o /tmp/p5 python bench.py --config C5_512 --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 1 > gpurun_out/ncu_r2u_c5.log 2>&1
python profiles/summarize_ncu.py full /tmp/p5.ncu-rep gpurun_out/ncu_r2u_c5.json > /dev/null
unset HYSCO_NO_GRAPH
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_smoke_r2u.csv python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
grep -o '"[a-z_0-9]*_kernel' gpurun_out/launches_smoke_r2u.csv | sort | uniq -c
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "flat_pcg and (5, 7, 37) or flat_pcg and (1, 3, 70)" > gpurun_out/memcheck_r2u_flat.log 2>&1; tail -4 gpurun_out/memcheck_r2u_flat.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_slab.py -m gpu -q -x > gpurun_out/memcheck_r2u_slab.log 2>&1; tail -4 gpurun_out/memcheck_r2u_slab.log
ls -la gpurun_out | grep r2u
