# round-2 GPU pass B: changed tests, smoke (+ its ncu launch list), the default bench, ncu of the 3T kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shipped.py tests/test_gpu_io.py -m gpu -q --timeout 600 > gpurun_out/pytest_r2b.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2b.log; tail -3 gpurun_out/pytest_r2b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2b.log 2>&1; tail -2 gpurun_out/smoke_r2b.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_smoke_r2b.csv python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
grep -c hysco gpurun_out/launches_smoke_r2b.csv; grep -o '"[a-z_]*_kernel' gpurun_out/launches_smoke_r2b.csv | sort | uniq -c
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err
tail -c 3000 gpurun_out/bench_r2b.json
export HYSCO_NO_GRAPH=1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:pcg_resident|eval_kernel|pcg_sync_floor" -s 2 -c 6 -o gpurun_out/prof_r2b_3t python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 --e2e-steps 2 > gpurun_out/ncu_r2b.log 2>&1
ls -la gpurun_out | grep r2b
