# L2-resident persistent PCG: parity (fp64 small shapes run it; forced on for f32 via HYSCO_L2PCG=1) + 7T bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -m gpu -q --timeout 600 -x > gpurun_out/pytest_r2d.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2d.log; tail -3 gpurun_out/pytest_r2d.log
HYSCO_NO_RESIDENT=1 HYSCO_L2PCG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -x -k "solve_fixed or pipeline or production or armijo_halving or resident_pcg_matches" > gpurun_out/pytest_r2d_forced.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2d_forced.log; tail -3 gpurun_out/pytest_r2d_forced.log
timeout 600 python -m pytest tests/test_gpu_shipped.py -m gpu -q --timeout 600 -k hcp7t > gpurun_out/pytest_r2d_7t.log 2>&1; tail -2 gpurun_out/pytest_r2d_7t.log
timeout 600 python bench.py --config C3_hcp7t --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_r2d.json 2> gpurun_out/bench7_r2d.err; tail -1 gpurun_out/bench7_r2d.json | cut -c1-400
HYSCO_L2PCG=0 timeout 600 python bench.py --config C3_hcp7t --steps 10 --warmup 3 --no-cpu-baseline | cut -c1-300
tail -5 gpurun_out/bench7_r2d.err
