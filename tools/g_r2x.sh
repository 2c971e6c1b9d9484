mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 900 -rf -k "admm" > gpurun_out/pytest_r2x.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2x.log; tail -4 gpurun_out/pytest_r2x.log
