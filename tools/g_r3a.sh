mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_slab.py -m gpu -q --timeout 900 -rf -k "admm" > gpurun_out/pytest_r3a.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r3a.log; tail -12 gpurun_out/pytest_r3a.log
