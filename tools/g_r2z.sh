mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_io.py -m gpu -q --timeout 600 -rf -k "cli_option" > gpurun_out/pytest_r2z.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2z.log; tail -4 gpurun_out/pytest_r2z.log
