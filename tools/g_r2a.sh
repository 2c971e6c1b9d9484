# round-2 GPU pass A: new shipped-config parity tests + the modified parity file
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_shipped.py tests/test_gpu_parity.py -m gpu -q --timeout 900 -rA > gpurun_out/pytest_r2a.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2a.log
tail -30 gpurun_out/pytest_r2a.log
