mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 900 -rf -k "flat or l2_persistent or resident_pcg_matches" > gpurun_out/pytest_r2l.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2l.log; tail -6 gpurun_out/pytest_r2l.log
