# full GPU suite after history + NVTX, smoke
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/pytest_r2y.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2y.log; tail -8 gpurun_out/pytest_r2y.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2y.log 2>&1; tail -2 gpurun_out/smoke_r2y.log
