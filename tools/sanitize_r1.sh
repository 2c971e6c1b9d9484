#!/bin/bash
# compute-sanitizer passes over the column kernels (diagnostic; run under gpurun)
mkdir -p gpurun_out
export HYSCO_NO_GRAPH=1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_lsq.py tests/test_gpu_io.py -q -x -k "not hcp3t and not cli" > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_memcheck.log | tail -3
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_lsq.py -q -x -k "parity and (37 or 144) and f32" > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" gpurun_out/san_racecheck.log | tail -3
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_lsq.py tests/test_gpu_io.py -q -x -k "parity and f32 and not hcp3t" > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_synccheck.log | tail -3
