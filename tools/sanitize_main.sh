#!/bin/bash
# compute-sanitizer passes over the main-path kernels on the small parity cases (diagnostic; run under gpurun)
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "not hcp3t" > gpurun_out/san_main_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_main_memcheck.log | tail -3
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "resident_pcg_matches or admm_fixed_parity or (solve_fixed_parity and f32)" > gpurun_out/san_main_racecheck.log 2>&1; echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" gpurun_out/san_main_racecheck.log | tail -3
