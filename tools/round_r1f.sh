bash tools/gpu_round.sh r1f ncu
timeout 300 python bench.py --stage cli --steps 5 --warmup 1 > gpurun_out/cli3_r1f.json 2>&1; tail -1 gpurun_out/cli3_r1f.json | cut -c1-200
timeout 300 python bench.py --stage lsq --steps 10 --warmup 3 > gpurun_out/lsq3_r1f.json 2>&1
timeout 300 python tools/timeline.py > gpurun_out/timeline_r1f_3t.txt 2>&1; tail -5 gpurun_out/timeline_r1f_3t.txt
