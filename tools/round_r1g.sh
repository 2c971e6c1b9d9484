bash tools/gpu_round.sh r1g
timeout 300 python bench.py --solver admm --steps 5 --warmup 2 > gpurun_out/admm3_r1g.json 2>/dev/null
timeout 300 python bench.py --stage lsq --steps 10 --warmup 3 > gpurun_out/lsq3_r1g.json 2>/dev/null
timeout 300 python bench.py --stage cli --steps 5 --warmup 1 > gpurun_out/cli3_r1g.json 2>/dev/null
timeout 300 python bench.py --config C3_hcp7t --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_r1g.json 2>/dev/null
for f in admm3_r1g lsq3_r1g cli3_r1g bench7_r1g; do tail -1 gpurun_out/$f.json | cut -c1-160; done
