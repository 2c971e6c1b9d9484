# 2-D tiled resident PCG: tiled-vs-strip test, full GPU suite, smoke, bench C2 (tiled and strips)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tiled" > gpurun_out/pytest_e_tiled.log 2>&1; tail -3 gpurun_out/pytest_e_tiled.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err
tail -1 gpurun_out/bench_e.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('tiled value',round(d['value'],2),'ms',round(d['ms_per_step'],3),'e2e',round(d['e2e']['value'],2),'solver',d['solver'],'res us/it',r['achieved'],'floor',r['peak'])"
HYSCO_RES_TILED=0 timeout 600 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_e_strip.json 2> gpurun_out/bench_e_strip.err
tail -1 gpurun_out/bench_e_strip.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('strip value',round(d['value'],2),'ms',round(d['ms_per_step'],3),'res us/it',r['achieved'],'floor',r['peak'])"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_e.log 2>&1; tail -3 gpurun_out/pytest_e.log
