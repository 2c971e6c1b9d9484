# slab path with the flat kernels applying the deferred decisions (no decide_kernel per PCG step)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_slab.py tests/test_gpu_parity.py -m gpu -q -x -k "slab or flat" > gpurun_out/pytest_p.log 2>&1; tail -2 gpurun_out/pytest_p.log
for v in 0 1; do
HYSCO_SLAB_NO_FUSE=$v timeout 900 python bench.py --no-cpu-baseline --config C3_hcp7t --slab > gpurun_out/bench_p_nofuse$v.json 2> gpurun_out/bench_p_nofuse$v.err
tail -1 gpurun_out/bench_p_nofuse$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('no_fuse=$v slab 7T', round(d['value'],2), d.get('ms_per_step'), d.get('solver'))"
done
