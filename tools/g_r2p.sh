# slab path as graph segments: slab tests (+ host-loop variant), 7T slab bench vs single
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_slab.py -m gpu -q --timeout 900 -rf > gpurun_out/pytest_r2p.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2p.log; tail -4 gpurun_out/pytest_r2p.log
HYSCO_NO_GRAPH=1 timeout 1200 python -m pytest tests/test_gpu_slab.py -m gpu -q --timeout 900 -rf > gpurun_out/pytest_r2p_ng.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2p_ng.log; tail -2 gpurun_out/pytest_r2p_ng.log
timeout 600 python bench.py --config C3_hcp7t --slab --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench7slab_r2p.json 2> gpurun_out/bench7slab_r2p.err
tail -1 gpurun_out/bench7slab_r2p.json | cut -c1-600; tail -3 gpurun_out/bench7slab_r2p.err
