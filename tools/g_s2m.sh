# round-2 final evidence: every bench mode line, memcheck of the resident tiled path
mkdir -p gpurun_out
B="--no-cpu-baseline"
timeout 900 python bench.py > gpurun_out/fin_c2.json 2> gpurun_out/fin_c2.err
timeout 900 python bench.py $B --config C3_hcp7t > gpurun_out/fin_c3.json 2> gpurun_out/fin_c3.err
timeout 1200 python bench.py $B --config C5_512 --steps 5 --warmup 3 > gpurun_out/fin_c5.json 2> gpurun_out/fin_c5.err
timeout 900 python bench.py $B --config C3_hcp7t --slab > gpurun_out/fin_slab7t.json 2> gpurun_out/fin_slab7t.err
timeout 900 python bench.py $B --solver admm > gpurun_out/fin_admm3t.json 2> gpurun_out/fin_admm3t.err
timeout 900 python bench.py $B --stage lsq > gpurun_out/fin_lsq3t.json 2> gpurun_out/fin_lsq3t.err
timeout 900 python bench.py $B --precond block --stop paper > gpurun_out/fin_blk3t.json 2> gpurun_out/fin_blk3t.err
timeout 900 python bench.py $B --batch 8 > gpurun_out/fin_b8.json 2> gpurun_out/fin_b8.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
for f in gpurun_out/fin_*.json; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d.get('value'), d.get('unit'), d.get('e2e',{}).get('value') if isinstance(d.get('e2e'),dict) else '')"; done
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tiled and 592" > gpurun_out/memcheck_r2_tiled.log 2>&1; tail -3 gpurun_out/memcheck_r2_tiled.log
