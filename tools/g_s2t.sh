# final bench lines after the streaming / slab changes
mkdir -p gpurun_out
B="--no-cpu-baseline"
timeout 900 python bench.py > gpurun_out/fin2_c2.json 2> gpurun_out/fin2_c2.err
timeout 900 python bench.py $B --config C3_hcp7t > gpurun_out/fin2_c3.json 2> gpurun_out/fin2_c3.err
timeout 1200 python bench.py $B --config C5_512 --steps 5 --warmup 3 > gpurun_out/fin2_c5.json 2> gpurun_out/fin2_c5.err
timeout 900 python bench.py $B --config C3_hcp7t --slab > gpurun_out/fin2_slab7t.json 2> gpurun_out/fin2_slab7t.err
for f in gpurun_out/fin2_*.json; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d.get('value'),3), d.get('e2e',{}).get('value') if isinstance(d.get('e2e'),dict) else '')"; done
