mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gla.py tests/test_gpu_ring.py -q -k "gla or generalised" 2>&1 | tail -2 > gpurun_out/r3m_gla.txt
for c in tnl04b tnl1b tnl7b; do timeout 300 python bench.py --config $c --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-layer 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['gla']; print('$c', round(g['value']/1e6,2), round(g['roofline']['frac'],3), {k:round(v*1e3) for k,v in g['stages_ms_per_step'].items() if 'gla' in k})" >> gpurun_out/r3m_gla.txt; done
