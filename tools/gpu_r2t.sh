mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_gla.py -q 2>&1 | tail -3 > gpurun_out/r2t_gla.txt
for w in 1 2 3 4; do for c in tnl04b tnl1b; do
LASP_GLA_WAVES=$w timeout 300 python bench.py --steps 5 --warmup 2 --config $c --no-e2e --no-cpu-baseline --no-layer 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['gla']; print('waves $w $c', round(g['value']/1e6,2), round(g['ms_per_step'],3), round(g['roofline']['frac'],3), {k:round(v*1e3) for k,v in g['stages_ms_per_step'].items()})" >> gpurun_out/r2t_waves.txt
done; done
