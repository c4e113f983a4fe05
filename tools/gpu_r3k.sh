mkdir -p gpurun_out
for i in 1 2; do for L in liblasp.so liblasp_gt16.so liblasp_gt32.so; do for c in tnl04b tnl1b; do
  LASP_LIB=$PWD/paper_2404_02882_b200/$L timeout 300 python bench.py --config $c --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-layer 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['gla']; print('$L $c', round(g['value']/1e6,2), round(g['roofline']['frac'],3), {k:round(v*1e3) for k,v in g['stages_ms_per_step'].items() if 'gla' in k})" >> gpurun_out/r3k_gla_gt.txt
done; done; done
