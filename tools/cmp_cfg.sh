# bench both head dims (short runs, no e2e / cpu baseline)
for cfg in tnl04b tnl1b; do
  timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), {k:round(v,4) for k,v in d['path']['stages_ms_per_step'].items()})"
done
