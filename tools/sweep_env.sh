# Sweep one environment knob of the library on the bench (same box), e.g.
#   bash tools/sweep_env.sh LASP_TARGET_CTAS "296 444 592 888" --config tnl1b
var=$1; vals=$2; shift 2
for i in 1 2; do for x in $vals; do
  env $var=$x timeout 200 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>/tmp/b.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$var=$x', round(d['value']/1e6,2), 'M tok/s', round(d['ms_per_step']*1e3,1), 'us', d['config'].get('segment_len'), {k: round(v*1e3,1) for k,v in d['path']['stages_ms_per_step'].items()})" || tail -2 /tmp/b.err
done; done
