# Same-box A/B of an environment switch without the test suite. usage: bash tools/ab_env2.sh VAR=value [bench args]
ab=$1; shift
b() { timeout 200 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-layer --no-gla "$@" 2>/tmp/b.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'M tok/s', round(d['ms_per_step']*1e3,1), 'us/step', {k: round(v*1e3,1) for k,v in d['path']['stages_ms_per_step'].items()})" || tail -3 /tmp/b.err; }
for i in 1 2; do
echo -n "default: "; b "$@"; echo -n "$ab: "; env $ab bash -c "$(declare -f b); b $*"
done
