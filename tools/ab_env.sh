# Same-box A/B of an environment switch (default: the fused prefix fold vs LASP_NO_FUSED_FOLD=1), after the
# GPU test suite. usage (on the GPU box): bash tools/ab_env.sh [VAR=value]
ab=${1:-LASP_NO_FUSED_FOLD=1}
b() { timeout 200 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>/tmp/b.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'M tok/s', round(d['ms_per_step']*1e3,1), 'us/step', {k: round(v*1e3,1) for k,v in d['path']['stages_ms_per_step'].items()})" || tail -3 /tmp/b.err; }
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do
echo default; b; echo $ab; env $ab bash -c "$(declare -f b); b"
echo default-tnl1b; b --config tnl1b; echo $ab-tnl1b; env $ab bash -c "$(declare -f b); b --config tnl1b"
done
