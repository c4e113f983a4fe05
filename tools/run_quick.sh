# Quick GPU check (on the box): full GPU test suite, then two bench lines (CUDA-graph replay and eager) and
# the TNL-1B shape. usage: bash tools/run_quick.sh
b() { timeout 200 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>/tmp/b.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'M tok/s', round(d['ms_per_step']*1e3,1), 'us/step', {k: round(v*1e3,1) for k,v in d['path']['stages_ms_per_step'].items()})" || tail -3 /tmp/b.err; }
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
echo graph; b
echo eager; b --no-graph
echo tnl1b; b --config tnl1b
