b() { timeout 200 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>/tmp/b.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), d['gpu_launches'], {k: round(v*1e3,1) for k,v in d['path']['stages_ms_per_step'].items()})" || tail -3 /tmp/b.err; }
echo eager; b; echo graph; b --graph; echo eager; b; echo graph; b --graph
echo graph-tnl1b; b --graph --config tnl1b; echo eager-tnl1b; b --config tnl1b
bash tools/cmp_variants.sh
