# head_dim 128 with the 28-block plan: the prefix fold fused into the core launches (LASP_FOLD_MAX_ROUNDS=4 / 8)
# vs the separate prefix kernel (default at these sizes)
b() { timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-layer --no-gla "$@" 2>/tmp/b.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'M tok/s', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['path']['stages_ms_per_step'].items()})" || tail -3 /tmp/b.err; }
{ for i in 1 2; do
  echo "default tnl1b"; b --config tnl1b; echo "rounds=4 tnl1b"; LASP_FOLD_MAX_ROUNDS=4 b --config tnl1b
  echo "default tnl7b"; b --config tnl7b --steps 10; echo "rounds=16 tnl7b"; LASP_FOLD_MAX_ROUNDS=16 b --config tnl7b --steps 10
done; } > gpurun_out/r4t_fold_d128.txt 2>&1
cat gpurun_out/r4t_fold_d128.txt
