# head_dim-128 plan: 28-block segments when the forward launch keeps >= 2 items per SM (default) vs the round-2 plan
# (LASP_LONG_SEG_BLOCKS=0); full GPU suite on the default
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r4r_pytest_gpu.txt 2>&1; tail -2 gpurun_out/r4r_pytest_gpu.txt
b() { timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-layer --no-gla "$@" 2>/tmp/b.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'M tok/s', round(d['ms_per_step']*1e3,1), 'us', d['config'].get('segment_len'), {k: round(v*1e3,1) for k,v in d['path']['stages_ms_per_step'].items()})" || tail -3 /tmp/b.err; }
{ for i in 1 2; do
  echo "default tnl1b"; b --config tnl1b; echo "LASP_LONG_SEG_BLOCKS=0 tnl1b"; LASP_LONG_SEG_BLOCKS=0 b --config tnl1b
  echo "default tnl7b"; b --config tnl7b --steps 10; echo "LASP_LONG_SEG_BLOCKS=0 tnl7b"; LASP_LONG_SEG_BLOCKS=0 b --config tnl7b --steps 10
done
echo "== seq sweep 16 x 128, default"; SWEEP_HD=128 timeout 900 python tools/seq_sweep.py 10 2>&1 | tail -6
echo "== seq sweep 16 x 128, LASP_LONG_SEG_BLOCKS=0"; LASP_LONG_SEG_BLOCKS=0 SWEEP_HD=128 timeout 900 python tools/seq_sweep.py 10 2>&1 | tail -6
} > gpurun_out/r4r_ab_longseg.txt 2>&1
cat gpurun_out/r4r_ab_longseg.txt
