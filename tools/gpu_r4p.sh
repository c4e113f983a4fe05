# head_dim 128, long local sequences: segment length capped (LASP_SEG_LEN 3584 / 4096) vs the ~5-items-per-SM plan
for sl in 0 3584 4096; do
  echo "== LASP_SEG_LEN=$sl"
  if [ $sl = 0 ]; then unset LASP_SEG_LEN; else export LASP_SEG_LEN=$sl; fi
  SWEEP_HD=128 SWEEP_N="32768,131072,524288,2097152" timeout 900 python tools/seq_sweep.py 10 2>&1 | tail -4
  timeout 300 python bench.py --config tnl7b --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-layer --no-gla 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tnl7b', round(d['value']/1e6,2), d['config'].get('segment_len'), {k:round(v*1e3,1) for k,v in d['path']['stages_ms_per_step'].items()})"
done > gpurun_out/r4p_seglen_d128.txt 2>&1
unset LASP_SEG_LEN
cat gpurun_out/r4p_seglen_d128.txt
