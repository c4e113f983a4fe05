# time experiment builds (liblasp_x*.so) against the production library; extra env (e.g. LASP_NO_FUSED=1)
# applies to every run. Two passes to expose run-to-run spread.
for pass in 1 2; do
for f in paper_2404_02882_b200/liblasp.so paper_2404_02882_b200/liblasp_x*.so; do L=$(basename $f)
  LASP_LIB=$PWD/paper_2404_02882_b200/$L timeout 200 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $CMP_ARGS > /tmp/v.out 2>&1
  tail -1 /tmp/v.out | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['value']/1e6,2), round(d['ms_per_step'],4), {k:round(v*1e3,1) for k,v in d['path']['stages_ms_per_step'].items()})" 2>/dev/null || { echo "$L failed"; tail -5 /tmp/v.out; }
done; done
