timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config4 or graph" 2>&1 | tail -2
bash tools/cmp_variants.sh
for f in liblasp.so liblasp_xseg128s3.so liblasp_xhead.so; do
  LASP_LIB=$PWD/paper_2404_02882_b200/$f timeout 200 python bench.py --config tnl1b --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tnl1b $f', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), {k:round(v*1e3,1) for k,v in d['path']['stages_ms_per_step'].items()})"
done
