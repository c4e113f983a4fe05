# Same-box A/B of two builds of the library (paper_2404_02882_b200/liblasp_old.so vs liblasp.so), alternating.
# usage (on the GPU box): bash tools/cmp_libs.sh [bench args, e.g. --config tnl1b]
for i in 1 2; do for L in liblasp_old.so liblasp.so; do LASP_LIB=$PWD/paper_2404_02882_b200/$L timeout 200 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['value']/1e6,2), round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['path']['stages_ms_per_step'].items()})"; done; done
