# Same-box A/B/C of library builds (alternating), e.g. r1 final vs this round's steps.
# usage (GPU box): bash tools/cmp3.sh "liblasp_r1.so liblasp_old.so liblasp.so" [bench args]
libs=${1:-"liblasp_old.so liblasp.so"}; shift
for i in 1 2; do for L in $libs; do LASP_LIB=$PWD/paper_2404_02882_b200/$L timeout 300 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-layer --no-gla "$@" 2>/tmp/cmp.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), {k:round(v*1e3,1) for k,v in d['path']['stages_ms_per_step'].items()})" || tail -2 /tmp/cmp.err; done; done
