# D = 128 analysis: ncu --set full with source of the fused backward and forward core launches at TNL-1B,
# and a CTA-0 timeline of the fused backward from a trace build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
LASP_TRACE_BUILD=1 python -c "from paper_2404_02882_b200 import build as b; b.build(force=True, out='paper_2404_02882_b200/liblasp_trace.so')" 2>&1 | tail -3
LASP_LIB=$PWD/paper_2404_02882_b200/liblasp_trace.so timeout 300 python tools/trace.py 40 bwd 128 > gpurun_out/r2i_trace_bwd128.txt 2>&1
LASP_LIB=$PWD/paper_2404_02882_b200/liblasp_trace.so timeout 300 python tools/trace.py 40 fwd 128 > gpurun_out/r2i_trace_fwd128.txt 2>&1
for sk in 4 5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:core_tc --launch-skip $sk --launch-count 1 \
    -o gpurun_out/r2i_tnl1b_core_skip$sk -f python bench.py --config tnl1b --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-layer > gpurun_out/r2i_ncu$sk.log 2>&1
done
ls -la gpurun_out
