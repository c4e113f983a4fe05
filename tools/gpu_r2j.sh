mkdir -p gpurun_out
./tools/tmem_bw > gpurun_out/r2j_tmem_bw.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
LASP_TRACE_BUILD=1 python -c "from paper_2404_02882_b200 import build as b; b.build(force=True, out='paper_2404_02882_b200/liblasp_trace.so')" 2>&1 | tail -3
LASP_LIB=$PWD/paper_2404_02882_b200/liblasp_trace.so timeout 300 python tools/trace.py 40 bwd 64 > gpurun_out/r2j_trace_bwd64.txt 2>&1
