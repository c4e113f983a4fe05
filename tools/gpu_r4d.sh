# S in two N = 64 halves (mask starts one half-product earlier) and the ring slot's c tile on its own barrier:
# A/B/C/D at both head dims, full GPU suite on the default build, trace at head_dim 128
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r4d_pytest_gpu.txt 2>&1; tail -2 gpurun_out/r4d_pytest_gpu.txt
bash tools/cmp3.sh "liblasp_xBOTHWHOLE.so liblasp_xSWHOLE.so liblasp_xFULLWHOLE.so liblasp.so" --config tnl1b > gpurun_out/r4d_ab_tnl1b.txt 2>&1; cat gpurun_out/r4d_ab_tnl1b.txt
bash tools/cmp3.sh "liblasp_xBOTHWHOLE.so liblasp_xSWHOLE.so liblasp_xFULLWHOLE.so liblasp.so" > gpurun_out/r4d_ab_tnl04b.txt 2>&1; cat gpurun_out/r4d_ab_tnl04b.txt
LASP_TRACE_BUILD=1 python -c "from paper_2404_02882_b200 import build as b; b.build(force=True, out='paper_2404_02882_b200/liblasp_trace.so')" 2>&1 | tail -1
LASP_LIB=$PWD/paper_2404_02882_b200/liblasp_trace.so timeout 300 python tools/trace.py 40 bwd 128 > gpurun_out/r4d_trace_bwd128.txt 2>&1
LASP_LIB=$PWD/paper_2404_02882_b200/liblasp_trace.so timeout 300 python tools/trace.py 40 bwd 64 > gpurun_out/r4d_trace_bwd64.txt 2>&1
