# per-chunk P readiness (default build) vs whole-P (xPWHOLE) A/B at both head dims, GPU tests, D = 128 / 64 traces
mkdir -p gpurun_out
LASP_TRACE_BUILD=1 python -c "from paper_2404_02882_b200 import build as b; b.build(force=True, out='paper_2404_02882_b200/liblasp_trace.so')" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r4b_pytest_gpu.txt 2>&1; tail -3 gpurun_out/r4b_pytest_gpu.txt
bash tools/cmp3.sh "liblasp_xPWHOLE.so liblasp.so" > gpurun_out/r4b_ab_pchunk_tnl04b.txt 2>&1; cat gpurun_out/r4b_ab_pchunk_tnl04b.txt
bash tools/cmp3.sh "liblasp_xPWHOLE.so liblasp.so" --config tnl1b > gpurun_out/r4b_ab_pchunk_tnl1b.txt 2>&1; cat gpurun_out/r4b_ab_pchunk_tnl1b.txt
LASP_LIB=$PWD/paper_2404_02882_b200/liblasp_trace.so timeout 300 python tools/trace.py 40 bwd 128 > gpurun_out/r4b_trace_bwd128.txt 2>&1
LASP_LIB=$PWD/paper_2404_02882_b200/liblasp_trace.so timeout 300 python tools/trace.py 40 bwd 64 > gpurun_out/r4b_trace_bwd64.txt 2>&1
head -45 gpurun_out/r4b_trace_bwd128.txt
