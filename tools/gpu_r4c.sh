# head_dim-128 item start: L2 prefetch of the next item's prefix state (producer) and the state loads overlapped
# with the first u . c scaling; A/B/C/D of the four builds at TNL-1B (and TNL-0.4B: no change expected), trace
mkdir -p gpurun_out
LASP_TRACE_BUILD=1 python -c "from paper_2404_02882_b200 import build as b; b.build(force=True, out='paper_2404_02882_b200/liblasp_trace.so')" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r4c_pytest_parity.txt 2>&1; tail -2 gpurun_out/r4c_pytest_parity.txt
bash tools/cmp3.sh "liblasp_xPREV.so liblasp_xNOPF.so liblasp_xPFONLY.so liblasp.so" --config tnl1b > gpurun_out/r4c_ab_state_tnl1b.txt 2>&1; cat gpurun_out/r4c_ab_state_tnl1b.txt
bash tools/cmp3.sh "liblasp_xPREV.so liblasp.so" > gpurun_out/r4c_ab_state_tnl04b.txt 2>&1; cat gpurun_out/r4c_ab_state_tnl04b.txt
LASP_LIB=$PWD/paper_2404_02882_b200/liblasp_trace.so timeout 300 python tools/trace.py 40 bwd 128 > gpurun_out/r4c_trace_bwd128.txt 2>&1
head -42 gpurun_out/r4c_trace_bwd128.txt; tail -6 gpurun_out/r4c_trace_bwd128.txt
