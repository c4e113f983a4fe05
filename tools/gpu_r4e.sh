# item-boundary L2 prefetch of a new item's first ring-depth blocks (default) vs none; segment target re-sweep at
# head_dim 128 with the new item start; GPU tests on the default build
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r4e_pytest_gpu.txt 2>&1; tail -2 gpurun_out/r4e_pytest_gpu.txt
bash tools/cmp3.sh "liblasp_xNOITEMPF.so liblasp.so" --config tnl1b > gpurun_out/r4e_ab_itempf_tnl1b.txt 2>&1; cat gpurun_out/r4e_ab_itempf_tnl1b.txt
bash tools/cmp3.sh "liblasp_xNOITEMPF.so liblasp.so" > gpurun_out/r4e_ab_itempf_tnl04b.txt 2>&1; cat gpurun_out/r4e_ab_itempf_tnl04b.txt
bash tools/cmp3.sh "liblasp_xNOITEMPF.so liblasp.so" --config tnl7b --steps 10 > gpurun_out/r4e_ab_itempf_tnl7b.txt 2>&1; cat gpurun_out/r4e_ab_itempf_tnl7b.txt
bash tools/sweep_env.sh LASP_TARGET_CTAS "444 592 740 888" --config tnl1b > gpurun_out/r4e_target_tnl1b.txt 2>&1; cat gpurun_out/r4e_target_tnl1b.txt
LASP_TRACE_BUILD=1 python -c "from paper_2404_02882_b200 import build as b; b.build(force=True, out='paper_2404_02882_b200/liblasp_trace.so')" 2>&1 | tail -1
LASP_LIB=$PWD/paper_2404_02882_b200/liblasp_trace.so timeout 300 python tools/trace.py 40 bwd 128 > gpurun_out/r4e_trace_bwd128.txt 2>&1
