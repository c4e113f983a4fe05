# head_dim-128 segment-state items split by value slice (2 items per segment, 4 x 48 KB stages) vs whole
# segments (xNOVSPLIT); full GPU suite on the default build
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r4g_pytest_gpu.txt 2>&1; tail -2 gpurun_out/r4g_pytest_gpu.txt
bash tools/cmp3.sh "liblasp_xNOVSPLIT.so liblasp.so" --config tnl1b > gpurun_out/r4g_ab_vsplit_tnl1b.txt 2>&1; cat gpurun_out/r4g_ab_vsplit_tnl1b.txt
bash tools/cmp3.sh "liblasp_xNOVSPLIT.so liblasp.so" --config tnl7b --steps 10 > gpurun_out/r4g_ab_vsplit_tnl7b.txt 2>&1; cat gpurun_out/r4g_ab_vsplit_tnl7b.txt
