# prefix kernel with compile-time D / direction and U sized to nseg (one wave of resident threads) vs the
# round-2 prefix kernel (xOLDPREFIX); GPU suite on the default build
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r4h_pytest_gpu.txt 2>&1; tail -2 gpurun_out/r4h_pytest_gpu.txt
bash tools/cmp3.sh "liblasp_xOLDPREFIX.so liblasp.so" --config tnl1b > gpurun_out/r4h_ab_prefix_tnl1b.txt 2>&1; cat gpurun_out/r4h_ab_prefix_tnl1b.txt
bash tools/cmp3.sh "liblasp_xOLDPREFIX.so liblasp.so" --config tnl7b --steps 10 > gpurun_out/r4h_ab_prefix_tnl7b.txt 2>&1; cat gpurun_out/r4h_ab_prefix_tnl7b.txt
