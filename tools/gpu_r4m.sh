# mask software-pipelined over half chunks (default) vs one chunk at a time (xSERIAL): parity, A/B both head dims
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r4m_pytest_parity.txt 2>&1; tail -2 gpurun_out/r4m_pytest_parity.txt
bash tools/cmp3.sh "liblasp_xSERIAL.so liblasp.so" > gpurun_out/r4m_ab_maskpipe_tnl04b.txt 2>&1; cat gpurun_out/r4m_ab_maskpipe_tnl04b.txt
bash tools/cmp3.sh "liblasp_xSERIAL.so liblasp.so" --config tnl1b > gpurun_out/r4m_ab_maskpipe_tnl1b.txt 2>&1; cat gpurun_out/r4m_ab_maskpipe_tnl1b.txt
