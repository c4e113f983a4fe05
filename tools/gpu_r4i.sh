# P chunk published after the next chunk's TMEM load (store latency hidden) vs the previous commit (xPREV)
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r4i_pytest_parity.txt 2>&1; tail -2 gpurun_out/r4i_pytest_parity.txt
bash tools/cmp3.sh "liblasp_xPREV.so liblasp.so" > gpurun_out/r4i_ab_defer_tnl04b.txt 2>&1; cat gpurun_out/r4i_ab_defer_tnl04b.txt
bash tools/cmp3.sh "liblasp_xPREV.so liblasp.so" --config tnl1b > gpurun_out/r4i_ab_defer_tnl1b.txt 2>&1; cat gpurun_out/r4i_ab_defer_tnl1b.txt
