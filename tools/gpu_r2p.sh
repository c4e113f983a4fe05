mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/r2p_parity.txt
bash tools/cmp3.sh "liblasp_old.so liblasp.so" --no-layer > gpurun_out/r2p_cmp_tnl04b.txt 2>&1
bash tools/cmp3.sh "liblasp_old.so liblasp.so" --config tnl1b --no-layer > gpurun_out/r2p_cmp_tnl1b.txt 2>&1
