mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ring.py tests/test_gpu_layer.py -x -q 2>&1 | tail -3 > gpurun_out/r2v_parity.txt
bash tools/cmp3.sh "liblasp_old.so liblasp.so" > gpurun_out/r2v_cmp_tnl04b.txt 2>&1
