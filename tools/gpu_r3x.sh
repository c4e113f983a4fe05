mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_gla.py -q -x -k "hybrid or autograd or processes" 2>&1 | tail -15 > gpurun_out/r3x.txt
