mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_layer.py -q -k "loopback and p2p" 2>&1 | tail -3 > gpurun_out/r3z.txt
timeout 300 python -m pytest tests/test_gpu_ring.py -q -k "p2p and not processes" 2>&1 | tail -3 >> gpurun_out/r3z.txt
timeout 300 python bench.py --loopback 2 --exchange p2p --steps 5 --warmup 3 --no-e2e 2>&1 | tail -2 | cut -c1-400 >> gpurun_out/r3z.txt
