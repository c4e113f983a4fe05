mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 300 python bench.py --loopback 2 --steps 3 --warmup 2 --no-e2e --exchange p2p > gpurun_out/r3r.json 2> gpurun_out/r3r.err
timeout 300 compute-sanitizer --tool memcheck python bench.py --loopback 2 --steps 2 --warmup 1 --no-e2e --exchange p2p --no-graph > gpurun_out/r3r_san.txt 2>&1
