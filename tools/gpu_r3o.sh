mkdir -p gpurun_out
timeout 600 python bench.py --loopback 4 --steps 10 --warmup 3 --no-e2e > gpurun_out/r3o_loop4.json 2> gpurun_out/r3o_loop4.err
timeout 600 python bench.py --loopback 2 --steps 10 --warmup 3 --no-e2e --config tnl1b > gpurun_out/r3o_loop2_tnl1b.json 2>> gpurun_out/r3o_loop4.err
