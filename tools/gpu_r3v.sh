mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_ring.py -q -x 2>&1 | tail -15 > gpurun_out/r3v_ring.txt
timeout 600 python bench.py --loopback 4 --steps 10 --warmup 3 --no-e2e > gpurun_out/r3v_loop4.json 2> gpurun_out/r3v_loop4.err
