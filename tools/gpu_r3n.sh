mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_ring.py -q -x 2>&1 | tail -25 > gpurun_out/r3n_ring.txt
