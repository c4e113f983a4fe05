mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_gla.py -q 2>&1 | tail -30 > gpurun_out/r2r_gla.txt
