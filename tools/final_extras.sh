timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "concurrent or fused_prefix" 2>&1 | tail -2
timeout 1200 python tools/seq_sweep.py > gpurun_out/r1i_seq_sweep.md 2> gpurun_out/r1i_seq_sweep.err; tail -3 gpurun_out/r1i_seq_sweep.md
