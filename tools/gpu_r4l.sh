# robustness on the final code (compute-sanitizer is closed on this pool): 1000-case seeded random-shape parity sweep
# (B 1-3, H 1-8, D 32/64/128, T 1-4 chained ranks, per-rank lengths up to 3000 tokens, ragged, bf16 and fp32)
LASP_LONG_SWEEP=1000 timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -k long_sweep > gpurun_out/r4l_long_sweep.txt 2>&1; tail -3 gpurun_out/r4l_long_sweep.txt
