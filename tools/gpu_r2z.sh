mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | grep -E "^E|FAILED|Error|assert" | head -30 > gpurun_out/r2z_fail.txt
