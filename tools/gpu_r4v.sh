# opt-in sweep: 24 random head_dim-128 shapes under the 28-block segment plan, against the fp64 oracle
LASP_PLAN_SWEEP=24 timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k long_segment_plan > gpurun_out/r4v_plan_sweep.txt 2>&1; grep -E "case|passed|failed" gpurun_out/r4v_plan_sweep.txt | tail -30
