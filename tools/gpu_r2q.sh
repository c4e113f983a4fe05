mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/r2q_parity.txt
LASP_CORE_SEG_DESC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 >> gpurun_out/r2q_parity.txt
bash tools/ab_env2.sh LASP_CORE_SEG_DESC=1 > gpurun_out/r2q_ab_tnl04b.txt 2>&1
bash tools/ab_env2.sh LASP_CORE_SEG_DESC=1 --config tnl1b > gpurun_out/r2q_ab_tnl1b.txt 2>&1
