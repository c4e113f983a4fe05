mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r3w_pytest.txt
bash tools/ab_env2.sh LASP_SEPARATE_ENTRY=1 > gpurun_out/r3w_ab_tnl04b.txt 2>&1
bash tools/ab_env2.sh LASP_SEPARATE_ENTRY=1 --config tnl1b > gpurun_out/r3w_ab_tnl1b.txt 2>&1
