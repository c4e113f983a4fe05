# u . c after the state copy in the head_dim-128 forward only (default) vs before it everywhere (xKUEARLY); plus
# segment targets that make every launch's item count a multiple of 148 at head_dim 128 (nseg = 37)
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_layer.py -m gpu -x -q > gpurun_out/r4o_pytest.txt 2>&1; tail -2 gpurun_out/r4o_pytest.txt
bash tools/cmp3.sh "liblasp_xKUEARLY.so liblasp.so" --config tnl1b > gpurun_out/r4o_ab_kulate_fwd_tnl1b.txt 2>&1; cat gpurun_out/r4o_ab_kulate_fwd_tnl1b.txt
bash tools/cmp3.sh "liblasp_xKUEARLY.so liblasp.so" --config tnl7b --steps 10 > gpurun_out/r4o_ab_kulate_fwd_tnl7b.txt 2>&1; cat gpurun_out/r4o_ab_kulate_fwd_tnl7b.txt
bash tools/sweep_env.sh LASP_TARGET_CTAS "740 1184" --config tnl1b > gpurun_out/r4o_target37_tnl1b.txt 2>&1; cat gpurun_out/r4o_target37_tnl1b.txt
bash tools/sweep_env.sh LASP_TARGET_CTAS "740 2368" --config tnl7b --steps 10 > gpurun_out/r4o_target37_tnl7b.txt 2>&1; cat gpurun_out/r4o_target37_tnl7b.txt
