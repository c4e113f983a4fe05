# head_dim 64 segment target re-swept on the final code (592 = 4 x 148 default)
bash tools/sweep_env.sh LASP_TARGET_CTAS "444 592 740 888 1184" --no-layer --no-gla > gpurun_out/r4u_target_tnl04b.txt 2>&1; cat gpurun_out/r4u_target_tnl04b.txt
