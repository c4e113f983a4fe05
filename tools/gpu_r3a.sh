mkdir -p gpurun_out
export SWEEP_N="524288,2097152" SWEEP_HD=64
for t in 592 1184 2368 4736; do echo "== target $t" >> gpurun_out/r3a_long.txt; LASP_TARGET_CTAS=$t timeout 600 python tools/seq_sweep.py 5 >> gpurun_out/r3a_long.txt 2>&1; done
