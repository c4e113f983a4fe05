for t in 592 1184 2368; do echo "target $t"; LASP_TARGET_CTAS=$t SWEEP_HD=64,128 SWEEP_N=524288,2097152 timeout 600 python tools/seq_sweep.py 5 | tail -4; done
