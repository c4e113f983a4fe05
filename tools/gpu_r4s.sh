# head_dim 64: longer segments (13 / 14 / 28 blocks) vs the 4 x 148-item plan (7 blocks) at TNL-0.4B, and 128K / 512K
bash tools/sweep_env.sh LASP_SEG_LEN "0 1664 1792 3584" > gpurun_out/r4s_seglen_tnl04b.txt 2>&1; cat gpurun_out/r4s_seglen_tnl04b.txt
for sl in 0 1792 3584; do echo "== LASP_SEG_LEN=$sl"; if [ $sl = 0 ]; then unset LASP_SEG_LEN; else export LASP_SEG_LEN=$sl; fi
  SWEEP_HD=64 SWEEP_N="131072,524288" timeout 600 python tools/seq_sweep.py 10 2>&1 | tail -2; done >> gpurun_out/r4s_seglen_tnl04b.txt 2>&1
unset LASP_SEG_LEN; tail -9 gpurun_out/r4s_seglen_tnl04b.txt
