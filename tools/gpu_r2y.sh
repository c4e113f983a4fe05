mkdir -p gpurun_out
export SWEEP_N="2048,4096,8192,16384,32768"
for v in 0 1; do
  if [ $v = 0 ]; then export LASP_MIN_SEG_BLOCKS=1; else unset LASP_MIN_SEG_BLOCKS; fi
  echo "== min_seg_blocks $v (0: old plan)" >> gpurun_out/r2y_short.txt
  timeout 600 python tools/seq_sweep.py 20 >> gpurun_out/r2y_short.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2 >> gpurun_out/r2y_short.txt
