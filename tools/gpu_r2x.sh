mkdir -p gpurun_out
export SWEEP_N="2048,4096,8192,32768"
for v in default fold; do
  if [ $v = fold ]; then export LASP_FOLD_MAX_ROUNDS=1000; else unset LASP_FOLD_MAX_ROUNDS; fi
  echo "== $v" >> gpurun_out/r2x_short.txt
  timeout 600 python tools/seq_sweep.py 20 >> gpurun_out/r2x_short.txt 2>&1
done
for t in 148 296 592; do echo "== target $t" >> gpurun_out/r2x_short.txt; LASP_TARGET_CTAS=$t SWEEP_N=2048,4096 timeout 300 python tools/seq_sweep.py 20 >> gpurun_out/r2x_short.txt 2>&1; done
