# one --set full capture each of the forward core launch and the fused backward launch (bench config tnl04b)
set -x
mkdir -p gpurun_out
for sk in 4 5; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:core_tc --launch-skip $sk --launch-count 1 \
    -o gpurun_out/core_skip$sk -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_core$sk.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
ls -la gpurun_out
