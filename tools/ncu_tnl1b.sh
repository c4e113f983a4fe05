# ncu --set full of the two core launches at the TNL-1B shape (16 x 128): forward (instance 4) and fused
# backward (instance 5) of the third step (-k regex:core_tc counts core launches only)
mkdir -p gpurun_out
for sk in 4 5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:core_tc --launch-skip $sk --launch-count 1 \
    -o gpurun_out/${TAG:-r1i}_tnl1b_core_skip$sk -f python bench.py --config tnl1b --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
ls -la gpurun_out | grep tnl1b
