mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gla_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/r3i_gla_f3 -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-layer > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gla_kernel --launch-skip 5 --launch-count 1 -o gpurun_out/r3i_gla_dk -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-layer > /dev/null 2>&1
ls -la gpurun_out | grep r3i
