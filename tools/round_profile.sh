# Round evidence: bench lines (both head dims), ncu launch list, ncu --set full of the top kernels.
# usage (on the GPU box): bash tools/round_profile.sh <tag>
tag=${1:-r}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --config tnl1b --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_bench_tnl1b.json 2> gpurun_out/${tag}_bench_tnl1b.err
timeout 900 python bench.py --config tnl7b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_tnl7b.json 2> gpurun_out/${tag}_bench_tnl7b.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"core_tc|seg_state|tag_kernel|prefix_kernel|combine|norm_apply|gla_" -c 40 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-layer --no-gla > /dev/null 2>&1
# launches per step (local path): seg_state(F) core(F, prefix fold fused) seg_state(R) core(bwd3, fold fused);
# -k regex:core_tc counts core launches only: instance 4 = fwd, 5 = bwd3 of the third step
for sk in 4 5; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:core_tc --launch-skip $sk --launch-count 1 \
    -o gpurun_out/${tag}_core_skip$sk -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-layer --no-gla > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_state_tc --launch-skip 4 --launch-count 1 \
  -o gpurun_out/${tag}_seg_skip4 -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-layer --no-gla > /dev/null 2>&1
ls -la gpurun_out | tail -12
# the same two core captures at the TNL-1B shape (head_dim 128)
for sk in 4 5; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:core_tc --launch-skip $sk --launch-count 1 \
    -o gpurun_out/${tag}_tnl1b_core_skip$sk -f python bench.py --config tnl1b --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-layer --no-gla > /dev/null 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"core_tc|seg_state|tag_kernel|prefix_kernel|combine|norm_apply|gla_" -c 40 --csv --log-file gpurun_out/${tag}_launches_tnl1b.csv \
  python bench.py --config tnl1b --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-layer --no-gla > /dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/${tag}_smoke.txt 2>&1
ls -la gpurun_out | tail -12
timeout 600 python bench.py --loopback 4 --steps 10 --warmup 3 --no-e2e > gpurun_out/${tag}_loop4.json 2> gpurun_out/${tag}_loop4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_reference.json 2> gpurun_out/${tag}_reference.err
