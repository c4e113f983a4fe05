mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5 > gpurun_out/r2k_parity.txt
for c in tnl04b tnl1b; do timeout 300 python bench.py --steps 20 --warmup 5 --config $c --no-e2e --no-cpu-baseline --no-layer > gpurun_out/r2k_bench_$c.json 2>> gpurun_out/r2k_bench.err; done
