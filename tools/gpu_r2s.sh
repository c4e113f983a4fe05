mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_gla.py -q 2>&1 | tail -3 > gpurun_out/r2s_gla.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-layer > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
timeout 300 python bench.py --steps 10 --warmup 3 --config tnl1b --no-e2e --no-cpu-baseline --no-layer > gpurun_out/r2s_bench_tnl1b.json 2>> gpurun_out/r2s_bench.err
