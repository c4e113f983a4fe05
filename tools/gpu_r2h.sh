mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_layer.py -q -s 2>&1 | tail -25 > gpurun_out/r2h_layer.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err
timeout 300 python bench.py --steps 20 --warmup 5 --config tnl1b --no-e2e --no-cpu-baseline > gpurun_out/r2h_bench_tnl1b.json 2>> gpurun_out/r2h_bench.err
