mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "128 or config3 or config4 or tnl or random" 2>&1 | tail -15 > gpurun_out/r3f_parity.txt
timeout 300 python bench.py --steps 10 --warmup 3 --config tnl1b --no-e2e --no-cpu-baseline --no-layer --no-gla > gpurun_out/r3f_bench_tnl1b.json 2> gpurun_out/r3f_bench.err
LASP_WIDE128=0 timeout 300 python bench.py --steps 10 --warmup 3 --config tnl1b --no-e2e --no-cpu-baseline --no-layer --no-gla > gpurun_out/r3f_bench_tnl1b_old.json 2>> gpurun_out/r3f_bench.err
