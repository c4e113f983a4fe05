set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2a_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
timeout 600 python bench.py --loopback 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/r2a_loop4.json 2> gpurun_out/r2a_loop4.err
timeout 600 python bench.py --config tnl1b --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2a_bench_tnl1b.json 2> gpurun_out/r2a_bench_tnl1b.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.txt 2>&1
tail -3 gpurun_out/*.err
