set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2b_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
timeout 600 python bench.py --config tnl1b --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2b_bench_tnl1b.json 2> gpurun_out/r2b_bench_tnl1b.err
timeout 600 python tools/overlap_exp.py --config tnl04b > gpurun_out/r2b_overlap_tnl04b.md 2>&1
timeout 600 python tools/overlap_exp.py --config tnl1b --hold-us 900 > gpurun_out/r2b_overlap_tnl1b.md 2>&1
timeout 600 python bench.py --loopback 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/r2b_loop4.json 2> gpurun_out/r2b_loop4.err
