# round-2 re-entry: state check of the restored tree (GPU tests + both bench shapes)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r4a_pytest_gpu.txt 2>&1; tail -3 gpurun_out/r4a_pytest_gpu.txt
timeout 300 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r4a_bench.json 2> gpurun_out/r4a_bench.err; tail -c 600 gpurun_out/r4a_bench.json
timeout 300 python bench.py --config tnl1b --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r4a_bench_tnl1b.json 2> gpurun_out/r4a_bench_tnl1b.err
python - <<'P'
import json
for f in ["gpurun_out/r4a_bench.json","gpurun_out/r4a_bench_tnl1b.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['value']/1e6,2), {k:round(v*1e3,1) for k,v in d['path']['stages_ms_per_step'].items()}, d['roofline']['frac'])
    except Exception as e: print(f, e)
P
