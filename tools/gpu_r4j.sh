# parity after dropping the whole-P variant code; loopback-4 line twice (ring-exchange variance check)
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ring.py -m gpu -x -q > gpurun_out/r4j_pytest.txt 2>&1; tail -2 gpurun_out/r4j_pytest.txt
for i in 1 2; do timeout 600 python bench.py --loopback 4 --steps 10 --warmup 3 --no-e2e > gpurun_out/r4j_loop4_$i.json 2> gpurun_out/r4j_loop4_$i.err
python -c "
import json; d=json.loads(open('gpurun_out/r4j_loop4_$i.json').read().strip().splitlines()[-1])
print({k:(round(v['value']/1e6,1), round(v['ms_per_step'],3), v['exchange_us_per_step']) for k,v in d['exchanges'].items()})"; done
timeout 600 python bench.py --loopback 4 --exchange ring --steps 10 --warmup 3 --no-e2e > gpurun_out/r4j_loop4_ringonly.json 2> gpurun_out/r4j_loop4_ringonly.err; tail -c 400 gpurun_out/r4j_loop4_ringonly.json
