mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_layer.py -x -q -s 2>&1 | tail -25 > gpurun_out/r2e_layer.txt
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2e_pytest.txt
bash tools/cmp3.sh "liblasp_old.so liblasp.so" > gpurun_out/r2e_cmp_tnl04b.txt 2>&1
bash tools/cmp3.sh "liblasp_old.so liblasp.so" --config tnl1b > gpurun_out/r2e_cmp_tnl1b.txt 2>&1
