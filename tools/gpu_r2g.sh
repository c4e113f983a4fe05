mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python scratch/diag_layer.py > gpurun_out/r2g_diag.txt 2>&1
