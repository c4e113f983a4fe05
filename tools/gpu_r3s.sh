mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --transport p2p --steps 5 --warmup 2 --no-e2e > gpurun_out/r3s_torchrun2.json 2> gpurun_out/r3s_torchrun2.err; echo "rc=$?" >> gpurun_out/r3s_torchrun2.err
