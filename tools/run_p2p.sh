python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 tools/p2p_probe.py > gpurun_out/p2p.txt 2>&1
nvidia-smi topo -m >> gpurun_out/p2p.txt 2>&1
