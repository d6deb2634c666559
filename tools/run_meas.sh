cd /root/repo
OD_TRACE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --no-lb-off --no-e2e > gpurun_out/trace4.json 2> gpurun_out/trace4.err
