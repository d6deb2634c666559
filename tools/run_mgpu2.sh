timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/pt_mr.txt 2>&1
OD_HALO=p2p timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e > gpurun_out/bench_n2_p2p.json 2> gpurun_out/bench_n2_p2p.err
