cd /root/repo
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pt.txt 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/bench_n4_4.json 2> gpurun_out/bench_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --no-lb-off > gpurun_out/bench_n4_1.json 2> gpurun_out/bench_n4.err
