cd /root/repo
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pt.txt 2>&1
T="timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29533"
$T --nproc-per-node 4 bench.py --gpus 4 --no-lb-off --no-e2e > gpurun_out/bench_n4_1.json 2> gpurun_out/bench_n4.err
$T --nproc-per-node 4 bench.py --gpus 4 --no-lb-off --no-e2e > gpurun_out/bench_n4_2.json 2> gpurun_out/bench_n4.err
$T --nproc-per-node 2 bench.py --gpus 2 --no-lb-off --no-e2e > gpurun_out/bench_n4_3.json 2> gpurun_out/bench_n2.err
$T --nproc-per-node 2 bench.py --gpus 2 --no-lb-off --no-e2e > gpurun_out/bench_n4_4.json 2> gpurun_out/bench_n2.err
