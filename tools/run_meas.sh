cd /root/repo
T="timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29533"
for i in 1 2; do
$T --nproc-per-node 4 bench.py --gpus 4 --no-lb-off --no-e2e --refine-adjacent > gpurun_out/adj_$i.json 2> gpurun_out/adj.err
$T --nproc-per-node 4 bench.py --gpus 4 --no-lb-off --no-e2e > gpurun_out/ref_$i.json 2> gpurun_out/ref.err
done
