cd /root/repo
T="timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29533"
for o in 0 1; do
  OD_OVERLAP=$o timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/ovl_n1_$o.json 2> gpurun_out/ovl.err
  OD_OVERLAP=$o $T --nproc-per-node 4 bench.py --gpus 4 --no-lb-off --no-e2e > gpurun_out/ovl_n4_$o.json 2> gpurun_out/ovl4.err
  OD_OVERLAP=$o $T --nproc-per-node 2 bench.py --gpus 2 --no-lb-off --no-e2e > gpurun_out/ovl_n2_$o.json 2> gpurun_out/ovl2.err
done
