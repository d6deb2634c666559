cd /root/repo
T="timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29533"
for c in 5 4 3 2; do
  echo "ctas=$c $(OD_PERSIST_CTAS=$c timeout 300 python tools/timeline.py 5 on 2>&1 | grep '"rank"')"
done > gpurun_out/ctas_sweep.txt 2>&1
for c in 5 4 3; do
  echo "ctas=$c N=4" >> gpurun_out/ctas_sweep.txt
  OD_PERSIST_CTAS=$c $T --nproc-per-node 4 tools/timeline.py 5 off 2>&1 | grep '"rank"' >> gpurun_out/ctas_sweep.txt
done
