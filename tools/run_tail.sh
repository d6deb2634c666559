cd /root/repo
for o in lpt spt lightwave shuffle lpt; do
  echo "order=$o $(OD_ORDER=$o timeout 300 python tools/timeline.py 5 on 2>&1 | grep '"rank"')"
done > gpurun_out/order_sweep.txt 2>&1
