cd /root/repo
T="timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29533"
timeout 300 python tools/timeline.py 5 on > gpurun_out/tl1.txt 2>&1
$T --nproc-per-node 4 tools/timeline.py 5 on > gpurun_out/tl4_on.txt 2>&1
$T --nproc-per-node 4 tools/timeline.py 5 on > gpurun_out/tl4_on2.txt 2>&1
$T --nproc-per-node 2 tools/timeline.py 5 on > gpurun_out/tl2_on.txt 2>&1
$T --nproc-per-node 2 tools/timeline.py 5 on > gpurun_out/tl2_on2.txt 2>&1
