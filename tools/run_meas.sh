cd /root/repo
timeout 600 python -m pytest tests/test_gpu_fields.py -q -x > gpurun_out/pt.txt 2>&1
for i in 1 2; do echo "N=1 $(timeout 300 python tools/timeline.py 5 on 2>&1 | grep '"rank"' | cut -c1-220)"; done > gpurun_out/mbar.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --no-lb-off --no-e2e > gpurun_out/bench_n4_1.json 2> gpurun_out/bench_n4.err
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench_n4_2.json 2> gpurun_out/bench_n1.err
