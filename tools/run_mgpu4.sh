for m in 6 5; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 --steps 30 --warmup 5 --no-e2e --kernel-mode $m > gpurun_out/bench_n4_m$m.json 2> gpurun_out/bench_n4_m$m.err
done
