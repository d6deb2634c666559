N=$1
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N > gpurun_out/r1_bench_n$N.json 2> gpurun_out/r1_bench_n$N.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --impl reference > gpurun_out/r1_bench_ref_n$N.json 2> gpurun_out/r1_bench_ref_n$N.err
