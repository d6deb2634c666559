# round-1 measurement set: bench N=1/2/4 (+ reference arm N=1), cfg5 sweeps N=1/N=4
cd /root/repo
T="timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 python bench.py > gpurun_out/r1_bench_n1.json 2> gpurun_out/r1_bench_n1.err
timeout 900 python bench.py --impl reference > gpurun_out/r1_bench_ref_n1.json 2> gpurun_out/r1_bench_ref_n1.err
$T --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/r1_bench_n2.json 2> gpurun_out/r1_bench_n2.err
$T --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/r1_bench_n4.json 2> gpurun_out/r1_bench_n4.err
timeout 900 python tools/sweep_cfg5.py 1,2,4,8,16,32 10 20 > gpurun_out/r1_cfg5_sweep_n1.jsonl 2> gpurun_out/cfg5.err
$T --nproc-per-node 4 tools/sweep_cfg5.py 1,4,16 10 20 > gpurun_out/r1_cfg5_sweep_n4.jsonl 2> gpurun_out/cfg5_4.err
