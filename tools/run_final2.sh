cd /root/repo
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pt.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1
bash tools/run_final.sh
T="timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29533"
$T --nproc-per-node 4 bench.py --gpus 4 --impl reference > gpurun_out/r1_bench_ref_n4.json 2> gpurun_out/ref4.err
