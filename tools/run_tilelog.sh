cd /root/repo
OD_TILELOG=gpurun_out/slog1 OD_TILELOG_STEP=19 timeout 300 python tools/timeline.py 5 on > gpurun_out/tl1.txt 2>&1
python tools/share_log.py gpurun_out/slog1.rank0.txt > gpurun_out/slog1_summary.txt 2>&1
OD_TILELOG=gpurun_out/slog4 OD_TILELOG_STEP=29 timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29533 --nproc-per-node 4 tools/timeline.py 5 on > gpurun_out/tl4.txt 2>&1
for r in 0 1 2 3; do python tools/share_log.py gpurun_out/slog4.rank$r.txt > gpurun_out/slog4_r$r.sum 2>&1; done
