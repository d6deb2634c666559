cd /root/repo
OD_TILELOG=gpurun_out/slog1 OD_TILELOG_STEP=19 timeout 300 python tools/timeline.py 5 on > gpurun_out/tl1.txt 2>&1
python tools/share_log.py gpurun_out/slog1.rank0.txt > gpurun_out/slog1_summary.txt 2>&1
