cd /root/repo
python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 256 -c 40 --csv --log-file gpurun_out/r1_launches_n1.csv python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:column_step_grid -s 3 -c 1 -o gpurun_out/r1_full_grid python tools/diag.py cfg4 > gpurun_out/ncu_f.log 2>&1
