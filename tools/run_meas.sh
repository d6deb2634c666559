cd /root/repo
timeout 600 python -m pytest tests/test_gpu_fields.py -q -x > gpurun_out/pt.txt 2>&1
ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum --clock-control none -k regex:column_step_grid -s 3 -c 2 --csv python tools/diag.py cfg4 2>/dev/null | grep '"ID"\|column_step_grid' > gpurun_out/shfl.csv
