python tools/diag.py cfg4 > gpurun_out/plain_f.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:column_step_persistent -s 3 -c 1 -o gpurun_out/prof_fused6 python tools/diag.py cfg4 > gpurun_out/ncu_f.log 2>&1
