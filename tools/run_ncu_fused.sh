export OD_FUSED_MINB=2
python tools/diag.py cfg4 overlap=3 > gpurun_out/plain_f.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:column_step2 -s 3 -c 1 -o gpurun_out/prof_fused4 python tools/diag.py cfg4 overlap=3 > gpurun_out/ncu_f.log 2>&1
