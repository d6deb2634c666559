python tools/diag.py cfg4 overlap=2 > gpurun_out/plain_f.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:column_step -s 3 -c 1 -o gpurun_out/prof_fused python tools/diag.py cfg4 overlap=2 > gpurun_out/ncu_f.log 2>&1
python tools/diag.py cfg4 overlap=0 > gpurun_out/plain_s.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"jacobi_step|physics_step" -s 6 -c 2 -o gpurun_out/prof_seq python tools/diag.py cfg4 overlap=0 > gpurun_out/ncu_s.log 2>&1
