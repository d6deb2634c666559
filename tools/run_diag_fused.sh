python -m pytest tests/test_gpu_fields.py -q -x > gpurun_out/pt.txt 2>&1 && python tools/diag.py cfg4 > gpurun_out/diag9.txt 2>&1 && \
ncu --set full --clock-control none -k regex:column_step_persistent -s 3 -c 1 -o gpurun_out/prof_fused7 python tools/diag.py cfg4 > gpurun_out/ncu_f.log 2>&1
