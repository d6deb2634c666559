python -m pytest tests/test_gpu_fields.py -q -x > gpurun_out/pt.txt 2>&1 && python tools/diag.py cfg4 overlap=5 > gpurun_out/diag8.txt 2>&1
