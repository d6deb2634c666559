python -m pytest tests/test_gpu_fields.py -q -x > gpurun_out/pt.txt 2>&1 && python tools/diag.py cfg4 overlap=6 > gpurun_out/diag7.txt 2>&1
