cd /root/repo
timeout 900 python -m pytest tests/test_gpu_fields.py -q -k "variants" > gpurun_out/pt.txt 2>&1
