cd /root/repo
timeout 600 python -m pytest tests/test_gpu_fields.py -q -x -k "few_levels" > gpurun_out/pt.txt 2>&1
