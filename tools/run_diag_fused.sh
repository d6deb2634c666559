python -m pytest tests -m gpu -x -q > gpurun_out/pt.txt 2>&1
for v in 2 3; do echo "cs3 minb=$v" >> gpurun_out/diag5.txt; OD_FUSED_MINB=$v python tools/diag.py cfg4 overlap=4 >> gpurun_out/diag5.txt 2>&1; done
