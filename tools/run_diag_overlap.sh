rm -f gpurun_out/diag2.txt
for c in 2 3 4; do for cv in 100 50; do echo "ctas=$c carve=$cv" >> gpurun_out/diag2.txt; OD_SMEM_CARVEOUT=$cv OD_PHYS_CTAS_PER_SM=$c python tools/diag.py cfg4 overlap=1 >> gpurun_out/diag2.txt 2>&1; done; done
