cd /root/repo
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/pt.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1
