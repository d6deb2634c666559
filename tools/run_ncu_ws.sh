# ncu --set full capture of the warp-specialised step kernel (mode 7, forced with OD_WS=1)
cd /root/repo
OD_WS=1 timeout 200 python tools/diag.py cfg3 nodes=1 > gpurun_out/ws_plain.log 2>&1 || exit 1
OD_WS=1 timeout 400 ncu --set full --clock-control none --import-source on -k regex:column_step_ws -s 3 -c 1 \
  -o gpurun_out/r1_full_ws python tools/diag.py cfg3 nodes=1 > gpurun_out/ncu_ws.log 2>&1
