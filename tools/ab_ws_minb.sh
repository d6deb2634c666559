# warp-specialised kernel occupancy A/B (OD_WS_MINB = 2, 3 (default), 4) by tile count
mkdir -p gpurun_out/abwm; rm -f gpurun_out/abwm/all.jsonl
for rep in 1 2; do
for sz in "1024 1024 16 16" "512 512 16 16" "512 256 8 4"; do set -- $sz
for w in 3 2 4; do
OD_WS_MINB=$w timeout 300 python tools/kexp.py nx=$1 ny=$2 kx=$3 ky=$4 mode=7 steps=20 | sed "s/^{/{\"ws_minb\": $w, /" >> gpurun_out/abwm/all.jsonl 2>>gpurun_out/abwm/err.log
done
timeout 300 python tools/kexp.py nx=$1 ny=$2 kx=$3 ky=$4 mode=4 steps=20 | sed "s/^{/{\"ws_minb\": 0, /" >> gpurun_out/abwm/all.jsonl 2>>gpurun_out/abwm/err.log
done; done
