# Grid (mode 4) vs warp-specialised (mode 7) step kernel by tile count on one GPU.
mkdir -p gpurun_out/wsx; rm -f gpurun_out/wsx/all.jsonl
IFS='|' read -ra SIZES <<< "${1:-256 256 8 8|512 256 16 8|512 384 16 12|512 512 16 16|512 256 8 4|768 256 12 4}"
for sz in "${SIZES[@]}"; do set -- $sz
for m in 4 7; do
timeout 300 python tools/kexp.py nx=$1 ny=$2 kx=$3 ky=$4 mode=$m steps=20 >> gpurun_out/wsx/all.jsonl 2>>gpurun_out/wsx/err.log
done; done
