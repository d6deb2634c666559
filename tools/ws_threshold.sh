mkdir -p gpurun_out/wsx; rm -f gpurun_out/wsx/all.jsonl
for sz in "256 256 8 8" "512 256 16 8" "512 384 16 12" "512 512 16 16"; do set -- $sz
for m in 4 7; do
timeout 300 python tools/kexp.py nx=$1 ny=$2 kx=$3 ky=$4 mode=$m steps=20 >> gpurun_out/wsx/all.jsonl 2>>gpurun_out/wsx/err.log
done; done
