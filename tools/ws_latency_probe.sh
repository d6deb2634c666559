# Latency regime: warp-specialised step time against the heavy column's serial
# chain (127 trips x 1537 units x 2 dependent DFMAs), alone on an SM or sharing it.
mkdir -p gpurun_out/wsl; rm -f gpurun_out/wsl/all.jsonl
run() { timeout 300 python tools/kexp.py "$@" steps=20 >> gpurun_out/wsl/all.jsonl 2>>gpurun_out/wsl/err.log; }
for m in 7 4; do
run nx=256 ny=128 kx=8 ky=4 F=1 mode=$m light=2      # 128 all-heavy tiles: one per SM
run nx=256 ny=256 kx=8 ky=8 F=1 mode=$m light=2      # 256 all-heavy tiles
run nx=256 ny=256 kx=8 ky=8 F=1 mode=$m               # 256 tiles, upper half heavy
run nx=256 ny=128 kx=8 ky=4 F=1 mode=$m light=2 n_inner=3072
done
