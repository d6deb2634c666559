# Latency regime, physics vs Jacobi vs co-residency: 128 all-heavy tiles (one per SM if
# the block scheduler spreads them), with and without the Jacobi (F=50 / F=1), and
# 128 heavy + 128 light tiles physics-only.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
rm -f gpurun_out/lat2.jsonl
run() { timeout 300 python tools/kexp.py steps=20 mode=5 "$@" 2>>gpurun_out/lat2.err | tail -1 >> gpurun_out/lat2.jsonl; }
run nx=256 ny=128 kx=8 ky=4 F=1 light=2
run nx=256 ny=128 kx=8 ky=4 F=50 light=2
run nx=256 ny=256 kx=8 ky=8 F=1
run nx=256 ny=256 kx=8 ky=8 F=1 light=2
run nx=256 ny=64 kx=8 ky=2 F=50 light=2
