cd "${GRAFT_REPO_ROOT:-/root/repo}"
run() { timeout 300 python tools/kexp.py nx=256 ny=256 kx=8 ky=8 steps=20 "$@" 2>>gpurun_out/lat.err | tail -1 >> gpurun_out/lat.jsonl; }
rm -f gpurun_out/lat.jsonl
for m in 5 4; do
run mode=$m F=50 light=1 heavy=1
run mode=$m F=1 light=1 heavy=1
run mode=$m F=50 n_inner=1 light=1 heavy=1
run mode=$m F=50 light=2 heavy=2
run mode=$m F=50
run mode=$m F=50 n_inner=1 nz=32
done
