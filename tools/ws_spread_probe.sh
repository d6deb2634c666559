# One tile per SM for grids that fit the GPU (column_step_ws with unused dynamic shared
# memory): A/B against OD_WS_SPREAD=0 on latency-regime shapes and the cfg1/cfg2 benches.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
rm -f gpurun_out/spread.jsonl
run() { sp=$1; shift; OD_WS_SPREAD=$sp timeout 300 python tools/kexp.py steps=20 mode=5 "$@" 2>>gpurun_out/spread.err | tail -1 | sed "s/^{/{\"spread\": $sp, /" >> gpurun_out/spread.jsonl; }
for sp in 0 1; do
run $sp nx=256 ny=128 kx=8 ky=4 F=50 light=2
run $sp nx=256 ny=128 kx=8 ky=4 F=50
run $sp nx=256 ny=256 kx=8 ky=8 F=50
run $sp nx=1024 ny=1024 kx=16 ky=16 F=50
done
for sp in 0 1; do
  for c in cfg2 cfg1; do
    OD_WS_SPREAD=$sp timeout 600 python bench.py --config $c --steps 100 --no-cpu --no-e2e > gpurun_out/spread_bench_${c}_$sp.json 2>>gpurun_out/spread.err
  done
done
