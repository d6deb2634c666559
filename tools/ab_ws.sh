# A/B of the warp-specialised kernel's unrolled Jacobi loop (OD_WS_UNROLL=1/0)
mkdir -p gpurun_out/abws; rm -f gpurun_out/abws/all.jsonl
OD_WS_UNROLL=1 timeout 600 python -m pytest -q -x tests/test_gpu_geometry.py tests/test_gpu_fields.py -k "ws or mode or geometry or variants" > gpurun_out/abws/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/abws/tests.log
for rep in 1 2; do for u in 1 0; do
for sz in "512 256 8 4" "512 256 16 8" "256 256 8 8"; do set -- $sz
OD_WS_UNROLL=$u timeout 300 python tools/kexp.py nx=$1 ny=$2 kx=$3 ky=$4 mode=7 steps=20 | sed "s/^{/{\"ws_unroll\": $u, /" >> gpurun_out/abws/all.jsonl 2>>gpurun_out/abws/err.log
done; done; done
