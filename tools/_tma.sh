cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_fields.py tests/test_gpu_geometry.py -q -x > gpurun_out/tma_tests.log 2>&1; tail -3 gpurun_out/tma_tests.log
for rep in 1 2; do for t in 1 0; do for args in "" "nx=512 ny=512"; do
  OD_TMA=$t timeout 300 python tools/kexp.py mode=4 $args 2>/dev/null | tail -1 | sed "s/^{/{\"tma\": $t, /"
done; done; done > gpurun_out/kexp_tma.jsonl
cat gpurun_out/kexp_tma.jsonl | cut -c1-200
