# Round-2 measurement set on one B200 (run from the repo root through gpurun).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
free -g | head -2 > gpurun_out/host_mem.txt; nproc >> gpurun_out/host_mem.txt
bash tools/gpu_suite.sh "bench cfg4" "bench cfg3" "bench cfg2 --steps 100" "bench cfg1 --steps 100" \
  "bench cfg5 --steps 20 --warmup 10" "ref cfg4" "ref cfg3" "ref cfg2 --steps 20" "ref cfg1 --steps 20" \
  "launches cfg4" "full cfg3 column_step_grid"
timeout 900 python tools/paper_presets.py > gpurun_out/paper_presets_n1.log 2>&1
timeout 900 python tools/cpu_full_grid_check.py cfg4 2 > gpurun_out/cpu_full_grid_cfg4.json 2> gpurun_out/cpu_full_grid_cfg4.err
echo campaign done
