# Round-2 measurement set on one B200 (run from the repo root through gpurun).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
free -g | head -2 > gpurun_out/host_mem.txt; nproc >> gpurun_out/host_mem.txt
bash tools/gpu_suite.sh smoke "bench cfg4" "bench cfg3" "bench cfg2 --steps 100" "bench cfg1 --steps 100" \
  "bench cfg5 --steps 20 --warmup 10" "ref cfg4" "ref cfg3" "ref cfg2 --steps 20" "ref cfg1 --steps 20" \
  "launches cfg4" "full cfg4 column_step_ws" "full cfg3 column_step_ws"
timeout 900 python tools/paper_presets.py > gpurun_out/paper_presets_n1.log 2>&1
timeout 900 python tools/load_spread.py cfg4 > gpurun_out/load_spread_cfg4.json 2>&1
timeout 1800 python tools/sweep_cfg5.py 1,2,4,8,16,32 10 20 > gpurun_out/cfg5_sweep_n1.jsonl 2> gpurun_out/cfg5_sweep_n1.err
echo campaign done
