# Round-2 multi-GPU measurement set: N GPUs of one box (gpurun --gpus N).
#   bash tools/campaign_mgpu.sh N [sweep]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=$1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
bash tools/gpu_suite.sh "mbench $N cfg4" "mbench $N cfg3"
timeout 900 $TR --master-port 29611 tools/migration_cost_check.py cfg3 \
  > gpurun_out/migcost_n$N.json 2> gpurun_out/migcost_n$N.err; echo "migcost rc=$?"
timeout 900 $TR --master-port 29612 tools/paper_presets.py expA expB expC cfg1 \
  > gpurun_out/paper_presets_n$N.log 2>&1; echo "presets rc=$?"
if [ "${2:-}" = sweep ]; then
  timeout 3000 $TR --master-port 29613 tools/sweep_cfg5.py 1,4,16,32 5,10,20,40 80 \
    > gpurun_out/cfg5_sweep_n$N.jsonl 2> gpurun_out/cfg5_sweep_n$N.err; echo "sweep rc=$?"
fi
echo campaign done
