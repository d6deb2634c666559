# N=4 timeline runs, one summary line per run (diagnostic)
cd /root/repo
out=gpurun_out/meas_matrix.txt; : > $out
run() {  # label nproc env...
  label=$1; np=$2; shift 2
  r=$(env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29533 --nproc-per-node $np tools/timeline.py 5 on ${MEAS:-1} 2>&1 | grep -E "^epoch|\"rank\": 0")
  echo "$label | $(echo "$r" | grep ^epoch | awk '{printf "%s->%s/%s ", $4, $6, $8}') | $(echo "$r" | grep rank | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["step_ms_median"], d["wait_ms_median"], d["total_ms"])')" >> $out
}
for rep in 1 2 3; do
  run "N4 firstwave" 4 OD_FIRSTWAVE=1
  run "N4 pureLPT" 4 OD_FIRSTWAVE=0
done
