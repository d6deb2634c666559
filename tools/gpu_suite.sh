#!/usr/bin/env bash
# One entry point for every GPU-box job of this repo (run through gpurun from
# the repo root; outputs land in gpurun_out/).  Stages run in the order given:
#
#   tests                  pytest -m gpu (all GPU parity tests)
#   smoke                  __graft_entry__.smoke()
#   bench CFG [ARGS..]     bench.py --config CFG ARGS  -> gpurun_out/bench_CFG[_TAG].json
#   mbench N CFG [ARGS..]  torchrun --nproc-per-node N bench.py --gpus N --config CFG ARGS
#   ref CFG [ARGS..]       bench.py --impl reference --config CFG ARGS
#   launches CFG           ncu launch list (gpu__time_duration) of a short bench run
#   full CFG REGEX         ncu --set full capture of one launch of kernel REGEX (diag run)
#   sanitize TOOL          compute-sanitizer --tool TOOL on smoke + one fused-step diag run
#
# TAG: environment variable appended to output names (default empty).
# Example:
#   gpurun --timeout 1800 -- 'bash tools/gpu_suite.sh tests "bench cfg4" "launches cfg4"'
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:+_$TAG}
rc=0
for stage in "$@"; do
  set -- $stage
  case "$1" in
    tests)
      timeout 3000 python -m pytest tests -m gpu -q -x -p no:cacheprovider \
        > gpurun_out/gputests$T.log 2>&1; r=$?; tail -3 gpurun_out/gputests$T.log ;;
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke$T.log 2>&1
      r=$?; tail -2 gpurun_out/smoke$T.log ;;
    bench)
      cfg=$2; shift 2
      timeout 1500 python bench.py --config "$cfg" "$@" > gpurun_out/bench_$cfg$T.json \
        2> gpurun_out/bench_$cfg$T.err; r=$?; tail -c 600 gpurun_out/bench_$cfg$T.json ;;
    mbench)
      n=$2; cfg=$3; shift 3
      timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus "$n" \
        --config "$cfg" "$@" > gpurun_out/bench_${cfg}_n$n$T.json 2> gpurun_out/bench_${cfg}_n$n$T.err
      r=$?; tail -c 600 gpurun_out/bench_${cfg}_n$n$T.json ;;
    ref)
      cfg=$2; shift 2
      timeout 1500 python bench.py --impl reference --config "$cfg" "$@" \
        > gpurun_out/ref_$cfg$T.json 2> gpurun_out/ref_$cfg$T.err; r=$?
      tail -c 400 gpurun_out/ref_$cfg$T.json ;;
    launches)
      cfg=$2
      timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/launches_$cfg$T.csv python bench.py --config "$cfg" --steps 10 \
        --warmup 10 --no-e2e --no-cpu --no-lb-off > gpurun_out/ncu_launches_$cfg$T.log 2>&1
      r=$? ;;
    full)
      cfg=$2; rx=$3
      timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s 12 \
        -c 1 -o gpurun_out/full_$cfg$T python tools/diag.py "$cfg" nodes=1 \
        > gpurun_out/ncu_full_$cfg$T.log 2>&1; r=$? ;;
    sanitize)
      tool=$2
      timeout 1500 compute-sanitizer --tool "$tool" --error-exitcode 9 \
        python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_${tool}_smoke$T.log 2>&1
      r=$?
      for shape in "sanA overlap=4" "sanA overlap=7" "sanB overlap=4" "sanB overlap=7"; do
        tagn=$(echo $shape | tr ' =' '__')
        timeout 1500 compute-sanitizer --tool "$tool" --error-exitcode 9 \
          python tools/diag.py $shape > gpurun_out/san_${tool}_${tagn}$T.log 2>&1
        r2=$?; [ $r -eq 0 ] && r=$r2
        tail -2 gpurun_out/san_${tool}_${tagn}$T.log
      done
      tail -3 gpurun_out/san_${tool}_smoke$T.log ;;
    *) echo "unknown stage $1"; r=2 ;;
  esac
  echo "[gpu_suite] $stage -> rc $r"
  [ $r -ne 0 ] && rc=$r
done
exit $rc
