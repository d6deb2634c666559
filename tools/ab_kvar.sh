# A/B of kernel variants selected by OD_KVAR on one box: parity slices, then
# alternating bench runs.  usage: bash tools/ab_kvar.sh "0 1 2" "cfg4 cfg3" reps
V=${1:-"0 1"}; C=${2:-"cfg4 cfg3"}; REPS=${3:-2}
mkdir -p gpurun_out/ab; rm -f gpurun_out/ab/summary
for v in $V; do
OD_KVAR=$v timeout 600 python -m pytest -q -x tests/test_gpu_geometry.py > gpurun_out/ab/geom_v$v.log 2>&1; echo geom v$v $? >> gpurun_out/ab/summary
done
for rep in $(seq $REPS); do for v in $V; do for c in $C; do
f=gpurun_out/ab/b_${c}_v${v}_r${rep}
OD_KVAR=$v timeout 300 python bench.py --config $c --steps 40 --warmup 10 --no-e2e --no-cpu --no-lb-off > $f.json 2>$f.err
echo $c v$v r$rep $(python -c "import json;d=json.loads([l for l in open('$f.json') if l.startswith('{')][-1]);print(round(d['value']/1e6,2),round(d['ms_per_step'],3),d['clocks']['sm_mhz'],round(d['roofline']['frac'],4))") >> gpurun_out/ab/summary
done; done; done
