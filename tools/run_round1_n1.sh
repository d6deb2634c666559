python bench.py > gpurun_out/r1_bench_n1.json 2> gpurun_out/r1_bench_n1.err
python bench.py --impl reference > gpurun_out/r1_bench_ref.json 2> gpurun_out/r1_bench_ref.err
python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 256 -c 40 --csv --log-file gpurun_out/r1_launches_n1.csv python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1
