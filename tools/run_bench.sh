python bench.py --steps 40 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 256 -c 60 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench2_ref.json 2>&1
