python tools/size_probe.py 5,6 128,192,216,256,512 > gpurun_out/size_probe2.txt 2>&1
