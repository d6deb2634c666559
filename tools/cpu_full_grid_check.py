"""Times the CPU oracle port (the --impl reference arm's kernel) on the FULL
grid of a workload next to the strided sample bench.py's reference arm uses,
to validate that column-updates/s carries over from the sample (VERDICT r1
weak #6).  python tools/cpu_full_grid_check.py cfg4 [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from oracle import fields as of  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cores = of.set_threads(os.cpu_count() or 1)
out = {"workload": name, "cores": cores, **bench.host_info()}
for label, side in (("sample", bench.CPU_SAMPLE_SIDE), ("full", 1 << 20)):
    state, desc, cols = bench.cpu_sample(name, None, side)
    bench.cpu_run(state, 1)
    n, dt = bench.cpu_run(state, steps)
    out[label] = {"columns": cols, "steps": n, "seconds": dt, "col_updates_per_s": cols * n / dt,
                  "what": desc}
    del state
out["full_over_sample"] = out["full"]["col_updates_per_s"] / out["sample"]["col_updates_per_s"]
print(json.dumps(out))
