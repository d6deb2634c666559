"""The paper's experiments on B200 with measured loads, side by side with the
reference simulator's modelled timelines (profiles/r2_paper_presets.json).

  python tools/paper_presets.py [expA expB expC cfg1 ...]

Per preset: our reference-format CSV (report.hpp:69-114; step_time_sum and
migration_cost are measured B200 seconds), the simulator's CSV (oracle/_ref,
K20-calibrated model), the measured per-VP loads of every epoch and the plans.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1310_4218_b200 as od  # noqa: E402
from oracle import ref as oref  # noqa: E402
from paper_1310_4218_b200 import configs  # noqa: E402

rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
local = int(os.environ.get("LOCAL_RANK", "0"))
if world > 1:  # torchrun: one rank per GPU, the presets' processors dealt to the GPUs
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
names = sys.argv[1:] or ["expA", "expB", "expC", "cfg1"]
out = {}
for name in names:
    cfg = configs.CONFIGS[name]()
    if cfg.proc_count() < world:
        continue
    nid = None
    if world > 1:
        obj = [od.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    t0 = time.perf_counter()
    with od.Engine(cfg, rank, world, local, nid) as eng:
        tl = eng.run()
    wall = time.perf_counter() - t0
    if rank != 0:
        continue
    row = {"config": od.config_to_json(cfg), "gpus": world, "host_wall_s": wall,
           "csv": od.render_report(tl, "csv"),
           "epochs": [{"epoch": e.epoch, "vp_loads": e.vp_loads, "proc_loads": e.proc_loads,
                       "moves": [tuple(m) for m in e.plan.moves],
                       "imbalance_before": e.imbalance_before,
                       "imbalance_after": e.imbalance_after,
                       "step_ms": [round(x * 1e3, 4) for x in e.step_times]}
                      for e in tl.epochs]}
    if name in ("expA", "expB", "expC"):
        row["reference_csv"] = oref.run_json({"preset": name})["csv"]
        row["reference_note"] = "the reference's own preset (K20-calibrated cost model)"
    else:
        # the same config through the reference simulator (default model, where
        # physics_cost_scale = 1: the Jacobi dominates and the hotspot hardly shows)
        j = {k: v for k, v in od.config_to_json(cfg).items() if k != "b200"}
        row["reference_csv"] = oref.run_json(j)["csv"]
        row["reference_note"] = "config through run_experiment with the default cost model"
    out[name] = row
    print(f"== {name} (B200 x{world}, measured)\n{row['csv']}== {name} (reference simulator)\n"
          f"{row['reference_csv']}", flush=True)
if rank == 0:
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"paper_presets_n{world}.json"), "w") as f:
        json.dump(out, f, indent=1)
if world > 1:
    dist.destroy_process_group()
