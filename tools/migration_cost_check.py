"""NVLink migration cost model vs measured migration:
run under torchrun (one rank per GPU).  cfg3-shaped run (GreedyLB re-places
most chunks every epoch, the worst case for migration volume); for every epoch
with moves, the measured migration seconds of the runtime (od_rt_run_epoch:
plan validation, NVLink pulls of U^t and A, table rebuild) against
od_plan_cost_nvlink (balancer.hpp:157-175's B200 replacement: per GPU
max(bytes out, bytes in) / link bandwidth + latency per transfer, GPUs in
parallel) at the nominal 900 GB/s per direction of NVLink 5.  Prints one JSON
line (rank 0)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
import paper_1310_4218_b200 as od  # noqa: E402
from paper_1310_4218_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
obj = [od.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
cfg = configs.CONFIGS[name](nodes=world, epochs=5)
d = cfg.domain
rows = []
with od.Engine(cfg, rank, world, local, obj[0]) as eng:
    subs = eng.subdomains()
    nbytes = []
    for s in subs:
        w, h = s.x_end - s.x_begin, s.y_end - s.y_begin
        pitch = (w + 15) // 16 * 16
        nbytes.append((d.fields + 1) * d.nz * h * pitch * 8)  # U^t and A move
    for e in range(1, cfg.epochs + 1):
        r = eng.run_epoch(e)
        if not r.plan.moves:
            continue
        ppg = cfg.proc_count() // world
        model = od.plan_cost_nvlink(r.plan, nbytes, ppg, world, 900e9, 2e-5)
        per_gpu_out = [0] * world
        per_gpu_in = [0] * world
        for m in r.plan.moves:
            a, b = m.from_ // ppg, m.to // ppg
            if a != b:
                per_gpu_out[a] += nbytes[m.vp]
                per_gpu_in[b] += nbytes[m.vp]
        worst = max(max(o, i) for o, i in zip(per_gpu_out, per_gpu_in))
        rows.append({"epoch": e, "moves": len(r.plan.moves), "cross_gpu_bytes_max": worst,
                     "measured_s": r.migration_cost, "model_s": model,
                     "measured_over_model": r.migration_cost / model if model else None,
                     "effective_GBps": worst / r.migration_cost / 1e9 if r.migration_cost else None})
if rank == 0:
    print(json.dumps({"config": name, "gpus": world, "epochs": rows,
                      "model": "od_plan_cost_nvlink, 900 GB/s per direction, 20 us per transfer"}),
          flush=True)
dist.destroy_process_group()
