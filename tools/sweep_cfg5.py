"""cfg5 sweep (BASELINE config 5): 2048x2048x96 sized to HBM, over-decomposition
1-32 chunks per GPU and LB period; run per rank under torchrun for N > 1.
Prints one JSON line per point (rank 0)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

rank = int(os.environ.get("RANK", "0"))
world = int(os.environ.get("WORLD_SIZE", "1"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
import paper_1310_4218_b200 as od  # noqa: E402
from paper_1310_4218_b200 import configs  # noqa: E402

cpgs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8,16,32").split(",")]
periods = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "10").split(",")]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
for cpg in cpgs:
    for period in periods:
        sync = max(1, period // 4)
        cfg = configs.cfg5(nodes=world, chunks_per_gpu=cpg, epochs=1 << 30,
                           window=od.MeasurementWindow(period - sync, sync))
        nid = None
        if world > 1:
            obj = [od.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nid = obj[0]
        eng = od.Engine(cfg, rank, world, local, nid)
        eng.advance(3)
        eng.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.advance(steps)
        eng.synchronize()
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        t = torch.tensor([ms], device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        hist = eng.epoch_history()
        if rank == 0:
            print(json.dumps({"gpus": world, "chunks_per_gpu": cpg, "chunks": cfg.vp_count(),
                              "lb_period": period, "ms_per_step": t.item() / steps,
                              "Mcol_per_s": 2048 * 2048 * steps / (t.item() * 1e-3) / 1e6,
                              "imbalance": [round(h["imbalance_before"], 3) for h in hist]}),
                  flush=True)
        eng.close()
if world > 1:
    dist.destroy_process_group()
