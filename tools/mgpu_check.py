"""Multi-rank correctness check (run under torchrun, one rank per GPU):
decomposed chunks over ranks, cross-rank halo exchange, greedy balancing every
epoch with real chunk migration; each rank compares the chunks it owns at the
end bitwise with the CPU field oracle.  Prints one JSON line per rank.
  torchrun --nproc-per-node N tools/mgpu_check.py MODE [small|cfg3]
cfg3: the full 512x512x64, F=50 bench grid (256 chunks, moving hotspot, GreedyLB
on N processors), two epochs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))

import paper_1310_4218_b200 as od  # noqa: E402
from tests.gpu_util import oracle_fields  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 4
obj = [od.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
shape = sys.argv[2] if len(sys.argv) > 2 else "small"
if shape == "cfg3":
    from paper_1310_4218_b200 import configs  # noqa: E402
    cfg = configs.cfg3(nodes=world, epochs=1000, overlap=mode)
    n_epochs = 2
else:
    cfg = od.ExperimentConfig(
        cluster=od.ClusterSpec(world, 2), domain=od.Domain(97, 61, 7, 3),
        decomposition=od.Decomposition(od.DecompositionKind.TwoD, 5, 4),
        window=od.MeasurementWindow(1, 1), epochs=1000, pattern=od.LoadPattern.UpperHalfHeavy,
        advection=od.AdvectionSchedule(17, 2, 2),
        policy=od.BalancePolicy(od.Strategy.Greedy, od.Strategy.RefineSwap, 1.0, 0.02),
        seed=99, n_inner=9, overlap=mode)
    n_epochs = 4
eng = od.Engine(cfg, rank, world, local, obj[0])
recs = [eng.run_epoch(e) for e in range(1, n_epochs + 1)]
U, A, own = eng.gather_fields()
st = eng.stats()
Uo, Ao = oracle_fields(cfg, n_epochs * cfg.window.epoch_steps())
ok_u = bool(np.array_equal(U[:, :, own], Uo[:, :, own]))
ok_a = bool(np.array_equal(A[:, own], Ao[:, own]))
maps = [r.mapping.assignment().tolist() for r in recs]
# every rank must hold identical mappings and plans
allm = [None] * world
dist.all_gather_object(allm, (maps, [[tuple(m) for m in r.plan.moves] for r in recs]))
same = all(x == allm[0] for x in allm)
owned = int(own.sum())
tot = [0] * world
dist.all_gather_object(tot, owned)
row = ({"rank": rank, "mode": mode, "fields_ok": ok_u and ok_a, "U_ok": ok_u,
                  "A_ok": ok_a, "consistent_plans": same, "owned_columns": owned,
                  "all_columns_covered": sum(tot) == cfg.domain.nx * cfg.domain.ny,
                  "moves": [len(r.plan.moves) for r in recs],
                  "halo_bytes": st["halo_bytes_sent"], "migrated_bytes": st["migrated_bytes"],
                  "imbalance": [[round(r.imbalance_before, 3), round(r.imbalance_after, 3)]
                                for r in recs]})
rows = [None] * world
dist.all_gather_object(rows, row)
if rank == 0:
    for r in rows:
        print(json.dumps(r), flush=True)
eng.close()
dist.destroy_process_group()
