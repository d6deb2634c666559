"""Device timeline of the cfg4 step under torchrun (diagnostic).

Runs `epochs` epochs of cfg4 with OD_TIMELINE set, then reads the per-step
globaltimer stamps every rank wrote (step begin, after halo pack, kernel
begin, kernel end) and prints, per rank, the average pack, kernel and
inter-step gap, plus the cross-rank skew of the kernel start.
  torchrun --nproc-per-node 4 tools/timeline.py [mode] [ny_override]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

rank = int(os.environ.get("RANK", 0))
world = int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
prefix = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", f"tl_w{world}")
os.environ["OD_TIMELINE"] = prefix
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))

import paper_1310_4218_b200 as od  # noqa: E402
from paper_1310_4218_b200 import configs  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 5
lb = (sys.argv[2] if len(sys.argv) > 2 else "on") == "on"
obj = [od.nccl_unique_id() if rank == 0 else None]
if world > 1:
    dist.broadcast_object_list(obj, src=0)
cfg = configs.cfg4(world, overlap=mode)
if len(sys.argv) > 3:
    cfg = cfg.replace(measure=od.MeasureMode(int(sys.argv[3])))
if not lb:
    import dataclasses
    cfg = cfg.replace(policy=dataclasses.replace(cfg.policy, trigger_threshold=1e9))
eng = od.Engine(cfg, rank, world, local, obj[0])
recs = [eng.run_epoch(e) for e in range(1, 5)]
eng.close()
if rank == 0:
    # measured chunk loads by class: heavy/light x (has a remote face or not), per GPU
    kx, ky = cfg.decomposition.kx, cfg.decomposition.ky
    for r in recs:
        m = np.array(r.mapping.assignment())
        L = np.array(r.vp_loads) * 1e3
        out = {}
        for v in range(len(L)):
            iy, ix = divmod(v, kx)
            heavy = iy < ky // 2
            nb = [(ix - 1, iy), (ix + 1, iy), (ix, iy - 1), (ix, iy + 1)]
            remote = sum(1 for (a, b) in nb if 0 <= a < kx and 0 <= b < ky and m[b * kx + a] != m[v])
            out.setdefault((int(m[v]), "H" if heavy else "L", remote), []).append(L[v])
        import hashlib
        print("epoch", r.epoch, "imb", round(r.imbalance_before, 4), "->", round(r.imbalance_after, 4),
              "moves", len(r.plan.moves), "map", hashlib.md5(bytes(m.astype(np.int8))).hexdigest()[:8],
              "plan", [tuple(x) for x in r.plan.moves][:30])
        if world == 1 and r.epoch == 2:
            Lh = L[: len(L) // 2].reshape(ky // 2, kx)
            print("heavy chunk loads (ms), rows of the chunk grid:")
            for row in Lh:
                print("   " + " ".join("%.3f" % x for x in row))
            print("light rows:")
            for row in L[len(L) // 2:].reshape(ky // 2, kx)[:3]:
                print("   " + " ".join("%.3f" % x for x in row))
        for k in sorted(out):
            a = np.array(out[k])
            print("   gpu%d %s remote=%d n=%3d mean %.4f ms sd %.4f" % (k[0], k[1], k[2], len(a), a.mean(), a.std()))
if world > 1:
    dist.barrier()
if rank == 0:
    rows = []
    for r in range(world):
        t = np.loadtxt(f"{prefix}.rank{r}.txt", dtype=np.float64).reshape(-1, 6)[:, 1:]
        rows.append(t)
    n = min(len(t) for t in rows)
    start = np.stack([t[:n, 2] for t in rows])  # kernel begin per rank
    end = np.stack([t[:n, 3] for t in rows])
    for r, t in enumerate(rows):
        t = t[:n]
        pack = (t[:, 1] - t[:, 0]) / 1e6
        pre = (t[:, 2] - t[:, 1]) / 1e6
        kern = (t[:, 3] - t[:, 2]) / 1e6
        gap = (t[1:, 0] - t[:-1, 3]) / 1e6
        step = (t[1:, 0] - t[:-1, 0]) / 1e6
        print(json.dumps({"rank": r, "steps": int(n), "pack_ms": round(float(np.median(pack)), 4),
                          "pre_ms": round(float(np.median(pre)), 4),
                          "kernel_ms": round(float(np.median(kern)), 4),
                          "kernel_ms_mean": round(float(kern[5:].mean()), 4),
                          "wait_ms_median": round(float(np.median(t[:, 4])) / 1e6, 4),
                          "wait_ms_max": round(float(t[:, 4].max()) / 1e6, 4),
                          "gap_ms_median": round(float(np.median(gap)), 4),
                          "gap_ms_max": round(float(gap.max()), 3),
                          "step_ms_median": round(float(np.median(step)), 4),
                          "total_ms": round(float((t[-1, 3] - t[0, 0]) / 1e6), 3)}))
    # per-epoch median kernel ms per rank
    for e in range(n // 10):
        print("epoch-kernels", e + 1, " ".join("%.3f" % np.median((rows[r][10 * e:10 * e + 10, 3] - rows[r][10 * e:10 * e + 10, 2]) / 1e6) for r in range(world)))
    # per-step detail for the last epoch
    for s in range(n - 10, n):
        print("step", s, " ".join(f"{(rows[r][s, 3] - rows[r][s, 2]) / 1e6:.3f}/w{rows[r][s, 4] / 1e6:.3f}"
                                  for r in range(world)))
if world > 1:
    dist.destroy_process_group()
