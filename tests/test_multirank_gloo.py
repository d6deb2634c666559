"""N>1 host logic on CPU (gloo, world_size 2): the product's cross-rank halo
schedule (od_exchange_schedule) drives a real point-to-point exchange of
packed face strips between two processes; each rank then rebuilds its chunks'
halo rings from local neighbours / received strips / zero-flux edges and runs
the Jacobi on them.  The result must equal the undecomposed CPU oracle bit for
bit, for scattered mappings like the ones GreedyLB produces."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

NX, NY, NZ, F = 37, 29, 4, 3
KX, KY = 4, 3


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def edge(block, side):
    """[f][k][e] strip of a chunk block (F, nz, h, w) on `side`."""
    if side == 0:
        return block[:, :, :, 0]
    if side == 1:
        return block[:, :, :, -1]
    if side == 2:
        return block[:, :, 0, :]
    return block[:, :, -1, :]


def worker(rank, world, port, rank_of_vp, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1310_4218_b200 as od
    from oracle import fields as of
    try:
        U, _ = of.init_state(NX, NY, NZ, F, seed)
        subs = od.decompose_2d(od.Domain(NX, NY, NZ, F), KX, KY)
        per_cell = NZ * F
        sends, recvs = od.exchange_schedule(subs, od.DecompositionKind.TwoD, KX, KY, rank_of_vp,
                                            world, rank, per_cell)
        block = {v: U[:, :, s.y_begin:s.y_end, s.x_begin:s.x_end].copy()
                 for v, s in enumerate(subs) if rank_of_vp[v] == rank}
        # pack (pack_faces semantics) and exchange per peer
        send_total = max([f.offset + per_cell * f.lenp for f in sends], default=0)
        recv_total = max([f.offset + per_cell * f.lenp for f in recvs], default=0)
        sbuf = np.zeros(send_total)
        for f in sends:
            strip = np.zeros((F, NZ, f.lenp))
            strip[:, :, :f.len] = edge(block[f.vp], f.side)
            sbuf[f.offset:f.offset + per_cell * f.lenp] = strip.reshape(-1)
        rbuf = torch.zeros(recv_total, dtype=torch.float64)
        reqs = []
        for q in range(world):
            if q == rank:
                continue
            ss = [f for f in sends if f.peer == q]
            rs = [f for f in recvs if f.peer == q]
            if ss:
                a, b = ss[0].offset, ss[-1].offset + per_cell * ss[-1].lenp
                reqs.append(dist.isend(torch.from_numpy(sbuf[a:b].copy()), q))
            if rs:
                a, b = rs[0].offset, rs[-1].offset + per_cell * rs[-1].lenp
                view = rbuf[a:b]
                reqs.append((dist.irecv(view, q), view, a))
        for r in reqs:
            (r[0] if isinstance(r, tuple) else r).wait()
        for r in reqs:
            if isinstance(r, tuple):
                rbuf[r[2]:r[2] + r[1].numel()] = r[1]
        rb = rbuf.numpy()
        remote = {}
        for f in recvs:  # strip of sender vp's side borders my chunk nbr on side ^ 1
            remote[(f.nbr, f.side ^ 1)] = rb[f.offset:f.offset + per_cell * f.lenp].reshape(
                F, NZ, f.lenp)[:, :, :f.len]
        # Jacobi on halo-padded chunks with the oracle, compare with the global oracle
        glob = np.empty_like(U)
        of.lib().oracle_jacobi(NX, NY, NZ, F, of._d(U), of._d(glob))
        ok = True
        for v, blk in block.items():
            s = subs[v]
            h, w = blk.shape[2], blk.shape[3]
            pad = np.zeros((F, NZ, h + 2, w + 2))
            pad[:, :, 1:-1, 1:-1] = blk
            for side in range(4):
                n = od.chunk_neighbor(od.DecompositionKind.TwoD, KX, KY, v, side)
                if n < 0:
                    strip = edge(blk, side)  # zero-flux: the cell itself
                elif rank_of_vp[n] == rank:
                    strip = edge(block[n], side ^ 1)
                else:
                    strip = remote[(v, side)]
                if side == 0:
                    pad[:, :, 1:-1, 0] = strip
                elif side == 1:
                    pad[:, :, 1:-1, -1] = strip
                elif side == 2:
                    pad[:, :, 0, 1:-1] = strip
                else:
                    pad[:, :, -1, 1:-1] = strip
            pad = np.ascontiguousarray(pad)
            res = np.empty_like(pad)
            of.lib().oracle_jacobi(w + 2, h + 2, NZ, F, of._d(pad), of._d(res))
            want = glob[:, :, s.y_begin:s.y_end, s.x_begin:s.x_end]
            ok = ok and np.array_equal(res[:, :, 1:-1, 1:-1], want)
        out[rank] = (ok, len(sends), len(recvs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mapping_kind", ["block", "scattered"])
def test_two_rank_halo_exchange_matches_oracle(mapping_kind):
    K = KX * KY
    if mapping_kind == "block":
        rank_of_vp = [v * 2 // K for v in range(K)]
    else:
        rng = np.random.default_rng(11)
        rank_of_vp = rng.integers(0, 2, K).tolist()
        rank_of_vp[0], rank_of_vp[1] = 0, 1
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, rank_of_vp, 31, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert out[0][0] and out[1][0], dict(out)
    # every face sent by one rank is received by the other
    assert out[0][1] == out[1][2] and out[1][1] == out[0][2] and out[0][1] > 0
