"""Multi-GPU path (one process per GPU, NCCL halo exchange and chunk
migration): runs tools/mgpu_check.py under torchrun on 2 GPUs when present,
and the main variants on 4 GPUs when present (three peers per GPU: per-face
halo flags from several senders, migration pulls from several sources)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(ngpus() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("mode,halo,extra", [(5, "p2p", {}), (5, "nccl", {}), (0, "p2p", {}),
                                             (4, "p2p", {}), (7, "p2p", {}),
                                             (5, "p2p", {"OD_OVERLAP": "0"}),
                                             (5, "p2p", {"OD_PACK_CTAS": "0"}),
                                             (5, "p2p", {"OD_LIB_VARIANT": "checked"}),
                                             (4, "p2p", {"OD_LIB_VARIANT": "checked"}),
                                             (4, "p2p", {"OD_TMA": "2"}),
                                             (4, "p2p", {"OD_TMA": "2",
                                                         "OD_LIB_VARIANT": "checked"})])
def test_two_gpus_fields_and_plans(mode, halo, extra):
    _run_ranks(2, mode, halo, extra)


@pytest.mark.skipif(ngpus() < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("mode,halo,extra", [(5, "p2p", {}), (5, "nccl", {}), (4, "p2p", {}),
                                             (5, "p2p", {"OD_PACK_CTAS": "0"}),
                                             (5, "p2p", {"OD_LIB_VARIANT": "checked"})])
def test_four_gpus_fields_and_plans(mode, halo, extra):
    _run_ranks(4, mode, halo, extra)


@pytest.mark.skipif(ngpus() < 2, reason="needs 2 GPUs")
def test_two_gpus_cfg3_full_grid():
    # the bench's cfg3 grid (512x512x64, F=50, 256 chunks) over 2 GPUs: GreedyLB
    # re-places ~half the chunks over NVLink every epoch, most faces remote
    _run_ranks(2, 5, "p2p", {}, shape="cfg3")


def _run_ranks(n, mode, halo, extra, shape="small"):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tools", "mgpu_check.py"), str(mode), shape]
    env = dict(os.environ, OD_HALO=halo, **extra)
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(rows) == n
    for r in rows:
        assert r["fields_ok"] and r["consistent_plans"] and r["all_columns_covered"], r
        assert sum(r["moves"]) > 0 and r["halo_bytes"] > 0 and r["migrated_bytes"] > 0
