"""bench.py's plain workload table (used by the reference arm, which must not
import the product package) matches paper_1310_4218_b200.configs."""
import importlib.util
import os

import pytest

from paper_1310_4218_b200 import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "expA", "expB", "expC"])
def test_workload_table_matches_configs(name):
    b = _bench()
    c = configs.CONFIGS[name]()
    d = c.domain
    want = (d.nx, d.ny, d.nz, d.fields, int(c.pattern), c.heavy_value, c.light_value,
            int(c.decomposition.kind), c.decomposition.kx, c.decomposition.ky,
            c.cluster.nodes, c.cluster.procs_per_node, c.n_inner, c.seed)
    got = b.WORKLOADS[name]
    # nodes of cfg3 (8 by default) only matter for static_node0, which cfg3 does not use
    assert got[:10] == want[:10] and got[11:] == want[11:], (got, want)


def test_reference_arm_imports_no_product_code():
    import subprocess
    import sys
    code = ("import sys, runpy; sys.argv=['bench.py']; import bench; "
            "b = bench; args = type('A', (), {'config': 'cfg2', 'n_inner': 4, 'steps': 1, "
            "'warmup': 0, 'gpus': 1})(); line = b.reference_arm(args); "
            "assert line['config']['same_config'], line; "
            "assert not any(m.startswith('paper_1310_4218_b200') for m in sys.modules), "
            "[m for m in sys.modules if m.startswith('paper')]; print('ok')")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
