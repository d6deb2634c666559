import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1310_4218_b200 as od
from tests.gpu_util import device_fields, oracle_fields
from tests.test_gpu_fields import small
mode = int(sys.argv[1])
ok = True
for kw in (dict(kx=1, ky=1, nz=2, F=1), dict(kx=4, ky=3),
           dict(nx=45, ny=30, kind=od.DecompositionKind.OneD, kx=1, ky=7),
           dict(nx=150, ny=70, nz=9, F=2, kx=3, ky=3, adv=(35, 1, 3), n_inner=7, ppn=3, threshold=1.0),
           dict(nx=33, ny=9, nz=1, F=1, kx=3, ky=2, heavy=3.0, n_inner=0)):
    cfg = small(overlap=mode, **kw)
    U, A, _ = device_fields(cfg, 6)
    Uo, Ao = oracle_fields(cfg, 6)
    du = int((U != Uo).sum()); da = int((A != Ao).sum())
    ok &= du == 0 and da == 0
    print(kw, "U diff", du, "A diff", da, flush=True)
print("ALL OK" if ok else "FAIL")
