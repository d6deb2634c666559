"""Helpers shared by the GPU parity tests: run a config on the device through
the C ABI and the same config through the CPU field oracle."""
import numpy as np

import paper_1310_4218_b200 as od
from oracle import fields as ofields
from oracle import ref as oref
from oracle import schedule as osched


def oracle_fields(cfg, n_steps, start_epoch=1):
    d = cfg.domain
    U, A = ofields.init_state(d.nx, d.ny, d.nz, d.fields, cfg.seed)
    base = oref.base_field(cfg)
    adv = cfg.advection
    sh = osched.shifts(adv.total_shift_rows, adv.epoch, adv.duration_steps,
                       cfg.window.async_steps, cfg.window.sync_steps, n_steps, d.ny, start_epoch)
    ofields.run(U, A, base, sh, cfg.n_inner)
    return U, A


def device_fields(cfg, n_steps, use_epochs=False):
    with od.Engine(cfg) as eng:
        if use_epochs:
            S = cfg.window.epoch_steps()
            assert n_steps % S == 0
            recs = [eng.run_epoch(e) for e in range(1, n_steps // S + 1)]
        else:
            eng.advance(n_steps)
            recs = None
        U, A, own = eng.gather_fields()
        assert own.all()
        return U, A, recs


def assert_bitwise(a, b, what):
    if not np.array_equal(a, b):
        diff = np.argwhere(a != b)
        first = tuple(diff[0])
        raise AssertionError(f"{what}: {len(diff)} values differ; first at {first}: "
                             f"{a[first]!r} vs {b[first]!r}")
