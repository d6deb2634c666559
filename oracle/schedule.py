"""TEST INFRASTRUCTURE ONLY: restatement of the reference epoch schedule.

advance_advection / set_shift (engine.hpp:323-342) and the Sync/Async window
split (measurement.hpp:33-36), so the field oracle can be driven with the same
per-step shifts as the runtime.
"""
from __future__ import annotations


def _round_half_away(x: float) -> int:  # std::lround
    return int(x + 0.5) if x >= 0 else -int(-x + 0.5)


def shifts(total_shift_rows: int, adv_epoch: int, duration_steps: int, async_steps: int,
           sync_steps: int, n_steps: int, ny: int, start_epoch: int = 1):
    """Per-step shift (mod ny) for n_steps timesteps starting at epoch start_epoch."""
    S = async_steps + sync_steps
    out, cur = [], 0
    for g in range(n_steps):
        e, s = start_epoch + g // S, g % S
        if adv_epoch != 0 and total_shift_rows != 0:
            tgt = cur
            if e > adv_epoch:
                tgt = total_shift_rows
            elif e == adv_epoch:
                k = min(s + 1, duration_steps)
                tgt = _round_half_away(float(total_shift_rows) * k / duration_steps)
            cur = tgt
        out.append(cur % ny)
    return out
