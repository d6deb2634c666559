"""Analyse an OD_TILELOG share-clock event log (diagnostic)."""
import sys
from collections import defaultdict

import numpy as np

ev = np.loadtxt(sys.argv[1])
t, v, n, tag, sm, d = ev.T
t0 = t.min()
open_ = {}
tiles = []
for i in np.argsort(t, kind="stable"):
    key = (int(tag[i]), int(sm[i]))
    if d[i] > 0:
        open_[key] = (t[i], v[i], n[i])
    else:
        ts, vs, ns = open_.pop(key)
        tiles.append((int(tag[i]) >> 20, (ts - t0) / 1e6, (t[i] - t0) / 1e6, (v[i] - vs) / 1e6, ns, int(sm[i])))
tiles = np.array(tiles)
print("tiles", len(tiles), "kernel span ms", (t.max() - t0) / 1e6, "SMs", len(set(sm)))
slot, ts, te, share, nin, smid = tiles.T
dur = te - ts
bins = np.linspace(0, te.max(), 13)
print("start-bin  ntiles  mean_dur  mean_share  share/dur  n_at_entry")
for a, b in zip(bins[:-1], bins[1:]):
    m = (ts >= a) & (ts < b)
    if m.any():
        print(f"{a:6.2f}-{b:6.2f} {m.sum():6d} {dur[m].mean():8.3f} {share[m].mean():9.4f} {np.mean(share[m] / dur[m]):8.3f} {nin[m].mean():6.2f}")
# per-SM concurrency over time
busy = defaultdict(float)
for s_ in set(smid.astype(int)):
    m = smid == s_
    busy[s_] = te[m].max() - ts[m].min()
b = np.array(list(busy.values()))
print("per-SM span ms: min %.3f median %.3f max %.3f" % (b.min(), np.median(b), b.max()))
order = np.argsort(te)[::-1][:12]
print("latest-ending tiles: slot start end dur share n_entry sm")
for i in order:
    print("  %4d %7.3f %7.3f %6.3f %6.3f %d %3d" % (slot[i], ts[i], te[i], dur[i], share[i], nin[i], smid[i]))
ends = np.array(sorted(te[smid == s_].max() for s_ in set(smid.astype(int))))
print("SM end times: p10 %.3f p50 %.3f p90 %.3f p99 %.3f max %.3f" % tuple(np.percentile(ends, [10, 50, 90, 99, 100])))
lastw = ts > ends.min() - 3
print("tiles starting within 3 ms of the first SM going idle:", int(lastw.sum()), "mean dur %.3f" % dur[lastw].mean())
