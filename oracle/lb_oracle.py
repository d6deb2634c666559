"""TEST INFRASTRUCTURE ONLY: pure-Python restatement of the reference's
balancers and bookkeeping, following
  greedy_lb          /root/reference/proj/include/overdeck/balancer.hpp:36-63
  refine_swap_lb     balancer.hpp:68-152
  should_balance     balancer.hpp:29-32
  proc_loads         cluster.hpp:142-148
  imbalance_ratio    cluster.hpp:151-157
  initial_block_mapping cluster.hpp:115-127
  apply_plan         cluster.hpp:130-139
  epoch_loads        measurement.hpp:75-91
  run_epoch policy   engine.hpp:257-268
Python floats are IEEE doubles and the operation order matches the reference,
so plans are bit-identical.  Pinned against the reference itself
(oracle/_ref via oracle/ref.py) and the reference unit-test vectors in
tests/test_oracle.py.  Small cases only (pure-Python loops).
"""
from __future__ import annotations


class StaleMove(Exception):
    pass


def initial_block_mapping(K, P):
    if P < 1 or K < P:
        raise ValueError("need K >= P >= 1")
    q, r = divmod(K, P)
    out = []
    for p in range(P):
        out += [p] * (q + (1 if p < r else 0))
    return out


def apply_plan(mapping, moves):
    out = list(mapping)
    for vp, frm, to in moves:
        if out[vp] != frm:
            raise StaleMove(vp)
        out[vp] = to
    return out


def proc_loads(loads, mapping, P):
    t = [0.0] * P
    for v, p in enumerate(mapping):
        t[p] += loads[v]
    return t


def imbalance_ratio(totals):
    s = 0.0
    for t in totals:
        s += t
    if s <= 0.0:
        return 1.0
    return max(totals) / (s / len(totals))


def should_balance(totals, threshold):
    return imbalance_ratio(totals) > threshold


def greedy_lb(loads, mapping, P):
    K = len(mapping)
    order = sorted(range(K), key=lambda v: (-loads[v], v))  # stable: desc load, asc id
    acc = [0.0] * P
    target = [0] * K
    for v in order:
        best = 0
        for p in range(1, P):
            if acc[p] < acc[best]:
                best = p
        target[v] = best
        acc[best] += loads[v]
    return [(v, mapping[v], target[v]) for v in range(K) if target[v] != mapping[v]]


def refine_swap_lb(loads, mapping, P, tol=0.02):
    K = len(mapping)
    cur = list(mapping)
    acc = proc_loads(loads, cur, P)
    total = 0.0
    for a in acc:
        total += a
    avg = total / P
    thr = avg * (1.0 + tol)
    plan = []

    def on(p):
        return [v for v in range(K) if cur[v] == p]

    for _ in range(K * P):
        over = -1
        for p in range(P):
            if acc[p] > thr and (over < 0 or acc[p] > acc[over]):
                over = p
        if over < 0:
            break
        dev = acc[over] - avg
        best = None
        for v in on(over):
            for q in range(P):
                if q == over or acc[q] >= avg:
                    continue
                src = acc[over] - loads[v]
                dst = acc[q] + loads[v]
                if abs(src - avg) >= dev or dst > thr:
                    continue
                score = max(abs(src - avg), abs(dst - avg))
                if best is None or score < best[2]:
                    best = (v, q, score)
        if best is not None:
            v, q, _ = best
            plan.append((v, over, q))
            acc[over] -= loads[v]
            acc[q] += loads[v]
            cur[v] = q
            continue
        sbest = None
        for q in range(P):
            if q == over or acc[q] >= avg:
                continue
            for a in on(over):
                for b in on(q):
                    d = loads[a] - loads[b]
                    if d <= 0:
                        continue
                    src = acc[over] - d
                    dst = acc[q] + d
                    if abs(src - avg) >= dev or dst > thr:
                        continue
                    score = max(abs(src - avg), abs(dst - avg))
                    if sbest is None or score < sbest[3]:
                        sbest = (a, b, q, score)
        if sbest is None:
            break
        a, b, q, _ = sbest
        plan.append((a, over, q))
        plan.append((b, q, over))
        d = loads[a] - loads[b]
        acc[over] -= d
        acc[q] += d
        cur[a] = q
        cur[b] = over
    return plan


def epoch_loads(K, samples):
    """samples: (vp, step, mode, value) in record order; mode 0 = Sync."""
    s = [0.0] * K
    n = [0] * K
    for vp, _step, mode, value in samples:
        if mode != 0:
            continue
        s[vp] += value
        n[vp] += 1
    if any(c == 0 for c in n):
        raise RuntimeError("incomplete measurement")
    return [s[v] / n[v] for v in range(K)]


def epoch_decision(loads, mapping, P, epoch, epochs, balance_calls, first, later, threshold,
                   tol):
    """-> (strategy or None, plan, balance_calls)"""
    totals = proc_loads(loads, mapping, P)
    if epoch < epochs and should_balance(totals, threshold):
        strategy = first if balance_calls == 0 else later
        plan = greedy_lb(loads, mapping, P) if strategy == 0 else \
            refine_swap_lb(loads, mapping, P, tol)
        return strategy, plan, balance_calls + 1
    return None, [], balance_calls
