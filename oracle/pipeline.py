"""Oracle of the intra-VW pipeline schedule (section 4, P:760-806;
SURVEY.md 8(f) NEXT-1). TEST INFRASTRUCTURE: only tests/, smoke() and
bench.py's cpu_baseline may import it; the product computes the same things
in paper_2005_14038_b200/csrc/pipeline.cpp, which shares no code with this.

Written plainly, in the paper's terms:
  * stage_depth / stage_memory -- "the actual memory requirement will vary
    depending on the stage of the pipeline": the first stage holds
    the forward results of every in-flight minibatch, the last only one.
    depth(q) = min(Nm, 2(k-q)+1) and mem = 3 x params + depth x resident
    activations (SPEC.md partition module's reading; readings Z21/Z22).
  * stage_time -- "the sum of the computation time of all the layers in the
    partition and the communication time needed for receiving the activations
    (in the forward pass) and local gradients (in the backward pass)".
  * partition_bruteforce -- "minimize the maximum execution time of the
    partitions within the bounds of satisfying the memory requirement"
    (P:791): every GPU order x every contiguous k-way split, smallest
    bottleneck, ties to the lexicographically smallest (order, cuts).
  * simulate -- scheduling conditions 1-3: per GPU forward tasks in
    minibatch order, backward tasks in minibatch order, FIFO among ready tasks
    (ties: backward first, then lower minibatch); the last partition runs
    forward+backward of a minibatch as one task. Minibatch p starts when
    p <= Nm or when p - Nm completes (local staleness Nm - 1).
All times are integer nanoseconds, so the product can match exactly.
"""
from __future__ import annotations

import itertools
from typing import Dict, List, Optional, Sequence, Tuple

PARAM_OVERHEAD = 3          # weights + gradients + optimizer state (reading Z22)


def stage_depth(q: int, k: int, Nm: int) -> int:
    """Minibatches whose forward results stage q (1-based) holds at once."""
    assert 1 <= q <= k and Nm >= 1
    return min(Nm, 2 * (k - q) + 1)


def stage_memory(units, lo: int, hi: int, q: int, k: int, Nm: int, batch: int = 32) -> int:
    """Bytes stage q needs for units[lo:hi] (fp32)."""
    params = sum(u.params for u in units[lo:hi])
    resident = sum(u.act_resident for u in units[lo:hi])
    return PARAM_OVERHEAD * 4 * params + stage_depth(q, k, Nm) * 4 * batch * resident


def compute_ns(units, lo: int, hi: int, flops_per_s: float, batch: int = 32) -> Tuple[int, int]:
    """(forward, backward) ns of units[lo:hi]; backward = 2 x forward."""
    f = sum(u.fwd_flops for u in units[lo:hi]) * batch
    fwd = int(round(f / flops_per_s * 1e9))
    return fwd, 2 * fwd


def comm_ns(units, cut: int, bw_bytes_per_s: float, batch: int = 32) -> int:
    """Transfer of the activation leaving unit cut-1 (same size as the gradient
    coming back across the same cut)."""
    return int(round(units[cut - 1].act_out * 4 * batch / bw_bytes_per_s * 1e9))


def stage_costs(units, cuts: Sequence[int], gpus: Sequence[dict], batch: int = 32):
    """Per stage q: fwd_ns, bwd_ns, comm_in_fwd_ns, comm_in_bwd_ns.
    gpus[q] = {"flops": F, "mem": bytes, "node": n} in stage order."""
    k = len(gpus)
    out = []
    for q in range(k):
        lo, hi = cuts[q], cuts[q + 1]
        fwd, bwd = compute_ns(units, lo, hi, gpus[q]["flops"], batch)
        cf = cb = 0
        if q > 0:
            bw = link_bw(gpus[q - 1], gpus[q])
            cf = comm_ns(units, lo, bw, batch)
        if q < k - 1:
            bw = link_bw(gpus[q], gpus[q + 1])
            cb = comm_ns(units, hi, bw, batch)
        out.append((fwd, bwd, cf, cb))
    return out


INTRA_BPS = 15.75e9
INTER_BPS = 56e9 / 8


def link_bw(a: dict, b: dict) -> float:
    return INTRA_BPS if a["node"] == b["node"] else INTER_BPS


def stage_time(cost) -> int:
    fwd, bwd, cf, cb = cost
    return fwd + bwd + cf + cb


def partition_bruteforce(units, gpus: Sequence[dict], Nm: int, batch: int = 32,
                         orders: Optional[Sequence[Sequence[int]]] = None):
    """Returns (bottleneck_ns, order, cuts) or None if no split fits memory."""
    L, k = len(units), len(gpus)
    best = None
    for order in (orders if orders is not None else itertools.permutations(range(k))):
        g = [gpus[i] for i in order]
        for inner in itertools.combinations(range(1, L), k - 1):
            cuts = (0,) + inner + (L,)
            ok = all(stage_memory(units, cuts[q], cuts[q + 1], q + 1, k, Nm, batch) <= g[q]["mem"]
                     for q in range(k))
            if not ok:
                continue
            b = max(stage_time(c) for c in stage_costs(units, cuts, g, batch))
            key = (b, tuple(order), cuts)
            if best is None or key < best:
                best = key
    return best


def simulate(costs, Nm: int, P: int):
    """Event-driven pipeline of one VW. costs[q] = (fwd, bwd, cf, cb) ns.
    Returns (start_ns[1..P], complete_ns[1..P], tasks) with tasks a list of
    (gpu, kind, p, t_start, t_end), kind in {"F", "B", "FB"}."""
    k = len(costs)
    st: Dict[int, int] = {}
    done: Dict[Tuple[str, int, int], int] = {}     # (kind, p, q) -> end time
    ready: Dict[Tuple[str, int, int], int] = {}    # (kind, p, q) -> ready time
    free = [0] * k
    comp: Dict[int, int] = {}
    tasks = []

    def admit(p, t):
        st[p] = t
        ready[("FB" if k == 1 else "F", p, 0)] = t

    for p in range(1, min(Nm, P) + 1):
        admit(p, 0)

    def eligible(key):
        kind, p, q = key
        if p > 1 and (kind, p - 1, q) not in done:        # conditions 1 and 2
            return False
        return True

    while len(comp) < P:
        cand = None
        for q in range(k):
            keys = [x for x in ready if x[2] == q and x not in done and eligible(x)]
            if not keys:
                continue
            s = max(free[q], min(ready[x] for x in keys))
            pick = min((x for x in keys if ready[x] <= s),
                       key=lambda x: (ready[x], 0 if x[0] != "F" else 1, x[1]))
            if cand is None or (s, q) < (cand[0], cand[1]):
                cand = (s, q, pick)
        assert cand is not None, "pipeline deadlock"
        s, q, key = cand
        kind, p, _ = key
        fwd, bwd, cf, cb = costs[q]
        dur = fwd if kind == "F" else bwd if kind == "B" else fwd + bwd
        end = s + dur
        free[q] = end
        done[key] = end
        del ready[key]
        tasks.append((q, kind, p, s, end))
        if kind == "F":                       # activation to stage q+1
            nxt = q + 1
            ready[("FB" if nxt == k - 1 else "F", p, nxt)] = end + costs[nxt][2]
        elif q > 0:                           # local gradient to stage q-1
            ready[("B", p, q - 1)] = end + costs[q - 1][3]
        else:                                 # backward reached stage 1: u_p exists
            comp[p] = end
            if p + Nm <= P:
                admit(p + Nm, end)            # START(p+Nm) at COMPLETE(p)
    return st, comp, tasks


def derive_tau_latency(costs, Nm: int, P: int = 0) -> Tuple[int, int]:
    """(tau_ns, L_ns): the mean completion interval over the middle half of a
    P-minibatch run (fill and drain excluded; floor to whole ns) and the first
    minibatch's start-to-complete time --
    the two numbers of the tick model complete(p) = max(start(p) + L,
    complete(p-1) + tau) (reading Z13)."""
    P = P or 24 * max(Nm, 1)
    _, comp, _ = simulate(costs, Nm, P)
    a, b = P // 4, 3 * P // 4
    tau = (comp[b] - comp[a]) // (b - a)
    return tau, comp[1]
