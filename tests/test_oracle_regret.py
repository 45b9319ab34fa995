"""Pins of Theorem 1 (section 6; Appendix A,
P:1614-1703) on oracle runs of the weight-dependent workload, CPU only.

The workload's minibatch functions are f_t(w) = a/2 ||w - b||^2 + sigma_n <xi_t, w>
(convex; gradient a (w - b) + sigma_n xi_t = the CONVEX gradient of the oracle),
t = one update u(v, p), T = N * W * N_m of them. Theorem 1: with
u_t = -eta_t grad f_t(w~_t), eta_t = sigma / sqrt(t),
sigma = M / (L sqrt((2 s_g + s_l) N)), the regret
R[W] = 1/T sum_t f_t(w~_t) - f(w*) <= 4 M L sqrt((2 s_g + s_l) N / T)
once T is large enough; Appendix A's last inequality before that
simplification holds for every T and every sigma:
T R <= sigma L^2 sqrt T + M^2/sigma sqrt T + sigma L^2 (2s_g+s_l)(s_g+s_l) N^2
       + 2 sigma L^2 (2s_g+s_l) N sqrt T.

w~_t is the weight minibatch p of VW v READ at its START (the oracle's
snapshot), f(w) = 1/T sum_t f_t, w* = b - sigma_n mean(xi) / a.
M and L (readings Z27): the domain is the box [-R0, R0]^P, R0 = 2; Assumption
2 as the proof uses it, D(w||w') = 1/2 ||w - w'||^2 <= M^2, gives M = R0 sqrt(2P);
L = sqrt(P) (a (R0 + 1) + sigma_n / 2) bounds ||grad f_t|| on the box. The test
asserts that every w~_t and w* lie in the box (the assumptions hold), then the
bounds. The step-size schedule itself is pinned by a closed form."""
import math
import random

import numpy as np
import pytest

from oracle import convex_target, initial_weights, run_schedule, s_global
from oracle.wsp import _draws
from workloads import GRAD_CONVEX, LR_THEOREM1, PULL_EAGER, PULL_LAZY, W0_PHILOX, WSPConfig

R0 = 2.0


def xi_of(idx, v, p, cfg):
    """The noise draw xi of u(v, p): the FLOAT draw of Philox stream 0."""
    x = _draws(idx, v, p, 0, cfg.seed)
    return (x >> 8).astype(np.float64) * 2.0 ** -24 - 0.5


def theorem_constants(cfg):
    P = cfg.nparams
    M = R0 * math.sqrt(2 * P)
    L = math.sqrt(P) * (cfg.conv_a * (R0 + 1) + cfg.conv_sigma / 2)
    sg, sl = s_global(cfg.Nm, cfg.D), cfg.Nm      # s_l = s_local + 1
    sigma = M / (L * math.sqrt((2 * sg + sl) * cfg.num_vw))
    return M, L, sg, sl, sigma


def regret(cfg, flip=False):
    """(R[W], T, max |w~|, max |w*|) of one oracle run."""
    idx = np.arange(cfg.nparams)
    run = run_schedule(cfg, record_snapshots=True)
    a, sn = float(cfg.conv_a), float(cfg.conv_sigma)
    b = convex_target(idx, cfg).astype(np.float64)
    f_sum, xi_sum, T, wmax = 0.0, np.zeros(cfg.nparams), 0, 0.0
    for (t, v, p, snap) in run.snapshots:
        w = snap.astype(np.float64)
        xi = xi_of(idx, v, p, cfg)
        f_sum += 0.5 * a * float(np.sum((w - b) ** 2)) + sn * float(np.dot(xi, w))
        xi_sum += xi
        T += 1
        wmax = max(wmax, float(np.max(np.abs(w))))
    assert T == cfg.num_vw * cfg.waves * cfg.Nm
    xbar = xi_sum / T
    wstar = b - sn * xbar / a
    f_star = 0.5 * a * float(np.sum((wstar - b) ** 2)) + sn * float(np.dot(xbar, wstar))
    return f_sum / T - f_star, T, wmax, float(np.max(np.abs(wstar)))


def theorem_cfg(N, Nm, D, W, tau, policy=PULL_EAGER, P=33, sigma_n=0.5, seed=7):
    base = WSPConfig("thm1", N, Nm, D, P, W, tau, grad_mode=GRAD_CONVEX, w0_mode=W0_PHILOX,
                     conv_a=0.5, conv_sigma=sigma_n, lr_schedule=LR_THEOREM1,
                     pull_policy=policy, seed=seed)
    M, L, sg, sl, sigma = theorem_constants(base)
    return base.replace(lr=sigma), (M, L, sg, sl, sigma)


@pytest.mark.parametrize("N", [1, 2, 3])
def test_schedule_closed_form_bsp(N):
    """BSP limit (N_m = 1, D = 0, sigma_n = 0, equal speeds): all N VWs
    read the same w_p, so w_{p+1} - b = (1 - a sum_v eta_{(p-1)N+v+1}) (w_p - b),
    eta_t = sigma / sqrt(t) -- the schedule and its worker-fastest numbering."""
    W = 12
    cfg = WSPConfig("bsp", N, 1, 0, 129, W, (7,) * N, lr=0.3, grad_mode=GRAD_CONVEX,
                    conv_a=0.5, conv_sigma=0.0, lr_schedule=LR_THEOREM1)
    idx = np.arange(cfg.nparams)
    r = run_schedule(cfg)
    b = convex_target(idx, cfg).astype(np.float64)
    e = initial_weights(idx, cfg).astype(np.float64) - b
    for p in range(1, W + 1):
        e = (1.0 - cfg.conv_a * sum(cfg.lr / math.sqrt((p - 1) * N + v + 1)
                                    for v in range(N))) * e
    got = r.wg.astype(np.float64) - b
    assert np.max(np.abs(got - e)) / np.max(np.abs(e)) < 1e-5
    # a plausible mistake -- the VW-major numbering t = v * W + p -- is caught
    e2 = initial_weights(idx, cfg).astype(np.float64) - b
    for p in range(1, W + 1):
        e2 = (1.0 - cfg.conv_a * sum(cfg.lr / math.sqrt(v * W + p) for v in range(N))) * e2
    if N > 1:
        assert np.max(np.abs(got - e2)) / np.max(np.abs(e2)) > 1e-3


def test_schedule_single_vw_pipelined():
    """One VW with N_m in flight: e_p = e_{p-1} - eta_{p-N_m}... each update
    u_q = -eta_q a e_q is applied to the weights N_m minibatches later
    (P:846-847), eta_q = sigma / sqrt(q)."""
    Nm, W = 3, 6
    cfg = WSPConfig("one", 1, Nm, 0, 65, W, (5,), lr=0.4, grad_mode=GRAD_CONVEX, conv_a=0.5,
                    conv_sigma=0.0, lr_schedule=LR_THEOREM1)
    idx = np.arange(cfg.nparams)
    r = run_schedule(cfg, record_snapshots=True)
    b = convex_target(idx, cfg).astype(np.float64)
    e = {p: initial_weights(idx, cfg).astype(np.float64) - b for p in range(0, Nm + 1)}
    for p in range(Nm + 1, W * Nm + 1):
        q = p - Nm
        e[p] = e[p - 1] - cfg.lr / math.sqrt(q) * cfg.conv_a * e[q]
    for (t, v, p, snap) in r.snapshots:
        d = snap.astype(np.float64) - b
        assert np.max(np.abs(d - e[p])) / np.max(np.abs(e[p])) < 1e-5, p


def min_waves(N, Nm, D):
    """Smallest W whose T = N W N_m is "large enough" for the simplified bound
    (App. A: 1/((2s_g+s_l)N) + (s_g+s_l)N/sqrt(T) <= 1); 40 if it never is (k = 1)."""
    sg = s_global(Nm, D)
    k = (2 * sg + Nm) * N
    if k == 1:
        return 40
    W = 1
    while 1.0 / k + (sg + Nm) * N / math.sqrt(N * W * Nm) > 1.0:
        W += 1
    return W


CASES = [
    # (N, Nm, D, tau, policy); W = min_waves + 4
    (1, 1, 0, (5,), PULL_EAGER),
    (2, 1, 0, (5, 5), PULL_EAGER),
    (2, 2, 0, (5, 7), PULL_EAGER),
    (2, 2, 1, (3, 8), PULL_LAZY),
    (3, 2, 1, (4, 6, 9), PULL_EAGER),
    (4, 1, 2, (2, 3, 5, 7), PULL_LAZY),
    (2, 3, 2, (3, 7), PULL_EAGER),
]


@pytest.mark.parametrize("case", CASES, ids=[f"N{c[0]}Nm{c[1]}D{c[2]}" for c in CASES])
def test_theorem1_regret_bound(case):
    N, Nm, D, tau, policy = case
    cfg, (M, L, sg, sl, sigma) = theorem_cfg(N, Nm, D, min_waves(N, Nm, D) + 4, tau, policy)
    R, T, wmax, wsmax = regret(cfg)
    # the assumptions hold on this run: every read weight and w* in the box
    assert wmax <= R0 and wsmax <= R0, (wmax, wsmax)
    k = (2 * sg + sl) * N
    sig = float(np.float32(cfg.lr))          # the sigma the run used (float32)
    general = (sig * L * L * math.sqrt(T) + M * M / sig * math.sqrt(T)
               + sig * L * L * k * (sg + sl) * N + 2 * sig * L * L * k * math.sqrt(T)) / T
    assert R <= general, (R, general)
    simplified = 4 * M * L * math.sqrt(k / T)
    if k > 1:
        # "T large enough" (App. A): 1/((2s_g+s_l)N) + (s_g+s_l)N/sqrt(T) <= 1
        # (never for k = 1, i.e. the serial case N = N_m = 1, D = 0)
        assert 1.0 / k + (sg + sl) * N / math.sqrt(T) <= 1.0, f"T={T}: raise W"
        assert R <= simplified, (R, simplified)
    # the regret is a real quantity here, not vacuous: it decays like 1/sqrt(T)
    assert R > 0


def test_regret_pin_catches_ascent():
    """A sign error in the update (gradient ascent) violates the bound."""
    cfg, (M, L, sg, sl, sigma) = theorem_cfg(2, 2, 0, min_waves(2, 2, 0) + 4, (5, 7))
    bad = cfg.replace(lr=-cfg.lr)
    R, T, wmax, _ = regret(bad)
    k = (2 * sg + sl) * cfg.num_vw
    assert wmax > R0 or R > 4 * M * L * math.sqrt(k / T)


@pytest.mark.parametrize("seed", range(6))
def test_theorem1_regret_random(seed):
    rng = random.Random(seed)
    N = rng.randint(1, 3)
    Nm = rng.randint(1, 3)
    D = rng.randint(0, 2)
    sg = s_global(Nm, D)
    k = (2 * sg + Nm) * N
    W = min_waves(N, Nm, D)
    tau = tuple(rng.randint(1, 9) for _ in range(N))
    cfg, (M, L, sg, sl, sigma) = theorem_cfg(N, Nm, D, W + rng.randint(0, 10), tau,
                                             rng.choice([PULL_EAGER, PULL_LAZY]),
                                             seed=rng.randint(1, 1 << 30))
    R, T, wmax, wsmax = regret(cfg)
    assert wmax <= R0 and wsmax <= R0
    assert 0 < R
    if k > 1:
        assert R <= 4 * M * L * math.sqrt(k / T)
