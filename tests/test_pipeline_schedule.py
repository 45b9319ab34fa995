"""Intra-VW pipeline schedule (section 4,
P:760-806): the oracle (oracle/pipeline.py: brute-force partition, plain event
loop) pinned by what the paper and arithmetic fix, and the library's native
partitioner / simulator (csrc/pipeline.cpp through include/hetpipe.h) checked
against it exactly (integer nanoseconds). Host code only: no GPU needed."""
import random
from types import SimpleNamespace as U

import pytest

from oracle import pipeline as op
from workloads import models as M


@pytest.fixture(scope="module")
def hp():
    from paper_2005_14038_b200 import hetpipe
    hetpipe.load()
    return hetpipe


def gpus_of(policy, vw):
    F = M.v_flops_per_s()
    return [{"flops": F * M.GPUS[t].speed, "mem": M.GPUS[t].mem_gb * 1e9, "node": n}
            for t, n in M.vw_gpus(policy, vw)]


# ---------------------------------------------------------------- oracle pins
def test_model_tables_match_paper_sizes():
    # P:203 "548MB" (VGG-19) and P:206 "230MB" (ResNet-152) of fp32 parameters
    assert sum(u.params for u in M.vgg19()) == 143_667_240
    assert sum(u.params for u in M.resnet152()) == 60_192_808
    assert round(sum(u.params for u in M.vgg19()) * 4 / 2 ** 20) == 548
    assert round(sum(u.params for u in M.resnet152()) * 4 / 2 ** 20) == 230
    # fc6 is 71.5% of VGG-19 (SURVEY.md 8(d) workload structure)
    assert abs(M.vgg19()[16].params / 143_667_240 - 0.715) < 0.001
    assert len(M.resnet152()) == 52 and len(M.vgg19()) == 19
    # Horovod moves 515MB across the 16-GPU cluster for VGG-19 = a ring
    # all-reduce's (n-1)/n of the 548 MB model (SURVEY.md reading Z19)
    assert abs(143_667_240 * 4 * 15 / 16 / 2 ** 20 - 515) / 515 < 0.005


def test_stage_depth_examples():
    # the last stage holds one minibatch, the first all in flight
    assert op.stage_depth(4, 4, 4) == 1
    assert op.stage_depth(1, 4, 4) == 4
    assert op.stage_depth(1, 1, 5) == 1
    assert op.stage_depth(1, 4, 9) == 7


def test_naive_model_parallelism_nm1():
    # Nm = 1: one minibatch in the VW at a time -> complete(p) = p x sum of stages
    costs = [(100, 200, 7, 5), (50, 100, 3, 0)]
    _, comp, _ = op.simulate(costs, 1, 6)
    one = 100 + 50 + 3 + 100 + 5 + 200
    assert [comp[p] for p in range(1, 7)] == [p * one for p in range(1, 7)]


def test_uniform_pipeline_saturates():
    # k uniform stages (fwd u, bwd 2u, no comm): with Nm >= k every GPU is busy,
    # one completion per 3u; latency of one minibatch = 4k - ... = (k-1)(u+2u) + 3u
    for k in (2, 3, 4):
        costs = [(100, 200, 0, 0)] * k
        tau, lat = op.derive_tau_latency(costs, k)
        assert lat == 300 * k
        assert tau == 300
        tau1, _ = op.derive_tau_latency(costs, 1)
        assert tau1 == 300 * k


def validate(tasks, k, Nm):
    """Conditions 1-3 of P:796-803 on a trace."""
    by_gpu = {}
    for g, kind, p, s, e in tasks:
        by_gpu.setdefault(g, []).append((s, e, kind, p))
    for g, ts in by_gpu.items():
        ts.sort()
        for a, b in zip(ts, ts[1:]):
            assert a[1] <= b[0], "GPU runs one task at a time"
        for kind in ("F", "B", "FB"):
            ps = [p for s, e, kd, p in ts if kd == kind]
            assert ps == sorted(ps), f"condition 1/2 ({kind}) on GPU {g}"
    # in flight: minibatches started on GPU 0 and not yet completed <= Nm
    first = {p: s for g, kind, p, s, e in tasks if g == 0 and kind in ("F", "FB")}
    done = {p: e for g, kind, p, s, e in tasks if g == 0 and kind in ("B", "FB")}
    for p, s in first.items():
        assert sum(1 for q in first if first[q] <= s < done[q]) <= Nm


@pytest.mark.parametrize("seed", range(20))
def test_simulated_traces_obey_conditions(seed):
    rng = random.Random(seed)
    k = rng.randint(1, 5)
    Nm = rng.randint(1, 2 * k)
    costs = [(rng.randint(1, 90), rng.randint(1, 150), rng.randint(0, 30), rng.randint(0, 30))
             for _ in range(k)]
    _, comp, tasks = op.simulate(costs, Nm, 30)
    validate(tasks, k, Nm)
    # bounds: a pipelined VW is never slower than naive model parallelism
    # (Nm = 1: one minibatch at a time, tau = the whole latency) and never
    # faster than its busiest GPU (each minibatch costs fwd + bwd there)
    t1, lat1 = op.derive_tau_latency(costs, 1, 48)
    # (the first stage receives no activation, the last no gradient)
    one = (sum(f + b for f, b, _, _ in costs) + sum(c[2] for c in costs[1:])
           + sum(c[3] for c in costs[:-1]))
    assert t1 == lat1 == one
    # (over a finite window completions may bunch: the busiest GPU can have done
    # part of the window's forward work before it; 10% slack at 200 minibatches)
    busiest = max(f + b for f, b, cf, cb in costs)
    for nm in range(1, 2 * k + 1):
        t, lat = op.derive_tau_latency(costs, nm, 200)
        assert 0.9 * busiest <= t <= t1 and lat >= lat1


def test_bruteforce_hand_example():
    # 3 units on 2 GPUs of one node, no memory limit, no comm (huge bw):
    # splits [0|1,2] -> max(10, 20+5)=25*3, [0,1|2] -> max(30, 5)*3 -> best first
    units = [U(params=1, fwd_flops=10, act_out=0, act_resident=0),
             U(params=1, fwd_flops=20, act_out=0, act_resident=0),
             U(params=1, fwd_flops=5, act_out=0, act_resident=0)]
    g = [{"flops": 1e9, "mem": 1e18, "node": 0}] * 2
    b, order, cuts = op.partition_bruteforce(units, g, 1, batch=1)
    assert cuts == (0, 1, 3) and b == 3 * 25 and order == (0, 1)


# ------------------------------------------------------ native vs oracle
def rand_profile(rng, L):
    return [U(params=rng.randint(0, 5_000_000), fwd_flops=rng.randint(1, 4_000_000_000),
              act_out=rng.randint(1, 2_000_000), act_resident=rng.randint(0, 8_000_000))
            for _ in range(L)]


@pytest.mark.parametrize("seed", range(60))
def test_partition_matches_bruteforce(hp, seed):
    rng = random.Random(1000 + seed)
    L = rng.randint(1, 9)
    k = rng.randint(1, min(4, L))
    Nm = rng.randint(1, 2 * k)
    units = rand_profile(rng, L)
    gpus = [{"flops": rng.choice([4e12, 3e12, 2.9e12, 2.4e12]),
             "mem": rng.choice([6e9, 8e9, 12e9, 24e9, 1e12]) * rng.choice([0.05, 1.0]),
             "node": rng.randint(0, 2)} for _ in range(k)]
    want = op.partition_bruteforce(units, gpus, Nm)
    got = hp.partition(units, gpus, Nm)
    if want is None:
        assert got is None
        return
    b, order, cuts, costs = got
    assert (b, order, cuts) == want
    g = [gpus[i] for i in order]
    assert costs == op.stage_costs(units, cuts, g)


@pytest.mark.parametrize("model,policy,vw", [("vgg19", "NP", 0), ("vgg19", "NP", 3),
                                             ("vgg19", "ED", 0), ("vgg19", "HD", 0),
                                             ("vgg19", "HD", 2), ("resnet152", "HD", 0)])
def test_partition_paper_models(hp, model, policy, vw):
    units = M.MODELS[model]()
    g = gpus_of(policy, vw)
    for Nm in (1, 4):
        want = op.partition_bruteforce(units, g, Nm)
        got = hp.partition(units, g, Nm)
        assert (got is None) == (want is None)
        if got is not None:
            assert got[:3] == want


@pytest.mark.parametrize("seed", range(30))
def test_simulation_matches_oracle(hp, seed):
    rng = random.Random(2000 + seed)
    k = rng.randint(1, 6)
    Nm = rng.randint(1, 2 * k + 1)
    P = rng.randint(1, 40)
    costs = [(rng.randint(0, 900), rng.randint(1, 1500), rng.randint(0, 300), rng.randint(0, 300))
             for _ in range(k)]
    st, comp, _ = op.simulate(costs, Nm, P)
    s, c = hp.pipeline_simulate(costs, Nm, P)
    assert list(s) == [st[p] for p in range(1, P + 1)]
    assert list(c) == [comp[p] for p in range(1, P + 1)]
    if P >= 8:
        assert hp.pipeline_tau_latency(costs, Nm, P) == op.derive_tau_latency(costs, Nm, P)


def test_max_m(hp):
    rng = random.Random(7)
    for _ in range(10):
        L = rng.randint(2, 7)
        k = rng.randint(1, min(3, L))
        units = rand_profile(rng, L)
        gpus = [{"flops": 3e12, "mem": rng.choice([2e9, 4e9, 8e9, 1e12]), "node": 0}
                for _ in range(k)]
        want = 0
        for nm in range(2 * k - 1, 0, -1):
            if op.partition_bruteforce(units, gpus, nm) is not None:
                want = nm
                break
        assert hp.max_m(units, gpus) == want


def test_bad_arguments(hp):
    units = M.vgg19()
    with pytest.raises(hp.HetPipeError):
        hp.partition(units, [gpus_of("NP", 0)[0]] * 9, 1)     # k > 8
    with pytest.raises(hp.HetPipeError):
        hp.pipeline_simulate([(0, 0, 0, 0)], 1, 4)             # zero-length stage
