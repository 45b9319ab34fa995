"""CPU oracle for the WSP hot path of HetPipe (arXiv 2005.14038).

TEST INFRASTRUCTURE ONLY. Nothing on the product path may import this package:
only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg
and `--impl reference`) use it. It shares no code with
`paper_2005_14038_b200/` (the CUDA path); both read only `workloads/`, which
holds sizes, seeds and speed vectors and none of the method's arithmetic.

Plain, slow, obviously correct: numpy float32 element-wise operations (one IEEE
binary32 round-to-nearest-even per operation, no fused multiply-add), a Python
event loop that follows PAPER.md section 5 step by step. Citations are
`P:n` = /root/reference/PAPER.md line n.

Pins (tests/test_oracle_*.py): Philox known-answer vectors, the paper's worked
examples, closed forms (BSP limit P:960 / P:819,
conservation P:928-929), invariants (D+1 clock bound P:942, p-Nm read bound
P:846-847, lockstep at D=0), brute force over every interleaving of
2 VW x 3 waves x 8 params (also with F = 2 and with heavy-ball momentum;
the s_global floor and the D+1 clock distance shown tight); the weight-dependent CONVEX
workload's BSP closed form and delayed recurrence, the section-6
decomposition and Lemma 1 (tests/test_oracle_convex.py); Theorem 1's step
sizes eta_t = sigma/sqrt(t) in closed form and its regret bound on oracle runs
(App. A; tests/test_oracle_regret.py); s_global with F
(tests/test_oracle_update_freq.py); the pipeline partitioner / simulator
oracle (oracle/pipeline.py, tests/test_pipeline_schedule.py). Parity
unpinned: the exact bits of FLOAT-mode intermediate w_local snapshots with
D>0 and heterogeneous speeds (their version sets are pinned exactly, their
values to within Higham's summation bound).
"""
from .philox import philox4x32_10, philox_words
from .wsp import (OracleRun, WSPOracle, convex_target, gradient, initial_weights,
                  run_schedule, s_global, step_size, version_floor, wave_range)

__all__ = ["philox4x32_10", "philox_words", "OracleRun", "WSPOracle", "convex_target",
           "gradient", "initial_weights", "run_schedule", "s_global", "step_size",
           "version_floor", "wave_range"]
