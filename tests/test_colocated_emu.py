"""Co-located ranks without NCCL on the host emulation: G ranks as threads of
one process, every arena caller-owned, connected by hp_connect_symmetric with
comm_id NULL (include/hetpipe.h) -- the same harness tests/test_gpu_colocated.py
runs on one B200. Checks the connect path itself (first flag barrier, refused
combinations) and parity of the exchange against the oracle."""
import numpy as np
import pytest

from placement_check import check, host_gradients, run_colocated
from workloads import C3, C5, GRAD_EXTERNAL, WSPConfig


@pytest.fixture(scope="module")
def emu():
    from emu import build_emu
    from paper_2005_14038_b200 import hetpipe
    return hetpipe, hetpipe.load_test_library(build_emu.build())


def host_alloc(nbytes):
    buf = np.zeros(nbytes + 256, dtype=np.uint8)
    addr = buf.ctypes.data
    return addr + (-addr) % 256, buf


CASES = [
    ("C3-G2-k1", C3.replace(nparams=4099, waves=5), 2, 1, {}),
    ("C3-G4-k2", C3.replace(nparams=4099, waves=5), 4, 2, {}),
    ("C5-G4-mom", C5.replace(nparams=3001, waves=3, D=4, num_vw=4, tau=C5.tau[:4]), 4, 1, {}),
    ("convexF", WSPConfig("cf", 3, 2, 1, 2053, 4, (3, 5, 4), grad_mode=3, lr=0.05, F=2), 3, 1, {}),
    ("split-F2", WSPConfig("sf", 3, 2, 1, 1030, 4, (3, 7, 4), F=2), 2, 1, {"split": "1"}),
    ("barriers", C3.replace(nparams=4099, waves=5), 4, 1, {"HP_P2P": "0"}),
    ("thm1", WSPConfig("t1", 3, 2, 1, 2053, 6, (3, 5, 4), lr=0.2, lr_schedule=1,
                       grad_mode=3), 3, 2, {}),
    ("reader-F3", WSPConfig("r3", 4, 1, 0, 333, 4, (3, 9, 4, 8), momentum=0.9, F=3), 3, 2,
     {"HP_PULL_PUSH": "0"}),
]


@pytest.mark.parametrize("name,cfg,G,k,env", CASES, ids=[c[0] for c in CASES])
def test_colocated_emu_parity(emu, monkeypatch, name, cfg, G, k, env):
    hetpipe, lib = emu
    if env.get("split"):
        monkeypatch.setenv("HP_SPLIT_FOLDS", "1")
    for k_, v_ in env.items():
        if k_.startswith("HP_"):
            monkeypatch.setenv(k_, v_)
    out = run_colocated(hetpipe, cfg, G, k, host_alloc, lib=lib, timeout=120)
    check(cfg, G, k, out)


def test_colocated_emu_external(emu):
    hetpipe, lib = emu
    cfg = C3.replace(nparams=2048, waves=3, D=1)
    out = run_colocated(hetpipe, cfg, 2, 1, host_alloc, lib=lib, grad_mode=GRAD_EXTERNAL,
                        host_grads=host_gradients(cfg), timeout=120)
    check(cfg, 2, 1, out)


def test_colocated_refuses_nccl_transport_and_nccl_barrier(emu, monkeypatch):
    hetpipe, lib = emu
    cfg = C3.replace(nparams=1024, waves=2)
    c = hetpipe.config_from(cfg, world=2, rank=0, vw_span=1, transport=hetpipe.XPORT_NCCL)
    addr, keep = host_alloc(hetpipe.arena_bytes(c, lib))
    c.arena = addr
    ctx = hetpipe.Context(c, lib=lib)
    with pytest.raises(hetpipe.HetPipeError, match="HP_ERR_STATE"):
        ctx.connect_symmetric([addr, addr + 256], 0, None)
    ctx.close()
    monkeypatch.setenv("HP_FLAG_BARRIER", "0")
    c = hetpipe.config_from(cfg, world=2, rank=0, vw_span=1)
    addr, keep = host_alloc(hetpipe.arena_bytes(c, lib))
    c.arena = addr
    ctx = hetpipe.Context(c, lib=lib)
    with pytest.raises(hetpipe.HetPipeError, match="HP_ERR_STATE"):
        ctx.connect_symmetric([addr, addr + 256], 0, None)
    ctx.close()
    del keep
