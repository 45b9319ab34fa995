"""CPU-side checks of the C-ABI boundary: the library loads, exports every
symbol include/hetpipe.h declares, and its closed forms match the paper's
(pure functions, no GPU needed). Building is __graft_entry__.build()'s job;
these tests build in-tree if the .so is stale."""
import os
import re

import pytest

from oracle import s_global as o_s_global, version_floor as o_floor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2005_14038_b200 import build, hetpipe
    build.build()
    return hetpipe.load()


def _declared():
    text = open(os.path.join(ROOT, "include", "hetpipe.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hp_[a-z_]+)\s*\(", text)))


def test_header_symbols_exported(lib):
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    from paper_2005_14038_b200.hetpipe import EXPORTS
    assert set(EXPORTS) == set(names)


def test_closed_forms_match_paper(lib):
    # P:999 s_global and P:998 floor, including the paper's example P:1001-1002
    assert lib.hp_s_global(4, 0) == 6 and lib.hp_version_floor(11, 4, 0) == 4
    for Nm in range(1, 9):
        for D in range(0, 6):
            assert lib.hp_s_global(Nm, D) == o_s_global(Nm, D)
            for p in range(1, 80):
                assert lib.hp_version_floor(p, Nm, D) == o_floor(p, Nm, D)


def test_init_without_gpu_fails_loudly(lib):
    """No CPU fallback: without a usable device hp_init_ex must return an error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2005_14038_b200 import hetpipe
    from workloads import C1
    with pytest.raises(hetpipe.HetPipeError):
        hetpipe.Context(hetpipe.config_from(C1))


def test_invalid_config_rejected(lib):
    from paper_2005_14038_b200 import hetpipe
    from workloads import C1
    for bad in (dict(num_vw=0), dict(num_vw=9), dict(Nm=0), dict(D=-1), dict(acc_slots=1),
                dict(param_begin=7), dict(param_count=10 ** 9)):
        with pytest.raises(hetpipe.HetPipeError) as e:
            hetpipe.Context(hetpipe.config_from(C1, **bad))
        assert e.value.status == hetpipe.HP_ERR_INVALID


def test_sources_share_nothing_with_oracle():
    """The CUDA path never imports/includes oracle/, and the oracle never
    imports the product package."""
    pkg = os.path.join(ROOT, "paper_2005_14038_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle|#include\s+\S*oracle", src, re.M), f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            src = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(from|import)\s+paper_2005_14038_b200", src, re.M), f


def test_config_layout_matches_library():
    import ctypes
    from paper_2005_14038_b200 import hetpipe
    lib = hetpipe.load()
    assert lib.hp_config_size() == ctypes.sizeof(hetpipe.hp_config)
    assert ctypes.sizeof(hetpipe.hp_stats) >= 8 * 4 + 8 * 16 + 8
