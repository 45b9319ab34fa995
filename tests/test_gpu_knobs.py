"""The tick kernel's scheduling knobs change no arithmetic.

Each knob is read once per process (a static in the engine), so every setting
runs the bit-exact random-config parity cases of test_gpu_parity.py in its own
pytest subprocess: the static grid stride (HP_DYN=0), no L2 prefetch
(HP_PREFETCH=0), dynamic tiles on every launch incl. the one-stream ones
(HP_DYN_MINLOADS=1), and non-persistent grids under dynamic tiles (HP_GRID=1).
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KNOBS = [
    {"HP_DYN": "0"},
    {"HP_PREFETCH": "0"},
    {"HP_DYN_MINLOADS": "1"},
    {"HP_DYN_MINLOADS": "1", "HP_GRID": "1"},
]


@pytest.mark.gpu
@pytest.mark.parametrize("knobs", KNOBS, ids=lambda k: "_".join(f"{a}={b}" for a, b in k.items()))
def test_parity_under_knob(knobs):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ, **knobs)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        "-k", "random_configs or convex_random or update_frequency_random"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
