"""The host engine, controller and emulated kernels under AddressSanitizer:
the emulation library rebuilt with -fsanitize=address and a subset of the
emulation tests re-run in a subprocess with libasan preloaded (compute-sanitizer
is not available on the GPU pool; this covers the host side and the
descriptors' bounds over the emulated buffers)."""
import glob
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _libasan():
    c = sorted(glob.glob("/usr/lib/gcc/x86_64-linux-gnu/*/libasan.so"))
    return c[-1] if c else None


def test_emulation_under_asan():
    asan = _libasan()
    if not asan:
        pytest.skip("libasan not available")
    from emu import build_emu
    lib = build_emu.build(asan=True)
    code = f"""
import sys
sys.path.insert(0, {os.path.dirname(HERE)!r}); sys.path.insert(0, {HERE!r})
import emu.build_emu as be
be.build = lambda asan=False: {lib!r}
import pytest
sys.exit(pytest.main(["-x", "-q", "-p", "no:cacheprovider",
                      {os.path.join(HERE, "test_placement_emu.py")!r},
                      {os.path.join(HERE, "test_transport_emu.py")!r},
                      {os.path.join(HERE, "test_engine_emu.py")!r},
                      "-k", "not random_configs and not replay"]))
"""
    env = dict(os.environ, LD_PRELOAD=asan, ASAN_OPTIONS="detect_leaks=0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "ERROR: AddressSanitizer" not in r.stderr
