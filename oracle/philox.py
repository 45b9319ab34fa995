"""Philox4x32-10 counter-based generator (Salmon et al., SC'11, "Parallel random
numbers: as easy as 1, 2, 3"), written out round by round in numpy uint64.

Stands in for the backward pass output: the paper computes u_p by processing
minibatch p; this build draws g(v,p,i) from a counter so that the
oracle and the CUDA path can each regenerate it without sharing buffers
(reading Z9). Pinned by the Random123 known-answer
vectors in tests/golden/philox_kat.txt.
"""
from __future__ import annotations

import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = 0x9E3779B9
_W1 = 0xBB67AE85
_MASK = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Ten Philox rounds on counter words (c0..c3, uint32 arrays or scalars) with
    key (k0, k1). Returns four uint32 arrays (the output words x0..x3)."""
    x0 = np.asarray(c0, dtype=np.uint64)
    x1 = np.asarray(c1, dtype=np.uint64)
    x2 = np.asarray(c2, dtype=np.uint64)
    x3 = np.asarray(c3, dtype=np.uint64)
    x0, x1, x2, x3 = np.broadcast_arrays(x0, x1, x2, x3)
    key0, key1 = int(k0) & 0xFFFFFFFF, int(k1) & 0xFFFFFFFF
    for rnd in range(10):
        if rnd > 0:                      # bump the key between rounds
            key0 = (key0 + _W0) & 0xFFFFFFFF
            key1 = (key1 + _W1) & 0xFFFFFFFF
        p0 = _M0 * x0                    # 64-bit products of 32-bit words
        p1 = _M1 * x2
        hi0, lo0 = p0 >> _S32, p0 & _MASK
        hi1, lo1 = p1 >> _S32, p1 & _MASK
        x0, x1, x2, x3 = (hi1 ^ x1 ^ np.uint64(key0), lo1,
                          hi0 ^ x3 ^ np.uint64(key1), lo0)
    return tuple(np.asarray(x, dtype=np.uint32) for x in (x0, x1, x2, x3))


def philox_words(idx, vw: int, p: int, stream: int, seed: int) -> np.ndarray:
    """The uint32 draw for each param index in `idx`: Philox4x32-10 with counter
    (i>>2, vw, p, stream) and key (seed lo32, seed hi32); param i takes word i&3."""
    idx = np.asarray(idx, dtype=np.int64)
    blk = (idx >> 2).astype(np.uint64)
    words = philox4x32_10(blk, np.uint64(vw), np.uint64(p), np.uint64(stream),
                          seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    stacked = np.stack(words, axis=0)                       # [4, n]
    return stacked[idx & 3, np.arange(idx.size)]
