"""Seeded input generation: std::mt19937_64 and the reference's uniform01.

The reference draws every random input from ``std::mt19937_64(seed)`` and maps
one 64-bit output to [0, 1) by its top 53 bits (proj/include/negf/synthetic.hpp:
18-20).  This is a vectorised restatement of the published MT19937-64
algorithm (Matsumoto & Nishimura; the C++ standard's parameters), so the same
seed yields bit-identical draws to the C++ generator.
"""
from __future__ import annotations

import numpy as np

_NN, _MM = 312, 156
_MATRIX_A = np.uint64(0xB5026F5AA96619E9)
_UM = np.uint64(0xFFFFFFF80000000)  # upper 33 bits
_LM = np.uint64(0x7FFFFFFF)         # lower 31 bits


class MT19937_64:
    """std::mt19937_64 with block generation (312 words per twist)."""

    def __init__(self, seed: int = 5489):
        mt = np.zeros(_NN, dtype=np.uint64)
        mt[0] = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        f = 6364136223846793005
        prev = int(mt[0])
        for i in range(1, _NN):
            prev = (f * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
            mt[i] = prev
        self._mt = mt
        self._buf = np.empty(0, dtype=np.uint64)
        self._pos = 0

    def _twist(self) -> None:
        mt = self._mt
        um = np.uint64(0xFFFFFFFF80000000)
        lm = np.uint64(0x7FFFFFFF)
        one = np.uint64(1)
        zero = np.uint64(0)
        with np.errstate(over="ignore"):
            # i in [0, NN-MM): uses old mt[i+MM]
            x = (mt[: _NN - _MM] & um) | (mt[1 : _NN - _MM + 1] & lm)
            mt[: _NN - _MM] = mt[_MM:_NN] ^ (x >> one) ^ np.where((x & one) == one, _MATRIX_A, zero)
            # i in [NN-MM, NN-1): uses new mt[i+MM-NN]
            lo, hi = _NN - _MM, _NN - 1
            while lo < hi:  # chunks whose source (i-156) is already final
                end = min(hi, lo + _MM)
                x = (mt[lo:end] & um) | (mt[lo + 1 : end + 1] & lm)
                mt[lo:end] = mt[lo - (_NN - _MM) : end - (_NN - _MM)] ^ (x >> one) ^ np.where(
                    (x & one) == one, _MATRIX_A, zero
                )
                lo = end
            x = (mt[_NN - 1] & um) | (mt[0] & lm)
            mt[_NN - 1] = mt[_MM - 1] ^ (x >> one) ^ (_MATRIX_A if (x & one) == one else zero)
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        self._buf = y
        self._pos = 0

    def next_u64(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        got = 0
        while got < count:
            if self._pos >= len(self._buf):
                self._twist()
            take = min(count - got, len(self._buf) - self._pos)
            out[got : got + take] = self._buf[self._pos : self._pos + take]
            self._pos += take
            got += take
        return out

    def uniform01(self, count: int | None = None):
        """Top 53 bits * 2^-53 (synthetic.hpp:18-20)."""
        c = 1 if count is None else count
        v = (self.next_u64(c) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        return float(v[0]) if count is None else v
