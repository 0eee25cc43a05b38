"""Host narrowing of the int64 edge weights to the upload width
(csrc/egs_narrow.cpp; AVX-512 on hosts that have it, scalar otherwise):
truncation and the |w| <= wmax range check against numpy, on every length
mod the vector width and at the range's edges.  CPU only."""
import ctypes as C

import numpy as np
import pytest

WIDTHS = [(np.int8, "_Z22egs_internal_narrow_i8PKlPaml"),
          (np.int16, "_Z23egs_internal_narrow_i16PKlPsml"),
          (np.int32, "_Z23egs_internal_narrow_i32PKlPiml")]


@pytest.fixture(scope="module")
def lib(egs):
    return egs._native.lib


@pytest.mark.parametrize("dt,sym", WIDTHS, ids=["i8", "i16", "i32"])
def test_narrow_matches_numpy(lib, dt, sym):
    fn = getattr(lib, sym)
    fn.restype = C.c_bool
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int64]
    rng = np.random.default_rng(5)
    wmax = int(np.iinfo(dt).max)
    for count in list(range(0, 40)) + [1000, 4099, 1 << 16]:
        for case in ("in", "edge", "over", "under"):
            w = rng.integers(-wmax, wmax + 1, size=count, dtype=np.int64)
            if count and case == "edge":
                w[rng.integers(count)] = wmax
                w[rng.integers(count)] = -wmax
            if count and case == "over":
                w[rng.integers(count)] = wmax + 1
            if count and case == "under":
                w[rng.integers(count)] = -wmax - 1 - int(rng.integers(1 << 40))
            out = np.zeros(count + 8, dtype=dt)  # guard past the end
            bad = fn(w.ctypes.data, out.ctypes.data, count, wmax)
            want_bad = bool(count) and bool((np.abs(w) > wmax).any())
            assert bad == want_bad, (count, case)
            assert np.array_equal(out[:count], w.astype(dt)), (count, case)
            assert not out[count:].any(), "wrote past the end"
        # an output not aligned to the vector store width (scalar head)
        for shift in (1, 3, 7):
            w = rng.integers(-wmax, wmax + 1, size=count, dtype=np.int64)
            buf = np.zeros(count + 16, dtype=dt)
            assert not fn(w.ctypes.data, buf[shift:].ctypes.data, count, wmax)
            assert np.array_equal(buf[shift:shift + count], w.astype(dt)), (count, shift)
            assert not buf[:shift].any() and not buf[shift + count:].any()
        # a tighter bound than the type's (packed records: 31 - tbits bits)
        w = np.full(max(count, 1), 100, dtype=np.int64)
        assert not fn(w.ctypes.data, np.zeros(w.size, dt).ctypes.data, w.size, 100)
        assert fn(w.ctypes.data, np.zeros(w.size, dt).ctypes.data, w.size, 99)


def test_widen_matches_numpy(lib):
    """The measure's 32-bit device values back to the raw int64 encoding
    (top = all ones -> INT64_MAX, energy.hpp:16)."""
    fn = lib._Z22egs_internal_widen_u32PKjPlm
    fn.restype = None
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    rng = np.random.default_rng(9)
    for count in list(range(0, 40)) + [1000, 4099, 1 << 16]:
        x = rng.integers(0, 1 << 31, size=count, dtype=np.uint32)
        x[rng.random(count) < 0.3] = 0xFFFFFFFF
        out = np.full(count + 4, 7, dtype=np.int64)
        fn(x.ctypes.data, out.ctypes.data, count)
        want = np.where(x == 0xFFFFFFFF, np.int64(2 ** 63 - 1), x.astype(np.int64))
        assert np.array_equal(out[:count], want), count
        assert (out[count:] == 7).all(), "wrote past the end"
