"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/egs_gpu.h declares, its host-side pieces (canonical generators, the
reference output format, GameArena::build mirror) agree bit-for-bit with the
oracle, and the solve path fails loudly instead of falling back to the CPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from arena_gen import random_arena
from oracle_bindings import ROOT

HEADER = os.path.join(ROOT, "include", "egs_gpu.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(egs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(egs):
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(egs.lib, name), name
    assert egs.lib.egs_version().startswith(b"egs_b200")


def test_library_is_sm100a_only(egs):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {egs.lib_path} 2>&1").read()
    assert "sm_100a" in out
    assert "sm_90" not in out


@pytest.mark.parametrize("args", [(10000, 4, 100, 1), (1000, 8, 100000, 1), (777, 3, 5, 42),
                                  (200000, 16, 100, 1)])
def test_fixed_generator_matches_oracle(egs, oracle, args):
    a = egs.GameArena.fixed(*args)
    g = oracle.fixed(*args)
    off, dst, w, own = g.csr()
    assert np.array_equal(a.csr_offsets, off)
    assert np.array_equal(a.csr_targets, dst)
    assert np.array_equal(a.csr_weights, w)
    assert np.array_equal(a.owners, own)
    assert a.credit_cap == g.a.credit_cap
    assert a.max_abs_weight == g.a.max_abs_weight


@pytest.mark.parametrize("args", [(10, 16, 100, 1), (14, 16, 100, 1), (12, 4, 7, 9)])
def test_rmat_generator_matches_oracle(egs, oracle, args):
    a = egs.GameArena.rmat(*args)
    g = oracle.rmat(*args)
    off, dst, w, own = g.csr()
    assert np.array_equal(a.csr_offsets, off)
    assert np.array_equal(a.csr_targets, dst)
    assert np.array_equal(a.csr_weights, w)
    assert np.array_equal(a.owners, own)
    assert a.credit_cap == g.a.credit_cap


def test_write_solution_matches_oracle(egs, oracle, golden):
    for key, rec in golden.items():
        if key.startswith("spec/"):
            edges = [tuple(e) for e in rec["edges"]]
            a = egs.GameArena.build(rec["n"], edges, rec["owners"])
            g = oracle.build(rec["n"], edges, rec["owners"])
            f, _ = oracle.solve_seq(g)
            assert egs.write_solution(a, f) == rec["solution"]
    a = egs.GameArena.fixed(10000, 4, 100, 1)
    g = oracle.fixed(10000, 4, 100, 1)
    f, _ = oracle.solve_sweep(g)
    assert egs.write_solution(a, f) == oracle.write_solution(g, f)


def test_python_build_matches_oracle(egs, oracle):
    for seed in range(100):
        n, edges, owners = random_arena(seed)
        a = egs.GameArena.build(n, edges, owners)
        g = oracle.build(n, edges, owners)
        off, dst, w, own = g.csr()
        assert np.array_equal(a.csr_offsets, off)
        assert np.array_equal(a.csr_targets, dst)
        assert np.array_equal(a.csr_weights, w)
        assert a.credit_cap == g.a.credit_cap


def test_build_rejects_non_total_and_dangling(egs):
    with pytest.raises(egs.EgsolveError):
        egs.GameArena.build(2, [(0, 1, 1)], [0, 1])
    with pytest.raises(egs.EgsolveError):
        egs.GameArena.build(1, [(0, 3, 1)], [0])
    with pytest.raises(egs.EgsolveError):
        egs.GameArena.build(2, [(0, 1, 1), (1, 0, 1)], [0])


def test_invalid_options_rejected_before_device(egs):
    a = egs.GameArena.build(2, [(0, 1, -1), (1, 0, 1)], [0, 1])
    with pytest.raises(egs.InvalidConfigError):
        egs.solve(a, options=egs.SolverOptions(mode="bogus"))
    with pytest.raises(egs.InvalidConfigError):
        egs.solve(a, options=egs.SolverOptions(workers=0))
    with pytest.raises(egs.InvalidConfigError):
        egs.solve(a, variant=egs.Variant.SWEEP)


def test_wide_weights_are_unsupported_not_wrong(egs):
    a = egs.GameArena.build(1, [(0, 0, -(2 ** 40))], [0])
    with pytest.raises(egs.OverflowError_):
        egs.solve(a)


def test_no_cpu_fallback_without_device(egs):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a CUDA device is present")
    except ImportError:
        pass
    a = egs.GameArena.build(2, [(0, 1, -1), (1, 0, 1)], [0, 1])
    with pytest.raises(egs.CudaError):
        egs.solve(a)
