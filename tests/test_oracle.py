"""Pin the C restatement (oracle/) against the reference: the published
splitmix64 stream, the SPEC fixtures, the compiled reference library
(oracle/_ref) and the golden vectors it produced (tests/golden/golden.json)."""
import ctypes as C

import numpy as np
import pytest

from arena_gen import chain_arena, random_arena
from oracle_bindings import INT64_MAX, fnv1a64


def test_splitmix64_seed0_stream(oracle):
    # proj/include/egsolve/rng.hpp:9-10
    s = C.c_uint64(0)
    got = [oracle.L.eo_splitmix64_next(C.byref(s)) for _ in range(3)]
    assert got == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


@pytest.mark.parametrize("solver", ["seq", "sweep", "frontier"])
def test_spec_fixtures(oracle, golden, solver):
    for key, rec in golden.items():
        if not key.startswith("spec/"):
            continue
        g = oracle.build(rec["n"], [tuple(e) for e in rec["edges"]], rec["owners"])
        f, _ = getattr(oracle, f"solve_{solver}")(g)
        assert oracle.write_solution(g, f) == rec["solution"], key


def test_spec_choose_chunk_examples():
    # bit_floor(clamp(llround(avg), 1, 64))
    def choose(avg):
        r = max(1, min(64, int(np.floor(avg + 0.5))))
        return 1 << (r.bit_length() - 1)
    assert [choose(2.76), choose(1.16), choose(6.14)] == [2, 1, 4]


SMALL_KEYS = [
    "fixed/10000/4/100/1", "fixed/1000/8/1000/1", "fixed/1000/8/100000/1",
    "fixed/2000/16/100/1", "fixed/3000/2/50/1", "rmat/12/16/100/1", "rmat/14/16/100/1",
]


def _gen(oracle, key):
    kind, a, b, W, seed = key.split("/")
    a, b, W, seed = int(a), int(b), int(W), int(seed)
    return oracle.fixed(a, b, W, seed) if kind == "fixed" else oracle.rmat(a, b, W, seed)


@pytest.mark.parametrize("key", SMALL_KEYS)
def test_oracle_matches_reference_golden(oracle, golden, key):
    rec = golden[key]
    g = _gen(oracle, key)
    arena_txt = oracle.write_arena(g).encode()
    assert (len(arena_txt), f"{fnv1a64(arena_txt):016x}") == (rec["arena_bytes"], rec["arena_fnv"])
    assert int(g.a.credit_cap) == rec["credit_cap"]
    f, st = oracle.solve_sweep(g)
    sol = oracle.write_solution(g, f).encode()
    assert (len(sol), f"{fnv1a64(sol):016x}") == (rec["solution_bytes"], rec["solution_fnv"])
    assert int((f == INT64_MAX).sum()) == rec["tops"]
    if key == "fixed/10000/4/100/1":
        assert st["rounds"] == rec["ref_rounds"] == 4508  # same in-order sweep


@pytest.mark.parametrize("key", [
    "fixed/100000/4/100/1", "fixed/100000/8/1000/1", "fixed/100000/16/100/1",
    "fixed/100000/8/100000/1", "rmat/16/16/100/1"])
def test_oracle_generators_match_big_golden(oracle, golden, key):
    if key not in golden:
        pytest.skip("big golden vectors not generated yet")
    rec = golden[key]
    g = _gen(oracle, key)
    txt = oracle.write_arena(g).encode()
    assert f"{fnv1a64(txt):016x}" == rec["arena_fnv"]
    assert int(g.a.credit_cap) == rec["credit_cap"]


def test_oracle_vs_compiled_reference_random(oracle, reflib):
    for seed in range(300):
        n, edges, owners = random_arena(seed)
        g = oracle.build(n, edges, owners)
        a = reflib.build(n, edges, owners)
        fr, _, _ = reflib.solve(a, reflib.SEQ)
        want = reflib.write_solution(a, fr)
        for solver in ("seq", "sweep", "frontier"):
            f, _ = getattr(oracle, f"solve_{solver}")(g)
            assert np.array_equal(f, fr), (seed, solver)
            assert oracle.write_solution(g, f) == want, (seed, solver)
        assert oracle.is_progress_measure(g, fr)


def test_oracle_vs_compiled_reference_generators(oracle, reflib):
    for args in [(50, 3, 5), (200, 2, 1000), (500, 8, 100000)]:
        g = oracle.fixed(*args, 7)
        a = reflib.fixed(*args, 7)
        assert oracle.write_arena(g) == reflib.write_arena(a)
        f, _ = oracle.solve_seq(g)
        fr, _, _ = reflib.solve(a, reflib.SWEEP, workers=2)
        assert np.array_equal(f, fr)
    g = oracle.rmat(10, 8, 100, 3)
    a = reflib.rmat(10, 8, 100, 3)
    assert oracle.write_arena(g) == reflib.write_arena(a)


def test_oracle_slow_climb_gadget(oracle, reflib):
    n, edges, owners = chain_arena(6)
    g = oracle.build(n, edges, owners)
    a = reflib.build(n, edges, owners)
    f, _ = oracle.solve_seq(g)
    fr, _, _ = reflib.solve(a, reflib.SEQ)
    assert np.array_equal(f, fr)
    assert (f[f != INT64_MAX] > 40).any()  # the climb reaches the exit cost


@pytest.mark.parametrize("key", ["fixed/1000000/8/1000/1", "fixed/1000000/8/100000/1"])
def test_full_size_golden_is_this_generator(oracle, golden, key):
    """The full-size C2/C5 golden records (tests/golden/make_golden_full.py,
    the reference run to its fixpoint) describe the canonical generator's
    arena: same size and credit_cap as the oracle's restatement builds."""
    if key not in golden:
        pytest.skip("full-size golden vectors not generated")
    rec = golden[key]
    g = _gen(oracle, key)
    assert (g.n, g.m, int(g.a.credit_cap)) == (rec["n"], rec["m"], rec["credit_cap"])
    assert rec["solution_bytes"] > 0 and len(rec["solution_sha256"]) == 64
