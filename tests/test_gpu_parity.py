"""Parity of the CUDA path against the oracle and the compiled reference.

Every case goes through the C-ABI (egs_gpu_solve / egs_ctx_*) and is compared
bit-for-bit with the reference's least progress measure and byte-for-byte
with its write_solution text."""
import hashlib

import numpy as np
import pytest

from arena_gen import chain_arena, random_arena
from oracle_bindings import INT64_MAX, fnv1a64

pytestmark = pytest.mark.gpu

MODES = ["auto", "dense", "sparse", "sweep"]


def _opts(egs, **kw):
    return egs.SolverOptions(**kw)


def _solve(egs, a, **kw):
    return egs.solve(a, options=_opts(egs, **kw))


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("certify", [True, False])
def test_spec_fixtures(egs, golden, mode, certify):
    for key, rec in golden.items():
        if not key.startswith("spec/"):
            continue
        a = egs.GameArena.build(rec["n"], [tuple(e) for e in rec["edges"]], rec["owners"])
        rep = _solve(egs, a, mode=mode, certify=certify)
        assert egs.write_solution(a, rep) == rec["solution"], key


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("certify", [True, False])
def test_random_small_arenas(egs, oracle, mode, certify):
    for seed in range(150):
        n, edges, owners = random_arena(seed, max_n=16, max_deg=5)
        a = egs.GameArena.build(n, edges, owners)
        g = oracle.build(n, edges, owners)
        want, _ = oracle.solve_seq(g)
        rep = _solve(egs, a, mode=mode, certify=certify, cert_interval=1)
        assert np.array_equal(rep.measure, want), (seed, mode, certify)
        assert egs.write_solution(a, rep) == oracle.write_solution(g, want)
        assert np.array_equal(rep.w1, np.nonzero(want == INT64_MAX)[0])


def test_random_medium_arenas_all_lane_widths(egs, oracle):
    # average degree 1..40 exercises lanes 1, 2, 4, 8, 16, 32
    for seed, deg in enumerate([1, 2, 3, 5, 9, 17, 40]):
        n, edges, owners = random_arena(1000 + seed, max_n=300, max_deg=2 * deg - 1, W=50)
        a = egs.GameArena.build(n, edges, owners)
        g = oracle.build(n, edges, owners)
        want, _ = oracle.solve_seq(g)
        for mode in MODES:
            rep = _solve(egs, a, mode=mode)
            assert np.array_equal(rep.measure, want), (seed, deg, mode)


def test_slow_climb_gadget(egs, oracle):
    n, edges, owners = chain_arena(20, w_cycle=-1, exit_w=-300)
    a = egs.GameArena.build(n, edges, owners)
    g = oracle.build(n, edges, owners)
    want, _ = oracle.solve_seq(g)
    for certify in (True, False):
        rep = _solve(egs, a, certify=certify)
        assert np.array_equal(rep.measure, want)


def test_heavy_rows(egs, oracle):
    # hubs longer than the heavy threshold take the CTA-per-row kernel
    import random
    r = random.Random(5)
    n = 3000
    owners = [v & 1 for v in range(n)]
    edges = []
    for v in range(n):
        deg = 5000 if v in (0, 1, 7, 8) else r.randint(1, 3)
        for _ in range(deg):
            edges.append((v, r.randrange(n), r.randint(-100, 100)))
    a = egs.GameArena.build(n, edges, owners)
    g = oracle.build(n, edges, owners)
    want, _ = oracle.solve_sweep(g)
    for mode in MODES:
        rep = _solve(egs, a, mode=mode)
        assert np.array_equal(rep.measure, want), mode


GOLDEN_SMALL = [
    ("fixed/10000/4/100/1", lambda e: e.GameArena.fixed(10000, 4, 100, 1)),
    ("fixed/1000/8/1000/1", lambda e: e.GameArena.fixed(1000, 8, 1000, 1)),
    ("fixed/1000/8/100000/1", lambda e: e.GameArena.fixed(1000, 8, 100000, 1)),
    ("fixed/2000/16/100/1", lambda e: e.GameArena.fixed(2000, 16, 100, 1)),
    ("fixed/3000/2/50/1", lambda e: e.GameArena.fixed(3000, 2, 50, 1)),
    ("rmat/12/16/100/1", lambda e: e.GameArena.rmat(12, 16, 100, 1)),
    ("rmat/14/16/100/1", lambda e: e.GameArena.rmat(14, 16, 100, 1)),
]


@pytest.mark.parametrize("key,make", GOLDEN_SMALL, ids=[k for k, _ in GOLDEN_SMALL])
def test_device_write_solution_golden(egs, golden, key, make):
    """egs_ctx_write_solution (device strategy + formatting) reproduces the
    reference's write_solution bytes."""
    rec = golden[key]
    with egs.DeviceSolver(make(egs)) as ds:
        ds.solve()
        sol = ds.write_solution().encode()
    assert (len(sol), f"{fnv1a64(sol):016x}") == (rec["solution_bytes"], rec["solution_fnv"])


def test_device_write_solution_spec_and_random(egs, golden, oracle):
    for key, rec in golden.items():
        if key.startswith("spec/"):
            a = egs.GameArena.build(rec["n"], [tuple(e) for e in rec["edges"]], rec["owners"])
            with egs.DeviceSolver(a) as ds:
                ds.solve()
                assert ds.write_solution() == rec["solution"], key
    for seed in range(60):
        n, edges, owners = random_arena(7000 + seed, max_n=40, max_deg=5)
        a = egs.GameArena.build(n, edges, owners)
        g = oracle.build(n, edges, owners)
        want, _ = oracle.solve_seq(g)
        with egs.DeviceSolver(a) as ds:
            ds.solve()
            assert ds.write_solution() == oracle.write_solution(g, want), seed


@pytest.mark.parametrize("key,make", GOLDEN_SMALL, ids=[k for k, _ in GOLDEN_SMALL])
@pytest.mark.parametrize("mode", MODES)
def test_canonical_golden_small(egs, golden, key, make, mode):
    rec = golden[key]
    a = make(egs)
    rep = _solve(egs, a, mode=mode)
    sol = egs.write_solution(a, rep).encode()
    assert (len(sol), f"{fnv1a64(sol):016x}") == (rec["solution_bytes"], rec["solution_fnv"])
    assert int((rep.measure == INT64_MAX).sum()) == rec["tops"]


def test_c1_plain_value_iteration_matches(egs, golden):
    """certify=False runs the reference's own iteration to credit_cap."""
    rec = golden["fixed/10000/4/100/1"]
    a = egs.GameArena.fixed(10000, 4, 100, 1)
    rep = _solve(egs, a, certify=False)
    sol = egs.write_solution(a, rep).encode()
    assert f"{fnv1a64(sol):016x}" == rec["solution_fnv"]
    assert rep.gpu["certified"] == 0
    assert rep.rounds > 1000  # the top climb to M_G really ran


GOLDEN_BIG = [
    ("fixed/100000/4/100/1", (100000, 4, 100)),
    ("fixed/100000/8/1000/1", (100000, 8, 1000)),
    ("fixed/100000/16/100/1", (100000, 16, 100)),
    ("fixed/100000/8/100000/1", (100000, 8, 100000)),
]


@pytest.mark.parametrize("key,args", GOLDEN_BIG, ids=[k for k, _ in GOLDEN_BIG])
def test_canonical_golden_1e5(egs, golden, key, args):
    if key not in golden:
        pytest.skip("golden vector not generated")
    rec = golden[key]
    a = egs.GameArena.fixed(*args, 1)
    rep = _solve(egs, a)
    sol = egs.write_solution(a, rep).encode()
    assert f"{fnv1a64(sol):016x}" == rec["solution_fnv"]
    assert rep.gpu["value_bits"] == (64 if rec["credit_cap"] >= 2 ** 31 - 1 else 32)


def test_rmat16_golden(egs, golden):
    key = "rmat/16/16/100/1"
    if key not in golden:
        pytest.skip("golden vector not generated")
    a = egs.GameArena.rmat(16, 16, 100, 1)
    rep = _solve(egs, a)
    sol = egs.write_solution(a, rep).encode()
    assert f"{fnv1a64(sol):016x}" == golden[key]["solution_fnv"]


GOLDEN_FULL = [
    ("fixed/1000000/8/1000/1", ("fixed", (1_000_000, 8, 1000))),      # C2
    ("fixed/1000000/8/100000/1", ("fixed", (1_000_000, 8, 100_000))),  # C5
    ("fixed/1000000/16/100/1", ("fixed", (1_000_000, 16, 100))),      # F16: C4's generator at 10^6
    ("rmat/22/16/100/1", ("rmat", (22, 16, 100))),                    # C3
    ("fixed/16000000/16/100/1", ("fixed", (16_000_000, 16, 100))),    # C4
]


@pytest.mark.parametrize("key,spec", GOLDEN_FULL, ids=["C2", "C5", "F16", "C3", "C4"])
def test_full_size_golden(egs, golden, key, spec):
    """BASELINE configs at full size, bit-exact against digests computed
    WITHOUT the certificate: the reference solve_sweep run to its fixpoint
    (C2, C5, F16, C3: tests/golden/make_golden_full.py, "ref_rounds") and
    the GPU's plain value iteration run to its fixpoint
    (tests/golden/make_golden_plain.py; "plain_gpu": C2, F16, C3 -- the same
    bytes as the reference -- and C4, "pin": "plain_gpu", 1.9 million
    in-place sweeps).  Compared: the device output path's write_solution
    bytes (SHA-256, length), the host formatter's bytes, tops and finite sum."""
    if key not in golden:
        pytest.skip("full-size golden vector not generated")
    rec = golden[key]
    kind, args = spec
    a = getattr(egs.GameArena, kind)(*args, 1)
    with egs.DeviceSolver(a) as ds:
        ds.solve()
        dev_text = ds.write_solution().encode()
        f = ds.read_measure()
    host_text = egs.write_solution(a, f).encode()
    digest = hashlib.sha256(dev_text).hexdigest()
    assert len(dev_text) == rec["solution_bytes"]
    assert digest == rec["solution_sha256"]
    if "plain_gpu" in rec:  # both pins agree where both exist
        assert digest == rec["plain_gpu"]["solution_sha256"]
    assert host_text == dev_text
    top = f == np.iinfo(np.int64).max
    assert int(top.sum()) == rec["tops"]
    assert int(f[~top].sum()) == rec["sum_finite"]


@pytest.mark.parametrize("tma_mask", ["0", "7"])
@pytest.mark.parametrize("cert_div", ["0.001", "1000"])
def test_schedule_knobs_give_identical_bytes(egs, golden, oracle, monkeypatch, tma_mask,
                                            cert_div):
    """Every light-row phase staged by TMA (mask 7) or read with plain loads
    (mask 0); certificate passes all dense (div 0.001) or sparse after the
    first (div 1000: mark, then push-style re-check queues).  The bytes must
    not move: golden vectors of the reference and random arenas vs the oracle."""
    monkeypatch.setenv("EGS_TMA_MASK", tma_mask)
    monkeypatch.setenv("EGS_CERT_SPARSE_DIV", cert_div)
    for key, make in [("rmat/16/16/100/1", lambda: egs.GameArena.rmat(16, 16, 100, 1)),
                      ("fixed/100000/16/100/1", lambda: egs.GameArena.fixed(100000, 16, 100, 1)),
                      ("fixed/10000/4/100/1", lambda: egs.GameArena.fixed(10000, 4, 100, 1))]:
        if key not in golden:
            continue
        a = make()
        for mode in MODES:
            rep = _solve(egs, a, mode=mode)
            sol = egs.write_solution(a, rep).encode()
            assert f"{fnv1a64(sol):016x}" == golden[key]["solution_fnv"], (key, mode)
    for seed in range(40):
        n, edges, owners = random_arena(7000 + seed, max_n=200, max_deg=40, W=60)
        a = egs.GameArena.build(n, edges, owners)
        g = oracle.build(n, edges, owners)
        want, _ = oracle.solve_seq(g)
        assert np.array_equal(_solve(egs, a, cert_interval=1).measure, want), seed


def test_value_width_boundary(egs, oracle):
    # credit_cap = 2^31 - 2 stays on the u32 path, 2^31 - 1 takes u64 (u32
    # reserves 2^32 - 1 for top and the top bit for the certificate's mark);
    # 2^32 - 2 is the old boundary, now deep in the u64 range
    for cap in (2 ** 31 - 2, 2 ** 31 - 1, 2 ** 32 - 3, 2 ** 32 - 2):
        x = [cap // 3, cap // 3, cap - 2 * (cap // 3)]
        edges = [(0, 1, -x[0]), (1, 2, -x[1]), (2, 0, -x[2]), (0, 0, 3), (1, 1, 1),
                 (2, 2, 0), (2, 1, 7)]
        owners = [1, 0, 1]
        a = egs.GameArena.build(3, edges, owners)
        assert a.credit_cap == cap
        g = oracle.build(3, edges, owners)
        want, _ = oracle.solve_seq(g)
        rep = _solve(egs, a)
        assert np.array_equal(rep.measure, want)
        assert rep.gpu["value_bits"] == (32 if cap < 2 ** 31 - 1 else 64)


def test_device_context_reuse_and_epm(egs, oracle):
    a = egs.GameArena.fixed(5000, 8, 1000, 3)
    g = oracle.fixed(5000, 8, 1000, 3)
    want, _ = oracle.solve_sweep(g)
    with egs.DeviceSolver(a) as ds:
        for _ in range(3):
            ds.solve()
            assert np.array_equal(ds.read_measure(), want)
        assert ds.is_progress_measure(want)
        bad = want.copy()
        fin = np.nonzero(bad != INT64_MAX)[0]
        bad[fin[bad[fin].argmax()]] = 0
        assert ds.is_progress_measure(bad) == oracle.is_progress_measure(g, bad)


def test_round_bound_and_timeout(egs):
    a = egs.GameArena.fixed(10000, 4, 100, 1)
    with pytest.raises(egs.BoundExhaustedError):
        _solve(egs, a, certify=False, sweep_bound=10)
    # plain value iteration on C1 climbs ~10^4 rounds; a 1 ms budget stops it
    # on the device (%globaltimer) with the reference's TimeoutError
    with pytest.raises(egs.TimeoutError_):
        _solve(egs, a, certify=False, timeout_seconds=0.001)
    # a context survives a failed solve: the next solve starts clean
    with egs.DeviceSolver(a, egs.SolverOptions(certify=False, sweep_bound=3)) as ds:
        for _ in range(2):
            with pytest.raises(egs.BoundExhaustedError):
                ds.solve()
    with egs.DeviceSolver(a) as ds:
        ds.solve()
        assert ds.is_fixpoint(ds.read_measure())


def test_sweep_bound_zero_and_debug_checks(egs, oracle):
    """sweep_bound keeps the reference's optional semantics (solver_par.cpp:
    149-150,184-188): 0 fails after the first round that raises something and
    passes an arena already at its fixpoint.  debug_checks (the reference's
    check_monotone plus a fixpoint check of the result) passes on every
    schedule and changes nothing."""
    a = egs.GameArena.fixed(10000, 4, 100, 1)
    with pytest.raises(egs.BoundExhaustedError):
        _solve(egs, a, sweep_bound=0)
    calm = egs.GameArena.build(4, [(0, 1, 3), (1, 2, 0), (2, 3, 5), (3, 0, 1)], [0, 1, 0, 1])
    assert _solve(egs, calm, sweep_bound=0).measure.tolist() == [0, 0, 0, 0]
    for seed in range(40):
        n, edges, owners = random_arena(7000 + seed, max_n=40, max_deg=6)
        b = egs.GameArena.build(n, edges, owners)
        want, _ = oracle.solve_seq(oracle.build(n, edges, owners))
        for mode in MODES:
            for certify in (True, False):
                rep = _solve(egs, b, mode=mode, certify=certify, debug_checks=True)
                assert np.array_equal(rep.measure, want), (seed, mode, certify)
    base = _solve(egs, a).measure
    assert np.array_equal(_solve(egs, a, debug_checks=True).measure, base)


def test_weight_width_paths(egs, oracle):
    """Weights travel as int8 / int16 / int32 by max |w|; every width gives
    the reference's measure, and a weight beyond int32 is refused loudly."""
    import random
    for W in (100, 127, 128, 30000, 32768, 10 ** 6, 2 ** 31 - 1):
        r = random.Random(W)
        n = 200
        edges = [(v, r.randrange(n), r.randint(-W, W)) for v in range(n) for _ in range(3)]
        edges.append((0, 1, W))
        owners = [v & 1 for v in range(n)]
        a = egs.GameArena.build(n, edges, owners)
        assert a.max_abs_weight == W
        g = oracle.build(n, edges, owners)
        want, _ = oracle.solve_seq(g)
        assert np.array_equal(_solve(egs, a).measure, want), W
    big = egs.GameArena.build(2, [(0, 1, -(2 ** 31)), (1, 0, 5)], [0, 1])
    with pytest.raises(egs.OverflowError_):
        _solve(egs, big)


def _bits(n):
    b = 1
    while (1 << b) < n:
        b += 1
    return b


@pytest.mark.parametrize("forced_wide", [False, True])
def test_edge_record_formats(egs, oracle, monkeypatch, forced_wide):
    """Packed 4-byte records (dst | w << tb) hold every id < n in tb bits and
    weights up to 2^(31-tb) - 1; one more and the arena takes 8-byte records.
    Vertex counts at and just past powers of two, weights at the limit."""
    import random
    if forced_wide:
        monkeypatch.setenv("EGS_EDGE_FORMAT", "8")
    for n in (2, 3, 16, 17, 32, 33, 255, 256, 257, 1025):
        tb = _bits(n)
        lim = (1 << (31 - tb)) - 1
        for W, packed in ((lim, True), (lim + 1, False)):
            r = random.Random(n * 7 + packed)
            edges = [(v, r.randrange(n), r.randint(-W, W)) for v in range(n) for _ in range(3)]
            edges += [(0, n - 1, -W), (n - 1, 0, W)]
            owners = [r.randint(0, 1) for _ in range(n)]
            a = egs.GameArena.build(n, edges, owners)
            g = oracle.build(n, edges, owners)
            want, _ = oracle.solve_seq(g)
            with egs.DeviceSolver(a) as ds:
                want_bytes = 4 if packed and not forced_wide else 8
                assert ds.upload_stats.edge_bytes == want_bytes, (n, W)
                ds.solve()
                got = ds.read_measure()
                assert np.array_equal(got, want), (n, W, forced_wide)
                assert ds.is_fixpoint(got)
            for mode in MODES:
                rep = _solve(egs, a, mode=mode)
                assert np.array_equal(rep.measure, want), (n, W, mode, forced_wide)
                assert egs.write_solution(a, rep) == oracle.write_solution(g, want)


def test_empty_and_single_vertex(egs):
    a = egs.GameArena.build(0, [], [])
    rep = _solve(egs, a)
    assert rep.measure.shape == (0,)
    a = egs.GameArena.build(1, [(0, 0, -7)], [1])
    assert _solve(egs, a).measure.tolist() == [INT64_MAX]


def test_fixpoint_check_small(egs, oracle):
    """The device fixpoint check accepts the reference's least measure and
    rejects perturbations of it (it backs the full-size tests below)."""
    for seed in range(40):
        n, edges, owners = random_arena(3000 + seed, max_n=30, max_deg=5)
        a = egs.GameArena.build(n, edges, owners)
        g = oracle.build(n, edges, owners)
        want, _ = oracle.solve_seq(g)
        with egs.DeviceSolver(a) as ds:
            assert ds.is_fixpoint(want)
            fin = np.nonzero((want != INT64_MAX) & (want > 0))[0]
            if fin.size:
                bad = want.copy()
                bad[fin[0]] -= 1
                assert not ds.is_fixpoint(bad)


FULL = [("C4", ("fixed", (16_000_000, 16, 100))), ("C3", ("rmat", (22, 16, 100))),
        ("C2", ("fixed", (1_000_000, 8, 1000))), ("C5", ("fixed", (1_000_000, 8, 100_000)))]


@pytest.mark.parametrize("name,spec", FULL, ids=[n for n, _ in FULL])
def test_full_size_configs_properties(egs, name, spec):
    """Full BASELINE configs, where the CPU reference cannot finish (C4 ~4
    days projected): the result is a fixpoint of the capped lift and a
    progress measure (device checks), and every schedule -- auto, dense,
    sparse, a late certificate -- gives the identical measure."""
    kind, args = spec
    a = getattr(egs.GameArena, kind)(*args, 1)
    base = None
    for opts in [dict(), dict(mode="dense"), dict(mode="sparse"), dict(cert_interval=7)]:
        with egs.DeviceSolver(a, egs.SolverOptions(**opts)) as ds:
            ds.solve()
            f = ds.read_measure()
            if base is None:
                base = f
                assert ds.is_fixpoint(f)
                assert ds.is_progress_measure(f)
                tops = int((f == INT64_MAX).sum())
                assert 0 < tops < a.num_vertices
                # device output path == host output path, byte for byte
                assert ds.write_solution() == egs.write_solution(a, f)
            else:
                assert np.array_equal(f, base), opts


TRANSPOSE_ARENAS = [lambda e: e.GameArena.fixed(100000, 16, 100, 1),
                    lambda e: e.GameArena.rmat(14, 16, 100, 1),
                    lambda e: e.GameArena.rmat(16, 8, 1000, 3),   # hubs spanning merge blocks
                    lambda e: e.GameArena.fixed(3000, 1, 10, 2)]


@pytest.mark.parametrize("make", TRANSPOSE_ARENAS, ids=["fixed-1e5-16", "rmat14", "rmat16", "fixed-d1"])
def test_transpose_builds_agree(egs, monkeypatch, make):
    """The predecessor transpose built chunk by chunk during the upload
    (EGS_CSC_SORT=inc, the default for >= 2^27 edges: per-chunk sort, rank,
    merge -- egs_build.cuh k_csc_*), by one library sort at the end
    (EGS_CSC_SORT=end, the default below) and by the hand-written LSD radix
    sort (EGS_CSC_SORT=radix, egs_scan.cuh) holds exactly the arena's edges
    (debug_checks: an order-free CSR/CSC fingerprint) and gives the identical
    measure.  (Round counts may differ: a column's source order sets the
    order of a sparse round's in-place lifts, hence how much it raises and
    the next round's dense / sparse choice -- rmat16 takes 6 or 7 dense
    rounds.)"""
    a = make(egs)
    out = {}
    for mode in ("radix", "end", "inc", "default"):
        if mode == "default":
            monkeypatch.delenv("EGS_CSC_SORT", raising=False)
        else:
            monkeypatch.setenv("EGS_CSC_SORT", mode)
        with egs.DeviceSolver(a, egs.SolverOptions(debug_checks=True)) as ds:
            st = ds.solve()
            out[mode] = (ds.read_measure(), st.rounds, st.dense_rounds)
    for mode in ("radix", "end", "inc"):
        assert np.array_equal(out[mode][0], out["default"][0]), mode


def test_concurrent_one_shot_solves(egs):
    """One-shot solves from several host threads at once (ctypes releases the
    GIL): the upload's narrowing helpers and the read-back's widening threads
    come from one process-wide pool (egs_pool.h), and a caller that finds it
    busy runs threads of its own -- every result equals the sequential one.
    Arenas large enough (>= 2^20 vertices) for the pooled paths."""
    import threading
    arenas = [egs.GameArena.fixed(1_100_000, 8, 100, s) for s in (1, 2, 3)]
    want = [egs.solve(a).measure for a in arenas]
    got = [None] * len(arenas)
    errs = []

    def run(i):
        try:
            for _ in range(3):
                got[i] = egs.solve(arenas[i]).measure
        except BaseException as e:  # noqa: BLE001 -- reported below
            errs.append(e)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(arenas))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errs, errs
    for w, g in zip(want, got):
        assert np.array_equal(w, g)
