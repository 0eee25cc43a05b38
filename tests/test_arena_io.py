"""Arena input/output of the solve path, host side:
the reference's text format (parse_arena / write_arena, io.cpp:87-176), the
GameArena::build semantics (arena.cpp:17-108) and the binary format.  The
compiled reference (oracle/_ref) is the oracle for texts, errors and spans.
CPU only: no device is touched."""
import os
import random

import numpy as np
import pytest

from arena_gen import random_arena


def _spans(a):
    return (np.asarray(a.csr_offsets, dtype=np.uint64), np.asarray(a.csr_targets, np.uint32),
            np.asarray(a.csr_weights, np.int64), np.asarray(a.owners, np.uint8))


def _same_as_ref(a, ref, r):
    ours = _spans(a)
    theirs = r.csr()  # offsets, targets, weights, owners of the reference's GameArena
    assert all(np.array_equal(x, y) for x, y in zip(ours, theirs))
    assert a.credit_cap == ref.credit_cap(r)


@pytest.mark.parametrize("gen,args", [("fixed", (2000, 4, 100)), ("fixed", (500, 8, 100_000)),
                                      ("rmat", (10, 16, 100))])
def test_write_and_parse_match_reference(egs, reflib, gen, args):
    a = getattr(egs.GameArena, gen)(*args, 1)
    r = getattr(reflib, gen)(*args, 1)
    text = a.write_text()
    assert text == reflib.write_arena(r)  # write_arena, byte for byte
    b = egs.GameArena.parse(text)
    _same_as_ref(b, reflib, r)
    assert b.write_text() == text


def test_parse_unsorted_edges_is_stable_like_build(egs, reflib):
    """Edges in any order: rows keep input order (the stable counting sort of
    GameArena::build)."""
    for seed in range(20):
        n, edges, owners = random_arena(seed, max_n=30, max_deg=5)
        random.Random(seed).shuffle(edges)
        lines = [f"eg {n} {len(edges)}"] + [f"v {v} {owners[v]}" for v in range(n)]
        lines += [f"e {s} {d} {w}" for s, d, w in edges]
        text = ("\n".join(lines) + "\n").encode()
        r, err = reflib.parse_arena(text)
        assert err is None
        a = egs.GameArena.parse(text)
        _same_as_ref(a, reflib, r)
        b = egs.GameArena.build(n, edges, owners)
        assert all(np.array_equal(x, y) for x, y in zip(_spans(a), _spans(b)))


def test_parse_comments_blank_lines_crlf(egs, reflib):
    text = b"# an arena\n\neg 2 3\r\nv 0 0\n# c\nv 1 1\n\ne 0 1 -3\ne 1 0 2\r\ne 1 1 -1\n"
    r, err = reflib.parse_arena(text)
    assert err is None
    _same_as_ref(egs.GameArena.parse(text), reflib, r)


BAD_TEXTS = [
    b"",
    b"# nothing\n",
    b"eg 2\n",
    b"eg  2 1\n",
    b"eg x 1\n",
    b"eg 2 -1\n",
    b"eg 2 1\nv 0 0\n",
    b"eg 2 1\nv 0 0\nv 2 1\ne 0 1 1\n",
    b"eg 2 1\nv 0 0\nv 1 2\ne 0 1 1\n",
    b"eg 2 1\nv 0 0\ne 0 1 1\n",
    b"eg 2 2\nv 0 0\nv 1 1\ne 0 1 1\n",
    b"eg 2 1\nv 0 0\nv 1 1\ne 0 1 1\ne 1 0 1\n",
    b"eg 2 2\nv 0 0\nv 1 1\ne 0 1 1\ne 1 5 1\n",
    b"eg 2 2\nv 0 0\nv 1 1\ne 0 1 1\ne 1 99999999999 1\n",
    b"eg 2 1\nv 0 0\nv 1 1\ne 0 1 1\n",
    b"eg 2 2\nv 0 0\nv 1 1\ne 0 1 1\ne 1 0 x\n",
    b"eg 2 2\nv 0 0\nv 1 1\ne 0 1 1\ne 1 0 1 1\n",
    b"eg 2 2\nv 0 0\nv 1 1\ne 0 1 1\ne 1 0 -9223372036854775808\n",
    b"eg 1 1\nv 0 0\ne 0 0 9223372036854775807\n",
]


@pytest.mark.parametrize("text", BAD_TEXTS, ids=range(len(BAD_TEXTS)))
def test_parse_errors_match_reference(egs, reflib, text):
    r, err = reflib.parse_arena(text)
    assert r is None, "fixture must be rejected by the reference"
    kind, _, msg = err.partition(": ")
    with pytest.raises(egs.EgsolveError) as ei:
        egs.GameArena.parse(text)
    want = {"SyntaxError": egs.SyntaxError_, "CountMismatchError": egs.CountMismatchError,
            "DanglingVertexIdError": egs.DanglingVertexIdError,
            "NonTotalArenaError": egs.NonTotalArenaError,
            "OverflowError": egs.OverflowError_}[kind]
    assert type(ei.value) is want, (err, repr(ei.value))
    assert str(ei.value) == msg


def test_parse_multithreaded_matches_reference(egs, reflib):
    """A text above the threading threshold (4 MiB): chunks split at line
    boundaries, the first error in file order wins."""
    a = egs.GameArena.fixed(60_000, 8, 1000, 3)
    text = a.write_text().encode()
    assert len(text) > (1 << 22)
    b = egs.GameArena.parse(text)
    assert all(np.array_equal(x, y) for x, y in zip(_spans(a), _spans(b)))
    lines = text.split(b"\n")
    bad = list(lines)
    bad[len(lines) // 2] = b"e 1 2"  # a syntax error in a middle chunk ...
    bad[len(lines) - 10] = b"e x 2 3"  # ... and a later one
    bt = b"\n".join(bad)
    r, err = reflib.parse_arena(bt)
    with pytest.raises(egs.SyntaxError_) as ei:
        egs.GameArena.parse(bt)
    assert r is None and str(ei.value) == err.partition(": ")[2]


@pytest.mark.parametrize("W", [100, 1000, 100_000, 3_000_000_000])
def test_binary_round_trip(egs, tmp_path, W):
    a = egs.GameArena.fixed(3000, 4, W, 7)
    p = str(tmp_path / "a.egb")
    a.save(p)
    b = egs.GameArena.load(p)
    assert all(np.array_equal(x, y) for x, y in zip(_spans(a), _spans(b)))
    assert (b.credit_cap, b.max_abs_weight) == (a.credit_cap, a.max_abs_weight)
    wb = 1 if W <= 127 else 2 if W <= 32767 else 4 if W < 2 ** 31 else 8
    n, m = a.num_vertices, a.num_edges
    pad = lambda x: (x + 7) // 8 * 8  # noqa: E731
    assert os.path.getsize(p) == 64 + pad(n) + pad((n + 1) * 8) + pad(m * 4) + pad(m * wb)
    assert b.write_text() == a.write_text()


def test_binary_rejects_corruption(egs, tmp_path):
    a = egs.GameArena.fixed(500, 4, 100, 1)
    p = str(tmp_path / "a.egb")
    a.save(p)
    raw = bytearray(open(p, "rb").read())
    n = a.num_vertices

    def load(buf):
        q = str(tmp_path / "b.egb")
        open(q, "wb").write(bytes(buf))
        return egs.GameArena.load(q)

    with pytest.raises(egs.InputError):
        load(raw[:-8])  # truncated
    bad = bytearray(raw)
    bad[0:8] = b"NOTARENA"
    with pytest.raises(egs.InputError):
        load(bad)
    bad = bytearray(raw)
    bad[32] ^= 1  # credit_cap in the header
    with pytest.raises(egs.InputError):
        load(bad)
    tgt0 = 64 + (n + 7) // 8 * 8 + (n + 1) * 8
    bad = bytearray(raw)
    bad[tgt0:tgt0 + 4] = (n + 5).to_bytes(4, "little")  # a dangling target
    with pytest.raises(egs.DanglingVertexIdError):
        load(bad)
    with pytest.raises(egs.InputError):
        egs.GameArena.load(str(tmp_path / "missing.egb"))


def test_build_errors(egs):
    with pytest.raises(egs.NonTotalArenaError):
        egs.GameArena.build(3, [(0, 1, 1), (1, 0, 1)], [0, 1, 0])
    with pytest.raises(egs.DanglingVertexIdError):
        egs.GameArena.build(2, [(0, 2, 1), (1, 0, 1)], [0, 1])
    with pytest.raises(egs.CountMismatchError):
        egs.GameArena.build(2, [(0, 1, 1), (1, 0, 1)], [0])
