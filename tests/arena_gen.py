"""Random small arenas for parity sweeps (test-only)."""
from __future__ import annotations

import random


def random_arena(seed: int, max_n: int = 12, max_deg: int = 4, W: int | None = None):
    """(n, edges, owners): total arena, random owners, row order = draw order.
    Weight ranges vary with the seed so both winning and losing regions,
    zero-weight cycles and long climbs appear."""
    r = random.Random(seed)
    n = r.randint(1, max_n)
    if W is None:
        W = r.choice([1, 2, 3, 10, 100, 1000, 10 ** 6])
    bias = r.choice([0, 0, -1, 1])
    owners = [r.randint(0, 1) for _ in range(n)]
    edges = []
    for v in range(n):
        for _ in range(r.randint(1, max_deg)):
            w = r.randint(-W, W) + bias * r.randint(0, max(1, W // 4))
            edges.append((v, r.randrange(n), w))
    r.shuffle(edges)  # rows keep this (input) order after the stable build
    return n, edges, owners


def chain_arena(length: int, w_cycle: int = -1, exit_w: int = -50):
    """A slow-climb gadget: a player-1 / player-0 two-cycle with weight
    w_cycle per lap and an expensive player-0 exit, repeated `length` times."""
    edges = []
    owners = []
    n = 3 * length
    for k in range(length):
        a, b, safe = 3 * k, 3 * k + 1, 3 * k + 2
        owners += [1, 0, 0]
        edges += [(a, b, w_cycle), (b, a, 0), (b, safe, exit_w), (safe, safe, 0)]
        if k + 1 < length:
            edges.append((safe, 3 * (k + 1), -1))
    return n, edges, owners
