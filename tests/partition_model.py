"""Test-only CPU model of one rank's partition steps (the semantics of
egs_part_step, include/egs_gpu.h) in numpy, so the multi-GPU orchestration
(paper_1710_03647_b200/distributed.py) can run under gloo on CPU.  Ids are
the arena's own (the device relabels internally; the orchestration never
looks at ids).  Never used by the product path."""
from __future__ import annotations

import numpy as np
import torch

from paper_1710_03647_b200.distributed import partition_layout

TOP = np.iinfo(np.int64).max
CAND = np.int64(1) << np.int64(62)  # the certificate's candidate mark in f (values < 2^62)


class NumpySteps:
    def __init__(self, off, dst, w, owners, cap, rank, world):
        self.off = np.asarray(off, dtype=np.int64)
        self.dst = np.asarray(dst, dtype=np.int64)
        self.w = np.asarray(w, dtype=np.int64)
        self.p0 = np.asarray(owners) == 0
        self.cap = int(cap)
        self.n = len(self.p0)
        self.slice, self.padded, self.own_lo, self.own_hi = partition_layout(self.n, world, rank)
        self.f = torch.zeros(max(self.padded, 1), dtype=torch.int64)
        self.stage = torch.zeros(max(self.padded, 1), dtype=torch.int64)
        self.chg = [np.zeros(self.n, bool), np.zeros(self.n, bool)]
        self.removed = np.zeros(self.n, bool)  # the last pruning pass's removals
        # sparse exchange buffers: (id, value) entries of 2 int64 words
        self.entry_words = 2
        self.send = torch.zeros(2 * max(self.slice, 1) + 1, dtype=torch.int64)
        self.recv = torch.zeros(2 * max(self.slice, 1) * world + 1, dtype=torch.int64)
        self.world, self.rank = world, rank

    def _ominus(self, ft, w):
        r = np.maximum(ft - w, 0)
        r = np.where(r > self.cap, TOP, r)
        return np.where(ft == TOP, TOP, r)

    @staticmethod
    def _is_cand(x):
        return (x != TOP) & ((x & CAND) != 0)

    def _rows(self):
        lo, hi = self.own_lo, self.own_hi
        return lo, hi, self.off[lo:hi + 1] if hi > lo else None

    def step(self, kind, parity):
        lo, hi, roff = self._rows()
        f = self.f.numpy()
        st = self.stage.numpy()
        chg = self.chg[parity & 1]
        if kind in (0, 1):  # round 1 / lift
            self.chg[(parity & 1) ^ 1][:] = False
            chg[:] = False
            if hi <= lo:
                return 0, 0
            b, e = roff[0], roff[-1]
            if kind == 0:
                ft = np.zeros(e - b, dtype=np.int64)
            else:
                ft = f[self.dst[b:e]]
            c = self._ominus(ft, self.w[b:e])
            seg = roff[:-1] - b
            mn = np.minimum.reduceat(c, seg)
            mx = np.maximum.reduceat(c, seg)
            val = np.where(self.p0[lo:hi], mn, mx)
            old = f[lo:hi] if kind == 1 else np.zeros(hi - lo, dtype=np.int64)
            live = old != TOP
            raised = live & (val > old)
            st[lo:hi][raised] = val[raised]
            chg[lo:hi] = raised
            return int(raised.sum()), 0
        if kind == 2:  # commit
            idx = np.nonzero(chg)[0]
            f[idx] = st[idx]
            return 0, 0
        if kind == 3:  # certificate init: raised, non-top vertices get the mark
            c = chg[lo:hi] & (f[lo:hi] != TOP)
            f[lo:hi][c] |= CAND
            return 0, 0
        if kind == 4:  # one pruning pass (snapshot semantics; same greatest fixpoint)
            if hi <= lo:
                return 0, 0
            b, e = roff[0], roff[-1]
            t = self.dst[b:e]
            ft = f[t]
            src = np.repeat(np.arange(lo, hi), np.diff(roff))
            fv = f[src] & ~CAND
            with np.errstate(over="ignore"):
                good = (ft == TOP) | (self._is_cand(ft) & (fv < (ft & ~CAND) - self.w[b:e]))
            seg = roff[:-1] - b
            allg = np.minimum.reduceat(good.astype(np.int8), seg).astype(bool)
            anyg = np.maximum.reduceat(good.astype(np.int8), seg).astype(bool)
            keep = np.where(self.p0[lo:hi], allg, anyg)
            own = f[lo:hi]
            drop = self._is_cand(own) & ~keep
            own[drop] &= ~CAND
            self.removed[:] = False
            self.removed[lo:hi] = drop
            return 0, int(drop.sum())
        if kind == 5:  # apply
            cand = self._is_cand(f[lo:hi])
            f[lo:hi][cand] = TOP
            chg[lo:hi] |= cand
            return int(cand.sum()), 0
        raise ValueError(kind)

    def pack(self, which, parity):
        lo, hi = self.own_lo, self.own_hi
        marks = self.chg[parity & 1] if which == 0 else self.removed
        ids = np.nonzero(marks[lo:hi])[0] + lo
        buf = self.send.numpy()
        buf[0:2 * len(ids):2] = ids
        buf[1:2 * len(ids):2] = self.f.numpy()[ids]
        return len(ids)

    def unpack(self, counts, stride):
        buf = self.recv.numpy()
        f = self.f.numpy()
        for r, cnt in enumerate(counts):
            if r == self.rank or cnt == 0:
                continue
            seg = buf[2 * r * stride: 2 * r * stride + 2 * cnt]  # stride in entries
            f[seg[0::2]] = seg[1::2]

    def read_measure(self):
        return self.f.numpy()[: self.n].copy()
