"""TEST DOUBLE of paper_2601_07628_b200.ops.CudaOps on CPU tensors.

Used only by the CPU test suite to exercise the engine's HOST logic (grid
plans, collective ledger, scalar tables, restart/termination decisions,
gloo multi-process runs) without a GPU. It mirrors each C-ABI op's
definition (include/gridlp_b200.h) with numpy/scipy arithmetic in the
reference's order. The package never imports it; the product path has no
CPU implementation.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import torch

from paper_2601_07628_b200.ops import Fused


def _clip(v, lo, hi):
    return np.clip(v, lo, hi)


class HostOps:
    kind = "host"

    def __init__(self, device, capacity, num_slots):
        self.device = device
        self.slots = np.zeros((max(num_slots, 1), 8))
        self.tau = self.sigma = self.gamma = 0.0
        self.k = 0
        self._mats = {}

    def _mat(self, dc):
        key = id(dc)
        hit = self._mats.get(key)
        if hit is None or hit[0] is not dc:
            h = dc.host
            a = sp.csr_matrix((h.val, h.col, h.ptr), shape=(h.num_rows, h.num_cols))
            hit = (dc, a)
            self._mats[key] = hit
        return hit[1]

    def _sums(self, src):
        if isinstance(src, Fused):
            return self._mat(src.mat).dot(src.gather.numpy())
        if not src.parts:
            return np.zeros(src.num_rows)
        acc = src.parts[0].numpy().copy()
        for p in src.parts[1:]:
            acc += p.numpy()
        return acc

    def set_step(self, tau, sigma, gamma, inner_k):
        self.tau, self.sigma, self.gamma, self.k = tau, sigma, gamma, inner_k

    def step_advance(self, delta):
        self.k += delta

    def read_slots(self, n):
        return self.slots[:n].copy()

    def _w(self, it):
        k = self.k + it
        return (1.0 + self.gamma) * (k + 1.0) / (k + 2.0), 1.0 / (k + 2.0)

    def store(self, src, out, slot=None):
        s = self._sums(src)
        out.numpy()[:len(s)] = s        # out may be a padded shard-exchange buffer
        if slot is not None:
            self.slots[slot, 0] = float(np.dot(s, s))

    def primal(self, src, col, it, halpern):
        aty = self._sums(src)
        x = col.x.numpy()
        xh = _clip(x - self.tau * (col.c.numpy() - aty), col.lo.numpy(), col.hi.numpy())
        col.xbar.numpy()[:] = 2.0 * xh - x
        if halpern:
            wm, wa = self._w(it)
            x[:] = (wm * xh - self.gamma * x) + wa * col.x0.numpy()
        else:
            x[:] = xh

    def _dual_map(self, y, z, lo, hi):
        v = y / self.sigma - z
        return self.sigma * (v - np.clip(v, -hi, -lo))

    def dual(self, src, row, it, halpern):
        z = self._sums(src)
        y = row.y.numpy()
        yh = self._dual_map(y, z, row.lo.numpy(), row.hi.numpy())
        if halpern:
            wm, wa = self._w(it)
            y[:] = (wm * yh - self.gamma * y) + wa * row.y0.numpy()
        else:
            y[:] = yh

    def kkt_rows(self, src, row, ax, slot):
        s = self._sums(src)
        if ax is not None:
            ax.numpy()[:] = s
        lo, hi, y = row.lo.numpy(), row.hi.numpy(), row.y.numpy()
        rv = np.maximum(s - hi, 0.0) - np.maximum(lo - s, 0.0)
        pos, neg = np.maximum(-y, 0.0), np.maximum(y, 0.0)
        fu, fl = np.isfinite(hi), np.isfinite(lo)
        bad = np.count_nonzero(pos[~fu] > 0.0) + np.count_nonzero(neg[~fl] > 0.0)
        self.slots[slot, :4] = [float(np.dot(rv, rv)), float(np.dot(hi[fu], pos[fu])),
                                float(np.dot(lo[fl], neg[fl])), float(bad)]

    def kkt_cols(self, src, col, slot):
        aty = self._sums(src)
        x, c = col.x.numpy(), col.c.numpy()
        shifted = x - self.tau * (c - aty)
        xp = np.clip(shifted, col.lo.numpy(), col.hi.numpy())
        rd = (xp - x) / self.tau
        rc = (xp - shifted) / self.tau
        dx = x - xp
        self.slots[slot, :4] = [float(np.dot(rd, rd)), float(np.dot(c, x)), float(np.dot(rc, x)),
                                float(np.dot(dx, dx))]
        col.xpb.numpy()[:] = 2.0 * xp - x

    def probe(self, src, row, ax, dy_out, slot):
        z = self._sums(src)
        y = row.y.numpy()
        yp = self._dual_map(y, z, row.lo.numpy(), row.hi.numpy())
        dy = y - yp
        self.slots[slot, 0] = float(np.dot(dy, dy))
        if ax is not None:
            self.slots[slot, 1] = float(np.dot(0.5 * (ax.numpy() - z), dy))
        if dy_out is not None:
            dy_out.numpy()[:] = dy

    def halfdiff_dot(self, a, b, d, slot):
        self.slots[slot, 0] = float(np.dot(0.5 * (a.numpy() - b.numpy()), d.numpy()))

    def anchor(self, v, anchor, slot):
        e = v.numpy() - anchor.numpy()
        self.slots[slot, 0] = float(np.dot(e, e))
        anchor.numpy()[:] = v.numpy()

    def dot(self, a, b, slot):
        self.slots[slot, 0] = float(np.dot(a.numpy(), b.numpy()))

    def div(self, inp, out, d):
        out.numpy()[:] = inp.numpy() / d

    def init_primal(self, col):
        v = np.clip(np.zeros(col.n), col.lo.numpy(), col.hi.numpy())
        col.x.numpy()[:] = v
        col.x0.numpy()[:] = v


def host_factory(device, capacity, num_slots):
    return HostOps(device, capacity, num_slots)
