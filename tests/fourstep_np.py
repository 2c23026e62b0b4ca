"""TEST INFRASTRUCTURE (never imported by the product): a NumPy restatement
of the distributed four-step NDCT's rank-local half (fl_fs_* in
include/fastleg_b200.h; kernels fs_* in paper_1505_00354_b200/csrc/fast_ndct.cu)
with the same layouts -- symmetric residue sets on the coefficient side, k2
blocks on the value side, the same exchange buffers -- so that
paper_1505_00354_b200/distributed.py's orchestration (term groups, NCCL-style
all-to-all / reduce-scatter / all-gather) runs over gloo on CPU with the real
collectives and is checked against the oracle's DLT / IDLT.

The arithmetic is the fast-mode NDCT the GPU runs: sum over the Chebyshev
(Jacobi-Anger) expansion terms l of the DCT-III (l even) / DST-III (l odd) of
T_l(n/N) c_n, weighted at output k by the Bessel weight of N delta'_k, with
every term's N/2-point complex FFT (Makhoul packing) split as L1 x L2."""
from __future__ import annotations

import numpy as np
from scipy.special import jv


def weight(l: int, y, swap: int = 0):
    """big_tables_kernel's term weight (fast_ndct.cu): +-eps_l J_l(y)."""
    j = jv(l, y)
    if l % 2 == 0:
        w = (1.0 if l == 0 else 2.0) * (-j if (l >> 1) & 1 else j)
    else:
        w = -2.0 * (-j if ((l - 1) >> 1) & 1 else j)
    return -w if swap and (l & 1) else w


def cheb_t(l: int, x):
    a, b = np.ones_like(x), x
    if l == 0:
        return a
    for _ in range(l - 1):
        a, b = b, 2.0 * x * b - a
    return b


def _tr_value(za, zc, c2, s2, ch, sh):
    ev = 0.5 * (za.real + zc.real) + 0.5j * (za.imag - zc.imag)
    od = 0.5 * (za.imag + zc.imag) - 0.5j * (za.real - zc.real)
    v = ev + od * (c2 + 1j * s2)
    return ch * v.real + sh * v.imag


class FourStepNP:
    """Drop-in for distributed.FourStep on CPU torch tensors."""

    def __init__(self, n: int, world: int, rank: int, delta, mult, terms: int = 14, swap: int = 0):
        L = n // 2
        lg = L.bit_length() - 1
        self.n, self.L = n, L
        self.L1 = 1 << (lg // 2)
        self.L2 = L // self.L1
        if world & (world - 1) or self.L1 < 2 * world:
            raise ValueError("four-step: bad world size")
        self.KB, self.B, self.U = self.L2 // world, n // world, self.L1 // (2 * world)
        self.world, self.rank, self.terms, self.swap = world, rank, terms, swap
        self.delta, self.mult = np.asarray(delta), np.asarray(mult)
        h = self.L1 // (2 * world)
        self.res = []
        for r in range(world):
            js = list(range(r * h, (r + 1) * h))
            lst = js + [self.L1 - j for j in js if j != 0] + ([self.L1 // 2] if r == world - 1 else [])
            self.res.append(np.array(lst, dtype=np.int64))
        self.nres_all = [len(r) for r in self.res]
        self.cum = np.concatenate([[0], np.cumsum(self.nres_all)])
        self.res_max = max(self.nres_all)
        self.owner = np.empty(self.L1, dtype=np.int64)
        self.lidx = np.empty(self.L1, dtype=np.int64)
        for r, lst in enumerate(self.res):
            self.owner[lst] = r
            self.lidx[lst] = np.arange(len(lst))
        self.nres = self.nres_all[rank]
        self.mirror = self.lidx[(self.L1 - self.res[rank]) % self.L1]
        self.slab = self.res_max * 2 * self.L2

    # ---- shared helpers -------------------------------------------------
    def k_of_q(self, q):
        return np.where(q < self.L, 2 * q, 2 * (self.n - 1 - q) + 1)

    def xpos(self, k0, k1, k2l):
        blk = k0 // self.B
        g = k0 & 1
        p0 = np.where(g == 1, self.L - (blk + 1) * (self.B // 4), blk * (self.B // 4))
        u = k1 - p0 // self.L2
        return blk * (self.B // self.world) + ((g * self.U + u) * self.KB + k2l) * 2

    def items(self):
        k1 = np.arange(self.L1)[:, None]
        k2l = np.arange(self.KB)[None, :]
        p = self.rank * self.KB + k2l + self.L2 * k1
        return k1, k2l, p

    def coef_counts(self, transpose: bool, send: bool):
        mine = (not send) if transpose else send
        return [(self.nres if mine else self.nres_all[peer]) * self.KB for peer in range(self.world)]

    def work_elems(self, terms: int) -> int:
        return terms * max(self.nres * self.L2, self.KB * self.L1)

    def groups(self, budget_bytes: int = 12 << 30, min_groups: int = 1):
        from paper_1505_00354_b200.distributed import FourStep
        return FourStep.groups(self, budget_bytes, min_groups)

    def check(self, transpose: bool, dev) -> None:
        return None

    # ---- layouts ---------------------------------------------------------
    def to_residue(self, full):
        import torch
        f = full.numpy()
        J = 2 * self.L2
        out = np.zeros((self.world, self.res_max, J))
        for d, r in enumerate(self.res):
            out[d, :len(r)] = f[r[:, None] + self.L1 * np.arange(J)[None, :]]
        return torch.from_numpy(out.ravel())

    def from_residue(self, slabs):
        import torch
        s = slabs.numpy().reshape(self.world, self.res_max, 2 * self.L2)
        out = np.empty(self.n)
        for d, r in enumerate(self.res):
            out[r[:, None] + self.L1 * np.arange(2 * self.L2)[None, :]] = s[d, :len(r)]
        return torch.from_numpy(out)

    def values(self, to_block: bool, x):
        import torch
        e = np.arange(self.B)
        per = self.B // self.world
        s, rem = e // per, e % per
        b, r2 = rem & 1, rem >> 1
        k2l, r3 = r2 % self.KB, r2 // self.KB
        u, g = r3 % self.U, r3 // self.U
        p0 = np.where(g == 1, self.L - (self.rank + 1) * (self.B // 4), self.rank * (self.B // 4))
        p = s * self.KB + k2l + self.L2 * (p0 // self.L2 + u)
        k = self.k_of_q(2 * p + b) - self.rank * self.B
        xv = x.numpy()
        out = np.empty(self.B)
        if to_block:
            out[k] = xv[e]
        else:
            out[e] = xv[k]
        return torch.from_numpy(out)

    # ---- the two halves of each direction -------------------------------
    def part(self, transpose, part, t0, t1, inp, out, work, first=True):
        nt = t1 - t0
        o = out.numpy()
        if not transpose and part == 1:
            V = self._fwd1(inp.numpy(), t0, t1)                         # [t][i][k2]
            send = V.reshape(nt, self.nres, self.world, self.KB).transpose(2, 0, 1, 3)
            o.view(np.complex128)[:] = send.ravel()
        elif not transpose and part == 2:
            self._fwd2(inp.numpy().view(np.complex128), t0, t1, o, first)
        elif transpose and part == 1:
            o.view(np.complex128)[:] = self._tr1(inp.numpy(), t0, t1)
        else:
            self._tr2(inp.numpy().view(np.complex128), t0, t1, o, first)

    def _fwd1(self, slab, t0, t1):
        J, L1, L2, n, L = 2 * self.L2, self.L1, self.L2, self.n, self.L
        chat = slab[:self.nres * J].reshape(self.nres, J)
        res = self.res[self.rank][:, None]
        m2 = np.arange(L2)[None, :]
        m = res + L1 * m2
        c0, c2 = chat[:, :L2], chat[:, L2:]
        zero = res == 0
        ic = np.where(zero, np.arange(self.nres)[:, None], self.mirror[:, None])
        j1 = np.where(zero, (J - m2) % J, J - 1 - m2)
        j3 = np.where(zero, L2 - m2, L2 - 1 - m2)
        c1 = np.where(m > 0, chat[ic, j1], 0.0)
        c3 = chat[ic, j3]
        xs = [m / n, (n - m) / n, (m + L) / n, (L - m) / n]
        sa, ca = np.sin(np.pi * m / (2 * n)), np.cos(np.pi * m / (2 * n))
        sb, cb = np.sin(np.pi * (m + L) / (2 * n)), np.cos(np.pi * (m + L) / (2 * n))
        tw4 = np.exp(2j * np.pi * m / n)
        k2 = np.arange(L2)[None, :]
        tw = np.exp(2j * np.pi * (res * k2) / L)
        out = []
        for l in range(t0, t1):
            odd = (l & 1) ^ self.swap
            r0, r1, r2, r3 = (cheb_t(l, x) for x in xs)
            st0, st1, st2, st3 = c0 * r0, np.where(m > 0, c1 * r1, 0.0), c2 * r2, c3 * r3
            if odd:
                xa, xan, xb, xbn = np.where(m > 0, 0.5 * st1, 0.0), np.where(m > 0, 0.5 * st0, 0.0), 0.5 * st3, 0.5 * st2
            else:
                xa, xan, xb, xbn = np.where(m > 0, 0.5 * st0, st0), np.where(m > 0, 0.5 * st1, 0.0), 0.5 * st2, 0.5 * st3
            wa = (ca * xa + sa * xan) + 1j * (sa * xa - ca * xan)
            wb = (cb * xb + sb * xbn) + 1j * (sb * xb - cb * xbn)
            z = (wa + wb) + 1j * (wa - wb) * tw4
            out.append(np.fft.ifft(z, axis=1) * L2 * tw)
        return np.stack(out)

    def _fwd2(self, recv, t0, t1, fx, first):
        nt = t1 - t0
        t = np.arange(nt)[:, None, None]
        k2l = np.arange(self.KB)[None, :, None]
        m1 = np.arange(self.L1)[None, None, :]
        s, i = self.owner[m1], self.lidx[m1]
        idx = self.cum[s] * self.KB * nt + (t * np.array(self.nres_all)[s] + i) * self.KB + k2l
        y = np.fft.ifft(recv[idx], axis=2) * self.L1                    # [t][k2l][k1]
        k1, k2l2, p = self.items()
        k0 = self.k_of_q(2 * p)
        acc = np.zeros((2,) + p.shape)
        for tt, l in enumerate(range(t0, t1)):
            odd = (l & 1) ^ self.swap
            yy = y[tt].T                                                  # [k1][k2l]
            for b, comp in ((0, yy.real), (1, yy.imag)):
                k = self.k_of_q(2 * p + b)
                v = np.where((k & 1) == 1, -comp, comp) if odd else comp
                acc[b] += weight(l, self.n * self.delta[k], self.swap) * v
        pos = self.xpos(k0, k1, k2l2)
        for b in range(2):
            if first:
                fx[pos + b] = acc[b]
            else:
                fx[pos + b] += acc[b]

    def _tr1(self, gx, t0, t1):
        nt = t1 - t0
        k1, k2l, p = self.items()
        k0 = self.k_of_q(2 * p)
        pos = self.xpos(k0, k1, k2l)
        gv = [gx[pos] * self.mult[k0], gx[pos + 1] * self.mult[self.k_of_q(2 * p + 1)]]
        m1 = np.arange(self.L1)[:, None]
        k2 = self.rank * self.KB + np.arange(self.KB)[None, :]
        tw = np.exp(-2j * np.pi * (m1 * k2) / self.L)                   # [m1][k2l]
        send = np.empty(nt * sum(self.coef_counts(True, True)), dtype=np.complex128)
        for tt, l in enumerate(range(t0, t1)):
            odd = (l & 1) ^ self.swap
            h = []
            for b in range(2):
                k = self.k_of_q(2 * p + b)
                v = weight(l, self.n * self.delta[k], self.swap) * gv[b]
                h.append(np.where((k & 1) == 1, -v, v) if odd else v)
            rows = (h[0] + 1j * h[1])                                    # [k1][k2l]
            X = np.fft.fft(rows, axis=0) * tw                            # [m1][k2l]
            d = self.owner[np.arange(self.L1)]
            base = self.cum[d] * self.KB * nt + (tt * np.array(self.nres_all)[d] + self.lidx) * self.KB
            send[base[:, None] + np.arange(self.KB)[None, :]] = X
        return send

    def _tr2(self, recv, t0, t1, out, first):
        nt = t1 - t0
        J = 2 * self.L2
        chunk = recv.reshape(self.world, nt, self.nres, self.KB)
        rows = chunk.transpose(1, 2, 0, 3).reshape(nt, self.nres, self.L2)   # k2 = s KB + k2l
        X = np.fft.fft(rows, axis=2)                                     # [t][i][m2]
        res = self.res[self.rank][:, None]
        m2 = np.arange(self.L2)[None, :]
        a = res + self.L1 * m2
        zero = res == 0
        ib = np.where(zero, np.arange(self.nres)[:, None], self.mirror[:, None])
        mb = np.where(zero, (self.L2 - m2) & (self.L2 - 1), self.L2 - 1 - m2)
        rr = [a, self.L + a]
        acc = [np.zeros(a.shape), np.zeros(a.shape)]
        for tt, l in enumerate(range(t0, t1)):
            odd = (l & 1) ^ self.swap
            za, zb = X[tt], X[tt][ib, mb]
            p0, p1 = (zb, za) if odd else (za, zb)
            for q in range(2):
                r = rr[q]
                c2, s2 = np.cos(-2 * np.pi * r / self.n), np.sin(-2 * np.pi * r / self.n)
                ch, sh = np.cos(np.pi * r / (2 * self.n)), np.sin(np.pi * r / (2 * self.n))
                if not odd:
                    x = _tr_value(p0, p1, c2, s2, ch, sh)
                else:
                    x = np.where(r == 0, 0.0, _tr_value(p0, p1, c2, -s2, sh, ch))
                acc[q] += cheb_t(l, r / self.n) * x
        o = out[:self.nres * J].reshape(self.nres, J)
        if first:
            o[:, :self.L2], o[:, self.L2:] = acc[0], acc[1]
        else:
            o[:, :self.L2] += acc[0]
            o[:, self.L2:] += acc[1]
