"""Generates the committed golden fixtures under tests/golden/ (run HERE, in the
build container, where /root/reference exists; the fixtures travel, the
reference does not).

* ref_vectors.json -- outputs of the UNMODIFIED reference headers, compiled in
  place by oracle/Makefile (oracle/_ref/libfastleg_ref.so), on small seeded
  inputs: nodes/weights, the four trig ops, NDCT forward/transpose, leg2cheb,
  DLT/IDLT (TransformConfig's own Newton grid). Stored as float.hex.
* nodes_truth.json -- Gauss-Legendre nodes/weights to 40 digits (mpmath Newton
  on the three-term recurrence), sampled k, for pinning the node kernel.

Usage: python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import REF, CHEB1, CHEBSTAR  # noqa: E402

EPS = 2.0 ** -52


def hx(a) -> list[str]:
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def ref_vectors() -> dict:
    assert REF is not None, "build oracle/_ref first (make -C oracle)"
    out: dict = {"source": "oracle/_ref/libfastleg_ref.so (reference headers compiled in place)"}
    nodes = {}
    for n in (1, 2, 3, 5, 8, 16, 17, 64, 100, 257):
        th, x, w = REF.nodes_weights(n)
        nodes[str(n)] = {"theta": hx(th), "x": hx(x), "w": hx(w)}
    out["nodes"] = nodes
    trig = []
    for n in (1, 2, 3, 4, 7, 13, 32, 64, 100):
        c = REF.random_decaying(n, 0.0, 100 + n)
        for kind in (CHEB1, CHEBSTAR):
            for op in range(4):
                trig.append({"n": n, "kind": kind, "op": op, "seed": 100 + n, "in": hx(c),
                             "out": hx(REF.trig(op, c, kind))})
    out["trig"] = trig
    ndct = []
    for n in (8, 13, 64, 256):
        th, x, w = REF.nodes_weights(n)
        c = REF.random_decaying(n, 1.0, 7 + n)
        for kind in (CHEB1, CHEBSTAR):
            for tol in (2.0 ** -23, EPS):
                L = REF.min_taylor_terms(kind, tol)
                from oracle import ORACLE
                delta = ORACLE.reference_delta(n, kind, th)
                ndct.append({"n": n, "kind": kind, "tol": tol, "L": L, "theta": hx(th),
                             "delta": hx(delta), "in": hx(c),
                             "fwd": hx(REF.ndct(c, kind, L, delta, False)),
                             "tr": hx(REF.ndct(c, kind, L, delta, True))})
    out["ndct"] = ndct
    l2c = []
    for n in (1, 2, 5, 16, 33, 128):
        c = REF.random_decaying(n, 0.5, 200 + n)
        l2c.append({"n": n, "in": hx(c), "fwd": hx(REF.leg2cheb(c, False)),
                    "tr": hx(REF.leg2cheb(c, True))})
    out["leg2cheb"] = l2c
    out["lambda"] = hx(REF.lambda_table(64))
    tr = []
    for n in (1, 2, 8, 64, 256):
        th, x, w = REF.nodes_weights(n)
        c = REF.random_decaying(n, 1.0, 42)
        for kind in (CHEB1, CHEBSTAR):
            f = REF.dlt_grid(c, kind, EPS, th, x, w)
            g = REF.idlt_grid(f, kind, EPS, th, x, w)
            tr.append({"n": n, "kind": kind, "theta": hx(th), "x": hx(x), "w": hx(w), "c": hx(c),
                       "f": hx(f), "back": hx(g)})
    out["transforms"] = tr
    return out


def nodes_truth() -> dict:
    import mpmath as mp
    mp.mp.dps = 40

    def pn(n, x):
        p0, p1 = mp.mpf(1), x
        for j in range(1, n):
            p0, p1 = p1, ((2 * j + 1) * x * p1 - j * p0) / (j + 1)
        return p1, p0

    def root(n, k):
        t = mp.mpf(k + 0.75) * mp.pi / (n + 0.5)
        for _ in range(60):
            x = mp.cos(t)
            p, q = pn(n, x)
            dp = n * (x * p - q) / mp.sin(t)
            step = p / dp
            t -= step
            if abs(step) < mp.mpf(10) ** -38:
                break
        x = mp.cos(t)
        p, q = pn(n, x)
        dp = n * (x * p - q) / mp.sin(t)
        return t, 2 / dp ** 2

    out = {}
    for n in (1, 2, 3, 5, 8, 16, 17, 64, 100, 129, 130, 257, 1000, 4096):
        ks = sorted(set(list(range(min(12, n // 2))) + [n // 4, max(n // 2 - 1, 0)]))
        ks = [k for k in ks if k < (n + 1) // 2]
        rows = []
        for k in ks:
            if n % 2 == 1 and k == (n - 1) // 2:
                t = mp.pi / 2
                _, p_prev = pn(n, mp.mpf(0))  # P_{n-1}(0)
                w = 2 / (n * p_prev) ** 2 if n > 1 else mp.mpf(2)
            else:
                t, w = root(n, k)
            rows.append({"k": k, "theta": mp.nstr(t, 36), "w": mp.nstr(w, 36)})
        out[str(n)] = rows
    return {"source": "mpmath 40-digit Newton on the three-term recurrence", "nodes": out}


if __name__ == "__main__":
    with open(os.path.join(HERE, "ref_vectors.json"), "w") as f:
        json.dump(ref_vectors(), f)
    with open(os.path.join(HERE, "nodes_truth.json"), "w") as f:
        json.dump(nodes_truth(), f, indent=0)
    print("wrote", os.listdir(HERE))
