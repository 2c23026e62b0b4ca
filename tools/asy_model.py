"""Cost model of the asymptotic-expansion Legendre->Chebyshev conversion
(Hale & Townsend 2014, the fast leg2cheb the paper cites)
against the Toeplitz-Hankel form this library runs for N >= 2^14
(development tool).

The expansion: P_n(cos t) = C_n sum_{m<M} h_{m,n} cos((n+m+1/2) t - (m+1/2) pi/2)
/ (2 sin t)^{m+1/2} + R, |R| <= C_n h_{M,n} 2 / (2 sin t)^{M+1/2}, with
C_n = (4/pi) prod_{j<=n} j/(j+1/2), h_{m,n} = prod_{j<=m} (j-1/2)^2/(j(n+j+1/2)).
Degrees are grouped in levels nu_0 < nu_1 < ... (ratio R); at level l the
expansion (for all n >= nu_l) is accurate to eps on |sin t| >= S_l; each level
costs 2M length-N transforms (a DCT-III and a DST-III per term, masked to
n >= nu_l: a transform over all n would multiply the FFT rounding of the
low degrees by (2 sin t)^{-(m+1/2)}), and every point t_j needs the
recurrence for the degrees below its level's cutoff.

  python tools/asy_model.py            # the table in DESIGN.md
  python tools/asy_model.py --check N  # accuracy of a NumPy evaluation vs the oracle
"""
import sys

import numpy as np
from scipy.special import gammaln


def levels(N, M=10, R=8, eps=2.0 ** -54):
    def logC(n):
        return np.log(4 / np.pi) + gammaln(n + 1) + gammaln(1.5) - gammaln(n + 1.5)

    def logh(m, n):
        return sum(np.log((j - 0.5) ** 2 / (j * (n + j + 0.5))) for j in range(1, m + 1))

    def smin(nu):
        return 0.5 * np.exp((np.log(2) + logC(nu) + logh(M, nu) - np.log(eps)) / (M + 0.5))

    nus, nu = [], 8
    while nu < N:
        if smin(nu) < 1:
            nus.append(nu)
        nu = nu * R if nus else nu + 8
    return nus, [smin(v) for v in nus]


def model(N, M, R):
    nus, S = levels(N, M, R)
    th = (np.arange(N // 2) + 0.5) * np.pi / N
    s = np.sin(th)
    lev = np.full(N // 2, len(nus))
    for l in range(len(nus) - 1, -1, -1):
        lev[s >= S[l]] = l
    nuj = np.array([nus[l] if l < len(nus) else N for l in lev])
    full = int((lev == len(nus)).sum() * 2)
    return len(nus), 2 * M * len(nus), 2 * nuj.sum() / N, full


def check(N, M=10, R=8):
    """NumPy evaluation (values at the cheb1 points by levels + the recurrence
    in y = 2 sin^2(t/2), then the scaled DCT-II) against the oracle's M c."""
    sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
    import scipy.fft as sf
    from oracle import ORACLE as O
    nus, S = levels(N, M, R)
    c = O.random_decaying(N, 0.5, 3)
    lam = O.lambda_table(N)
    n = np.arange(N)
    Cn = 2.0 / (np.sqrt(np.pi) * (n + 1) * lam[1:])
    th = (n + 0.5) * np.pi / N
    s = np.sin(th)
    lev = np.full(N, len(nus))
    for l in range(len(nus) - 1, -1, -1):
        lev[s >= S[l]] = l
    nuj = np.array([nus[l] if l < len(nus) else N for l in lev])
    f = np.zeros(N)
    for l, nu in enumerate(nus):
        pts = lev == l
        h, acc = np.ones(N), np.zeros(N)
        for m in range(M):
            if m:
                h = h * (m - 0.5) ** 2 / (m * (n + m + 0.5))
            u = np.where(n >= nu, c * Cn * h, 0.0)
            dc = sf.dct(np.concatenate([[u[0]], 0.5 * u[1:]]), type=3)
            ds = sf.dst(np.concatenate([0.5 * u[1:], [0.0]]), type=3)
            ph = (m + 0.5) * (th - np.pi / 2)
            acc += (np.cos(ph) * dc - np.sin(ph) * ds) / (2 * s) ** (m + 0.5)
        f[pts] += acc[pts]
    flip = th > np.pi / 2
    t = np.where(flip, np.pi - th, th)
    y = 2 * np.sin(t / 2) ** 2
    sg = np.where(flip, -1.0, 1.0)
    acc = np.where(nuj > 0, c[0], 0.0) + np.where(nuj > 1, c[1] * (1 - y) * sg, 0.0)
    P, d = 1 - y, -y
    for k in range(1, nuj.max() - 1):
        d = (k * d - (2 * k + 1) * y * P) / (k + 1)
        P = P + d
        acc += np.where(nuj > k + 1, c[k + 1] * P * sg ** (k + 1), 0.0)
    f += acc
    chat = sf.dct(f, type=2) / N
    chat[0] *= 0.5
    return np.max(np.abs(chat - O.leg2cheb(c))) / np.abs(c).sum()


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--check":
        print(f"max |asy - oracle| / ||c||_1 = {check(int(sys.argv[2])):.2e}")
    else:
        print("N      M  R  levels  length-N transforms  recurrence steps/N  full-recurrence points")
        for N in (2 ** 20, 2 ** 26):
            for M, R in ((10, 8), (14, 4), (18, 8)):
                lv, tr, rec, full = model(N, M, R)
                print(f"2^{int(np.log2(N)):<4d} {M:2d} {R:2d} {lv:6d} {tr:20d} {rec:19.0f} {full:23d}")
