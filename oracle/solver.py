"""CPU restatement of the ChebFD driver -- TEST INFRASTRUCTURE ONLY.

Restates /root/reference/proj/src/solver.cpp (svqb_orthonormalize :32-61,
rayleigh_ritz :63-91, solve :93-214) and src/spectral.cpp (lanczos_bounds
:96-154, kpm_dos :156-205, ChebSeriesDensity::count :46-57) on top of the
C oracle's kernels (chebfd_oracle.c) with numpy.linalg.eigh in place of
Eigen's SelfAdjointEigenSolver.  Eigenvectors are only defined up to a
unitary rotation inside (near-)degenerate eigenspaces, so Ritz VALUES,
residuals, iteration counts and accept/ghost decisions are what this
restatement pins (against the compiled reference: tests/test_oracle_solver.py).
Small problems only (the C oracle is single-threaded).
"""
from __future__ import annotations

import math

import numpy as np

from . import CSR, Oracle


def _sym(g):
    return 0.5 * (g + g.conj().T)


def svqb(orc: Oracle, y, drop_tol=1e-14):
    """solver.cpp:32-61 -> (q, rank)"""
    if y.shape[1] < 1:
        raise ValueError("svqb: empty block")
    g = _sym(orc.gram(y, y))
    lam, v = np.linalg.eigh(g)
    lmax, trace = lam[-1], lam.sum()
    if lam[0] < -1e-12 * max(trace, 0.0):
        raise RuntimeError("svqb: Gram matrix indefinite, corrupted input")
    keep = [i for i in range(len(lam)) if lam[i] > drop_tol * lmax and lam[i] > 0.0]
    if not keep:
        raise RuntimeError("svqb: block numerically zero")
    c = v[:, keep] / np.sqrt(lam[keep])[None, :]
    return orc.block_mult_small(y, np.ascontiguousarray(c, dtype=y.dtype)), len(keep)


def rayleigh_ritz(orc: Oracle, a: CSR, q):
    """solver.cpp:63-91 -> (values, vectors, residual_norms)"""
    aq = orc.spmmvm(a, q, 1.0, 0.0)
    vals, z = np.linalg.eigh(_sym(orc.gram(q, aq)))
    z = np.ascontiguousarray(z, dtype=q.dtype)
    v = orc.block_mult_small(q, z)
    av = orc.block_mult_small(aq, z)
    av -= v * vals[None, :]
    return vals, v, orc.column_norms(av)


def lanczos_bounds(orc: Oracle, a: CSR, iters=30, seed=1):
    """spectral.cpp:96-154"""
    if iters < 2:
        raise ValueError("lanczos_bounds: iters must be >= 2")
    d = a.dim
    m = min(iters, d)
    cx = a.kind == 1
    for restart in range(4):
        v = orc.randomize(d, 1, seed + 977 * restart, cx)
        v /= orc.column_norms(v)[0]
        basis, al, be = [], [], []
        breakdown = False
        for j in range(m):
            basis.append(v)
            w = orc.spmmvm(a, v, 1.0, 0.0)
            for pas in range(2):
                for qi, q in enumerate(basis):
                    h = orc.column_dots(q, w)[0]
                    w = w - h * q
                    if pas == 0 and qi == len(basis) - 1:
                        al.append(float(np.real(h)))
            b_j = orc.column_norms(w)[0]
            if j + 1 == m or len(basis) == d:
                break
            if b_j < 1e-14:
                breakdown = True
                break
            be.append(b_j)
            v = w / b_j
        if breakdown and len(al) < 2 and restart < 3:
            continue
        if not al:
            continue
        k = len(al)
        t = np.diag(al) + (np.diag(be[:k - 1], 1) + np.diag(be[:k - 1], -1) if k > 1 else 0)
        ev = np.linalg.eigvalsh(t)
        rmin, rmax = ev.min(), ev.max()
        pad = 0.01 * (rmax - rmin) + 1e-12 * (1.0 + abs(rmin) + abs(rmax))
        return rmin - pad, rmax + pad
    raise RuntimeError("lanczos_bounds: repeated breakdown")


def kpm_dos(orc: Oracle, a: CSR, bounds, order, samples, seed=1):
    """spectral.cpp:156-205 -> raw moments mu[0..order]"""
    d = a.dim
    alpha = 2.0 / (bounds[1] - bounds[0])
    beta = (bounds[0] + bounds[1]) / (bounds[0] - bounds[1])
    z = orc.randomize(d, samples, seed, a.kind == 1)
    z /= orc.column_norms(z)[None, :]
    scale = d / samples
    mu = np.zeros(order + 1)
    mu[0] = d

    def acc(n, w):
        s = 0.0
        for v in orc.column_dots(z, w):
            s += float(np.real(v))
        mu[n] = scale * s
        if not math.isfinite(mu[n]) or abs(mu[n]) > 4.0 * d:
            raise RuntimeError("kpm_dos: moment growth indicates spectrum outside bounds")

    u = orc.spmmvm(a, z, alpha, beta)
    acc(1, u)
    w = z.copy()
    orc.recurrence_step(a, u, w, alpha, beta)
    acc(2, w)
    pu, pw = u, w
    for n in range(3, order + 1):
        pu, pw = pw, pu
        orc.recurrence_step(a, pu, pw, alpha, beta)
        acc(n, pw)
        if n % 128 == 0 and np.any(~np.isfinite(orc.column_norms(pw)) | (orc.column_norms(pw) > 4)):
            raise RuntimeError("kpm_dos: recurrence growth, bounds violated")
    return mu


def dos_count(orc: Oracle, mu, bounds, lo, hi):
    """ChebSeriesDensity::count (spectral.cpp:46-57), Jackson damping."""
    if hi < lo:
        return -dos_count(orc, mu, bounds, hi, lo)
    order = len(mu) - 1
    g = orc.kernel_coeffs("jackson", max(order, 1))
    damped = g[:order + 1] * mu
    alpha = 2.0 / (bounds[1] - bounds[0])
    beta = (bounds[0] + bounds[1]) / (bounds[0] - bounds[1])
    th = lambda l: math.acos(min(1.0, max(-1.0, alpha * l + beta)))  # noqa: E731
    tl, tu = th(lo), th(hi)
    acc = damped[0] * (tl - tu)
    for n in range(1, order + 1):
        acc += 2.0 * damped[n] * (math.sin(n * tl) - math.sin(n * tu)) / n
    return acc / math.pi


def solve(orc: Oracle, a: CSR, target, degree, n_search=0, epsilon=1e-10, kernel="lanczos2",
          max_iters=40, seed=1, dos_moments=2000, dos_samples=32, bounds=None):
    """solver.cpp:93-214 with an imposed degree (the automatic rule is pinned
    separately in tests/test_design.py)."""
    b = bounds if bounds is not None else lanczos_bounds(orc, a, 30, seed)
    mu = kpm_dos(orc, a, b, dos_moments, dos_samples, seed + 1)
    nt = dos_count(orc, mu, b, target[0], target[1])
    rep = dict(bounds=b, n_target_estimate=nt, converged=False, iterations=0)
    if nt < 0.5:
        rep.update(converged=True, values=np.zeros(0), residual_norms=np.zeros(0),
                   accepted=np.zeros(0, bool))
        return rep
    ns = n_search if n_search > 0 else 2 * int(math.ceil(nt))
    comb, alpha, beta = orc.make_filter(target, b, degree, kernel)
    sqrt_eps = math.sqrt(epsilon)
    required = max(1.0, math.ceil(nt - 3.0 * math.sqrt(nt)))
    x = orc.randomize(a.dim, ns, seed + 2, a.kind == 1)
    x /= orc.column_norms(x)[None, :]
    for it in range(1, max_iters + 1):
        x, _ = orc.apply_filter(a, x, comb, alpha, beta)
        q, rank = svqb(orc, x)
        repair = 0
        while rank < ns and repair < 5:
            fresh = orc.randomize(a.dim, ns - rank, seed + 1000 + it * 13 + repair, a.kind == 1)
            q, rank = svqb(orc, np.ascontiguousarray(np.concatenate([q[:, :rank], fresh], axis=1)))
            repair += 1
        vals, v, res = rayleigh_ritz(orc, a, q)
        inside = (vals >= target[0]) & (vals <= target[1])
        real = inside & (res <= sqrt_eps)
        accepted = real & (res <= epsilon)
        pending = int((real & ~accepted).sum())
        rep.update(iterations=it, values=vals, residual_norms=res, accepted=accepted, n_search=ns)
        if pending == 0 and accepted.sum() >= required:
            rep["converged"] = True
            break
        x = np.ascontiguousarray(v)
    return rep
