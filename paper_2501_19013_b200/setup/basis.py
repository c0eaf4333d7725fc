"""1D quadrature and shape functions for the host-side set-up.

Restates the reference's 1D ingredients (src/basis.py) -- Gauss-Legendre and
Gauss-Lobatto-Legendre rules, Lagrange polynomials on GLL nodes, open uniform
knot vectors and Cox-de Boor B-splines -- with independent implementations.
They are pinned value-for-value against the reference's own outputs in
tests/test_setup_basis.py (golden vectors, ~1e-14).
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np
from numpy.polynomial import legendre as npleg


@lru_cache(maxsize=None)
def gl_rule(q: int):
    """Gauss-Legendre nodes/weights with q points (src/basis.py:31-36)."""
    if q < 1:
        raise ValueError("need at least one quadrature point")
    x, w = npleg.leggauss(q)
    return x, w


def _legendre(p: int, x):
    """P_p(x) and P_{p-1}(x) by the three-term recurrence."""
    x = np.asarray(x, dtype=float)
    a, b = np.ones_like(x), x.copy()
    if p == 0:
        return a, np.zeros_like(x)
    for k in range(1, p):
        a, b = b, ((2 * k + 1) * x * b - k * a) / (k + 1)
    return b, a


@lru_cache(maxsize=None)
def gll_rule(p: int):
    """GLL nodes/weights, p+1 points incl. the end points (src/basis.py:54-79).

    Interior nodes are the roots of P_p'; they are polished by Newton steps on
    (1 - x^2) P_p'(x) = p (x P_p - P_{p-1}) starting from Chebyshev-Lobatto
    points.  Weights 2 / (p (p+1) P_p(x)^2).
    """
    if p < 1:
        raise ValueError("GLL rule needs polynomial degree >= 1")
    if p == 1:
        return np.array([-1.0, 1.0]), np.array([1.0, 1.0])
    if p == 2:
        return np.array([-1.0, 0.0, 1.0]), np.array([1.0, 4.0, 1.0]) / 3.0
    x = -np.cos(np.pi * np.arange(1, p) / p)
    for _ in range(100):
        P, Pm = _legendre(p, x)
        dP = p * (x * P - Pm) / (x * x - 1.0)           # P_p'
        # f = (1-x^2) P_p' ; f' = -p(p+1) P_p (Legendre ODE)
        step = (1.0 - x * x) * dP / (p * (p + 1) * P)
        x = x + step
        if np.max(np.abs(step)) < 1e-15:
            break
    nodes = np.concatenate(([-1.0], x, [1.0]))
    P, _ = _legendre(p, nodes)
    return nodes, 2.0 / (p * (p + 1) * P * P)


def lagrange_eval(nodes, x):
    """Values V[i, j] = L_j(x_i) and derivatives D[i, j] = L_j'(x_i) of the
    Lagrange basis on ``nodes`` (src/basis.py:82-119)."""
    nodes = np.asarray(nodes, dtype=float)
    x = np.atleast_1d(np.asarray(x, dtype=float))
    n = nodes.shape[0]
    dx = x[:, None] - nodes[None, :]
    den = np.array([np.prod([nodes[j] - nodes[m] for m in range(n) if m != j])
                    for j in range(n)])
    V = np.empty((x.shape[0], n))
    D = np.empty((x.shape[0], n))
    for j in range(n):
        others = [m for m in range(n) if m != j]
        V[:, j] = np.prod(dx[:, others], axis=1) / den[j]
        acc = np.zeros(x.shape[0])
        for k in others:
            rest = [m for m in others if m != k]
            acc += np.prod(dx[:, rest], axis=1) if rest else 1.0
        D[:, j] = acc / den[j]
    return V, D


def open_uniform_knots(n_e: int, p: int, a: float = 0.0, b: float = 1.0) -> np.ndarray:
    """Open uniform knot vector with n_e spans (src/basis.py:122-133)."""
    if n_e < 1 or p < 1:
        raise ValueError("need n_e >= 1 and p >= 1")
    inner = a + (b - a) * np.arange(1, n_e) / n_e
    return np.concatenate((np.full(p + 1, a), inner, np.full(p + 1, b)))


def bspline_eval(knots, p: int, x):
    """Nonzero B-splines of degree p and their derivatives at x, by the
    Cox-de Boor triangle (src/basis.py:144-188).  Returns (span, V, D)."""
    knots = np.asarray(knots, dtype=float)
    x = np.atleast_1d(np.asarray(x, dtype=float))
    nb = knots.shape[0] - p - 1
    span = np.clip(np.searchsorted(knots, x, side="right") - 1, p, nb - 1)
    m = x.shape[0]
    # N[d] holds the degree-d functions span-d..span
    N = np.ones((m, 1))
    lower = None
    for d in range(1, p + 1):
        new = np.zeros((m, d + 1))
        for r in range(d):
            # old column r is N_{i,d-1}, i = span-d+1+r; it feeds N_{i,d}
            # (rising term) and N_{i-1,d} (falling term), both over t_{i+d}-t_i
            i = span - d + 1 + r
            den = knots[i + d] - knots[i]
            safe = np.where(den > 0, den, 1.0)
            up = np.where(den > 0, (x - knots[i]) / safe, 0.0)
            down = np.where(den > 0, (knots[i + d] - x) / safe, 0.0)
            new[:, r + 1] += up * N[:, r]
            new[:, r] += down * N[:, r]
        if d == p:
            lower = N
        N = new
    if p == 0:
        lower = np.ones((m, 1))
    # shift: after the loop column c of N is function span - p + c
    # derivative: N'_{i,p} = p/(t_{i+p}-t_i) N_{i,p-1} - p/(t_{i+p+1}-t_{i+1}) N_{i+1,p-1}
    D = np.zeros((m, p + 1))
    for c in range(p + 1):
        i = span - p + c
        if c > 0:
            den = knots[i + p] - knots[i]
            D[:, c] += np.where(den > 0, p * lower[:, c - 1] / np.where(den > 0, den, 1.0), 0.0)
        if c < p:
            den = knots[i + p + 1] - knots[i + 1]
            D[:, c] -= np.where(den > 0, p * lower[:, c] / np.where(den > 0, den, 1.0), 0.0)
    return span, N, D


class Basis1D:
    """Per-direction basis: 'lagrange' (GLL nodal) or 'bspline' (C^{p-1})."""

    def __init__(self, family: str, p: int, n_e: int):
        if family not in ("lagrange", "bspline"):
            raise ValueError(f"unknown basis family {family!r}")
        self.family, self.p, self.n_e = family, int(p), int(n_e)
        self.knots = open_uniform_knots(n_e, p) if family == "bspline" else None

    @property
    def n_funcs(self) -> int:
        """Global functions per direction (src/basis.py:205-210)."""
        return self.n_e * self.p + 1 if self.family == "lagrange" else self.n_e + self.p

    def first_func(self, e):
        """Index of the first function supported on cell e (src/basis.py:217-221)."""
        return np.asarray(e) * self.p if self.family == "lagrange" else np.asarray(e)

    def eval(self, e: int, xi):
        """Values/derivatives (w.r.t. xi in [-1,1]) of the p+1 functions of
        cell e (src/basis.py:223-244, src/assembly.py:439-444)."""
        xi = np.atleast_1d(np.asarray(xi, dtype=float))
        if self.family == "lagrange":
            return lagrange_eval(gll_rule(self.p)[0], xi)
        a = self.knots[self.p + e]
        b = self.knots[self.p + e + 1]
        x = a + (b - a) * (xi + 1.0) / 2.0
        x = np.clip(x, a, np.nextafter(b, a))
        span, V, D = bspline_eval(self.knots, self.p, x)
        if not np.all(span == self.p + e):
            raise RuntimeError("evaluation points left the requested span")
        return V, D * (b - a) / 2.0

    def signature(self, e: int):
        """Cells with equal signatures share 1D tables (src/assembly.py:256-261)."""
        if self.family == "lagrange":
            return 0
        return (min(e, self.p), min(self.n_e - 1 - e, self.p))


def uncut_1d(basis: Basis1D, e: int, q: int | None = None):
    """Exact 1D reference mass/stiffness of cell e with a q-point GL rule
    (src/assembly.py:263-272)."""
    q = basis.p + 1 if q is None else q
    x, w = gl_rule(q)
    V, D = basis.eval(e, x)
    return (V * w[:, None]).T @ V, (D * w[:, None]).T @ D


def uncut_g1(basis: Basis1D, e: int, q: int | None = None):
    """Exact 1D reference "gradient-mass" G[a][b] = int phi_a' phi_b of cell e
    (the mixed-derivative factor of the plane-strain operator)."""
    q = basis.p + 1 if q is None else q
    x, w = gl_rule(q)
    V, D = basis.eval(e, x)
    return (D * w[:, None]).T @ V


def dyadic_intervals(max_depth: int):
    """Start, length and id offset of every dyadic subinterval of [-1, 1]
    up to max_depth (src/assembly.py:447-459)."""
    starts, lengths, offsets = [], [], np.zeros(max_depth + 1, dtype=np.int64)
    acc = 0
    for d in range(max_depth + 1):
        m = 2 ** d
        offsets[d] = acc
        acc += m
        starts.append(-1.0 + (2.0 / m) * np.arange(m))
        lengths.append(np.full(m, 2.0 / m))
    return np.concatenate(starts), np.concatenate(lengths), offsets


def dyadic_tables(basis: Basis1D, e: int, max_depth: int, q: int | None = None):
    """Per dyadic interval: mapped GL nodes, weights, basis values and the 1D
    partial mass/stiffness (src/assembly.py:310-330)."""
    q = basis.p + 1 if q is None else q
    x, w = gl_rule(q)
    starts, lengths, offsets = dyadic_intervals(max_depth)
    xi = starts[:, None] + (x[None, :] + 1.0) / 2.0 * lengths[:, None]
    V, D = basis.eval(e, xi.ravel())
    n = basis.p + 1
    V = V.reshape(-1, q, n)
    D = D.reshape(-1, q, n)
    wq = w[None, :] * (lengths[:, None] / 2.0)
    m1 = np.einsum("lqa,lq,lqb->lab", V, wq, V)
    k1 = np.einsum("lqa,lq,lqb->lab", D, wq, D)
    g1 = np.einsum("lqa,lq,lqb->lab", D, wq, V)     # int phi_a' phi_b (elasticity)
    return {"xi": xi, "w": wq, "V": V, "D": D, "m1": m1, "k1": k1, "g1": g1, "offsets": offsets}
