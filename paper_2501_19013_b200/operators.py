"""Device-resident stiffness operators (the ``K`` the integrators consume).

The reference integrators accept anything with ``K @ x`` (scipy CSR from
``assemble``, src/assembly.py:518-612, or the separable ``LinearOperator`` of
``TensorSystem``, src/assembly.py:674-690).  Here ``K`` is uploaded once into
HBM and stays there across every step of every run:

* :class:`CsrOperator` -- any scipy sparse / dense matrix (IGA B-spline path,
  generic systems).
* :class:`ScmOperator` -- matrix-free spectral-cell stiffness on a Cartesian
  grid: sum-factorised uncut cells plus dense cut cells.

``op @ x`` works on host vectors (one device round trip) so an operator can be
handed to any code written against the reference's duck type.
"""

from __future__ import annotations

import weakref

import numpy as np
import scipy.sparse as sp

from . import _lib


class DeviceOperator:
    """Base class: an opaque ``wcb_operator`` handle on one device."""

    kind = "abstract"

    def __init__(self, handle, n: int, ctx: _lib.Context):
        self._h = handle
        self.n = int(n)
        self.ctx = ctx
        self.shape = (self.n, self.n)
        self.dtype = np.dtype(np.float64)

    @property
    def handle(self):
        return self._h

    @property
    def step_kernel(self) -> str:
        """The kernel(s) one fused time step of this operator launches."""
        buf = _lib.C.create_string_buffer(256)
        _lib.check(_lib.load().wcb_operator_step_kernel(self._h, buf, 256))
        return buf.value.decode()

    def matvec(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError(f"expected shape ({self.n},), got {x.shape}")
        y = np.empty(self.n)
        _lib.check(_lib.load().wcb_operator_apply(self._h, _lib.dptr(x), _lib.dptr(y)))
        return y

    def __matmul__(self, x):
        x = np.asarray(x, dtype=np.float64)
        if x.ndim == 2:
            return np.stack([self.matvec(x[:, j]) for j in range(x.shape[1])], axis=1)
        return self.matvec(x)

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().wcb_operator_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CsrOperator(DeviceOperator):
    """CSR ``K`` in HBM (int64 row pointers, int32 columns, fp64 values)."""

    kind = "csr"

    def __init__(self, K, device: int | None = None):
        A = sp.csr_matrix(K, dtype=np.float64)
        if A.shape[0] != A.shape[1]:
            raise ValueError("matrix must be square")
        A.sum_duplicates()
        n = A.shape[0]
        indptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(A.indices, dtype=np.int32)
        data = np.ascontiguousarray(A.data, dtype=np.float64)
        ctx = _lib.context(device)
        h = _lib.C.c_void_p()
        _lib.check(_lib.load().wcb_operator_csr_create(
            ctx.handle, n, _lib.i64ptr(indptr), _lib.i32ptr(indices), _lib.dptr(data),
            _lib.C.byref(h)))
        super().__init__(h, n, ctx)
        self.nnz = int(data.shape[0])


class ScmOperator(DeviceOperator):
    """Matrix-free spectral-cell-method stiffness on a Cartesian cell grid.

    Parameters mirror what ``assemble`` consumes (src/assembly.py:518-583):
    the shared uncut 1D factors ``m1, k1`` (src/assembly.py:263-272), the cell
    classification (src/geometry.py:36-41, 0 outside / 1 inside / 2 cut), the
    compact DOF map (src/assembly.py:159-180) and the physical cut-cell
    stiffness matrices ``sk (K_in + alpha K_out)`` (src/assembly.py:582).
    """

    kind = "scm"

    def __init__(self, dim: int, p: int, n_e, k1, m1, sk: float, cell_class,
                 lex_of_compact, cut_cells, cut_K, device: int | None = None, slab=None):
        dim = int(dim)
        p = int(p)
        n_e = tuple(int(v) for v in n_e)
        if len(n_e) != dim:
            raise ValueError("n_e must have dim entries")
        L = (p + 1) ** dim
        self._k1 = np.ascontiguousarray(k1, dtype=np.float64).reshape(p + 1, p + 1)
        self._m1 = np.ascontiguousarray(m1, dtype=np.float64).reshape(p + 1, p + 1)
        self._cls = np.ascontiguousarray(cell_class, dtype=np.int8).reshape(-1)
        lo, hi, last = (0, n_e[0], True) if slab is None else (int(slab[0]), int(slab[1]),
                                                               bool(slab[2]))
        rows = hi - (lo - 1 if lo > 0 else lo)
        if self._cls.shape[0] != rows * int(np.prod(n_e[1:])):
            raise ValueError("cell_class must cover the cell rows of the operator")
        self._lex = np.ascontiguousarray(lex_of_compact, dtype=np.int64)
        self._cut = np.ascontiguousarray(cut_cells, dtype=np.int64).reshape(-1)
        self._cutK = np.ascontiguousarray(cut_K, dtype=np.float64).reshape(-1)
        if self._cutK.shape[0] != self._cut.shape[0] * L * L:
            raise ValueError("cut_K must hold n_cut * L * L values")
        desc = _lib.ScmDesc()
        desc.dim = dim
        desc.p = p
        for i in range(3):
            desc.n_e[i] = n_e[i] if i < dim else 1
        desc.k1 = _lib.dptr(self._k1)
        desc.m1 = _lib.dptr(self._m1)
        desc.sk = float(sk)
        desc.cell_class = _lib.i8ptr(self._cls)
        desc.n_dof = self._lex.shape[0]
        desc.lex_of_compact = _lib.i64ptr(self._lex)
        desc.n_cut = self._cut.shape[0]
        desc.cut_cells = _lib.i64ptr(self._cut) if self._cut.size else None
        desc.cut_K = _lib.dptr(self._cutK) if self._cutK.size else None
        desc.x_cell_lo = lo
        desc.x_cell_hi = hi
        desc.x_owns_last = 1 if last else 0
        ctx = _lib.context(device)
        h = _lib.C.c_void_p()
        _lib.check(_lib.load().wcb_operator_scm_create(ctx.handle, _lib.C.byref(desc),
                                                       _lib.C.byref(h)))
        super().__init__(h, self._lex.shape[0], ctx)
        self.dim, self.p, self.n_e, self.sk = dim, p, n_e, float(sk)
        self.n_cut = int(self._cut.shape[0])


class ElasticOperator(DeviceOperator):
    """Matrix-free plane-strain stiffness on the SCM node grid (BASELINE
    config 4; setup/elastic.py documents the operator).  DOFs are component
    major: ``dof = comp * n_node + node``."""

    kind = "elastic"

    def __init__(self, p: int, n_e: int, lam: float, mu: float, m1, k1, g1, cell_class,
                 lex_of_compact, cut_cells, cut_K, device: int | None = None, slab=None):
        p = int(p)
        n_e = int(n_e)
        N = p + 1
        L = 2 * N * N
        self._m1 = np.ascontiguousarray(m1, dtype=np.float64).reshape(N, N)
        self._k1 = np.ascontiguousarray(k1, dtype=np.float64).reshape(N, N)
        self._g1 = np.ascontiguousarray(g1, dtype=np.float64).reshape(N, N)
        self._cls = np.ascontiguousarray(cell_class, dtype=np.int8).reshape(-1)
        if slab is None and self._cls.shape[0] != n_e * n_e:
            raise ValueError("cell_class must hold n_e^2 entries")
        self._lex = np.ascontiguousarray(lex_of_compact, dtype=np.int64)
        self._cut = np.ascontiguousarray(cut_cells, dtype=np.int64).reshape(-1)
        self._cutK = np.ascontiguousarray(cut_K, dtype=np.float64).reshape(-1)
        if self._cutK.shape[0] != self._cut.shape[0] * L * L:
            raise ValueError("cut_K must hold n_cut * L * L values, L = 2 (p+1)^2")
        desc = _lib.ElasticDesc()
        desc.p = p
        desc.n_e[0] = desc.n_e[1] = n_e
        desc.lam, desc.mu = float(lam), float(mu)
        desc.m1, desc.k1, desc.g1 = _lib.dptr(self._m1), _lib.dptr(self._k1), _lib.dptr(self._g1)
        desc.cell_class = _lib.i8ptr(self._cls)
        desc.n_node = self._lex.shape[0]
        desc.lex_of_compact = _lib.i64ptr(self._lex)
        desc.n_cut = self._cut.shape[0]
        desc.cut_cells = _lib.i64ptr(self._cut) if self._cut.size else None
        desc.cut_K = _lib.dptr(self._cutK) if self._cutK.size else None
        if slab is not None:
            lo, hi, last = slab
            desc.x_cell_lo, desc.x_cell_hi, desc.x_owns_last = int(lo), int(hi), 1 if last else 0
        ctx = _lib.context(device)
        h = _lib.C.c_void_p()
        _lib.check(_lib.load().wcb_operator_elastic_create(ctx.handle, _lib.C.byref(desc),
                                                           _lib.C.byref(h)))
        super().__init__(h, 2 * self._lex.shape[0], ctx)
        self.dim, self.p, self.n_e = 2, p, (n_e, n_e)
        self.lam, self.mu = float(lam), float(mu)
        self.n_cut = int(self._cut.shape[0])


def _tensor_system_of(K):
    """The reference ``TensorSystem`` behind ``K`` when ``K`` is its
    ``stiffness_operator()`` (a scipy LinearOperator whose matvec is the bound
    ``k_matvec``, src/assembly.py:674-690), else None."""
    f = getattr(K, "_CustomLinearOperator__matvec_impl", None)
    owner = getattr(f, "__self__", None)
    if owner is None or getattr(f, "__name__", "") != "k_matvec":
        return None
    if not all(hasattr(owner, a) for a in ("m1", "k1", "grid", "rho", "c")):
        return None
    return owner


def _element_1d(glob: np.ndarray, p: int, n_e: int) -> np.ndarray:
    """Element matrix of a uniform 1D Lagrange assembly ``glob`` (sum of
    n_e equal (p+1)^2 blocks overlapping in one node): the first block, whose
    last diagonal entry (shared with the second block) is restored from the
    persymmetry of the GLL element matrices."""
    e = np.array(glob[: p + 1, : p + 1], dtype=np.float64)
    if n_e > 1:
        e[p, p] = glob[0, 0]
    re = np.zeros_like(glob)
    for c in range(n_e):
        re[c * p: c * p + p + 1, c * p: c * p + p + 1] += e
    if not np.allclose(re, glob, rtol=1e-13, atol=1e-13 * np.abs(glob).max()):
        raise TypeError("TensorSystem 1D factors are not a uniform Lagrange assembly")
    return e


def tensor_csr(tensor) -> sp.csr_matrix:
    """The separable stiffness of a ``TensorSystem`` as CSR:
    ``rho c^2 (k1 x m1 x m1 + m1 x k1 x m1 + m1 x m1 x k1)`` (src/assembly.py:674-684)."""
    m = sp.csr_matrix(np.asarray(tensor.m1, dtype=np.float64))
    k = sp.csr_matrix(np.asarray(tensor.k1, dtype=np.float64))
    K = (sp.kron(sp.kron(k, m), m) + sp.kron(sp.kron(m, k), m) + sp.kron(sp.kron(m, m), k))
    return (float(tensor.rho) * float(tensor.c) ** 2 * K).tocsr()


def tensor_operator(tensor, device: int | None = None) -> DeviceOperator:
    """Device form of the reference's separable stiffness
    ``rho c^2 (k1 x m1 x m1 + m1 x k1 x m1 + m1 x m1 x k1)`` of a fully uncut
    grid (``TensorSystem``, src/assembly.py:615-690).

    Lagrange: the global 1D factors are sums of one element matrix, so the
    Kronecker sum equals the sum of uncut element operators and runs in the
    matrix-free SCM kernel (every cell uncut, all nodes DOFs, lex order =
    ``P.reshape(n1, n1, n1)``).  B-splines: the Kronecker sum is formed as
    CSR once (entries are products of the 1D factors) and applied by the CSR
    kernel."""
    grid = tensor.grid
    spec = grid.spec
    rho_c2 = float(tensor.rho) * float(tensor.c) ** 2
    m1g = np.asarray(tensor.m1, dtype=np.float64)
    k1g = np.asarray(tensor.k1, dtype=np.float64)
    n1 = m1g.shape[0]
    if getattr(spec, "family", "") == "lagrange":
        p, n_e = int(spec.p), int(spec.n_e)
        h = float(grid.h)
        m1 = _element_1d(m1g, p, n_e) / (h / 2.0)
        k1 = _element_1d(k1g, p, n_e) * (h / 2.0)
        op = ScmOperator(dim=3, p=p, n_e=(n_e,) * 3, k1=k1, m1=m1, sk=rho_c2 * (h / 2.0),
                         cell_class=np.ones(n_e ** 3, dtype=np.int8),
                         lex_of_compact=np.arange(n1 ** 3, dtype=np.int64),
                         cut_cells=np.zeros(0, dtype=np.int64), cut_K=np.zeros(0),
                         device=device)
    else:
        op = CsrOperator(tensor_csr(tensor), device=device)
    op.tensor = tensor
    return op


_cache: dict[int, tuple] = {}


def _words(a: np.ndarray) -> int:
    """Wrapping 64-bit sum of the array's bytes (one vectorised pass)."""
    b = np.ascontiguousarray(a).reshape(-1).view(np.uint8)
    head = b[: b.shape[0] // 8 * 8].view(np.uint64)
    tail = b[head.shape[0] * 8:]
    return int(np.add.reduce(head, dtype=np.uint64)) ^ int(tail.sum()) ^ (b.shape[0] << 1)


def _fingerprint(K) -> tuple | None:
    """Content fingerprint of a host matrix: shape, buffers and a checksum of
    every stored value and index.  The reference reads ``K`` on every call,
    so an in-place change (``K *= s``, ``K.data[:] = ...``) must not reuse a
    stale device copy."""
    if sp.issparse(K):
        A = K if K.format in ("csr", "csc", "bsr") else None
        if A is None:
            return None
        return (K.format, K.shape, A.data.ctypes.data, A.indices.ctypes.data,
                A.indptr.ctypes.data, _words(A.data), _words(A.indices), _words(A.indptr))
    if isinstance(K, np.ndarray):
        return ("dense", K.shape, K.dtype.str, K.ctypes.data, _words(K))
    return None


def as_device_operator(K, device: int | None = None) -> DeviceOperator:
    """Device operator for ``K``.  Host matrices are uploaded once and reused
    while the same object lives with unchanged contents (checked by a content
    fingerprint on every call); a reference ``TensorSystem`` stiffness
    ``LinearOperator`` (src/assembly.py:686-690) becomes the matrix-free
    operator of its grid."""
    if isinstance(K, DeviceOperator):
        return K
    tensor = _tensor_system_of(K)
    obj = K if tensor is None else tensor
    key = id(obj)
    fp = _fingerprint(K) if tensor is None else (
        "tensor", _words(np.asarray(tensor.m1)), _words(np.asarray(tensor.k1)),
        float(tensor.rho), float(tensor.c))
    hit = _cache.get(key)
    if hit is not None:
        ref, op, fp0 = hit
        if ref() is obj and fp is not None and fp == fp0 and (device is None or op.ctx.device == device):
            return op
        _cache.pop(key, None)
    if tensor is not None:
        op = tensor_operator(tensor, device=device)
    elif sp.issparse(K) or isinstance(K, np.ndarray) or isinstance(K, np.matrix):
        op = CsrOperator(K, device=device)
    else:
        raise TypeError(
            f"unsupported stiffness operator type {type(K).__name__}: pass a scipy "
            "sparse matrix, a dense array, a TensorSystem stiffness operator or a "
            "paper_2501_19013_b200 DeviceOperator")
    if fp is None:
        return op
    try:
        ref = weakref.ref(obj)
    except TypeError:
        return op
    _cache[key] = (ref, op, fp)
    weakref.finalize(obj, _cache.pop, key, None)
    return op
