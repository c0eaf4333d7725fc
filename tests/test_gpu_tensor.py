"""Boundary-fitted grids through the reference's separable operators
(``TensorSystem``, src/assembly.py:615-770) -- the path ``harness.prepare``
takes for uncut Lagrange / B-spline grids (src/harness.py:317-324, 364-370):

* ``cdm_run`` with ``K = TensorSystem.stiffness_operator()`` (a scipy
  LinearOperator): the device recognises it and runs the matrix-free SCM
  kernel (Lagrange) or the Kronecker CSR (B-splines);
* B-splines carry the consistent Kronecker mass: ``cdm_run`` and
  ``max_gen_eig`` go through the device consistent-mass plan;
* ``newmark_run(s_factory=...)``: the factory is called as in the reference,
  the device factorises the same S.

Goldens: tests/golden/make_golden.py ``gen_tensor`` (the reference itself).
The TensorSystem here is a stand-in with the same attributes (the reference
package does not exist on the GPU box)."""

from types import SimpleNamespace

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from conftest import csr_from, load_golden

pytestmark = pytest.mark.gpu

from paper_2501_19013_b200 import cdm_run, max_gen_eig, newmark_run  # noqa: E402
from paper_2501_19013_b200.operators import ScmOperator, as_device_operator  # noqa: E402
from paper_2501_19013_b200.setup.configs import ricker  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


class Tensor:
    """Duck-typed TensorSystem: the attributes the device adapter reads."""

    def __init__(self, g, k):
        fam = {"l": "lagrange", "b": "bspline"}[k]
        self.m1, self.k1 = g[f"{k}_m1"], g[f"{k}_k1"]
        self.rho, self.c = 1.0, 1.0
        spec = SimpleNamespace(family=fam, p=int(g[f"{k}_p"]), n_e=int(g[f"{k}_n_e"]))
        self.grid = SimpleNamespace(spec=spec, h=float(g[f"{k}_h"]))
        m, kk = sp.csr_matrix(self.m1), sp.csr_matrix(self.k1)
        self._K = (sp.kron(sp.kron(kk, m), m) + sp.kron(sp.kron(m, kk), m)
                   + sp.kron(sp.kron(m, m), kk)).tocsr()

    def k_matvec(self, x):
        return self._K @ x

    def stiffness_operator(self):
        n = self._K.shape[0]
        return spla.LinearOperator((n, n), matvec=self.k_matvec, rmatvec=self.k_matvec, dtype=float)


class Fact:
    """What s_factory returns: anything with solve / n."""

    def __init__(self, n):
        self.n = n
        self.calls = 0

    def solve(self, b):   # never called by the device loop
        self.calls += 1
        raise AssertionError("host solve called")


@pytest.mark.parametrize("k", ["l", "b"])
def test_tensor_stiffness_operator_cdm_matches_reference(k):
    g = load_golden("tensor")
    ts = Tensor(g, k)
    K = ts.stiffness_operator()
    M = csr_from(g, f"{k}_M")
    op = as_device_operator(K)
    if k == "l":
        assert isinstance(op, ScmOperator) and op.n_cut == 0
    x = np.random.default_rng(0).standard_normal(op.n)
    assert rel(op @ x, ts.k_matvec(x)) <= 1e-13
    assert as_device_operator(K) is op          # cached per TensorSystem
    lam, it = max_gen_eig(K, M, tol=1e-7, seed=0)
    assert abs(lam - float(g[f"{k}_lam"])) <= 1e-12 * float(g[f"{k}_lam"])
    assert it == int(g[f"{k}_it"])
    f = lambda t: ricker(t, 10.0)  # noqa: E731
    r = cdm_run(M, K, g[f"{k}_F"], f, float(g[f"{k}_dt"]), 150, obs_mat=csr_from(g, f"{k}_obs"))
    assert rel(r.psi, g[f"{k}_psi"]) <= 1e-10
    assert rel(r.obs, g[f"{k}_obs"]) <= 1e-10
    # consistent Kronecker mass (B-splines): the reference factorises M
    assert r.fact_dim == (0 if k == "l" else M.shape[0])


@pytest.mark.parametrize("k", ["l", "b"])
def test_tensor_newmark_with_s_factory(k):
    """The reference's factories solve S by CG to a 1e-13 relative residual
    (Lagrange) or by fast diagonalisation (B-splines); the device solves the
    same S exactly through its SuperLU factors, so the fields agree to the
    CG tolerance, not to rounding."""
    g = load_golden("tensor")
    ts = Tensor(g, k)
    K = ts.stiffness_operator()
    M = csr_from(g, f"{k}_M")
    made = []

    def factory():
        made.append(Fact(M.shape[0]))
        return made[-1]

    f = lambda t: ricker(t, 10.0)  # noqa: E731
    r = newmark_run(M, K, g[f"{k}_F"], f, float(g[f"{k}_dtn"]), 60, obs_mat=csr_from(g, f"{k}_obs"),
                    s_factory=factory)
    assert len(made) == 1 and made[0].calls == 0
    tol = 1e-9 if k == "l" else 1e-11
    assert rel(r.psi, g[f"{k}_nm_psi"]) <= tol
    assert rel(r.obs, g[f"{k}_nm_obs"]) <= tol
    assert rel(r.psi_dot, g[f"{k}_nm_v"]) <= tol
    with pytest.raises(TypeError):
        newmark_run(M, K, g[f"{k}_F"], f, 1e-3, 3, s_factory=lambda: None)
