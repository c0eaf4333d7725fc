"""Generate golden vectors by running the REFERENCE package (read-only at
/root/reference/pkg/src) in this container.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The fixtures pin the CPU oracle (oracle/timeint.py) and the device parity
tests to the reference's own outputs.  The reference does not exist on the GPU
box; only the committed .npz files travel.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import scipy.sparse as sp

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.dont_write_bytecode = True

from wavecell import assembly as A                      # noqa: E402
from wavecell import assembly as A_                     # noqa: E402
from wavecell import basis as B                         # noqa: E402
from wavecell import basis as B_                        # noqa: E402
from wavecell import geometry as G                      # noqa: E402
from wavecell import harness as H                       # noqa: E402
from wavecell import linalg as LA                       # noqa: E402
from wavecell import stabilization as S                 # noqa: E402
from wavecell import timeint as T                       # noqa: E402

OUT = Path(__file__).resolve().parent


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    size = (OUT / f"{name}.npz").stat().st_size
    print(f"{name}.npz  {size / 1024:.1f} KiB")


def csr_parts(prefix, M):
    M = sp.csr_matrix(M)
    return {f"{prefix}_indptr": M.indptr.astype(np.int64),
            f"{prefix}_indices": M.indices.astype(np.int64),
            f"{prefix}_data": M.data, f"{prefix}_shape": np.array(M.shape)}


def bar_system():
    h = 1.0 / 3.0
    M = sp.diags([h / 2.0, h, h, h / 2.0]).tocsr()
    K1 = np.array([[1.0, -1.0], [-1.0, 1.0]]) / h
    K = np.zeros((4, 4))
    for e in range(3):
        K[e:e + 2, e:e + 2] += K1
    return M, sp.csr_matrix(K)


def gen_bar():
    M, K = bar_system()
    F = np.array([0.0, 1.0, 0.5, 0.2])
    obs = sp.identity(4, format="csr")
    f = lambda t: np.sin(6.0 * t)           # noqa: E731
    dt, n_t = 5e-3, 200
    r_cdm = T.cdm_run(M, K, F, f, dt, n_t, obs_mat=obs)
    r_nm = T.newmark_run(M, K, F, f, dt, n_t, obs_mat=obs)
    r_imex = T.imex_run(M, K, F, f, dt, n_t, np.array([1, 2]), np.array([0, 3]), obs_mat=obs)
    psi0 = np.array([0.1, 0.0, -0.2, 0.05])
    v0 = np.array([0.0, 0.3, 0.1, -0.1])
    r_init = T.cdm_run(M, K, F, np.cos, 1e-2, 100, obs_mat=obs, psi0=psi0, v0=v0)
    Mc = sp.csr_matrix(M.toarray() + 0.05 * np.ones((4, 4)))
    r_imex_c = T.imex_run(Mc, K, F, f, dt, n_t, np.arange(4), np.array([], dtype=int),
                          obs_mat=obs)
    save("bar", M=M.toarray(), Mc=Mc.toarray(), K=K.toarray(), F=F, dt=dt, n_t=n_t,
         cdm_obs=r_cdm.obs, cdm_psi=r_cdm.psi, nm_obs=r_nm.obs, imex_obs=r_imex.obs,
         imex_psi=r_imex.psi, imexc_obs=r_imex_c.obs, imexc_vdot=r_imex_c.psi_dot,
         psi0=psi0, v0=v0, init_obs=r_init.obs, init_psi=r_init.psi)


def gen_scalar():
    M = sp.csr_matrix(np.array([[1.0]]))
    K = sp.csr_matrix(np.array([[1.0]]))
    r = T.cdm_run(M, K, np.zeros(1), lambda t: 0.0, 1.99, 10000,
                  obs_mat=sp.identity(1, format="csr"), psi0=[1.0])
    try:
        T.cdm_run(M, K, np.zeros(1), lambda t: 0.0, 2.01, 10000, psi0=[1.0])
        raise AssertionError("expected divergence")
    except T.DivergenceError as e:
        step, amp = e.step, e.amplitude
    save("scalar", stable_obs=r.obs, stable_psi=r.psi, div_step=step, div_amp=amp)


def gen_rand10():
    rng = np.random.default_rng(6)
    n = 10
    M = sp.diags(rng.uniform(0.5, 2.0, n)).tocsr()
    Am = rng.standard_normal((n, n))
    K = sp.csr_matrix(Am @ Am.T + n * np.eye(n))
    F = rng.standard_normal(n)
    psi0 = rng.standard_normal(n)
    lam, it = LA.max_gen_eig(K, M)
    dt = 0.5 * LA.dt_crit(K, M)
    r = T.cdm_run(M, K, F, lambda t: np.sin(3.0 * t), dt, 200,
                  obs_mat=sp.identity(n, format="csr"), psi0=psi0)
    save("rand10", M=M.diagonal(), K=K.toarray(), F=F, psi0=psi0, lam=lam, iters=it, dt=dt,
         obs=r.obs, psi=r.psi)


def scm_desc(grid, cache, params, rho=1.0, c=1.0):
    """The matrix-free description of a reference Lagrange system."""
    spec = grid.spec
    n = spec.p + 1
    h = grid.h
    sk = rho * c * c * (h / 2.0)
    m1, k1 = cache._uncut_1d(0)
    cut = [tuple(int(v) for v in ijk) for ijk in grid.kept
           if grid.classes[tuple(ijk)] == G.ElementClass.CUT]
    n_e = spec.n_e
    cut_lex = np.array([(i * n_e + j) * n_e + k for i, j, k in cut], dtype=np.int64)
    order = np.argsort(cut_lex)
    cut_K = np.stack([sk * (cache.cut_element(cut[o]).K_in
                            + params.alpha * cache.cut_element(cut[o]).K_out)
                      for o in order]) if cut else np.zeros((0, n ** 3, n ** 3))
    return dict(dim=3, p=spec.p, n_e=np.array([n_e] * 3), k1=k1, m1=m1, sk=sk,
                cell_class=np.asarray(grid.classes, dtype=np.int8).ravel(),
                lex_of_compact=grid.dofmap.lex_of_compact.astype(np.int64),
                cut_cells=cut_lex[order], cut_K=cut_K,
                c_idx=grid.dofmap.c_idx.astype(np.int64),
                d_idx=grid.dofmap.d_idx.astype(np.int64))


def gen_cube(name, p, n_e, alpha, depth, n_t, store_csr, lumping="hrz"):
    geom = G.ImmersedGeometry.from_angles(0.3, 0.5, (10.0, 10.0, 10.0))
    grid = G_grid = A.Grid.build(geom, B.BasisSpec(family="lagrange", p=p, n_e=n_e))
    cache = A.ElementIntegralCache(G_grid, octree_depth=depth)
    params = S.StabilizationParams(alpha=alpha, lumping=lumping)
    system = A.assemble(grid, params, source=A.benchmark_source(0.3), cache=cache)
    obs = H.observer_matrix(grid)
    desc = scm_desc(grid, cache, params)
    lam, it = LA.max_gen_eig(system.K, system.M, tol=1e-7, seed=0)
    dt = T.select_dt(2.0 / np.sqrt(lam))
    f = lambda t: A.ricker(t, 10.0)         # noqa: E731
    r = T.cdm_run(system.M, system.K, system.F_s, f, dt, n_t, obs_mat=obs)
    rng = np.random.default_rng(123)
    X = rng.standard_normal((system.n_dof, 2))
    KX = system.K @ X
    extra = csr_parts("K", system.K) if store_csr else {}
    save(name, **desc, M=system.M.diagonal(), F=system.F_s, **csr_parts("obs", obs),
         lam=lam, iters=it, dt=dt, n_t=n_t, psi=r.psi, obs=r.obs, X=X, KX=KX,
         K_abs_sum=np.abs(system.K).sum(axis=1).A1, **extra)


def gen_cube_imex(name, p, n_e, alpha, depth, n_t):
    geom = G.ImmersedGeometry.from_angles(0.3, 0.5, (10.0, 10.0, 10.0))
    grid = A.Grid.build(geom, B.BasisSpec(family="lagrange", p=p, n_e=n_e))
    cache = A.ElementIntegralCache(grid, octree_depth=depth)
    params = S.StabilizationParams(alpha=alpha)
    system = A.assemble(grid, params, source=A.benchmark_source(0.3), cache=cache)
    obs = H.observer_matrix(grid)
    dm = grid.dofmap
    dtd = T.imex_critical_time_step(system.K, system.M, dm.d_idx, tol=1e-7)
    dt = 0.9 * dtd
    f = lambda t: A.ricker(t, 10.0)         # noqa: E731
    r = T.imex_run(system.M, system.K, system.F_s, f, dt, n_t, dm.c_idx, dm.d_idx,
                   obs_mat=obs)
    desc = scm_desc(grid, cache, params)
    save(name, **desc, **csr_parts("M", system.M), **csr_parts("K", system.K),
         F=system.F_s, **csr_parts("obs", obs), dtd=dtd, dt=dt, n_t=n_t, psi=r.psi,
         obs=r.obs)


def gen_bspline_cube(name, p, n_e, alpha, depth):
    """Reference IGA-FCM system (B-splines, row-sum lumping) on the rotated cube."""
    geom = G.ImmersedGeometry.from_angles(0.3, 0.5, (10.0, 10.0, 10.0))
    grid = A.Grid.build(geom, B.BasisSpec(family="bspline", p=p, n_e=n_e))
    cache = A.ElementIntegralCache(grid, octree_depth=depth)
    params = S.StabilizationParams(alpha=alpha, lumping="row_sum")
    system = A.assemble(grid, params, source=A.benchmark_source(0.3), cache=cache)
    lam, it = LA.max_gen_eig(system.K, system.M, tol=1e-7, seed=0)
    dt = T.select_dt(2.0 / np.sqrt(lam))
    f = lambda t: A.ricker(t, 10.0)         # noqa: E731
    r = T.cdm_run(system.M, system.K, system.F_s, f, dt, 200)
    save(name, **csr_parts("K", system.K), M=system.M.diagonal(), F=system.F_s,
         lex_of_compact=grid.dofmap.lex_of_compact.astype(np.int64), lam=lam, iters=it,
         dt=dt, psi=r.psi)


def gen_basis():
    """1D ingredients of the spectral-cell / B-spline discretisation."""
    out = {}
    x = np.linspace(-1.0, 1.0, 13)
    for p in range(1, 8):
        g = B.gll_rule(p)
        out[f"gll{p}_x"], out[f"gll{p}_w"] = g.nodes, g.weights
        V, D = B.lagrange_eval(g.nodes, x)
        out[f"lag{p}_V"], out[f"lag{p}_D"] = V, D
        gl = B.gl_rule(p + 1)
        out[f"gl{p + 1}_x"], out[f"gl{p + 1}_w"] = gl.nodes, gl.weights
    for p in range(1, 6):
        spec = B.BasisSpec("lagrange", p, 2)
        geom = G.ImmersedGeometry.from_angles(0.3, 0.5, (0.0, 0.0, 0.0))
        grid = A.Grid.build(geom, spec, boundary_fitted=True)
        cache = A.ElementIntegralCache(grid, octree_depth=2)
        m1, k1 = cache._uncut_1d(0)
        out[f"m1_{p}"], out[f"k1_{p}"] = m1, k1
        tabs = cache._dyadic_tables(0)
        out[f"dy{p}_m1"], out[f"dy{p}_k1"] = tabs["m1"], tabs["k1"]
    for p in (2, 3):
        knots = B.open_uniform_knots(7, p)
        pts = np.linspace(0.0, 1.0, 29)
        span, V, D = B.bspline_eval(knots, p, pts)
        out[f"bs{p}_span"], out[f"bs{p}_V"], out[f"bs{p}_D"] = span, V, D
        spec = B.BasisSpec("bspline", p, 7)
        for e in (0, 1, 3, 6):
            Ve, De = spec.eval_element(e, x, knots=knots)
            out[f"bs{p}_e{e}_V"], out[f"bs{p}_e{e}_D"] = Ve, De
    save("basis", **out)


def gen_lumping():
    rng = np.random.default_rng(3)
    C = rng.standard_normal((5, 8, 8))
    Ms = np.einsum("bij,bkj->bik", C, C) + 8.0 * np.eye(8)
    save("lumping", M=Ms, hrz=S.hrz_lump(Ms), rowsum=S.row_sum_lump(Ms))


def gen_paper():
    """The reference's own benchmark (PAPER section 4, tests/test_acceptance.py
    criteria 2-4): rotated cube, SCM p=3, n_e=13 (alpha 1e-8 CDM, alpha 1e-12
    IMEX) and n_e=10 (stability dichotomy), octree depth 4, consistent cut
    mass (lumping 'none', the StabilizationParams default).  Only compact
    fingerprints of the operators are stored (K X, M X, the load, the
    observers); the device tests rebuild the system with the host set-up
    restatement and check it against them."""
    geom = G.ImmersedGeometry.from_angles(0.3, 0.5, (10.0, 10.0, 10.0))
    src = A.benchmark_source(0.3)
    f = lambda t: A.ricker(t, 10.0)          # noqa: E731
    out = {}
    grid = A.Grid.build(geom, B.BasisSpec(family="lagrange", p=3, n_e=13))
    cache = A.ElementIntegralCache(grid, octree_depth=4)
    obs = H.observer_matrix(grid)
    n = grid.dofmap.n_dof
    X = np.random.default_rng(7).standard_normal((n, 2))
    out["X"] = X
    out.update(csr_parts("obs", obs))
    # criterion 2 (explicit): dt_crit of the full system, consistent M
    s8 = A.assemble(grid, S.StabilizationParams(alpha=1e-8), source=src, cache=cache)
    lam, it = LA.max_gen_eig(s8.K, s8.M, tol=1e-7, seed=0)
    out.update(F8=s8.F_s, KX8=s8.K @ X, MX8=s8.M @ X, lam8=lam, it8=it, dtc8=2.0 / np.sqrt(lam),
               Mdiag8=s8.M.diagonal(), Mnnz8=s8.M.nnz)
    dt8 = T.select_dt(2.0 / np.sqrt(lam))
    r = T.cdm_run(s8.M, s8.K, s8.F_s, f, dt8, 300, obs_mat=obs)
    out.update(dt8=dt8, psi8=r.psi, obs8=r.obs)
    print("n13 alpha 1e-8:", 2.0 / np.sqrt(lam), it)
    # criteria 2 and 4 (IMEX): explicit-subsystem step, 2000 IMEX steps at 0.9x
    s12 = A.assemble(grid, S.StabilizationParams(alpha=1e-12), source=src, cache=cache)
    dm = grid.dofmap
    dtd = T.imex_critical_time_step(s12.K, s12.M, dm.d_idx, tol=1e-7)
    Kr = sp.csr_matrix(s12.K)
    lam_d, it_d = LA.max_gen_eig(Kr[dm.d_idx][:, dm.d_idx], sp.csr_matrix(s12.M)[dm.d_idx][:, dm.d_idx],
                                 tol=1e-7, seed=0)
    lam_lb, it_lb = LA.max_gen_eig(s12.K, s12.M, tol=1e-3, seed=0)
    r = T.imex_run(s12.M, s12.K, s12.F_s, f, 0.9 * dtd, 2000, dm.c_idx, dm.d_idx, obs_mat=obs)
    out.update(F12=s12.F_s, KX12=s12.K @ X, MX12=s12.M @ X, dtd12=dtd, lamd12=lam_d, itd12=it_d,
               lamlb12=lam_lb, itlb12=it_lb, psi12=r.psi, obs12=r.obs,
               c_idx=dm.c_idx.astype(np.int64))
    print("n13 alpha 1e-12:", dtd, it_d)
    save("paper_n13", **out)
    # criterion 3: stability dichotomy on n_e = 10
    grid = A.Grid.build(geom, B.BasisSpec(family="lagrange", p=3, n_e=10))
    cache = A.ElementIntegralCache(grid, octree_depth=4)
    obs = H.observer_matrix(grid)
    n = grid.dofmap.n_dof
    X = np.random.default_rng(8).standard_normal((n, 2))
    s10 = A.assemble(grid, S.StabilizationParams(alpha=1e-8), source=src, cache=cache)
    lam, it = LA.max_gen_eig(s10.K, s10.M, tol=1e-7, seed=0)
    dtc = 2.0 / np.sqrt(lam)
    stable = T.cdm_run(s10.M, s10.K, s10.F_s, f, 0.99 * dtc, 2000, obs_mat=obs)
    try:
        T.cdm_run(s10.M, s10.K, s10.F_s, f, 1.05 * dtc, 2000, obs_mat=obs)
        raise AssertionError("expected divergence")
    except T.DivergenceError as e:
        step, amp = e.step, e.amplitude
    print("n10:", dtc, it, "diverged at", step)
    save("paper_n10", X=X, **csr_parts("obs", obs), F=s10.F_s, KX=s10.K @ X, MX=s10.M @ X,
         lam=lam, it=it, dtc=dtc, psi=stable.psi, obs=stable.obs, div_step=step, div_amp=amp)


def gen_tensor():
    """Boundary-fitted grids through the reference's separable operators
    (TensorSystem, src/assembly.py:615-770): the stiffness LinearOperator in
    cdm_run and newmark_run with its s_factory (Lagrange: diagonal M and CG
    inverse; B-splines: consistent Kronecker M and fast diagonalisation)."""
    geom = G.ImmersedGeometry.from_angles(0.3, 0.5, (10.0, 10.0, 10.0))
    src = A.benchmark_source(0.3)
    f = lambda t: A.ricker(t, 10.0)          # noqa: E731
    out = {}
    for fam, p, n_e in (("lagrange", 3, 4), ("bspline", 2, 4)):
        grid = A.Grid.build(geom, B.BasisSpec(family=fam, p=p, n_e=n_e), boundary_fitted=True)
        ts = A.TensorSystem(grid)
        M = ts.mass_matrix()
        K = ts.stiffness_operator()
        F = A.spatial_load(grid, src, alpha=1.0)
        obs = H.observer_matrix(grid)
        lam, it = LA.max_gen_eig(tensor_csr_ref(ts), M,
                                 tol=1e-7, seed=0)
        dt = 0.9 * 2.0 / np.sqrt(lam)
        r = T.cdm_run(M, K, F, f, dt, 150, obs_mat=obs)
        dtn = 4.0 * dt
        rn = T.newmark_run(M, K, F, f, dtn, 60, obs_mat=obs,
                           s_factory=lambda: ts.newmark_factorization(0.25, dtn))
        k = fam[0]
        out.update({f"{k}_m1": ts.m1, f"{k}_k1": ts.k1, f"{k}_p": p, f"{k}_n_e": n_e, f"{k}_h": grid.h,
                    f"{k}_F": F, f"{k}_lam": lam, f"{k}_it": it, f"{k}_dt": dt, f"{k}_psi": r.psi,
                    f"{k}_obs": r.obs, f"{k}_dtn": dtn, f"{k}_nm_psi": rn.psi, f"{k}_nm_obs": rn.obs,
                    f"{k}_nm_v": rn.psi_dot},
                   **csr_parts(f"{k}_obs", obs), **csr_parts(f"{k}_M", M))
        print(fam, sp.csr_matrix(M).nnz, lam, it)
    save("tensor", **out)


def gen_evs():
    """jacobi_eig and evs_stabilize of the reference on a batch of SPD
    matrices with clustered small eigenvalues (badly cut cell masses) and on
    real cut-cell masses of the rotated cube (p=2, n_e=4, alpha 1e-8)."""
    rng = np.random.default_rng(11)
    n, B = 27, 12
    Q = np.linalg.qr(rng.standard_normal((B, n, n)))[0]
    lam = np.exp(rng.uniform(np.log(1e-9), 0.0, (B, n)))
    A = np.einsum("bik,bk,bjk->bij", Q, lam, Q)
    Mf = A + 0.1 * np.eye(n)
    lam_r, V_r = LA.jacobi_eig(A)
    evs = S.evs_stabilize(A, Mf, 0.1, 1e-2)
    geom = G.ImmersedGeometry.from_angles(0.3, 0.5, (10.0, 10.0, 10.0))
    grid = A_.Grid.build(geom, B_.BasisSpec(family="lagrange", p=2, n_e=4))
    cache = A_.ElementIntegralCache(grid, octree_depth=2)
    cut = [tuple(int(v) for v in ijk) for ijk in grid.kept
           if grid.classes[tuple(ijk)] == G.ElementClass.CUT][:16]
    Mo_c, Mf_c = [], []
    for ijk in cut:
        M_o, K_o, M_f, K_f = A_.element_matrices(grid, ijk, 1e-8, cache=cache)
        Mo_c.append(M_o)
        Mf_c.append(M_f)
    Mo_c, Mf_c = np.array(Mo_c), np.array(Mf_c)
    evs_c = S.evs_stabilize(Mo_c, Mf_c, 0.01, 1e-2)
    save("evs", A=A, Mf=Mf, lam=lam_r, V=V_r, evs=evs, Mo_c=Mo_c, Mf_c=Mf_c, evs_c=evs_c)


def tensor_csr_ref(ts):
    m, k = sp.csr_matrix(ts.m1), sp.csr_matrix(ts.k1)
    return ts.rho * ts.c ** 2 * (sp.kron(sp.kron(k, m), m) + sp.kron(sp.kron(m, k), m)
                                 + sp.kron(sp.kron(m, m), k)).tocsr()


if __name__ == "__main__" and len(sys.argv) > 1:
    for name in sys.argv[1:]:
        globals()[f"gen_{name}"]()
elif __name__ == "__main__":
    gen_bar()
    gen_scalar()
    gen_rand10()
    gen_basis()
    gen_lumping()
    gen_cube("cube_p2n4", p=2, n_e=4, alpha=1e-6, depth=2, n_t=300, store_csr=True)
    gen_cube("cube_p3n6", p=3, n_e=6, alpha=1e-8, depth=3, n_t=200, store_csr=False)
    gen_cube_imex("cube_imex_p2n4", p=2, n_e=4, alpha=1e-12, depth=2, n_t=150)
    gen_cube_imex("cube_imex_p2n4_a4", p=2, n_e=4, alpha=1e-4, depth=2, n_t=150)
    gen_bspline_cube("bspline_cube_p2n5", p=2, n_e=5, alpha=1e-6, depth=2)
    gen_tensor()
    gen_paper()
    gen_evs()
