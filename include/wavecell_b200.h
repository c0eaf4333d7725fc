/*
 * wavecell_b200.h -- C ABI of the B200 (sm_100a) explicit wave-stepping hot path.
 *
 * The reference (`wavecell`, arXiv 2501.19013) is a pure-Python package whose
 * time-marching loop runs in SciPy's C++ CSR matvec.  Its "FFI boundary" is the
 * Python function API of `wavecell.timeint` / `wavecell.linalg`; every entry
 * point below replaces one of those functions (or the operator object it
 * consumes) and is bound from Python through ctypes by
 * `paper_2501_19013_b200/_lib.py` (see INTEGRATION.md for the binding stub).
 *
 * Conventions
 *   - Plain C types only: host pointers, int64 sizes, fp64 values.  No torch
 *     or CUDA types cross the boundary (the stream is exported as void*).
 *   - Vectors are in the reference's *compact DOF order*
 *     (src/assembly.py:159-180, lex = (fx*n1 + fy)*n1 + fz, x slowest).
 *   - All inputs are deep-copied to the device; inputs are never mutated
 *     (the reference copies psi0/v0, src/timeint.py:162-164).
 *   - Every function returns a WCB_* status code; wcb_last_error() gives a
 *     thread-local message.  The Python shim re-raises the reference's
 *     exception types (DivergenceError, RuntimeError, ValueError).
 *   - Calls are synchronous with respect to the host: when a call returns,
 *     its outputs are in the caller's buffers.
 */
#ifndef WAVECELL_B200_H
#define WAVECELL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WCB_ABI_VERSION 2

enum wcb_status {
    WCB_OK = 0,
    WCB_E_ARG = 1,          /* invalid argument -> ValueError                        */
    WCB_E_CUDA = 2,         /* CUDA runtime failure -> RuntimeError                  */
    WCB_E_DIVERGED = 3,     /* max|psi| > 1e12 or non-finite -> DivergenceError       */
    WCB_E_NOCONV = 4,       /* power iteration hit max_iter -> RuntimeError           */
    WCB_E_UNSUPPORTED = 5   /* operator/shape combination not built -> NotImplemented */
};

typedef struct wcb_context wcb_context;    /* one device + one stream + events      */
typedef struct wcb_operator wcb_operator;  /* device-resident stiffness K            */
typedef struct wcb_cdm_plan wcb_cdm_plan;  /* device-resident M, F_s, observers      */
typedef struct wcb_imex_plan wcb_imex_plan;/* device-resident IMEX split + S_cc LU   */

/* StageTimings, src/timeint.py:46-56 (seconds, from CUDA events). */
typedef struct {
    double factorization;
    double rhs;
    double backward_insertion;
} wcb_timings;

/* DivergenceError(step, amplitude), src/timeint.py:36-43,91-94. */
typedef struct {
    int64_t step;        /* first step k with max|psi_k| > 1e12 or non-finite; -1 if none */
    double amplitude;    /* max|psi_k| at that step                                   */
} wcb_divergence;

/* Observer matrix obs_mat (CSR, n_obs x n_dof), src/timeint.py:97-106,
 * src/harness.py:59-98.  Entries are summed in stored order. */
typedef struct {
    int64_t n_obs;
    const int64_t* indptr;   /* n_obs + 1 */
    const int64_t* indices;  /* nnz, compact DOF ids */
    const double* data;      /* nnz */
} wcb_observer;

/* Matrix-free spectral-cell (GLL Lagrange) stiffness on a Cartesian grid.
 * Uncut cells: sk * (k1 (x) m1 [(x) m1] + ...) applied by sum factorisation
 *   (src/assembly.py:263-295, TensorSystem.k_matvec src/assembly.py:674-684).
 * Cut cells: dense physical K_o = sk (K_in + alpha K_out) per cell
 *   (src/assembly.py:575-583), local DOF order z fastest (src/assembly.py:85-89). */
typedef struct {
    int32_t dim;                 /* 2 or 3                                              */
    int32_t p;                   /* polynomial degree (2D: 1..6, 3D: 1..4)              */
    int64_t n_e[3];              /* cells per axis, axis 0 slowest (x)                 */
    const double* k1;            /* (p+1)^2 row-major 1D GL-exact stiffness (reference) */
    const double* m1;            /* (p+1)^2 row-major 1D GL-exact mass (reference)      */
    double sk;                   /* rho c^2 (h/2)^(dim-2), src/assembly.py:504-505      */
    const int8_t* cell_class;    /* prod(n_e) ElementClass (0 out,1 in,2 cut), lex      */
    int64_t n_dof;               /* compact DOFs                                        */
    const int64_t* lex_of_compact; /* n_dof node lex ids (src/assembly.py:173)          */
    int64_t n_cut;               /* number of cut cells                                 */
    const int64_t* cut_cells;    /* n_cut cell lex ids, ascending                       */
    const double* cut_K;         /* n_cut * L * L physical element stiffness, L=(p+1)^dim */
    /* x slab (multi-GPU); x_cell_hi = 0 means the whole grid.  A
     * slab owns cell rows [x_cell_lo, x_cell_hi) and node rows
     * [x_cell_lo*p, x_cell_hi*p) (+ row n_e*p if x_owns_last).  cell_class then
     * covers the existing cell rows of [x_cell_lo-1, x_cell_hi), lex_of_compact
     * the owned DOFs (global lex), cut_cells the cut cells of those rows. */
    int64_t x_cell_lo;
    int64_t x_cell_hi;
    int32_t x_owns_last;
} wcb_scm_desc;

/* Matrix-free plane-strain elastic stiffness on the SCM node grid (BASELINE
 * config 4; the reference has no vector operator).  DOFs are
 * component major: dof = comp * n_node + node (node = scalar compact id).
 * Uncut cells: [[(l+2m) k1(x)m1 + m m1(x)k1, l g1(x)g1^T + m (g1(x)g1^T)^T],
 * [.^T, m k1(x)m1 + (l+2m) m1(x)k1]] by sum factorisation, g1[a][b] =
 * int phi_a' phi_b.  Cut cells: dense physical matrices, L = 2 (p+1)^2,
 * local order (comp, x-node, y-node), src/assembly.py:575-583 applied to
 * each derivative pairing. */
typedef struct {
    int32_t p;                   /* 1..5                                                */
    int64_t n_e[2];              /* cells per axis (equal)                              */
    double lam, mu;              /* Lame parameters (plane strain)                      */
    const double* m1;            /* (p+1)^2 GL-exact 1D mass                             */
    const double* k1;            /* (p+1)^2 GL-exact 1D stiffness                        */
    const double* g1;            /* (p+1)^2 GL-exact int phi_a' phi_b                    */
    const int8_t* cell_class;    /* n_e^2 ElementClass, lex                              */
    int64_t n_node;              /* compact nodes (DOFs = 2 n_node)                      */
    const int64_t* lex_of_compact; /* n_node node lex ids, ascending                     */
    int64_t n_cut;
    const int64_t* cut_cells;    /* n_cut cell lex ids, ascending                        */
    const double* cut_K;         /* n_cut * L * L, L = 2 (p+1)^2                          */
    /* x slab as in wcb_scm_desc (x_cell_hi == 0: the whole grid); n_node,
     * lex_of_compact, cell_class and cut_cells then describe the slab's nodes
     * and the cell rows [x_cell_lo-1, x_cell_hi) */
    int64_t x_cell_lo;
    int64_t x_cell_hi;
    int32_t x_owns_last;
} wcb_elastic_desc;

/* ---- library / context ------------------------------------------------- */
int wcb_abi_version(void);
const char* wcb_last_error(void);
int wcb_device_count(int* out);
int wcb_context_create(int device, wcb_context** out);
int wcb_context_destroy(wcb_context* ctx);
void* wcb_context_stream(wcb_context* ctx);        /* cudaStream_t of the context          */
int64_t wcb_context_launches(wcb_context* ctx);    /* kernels launched so far (counter)     */

/* ---- operators: replace the K consumed by the integrators ---------------- */
/* scipy CSR K from assemble()/_to_csr, src/assembly.py:518-612 (IGA and generic path). */
int wcb_operator_csr_create(wcb_context* ctx, int64_t n, const int64_t* indptr,
                            const int32_t* indices, const double* data,
                            wcb_operator** out);
/* Matrix-free SCM K (replaces the CSR K of Lagrange systems, src/assembly.py:554-583). */
int wcb_operator_scm_create(wcb_context* ctx, const wcb_scm_desc* desc, wcb_operator** out);
/* Matrix-free plane-strain K (config 4; used by imex_run / cdm_run as any K). */
int wcb_operator_elastic_create(wcb_context* ctx, const wcb_elastic_desc* desc, wcb_operator** out);
int wcb_operator_destroy(wcb_operator* op);
int64_t wcb_operator_n(const wcb_operator* op);
/* y = K @ x on host buffers (K.__matmul__, src/timeint.py:175,182). */
int wcb_operator_apply(wcb_operator* op, const double* x, double* y);
/* Halo layout of a slab operator (state rows of xstride doubles):
 * out[0] xstride, out[1] top halo first row, out[2] top halo rows (p or 0),
 * out[3] bottom halo row, out[4] bottom halo rows (1 or 0), out[5] first row
 * sent to the next slab, out[6] rows sent (p or 0), out[7] row sent to the
 * previous slab (1 row).  Returns 1 for a slab of a larger grid, else 0. */
int wcb_operator_halo(const wcb_operator* op, int64_t* out8);
/* Name of the kernel(s) one fused time step of this operator launches
 * (NUL-terminated, truncated to cap bytes) -- for bench and profile labels. */
int wcb_operator_step_kernel(const wcb_operator* op, char* out, int64_t cap);

/* ---- multi-GPU slabs: NCCL communicator per context -------- */
/* imex_run over consecutive x slabs of one plane-strain grid emulated in one
 * process (plans share one context; halos by device copies after every step).
 * Per plan: psi_out (its DOFs), psi_dot_out (its v_c, may be NULL), obs_out
 * (its observer partial sums, n_obs x (n_t+1), may be NULL). */
int wcb_imex_group_run(int n_plans, wcb_imex_plan** plans, double f0, const double* ft_k,
                       const double* ft_new, double dt, int64_t n_t, double beta, double gamma,
                       double** psi_out, double** psi_dot_out, double** obs_out,
                       wcb_divergence* div, wcb_timings* tm);
/* Halo exchange with the +-1 slab neighbours after every step and all-reduces
 * of the divergence amplitude / observer partial sums run on the context's
 * stream.  NCCL is loaded with dlopen("libnccl.so.2"). */
int wcb_dist_unique_id(char* out128);
int wcb_dist_init(wcb_context* ctx, int rank, int world, const char* id128);
int wcb_dist_finalize(wcb_context* ctx);
/* Single-process emulation of a slab group (all plans on one context): the
 * same kernels and halo layout, exchanges done by device copies.  Outputs are
 * per plan (owned DOFs); obs_out receives the sum of the partial observers. */
int wcb_cdm_group_run(int n_plans, wcb_cdm_plan** plans, const double* ft, double dt,
                      int64_t n_t, double** psi_out, double* obs_out,
                      wcb_divergence* div, wcb_timings* tm);

/* ---- critical time step: max_gen_eig, src/linalg.py:89-122 --------------- */
/* Power iteration on M^-1 K with diagonal M; x0 is the normalised seeded start
 * vector (src/linalg.py:103-105).  Returns WCB_E_NOCONV after max_iter. */
int wcb_max_gen_eig(wcb_operator* K, const double* m_diag, const double* x0,
                    double tol, int64_t max_iter, double* lam, int64_t* n_iter);
/* Power iteration on the principal sub-problem (K_ss, M_ss), s = sub_idx
 * (ascending compact ids): imex_critical_time_step's d subsystem,
 * src/timeint.py:80-88, without forming K_dd.  m_diag holds n entries (only
 * the sub entries are read), x0_sub the n_sub-long start vector. */
int wcb_max_gen_eig_sub(wcb_operator* op, const double* m_diag, int64_t n_sub,
                        const int64_t* sub_idx, const double* x0_sub, double tol,
                        int64_t max_iter, double* out_lambda, int64_t* out_iters);

/* Host-side check of factorize()'s diagonal fast path (src/linalg.py:63-69)
 * for a CSR mass matrix, multi-threaded: returns 1 when the pattern is exactly
 * the diagonal in order and every stored value is positive and finite, 0 when
 * the pattern is the diagonal but a value is not positive/finite, -1 when the
 * pattern is not the identity (the caller falls back to a general check).
 * index_bytes = 4 or 8 for indptr / indices. */
int wcb_csr_diagonal_check(int64_t n, const void* indptr, const void* indices, int index_bytes,
                           const double* data);

/* ---- central difference method: cdm_run, src/timeint.py:159-193 ---------- */
/* Diagonal M only (the factorize() fast path, src/linalg.py:63-69).  F_s may be
 * sparse: only its nonzeros are kept on the device. */
int wcb_cdm_plan_create(wcb_operator* K, const double* m_diag, const double* F_s,
                        const wcb_observer* obs, wcb_cdm_plan** out);
int wcb_cdm_plan_destroy(wcb_cdm_plan* plan);
/* ft[k] = f_t(k*dt) for k = 0..n_t-1 (f_t(0.0) == ft[0] is the bootstrap force).
 * psi0 / v0 may be NULL (zeros).  obs_out is n_obs x (n_t+1) row-major or NULL.
 * Returns WCB_E_DIVERGED with *div filled on divergence. */
int wcb_cdm_plan_run(wcb_cdm_plan* plan, const double* ft, double dt, int64_t n_t,
                     const double* psi0, const double* v0, double* psi_out,
                     double* obs_out, wcb_divergence* div, wcb_timings* tm);
/* Same run with the observers recorded every record_every steps only:
 * obs_out is n_obs x (n_t / record_every + 1), column j = obs at step
 * j * record_every -- the exact-hit samples of sample_observers
 * (src/harness.py:101-131) without moving the full history. */
int wcb_cdm_plan_run_sampled(wcb_cdm_plan* plan, const double* ft, double dt, int64_t n_t,
                             int64_t record_every, const double* psi0, const double* v0,
                             double* psi_out, double* obs_out, wcb_divergence* div, wcb_timings* tm);
/* Algorithmic bytes one fused time step of this plan moves: 32 B per DOF
 * (psi_k, psi_{k-1}, 1/m, psi_{k+1}) less 8 B per DOF whose 1/m the kernel
 * takes from the interior-cell table (bitwise-checked at plan creation), plus
 * the operator's own data (cut-cell matrices, CSR arrays). */
int wcb_cdm_plan_step_bytes(const wcb_cdm_plan* plan, double* out);
/* Same loop on device-resident buffers (cudaMalloc'd by the caller on the
 * context's device): d_ft (n_t), d_psi0/d_v0 (n, may be NULL), d_psi_out (n),
 * d_obs_out (n_obs*(n_t+1) or NULL).  Used by bench.py for the HBM-resident
 * number; synchronous on return. */
int wcb_cdm_plan_run_device(wcb_cdm_plan* plan, const double* d_ft, double dt,
                            int64_t n_t, const double* d_psi0, const double* d_v0,
                            double* d_psi_out, double* d_obs_out,
                            wcb_divergence* div, wcb_timings* tm);

/* ---- implicit-explicit split: imex_run, src/timeint.py:196-292 ----------- */
/* d rows: diagonal mass m_d (src/timeint.py:223-236); c rows: S_cc = M_cc +
 * beta dt^2 K_cc prefactorised on the host as Pr S_cc Pc = L U (SuperLU,
 * src/linalg.py:70-80) and M_cc likewise; both triangular solves run on the
 * device every step.  Factors are CSR (L unit-lower, U upper incl. diagonal). */
typedef struct {
    int64_t n;                      /* factor dimension                           */
    const int64_t* perm_r;          /* row permutation: (Pr b)[perm_r[i]] = b[i]    */
    const int64_t* perm_c;          /* col permutation: x[i] = z[perm_c[i]]         */
    const int64_t* L_indptr; const int32_t* L_indices; const double* L_data;
    const int64_t* U_indptr; const int32_t* U_indices; const double* U_data;
} wcb_lu;

/* S_cc may be NULL (a mass-only plan, see wcb_mass_plan_create). */
int wcb_imex_plan_create(wcb_operator* K, int64_t n_c, const int64_t* c_idx,
                         int64_t n_d, const int64_t* d_idx, const double* m_d,
                         const wcb_lu* S_cc, const wcb_lu* M_cc, const double* F_s,
                         const wcb_observer* obs, wcb_imex_plan** out);
int wcb_imex_plan_destroy(wcb_imex_plan* plan);
/* ft_k[k] = f_t(k*dt), ft_new[k] = f_t(k*dt + dt) (src/timeint.py:259-260),
 * f0 = f_t(0.0).  psi_dot_out (n_c, may be NULL) receives the final v_c in
 * c order (the reference returns it scattered when d is empty, :285-288). */
int wcb_imex_plan_run(wcb_imex_plan* plan, double f0, const double* ft_k,
                      const double* ft_new, double dt, int64_t n_t, double beta,
                      double gamma, const double* psi0, const double* v0,
                      double* psi_out, double* psi_dot_out, double* obs_out,
                      wcb_divergence* div, wcb_timings* tm);

/* ---- consistent (non-diagonal) mass: factorize()'s SuperLU path ------------
 * src/linalg.py:70-80 as used by cdm_run (src/timeint.py:166-176) and
 * max_gen_eig (src/linalg.py:106-116) when M is not diagonal.  A symmetric M
 * splits into the rows that store only their diagonal (d, m_d) and the rest
 * (c); M = blockdiag(diag(m_d), M_cc) after permutation, M_cc prefactorised on
 * the host (wcb_lu) and also passed as CSR in c order (for x'Mx).  The plan is
 * an IMEX plan without S_cc factors. */
int wcb_mass_plan_create(wcb_operator* K, int64_t n_c, const int64_t* c_idx, int64_t n_d,
                         const int64_t* d_idx, const double* m_d, const wcb_lu* M_cc,
                         const int64_t* Mcc_indptr, const int32_t* Mcc_indices, const double* Mcc_data,
                         const double* F_s, const wcb_observer* obs, wcb_imex_plan** out);
/* cdm_run with that mass: ft[k] = f_t(k*dt), k = 0..n_t-1 (as wcb_cdm_plan_run);
 * per step the d rows by the fused explicit step, the c rows by
 * (f F - K psi_k)_c, the two M_cc triangular solves and the leapfrog update. */
int wcb_imex_plan_cdm_run(wcb_imex_plan* plan, const double* ft, double dt, int64_t n_t,
                          const double* psi0, const double* v0, double* psi_out, double* obs_out,
                          wcb_divergence* div, wcb_timings* tm);
/* max_gen_eig(K, M) with that mass (x0 = the seeded start vector, n entries). */
int wcb_imex_plan_max_gen_eig(wcb_imex_plan* plan, const double* x0, double tol, int64_t max_iter,
                              double* lam, int64_t* n_iter);

/* ---- eigenvalue stabilisation -----------------------------
 * jacobi_eig, src/linalg.py:133-212: batched cyclic Jacobi on the device (n
 * symmetric L x L matrices, L <= 100): lam (n x L ascending), V (n x L x L,
 * eigenvectors as columns).  WCB_E_NOCONV after max_sweeps. */
int wcb_jacobi_eig(wcb_context* ctx, int64_t n, int L, const double* A, int max_sweeps, double tol,
                   double* lam, double* V);
/* evs_stabilize, src/stabilization.py:73-102, in place on the n consistent
 * cut-cell masses M_o (n x L x L); mf_absmax[b] = max |M_f| of cell b. */
int wcb_evs_stabilize(wcb_context* ctx, int64_t n, int L, double* M_o, const double* mf_absmax,
                      double epsilon, double f_lambda);

/* ---- native host set-up, voids = union of open balls in [0,1]^d ----
 * Host-only, multi-threaded C++ (no device).  Replaces the Python set-up of
 * the ball-void geometries (setup/geometry.py BallVoids, setup/cutcell.py),
 * restating src/geometry.py:36-41,316-346 and src/assembly.py:310-423,575-592. */
/* cls[n_e^dim] = 0 outside / 1 inside / 2 cut (before the sliver rule). */
int wcb_setup_ball_classify(int dim, int64_t n_e, int64_t n_balls, const double* centers, const double* radii,
                            int8_t* cls);
/* The sliver rule (src/assembly.py:187-211) on the cut cells (lex ids): sample
 * certificate, then the physical fraction by 2^dim-section to `depth`;
 * discard[i] = 1 when cut cell i keeps less than min_fraction. */
int wcb_setup_ball_slivers(int dim, int64_t n_e, int64_t n_balls, const double* centers, const double* radii,
                           int64_t n_cut, const int64_t* cut_cells, double min_fraction, int depth,
                           uint8_t* discard);
/* Compact DOF map of a classified Lagrange grid (src/assembly.py:159-180):
 * lex_of_compact = NULL counts (returns n_dof, *n_c = number of c DOFs);
 * then lex_of_compact (n_dof), c_idx (n_c, compact ids) and optionally d_idx
 * (n_dof - n_c) and compact_of_lex ((p n_e + 1)^dim, -1 off the DOFs) are
 * filled.  Negative return: -WCB_E_ARG. */
int64_t wcb_setup_dofmap(int dim, int p, int64_t n_e, const int8_t* cls, int64_t* lex_of_compact,
                         int64_t* c_idx, int64_t* n_c, int64_t* d_idx, int64_t* compact_of_lex);
/* Lumped diagonal mass: sm * GLL weight products from the inside cells of
 * every DOF plus the lumped cut-cell vectors cut_M (n_cut x L) in cut-cell
 * order (src/assembly.py:586-592). */
int wcb_setup_lumped_mass(int dim, int p, int64_t n_e, const int8_t* cls, const double* w, double sm,
                          int64_t n_dof, const int64_t* lex_of_compact, int64_t n_cut, const int64_t* cut_cells,
                          const double* cut_M, const int64_t* compact_of_lex, double* m);
/* Cut-cell integrals of the listed cells (lex ids): K_out (n_cells x L x L)
 * = sk (K_in + alpha K_out); M_out = sm (M_in + alpha M_out) consistent
 * (lumping 0, n_cells x L x L), HRZ (1) or row-sum (2) lumped (n_cells x L).
 * Tables: the dyadic 1D tables of setup/basis.py (offsets[depth+1]; per
 * interval q GL points xi, weights w, values V and derivatives D (q x N),
 * m1 / k1 (N x N)).  nthreads <= 0: all host threads (capped at 32). */
int wcb_setup_ball_cut_cells(int dim, int p, int64_t n_e, int64_t n_balls, const double* centers,
                             const double* radii, int depth, int q, const int64_t* offsets, const double* xi,
                             const double* w, const double* V, const double* D, const double* m1,
                             const double* k1, int64_t n_cells, const int64_t* cells, double alpha, double sk,
                             double sm, int lumping, int nthreads, double* K_out, double* M_out);

#ifdef __cplusplus
}
#endif
#endif /* WAVECELL_B200_H */
