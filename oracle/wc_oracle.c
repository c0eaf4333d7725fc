/*
 * wc_oracle.c -- CPU restatement of the reference hot path (TEST
 * INFRASTRUCTURE / CPU BASELINE ONLY; never linked into the product).
 *
 *  - wco_scm_csr: global CSR stiffness of a spectral-cell system from its
 *    structured description, i.e. the reference's assemble()/_to_csr
 *    (src/assembly.py:518-612): uncut kept cells contribute
 *    sk * sum_k (m1 (x) .. k1 (x) .. m1) (src/assembly.py:285-288), cut cells
 *    their dense K_o (src/assembly.py:582); duplicate entries are summed.
 *  - wco_cdm_run: the CDM loop of src/timeint.py:159-193 on that CSR with a
 *    diagonal mass (factorize() fast path, src/linalg.py:63-69), row-parallel
 *    with OpenMP (SciPy's csr_matvec is the same row loop, single-threaded).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* local index of node coordinate along one axis inside cell e: a in 0..p */
static inline double kron_entry(int dim, int p, const double* k1, const double* m1,
                                const int* ra, const int* ca) {
    /* sum_k prod_j (j == k ? k1 : m1)[ra[j], ca[j]] */
    const int N = p + 1;
    double s = 0.0;
    for (int k = 0; k < dim; ++k) {
        double prod = 1.0;
        for (int j = 0; j < dim; ++j) {
            const double* A = (j == k) ? k1 : m1;
            prod *= A[ra[j] * N + ca[j]];
        }
        s += prod;
    }
    return s;
}

/* Count (pass 0) or fill (pass 1) the CSR of a Lagrange SCM system.
 * cell_class: n_e^dim (0 out, 1 in, 2 cut); compact_of_lex: n1^dim (-1 none);
 * cut_index: n_e^dim -> index into cut_K or -1. */
int64_t wco_scm_csr(int dim, int p, int64_t n_e, const double* k1, const double* m1, double sk,
                    const int8_t* cell_class, const int64_t* compact_of_lex,
                    const int64_t* lex_of_compact, int64_t n_dof, const int64_t* cut_index,
                    const double* cut_K, int64_t* indptr, int64_t* indices, double* data) {
    const int N = p + 1;
    int L = 1;
    for (int k = 0; k < dim; ++k) L *= N;
    const int64_t n1 = n_e * p + 1;
    const int pass = indices != NULL;
    int64_t total = 0;
#pragma omp parallel
    {
        const int cap = 1 << 14;
        int64_t* cols = (int64_t*)malloc(sizeof(int64_t) * cap);
        double* vals = (double*)malloc(sizeof(double) * cap);
        int64_t* uniq = (int64_t*)malloc(sizeof(int64_t) * cap);
#pragma omp for schedule(dynamic, 256) reduction(+ : total)
        for (int64_t r = 0; r < n_dof; ++r) {
            int64_t lex = lex_of_compact[r];
            int64_t I[3] = {0, 0, 0};
            for (int k = dim - 1; k >= 0; --k) { I[k] = lex % n1; lex /= n1; }
            int nc = 0;
            /* incident cells: per axis e = I/p and (I%p==0) e = I/p - 1 */
            int64_t ce[3][2];
            int cn[3];
            for (int k = 0; k < dim; ++k) {
                cn[k] = 0;
                int64_t e = I[k] / p;
                if (I[k] % p == 0 && e - 1 >= 0) ce[k][cn[k]++] = e - 1;
                if (e < n_e) ce[k][cn[k]++] = e;
            }
            int idx[3] = {0, 0, 0};
            for (;;) {
                int64_t cell[3] = {0, 0, 0};
                int64_t clex = 0;
                for (int k = 0; k < dim; ++k) { cell[k] = ce[k][idx[k]]; clex = clex * n_e + cell[k]; }
                int8_t cls = cell_class[clex];
                if (cls != 0) {
                    int ra[3];
                    int rloc = 0;
                    for (int k = 0; k < dim; ++k) { ra[k] = (int)(I[k] - cell[k] * p); rloc = rloc * N + ra[k]; }
                    for (int m = 0; m < L; ++m) {
                        int ca[3];
                        int t = m;
                        for (int k = dim - 1; k >= 0; --k) { ca[k] = t % N; t /= N; }
                        int64_t clx = 0;
                        for (int k = 0; k < dim; ++k) clx = clx * n1 + cell[k] * p + ca[k];
                        double v;
                        if (cls == 1) v = sk * kron_entry(dim, p, k1, m1, ra, ca);
                        else v = cut_K[(cut_index[clex] * L + rloc) * (int64_t)L + m];
                        cols[nc] = compact_of_lex[clx];
                        vals[nc] = v;
                        nc++;
                    }
                }
                int k = dim - 1;
                while (k >= 0 && ++idx[k] >= cn[k]) { idx[k] = 0; --k; }
                if (k < 0) break;
            }
            /* unique sorted columns, summing duplicates in cell order */
            memcpy(uniq, cols, sizeof(int64_t) * nc);
            qsort(uniq, nc, sizeof(int64_t), cmp_i64);
            int nu = 0;
            for (int i = 0; i < nc; ++i)
                if (nu == 0 || uniq[nu - 1] != uniq[i]) uniq[nu++] = uniq[i];
            if (!pass) {
                indptr[r + 1] = nu;
            } else {
                int64_t base = indptr[r];
                for (int i = 0; i < nu; ++i) { indices[base + i] = uniq[i]; data[base + i] = 0.0; }
                for (int i = 0; i < nc; ++i) {
                    int lo = 0, hi = nu - 1;
                    while (lo < hi) { int mid = (lo + hi) / 2; if (uniq[mid] < cols[i]) lo = mid + 1; else hi = mid; }
                    data[base + lo] += vals[i];
                }
            }
            total += nu;
        }
        free(cols); free(vals); free(uniq);
    }
    if (!pass) {
        indptr[0] = 0;
        for (int64_t r = 0; r < n_dof; ++r) indptr[r + 1] += indptr[r];
    }
    return total;
}

/* CDM, src/timeint.py:159-193.  Observers (CSR obs_ptr/obs_idx/obs_val,
 * n_obs rows; NULL for none) are recorded into obs_out (n_obs x (n_t+1))
 * every step as _Recorder does (src/timeint.py:97-106).  Returns the first
 * diverged step (max|psi| > 1e12 or non-finite) or 0. */
int64_t wco_cdm_run_obs(int64_t n, const int64_t* indptr, const int64_t* indices, const double* data,
                        const double* m, const double* F, const double* ft, double dt, int64_t n_t,
                        const double* psi0, const double* v0, double* psi_out, int nthreads,
                        int64_t n_obs, const int64_t* obs_ptr, const int64_t* obs_idx, const double* obs_val,
                        double* obs_out) {
    if (nthreads > 0) omp_set_num_threads(nthreads);
    double* psi = (double*)malloc(sizeof(double) * (n ? n : 1));
    double* prev = (double*)malloc(sizeof(double) * (n ? n : 1));
    double* nxt = (double*)malloc(sizeof(double) * (n ? n : 1));
    const double c = 0.5 * dt * dt, dt2 = dt * dt;
    int64_t diverged = 0;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double Ku = 0.0;
        const double p0 = psi0 ? psi0[i] : 0.0;
        for (int64_t j = indptr[i]; j < indptr[i + 1]; ++j) Ku += data[j] * (psi0 ? psi0[indices[j]] : 0.0);
        double a = (ft[0] * F[i] - Ku) / m[i];
        psi[i] = p0;
        prev[i] = p0 - dt * (v0 ? v0[i] : 0.0) + c * a;
    }
#define WCO_RECORD(col)                                                                    \
    for (int64_t r = 0; r < n_obs; ++r) {                                                  \
        double s = 0.0;                                                                    \
        for (int64_t j = obs_ptr[r]; j < obs_ptr[r + 1]; ++j) s += obs_val[j] * psi[obs_idx[j]]; \
        obs_out[r * (n_t + 1) + (col)] = s;                                                \
    }
    if (obs_out) { WCO_RECORD(0) }
    for (int64_t k = 0; k < n_t && !diverged; ++k) {
        const double f = ft[k];
        double amp = 0.0;
#pragma omp parallel for schedule(static) reduction(max : amp)
        for (int64_t i = 0; i < n; ++i) {
            double Ku = 0.0;
            for (int64_t j = indptr[i]; j < indptr[i + 1]; ++j) Ku += data[j] * psi[indices[j]];
            double rhs = f * F[i] - Ku;
            double v = 2.0 * psi[i] - prev[i] + dt2 * (rhs / m[i]);
            nxt[i] = v;
            double av = fabs(v);
            if (!(av <= 1.0e12)) av = INFINITY;
            if (av > amp) amp = av;
        }
        double* t = prev; prev = psi; psi = nxt; nxt = t;
        if (obs_out) { WCO_RECORD(k + 1) }
        if (amp > 1.0e12) diverged = k + 1;
    }
#undef WCO_RECORD
    memcpy(psi_out, psi, sizeof(double) * n);
    free(psi); free(prev); free(nxt);
    return diverged;
}

int64_t wco_cdm_run(int64_t n, const int64_t* indptr, const int64_t* indices, const double* data,
                    const double* m, const double* F, const double* ft, double dt, int64_t n_t,
                    const double* psi0, const double* v0, double* psi_out, int nthreads) {
    return wco_cdm_run_obs(n, indptr, indices, data, m, F, ft, dt, n_t, psi0, v0, psi_out, nthreads, 0, NULL,
                           NULL, NULL, NULL);
}

int wco_max_threads(void) { return omp_get_max_threads(); }
