// Native host set-up for void geometries made of balls:
// cell classification of the Cartesian grid and the alpha-independent
// cut-cell integrals, multi-threaded C++ (host code only).
//
// Restates, for the BallVoids plug-in of setup/geometry.py:
//   * BallVoids.classify_boxes (src/geometry.py:36-41 classes): a closed box
//     is CUT when it meets an open ball, OUTSIDE when one ball covers it,
//     INSIDE otherwise -- per ball over the cells of its bounding box;
//   * CutCellIntegrator.integrate (setup/cutcell.py; src/assembly.py:310-423):
//     recursive 2^d-section of the cell (src/geometry.py:316-346), settled
//     leaves as Kronecker products of the per-interval 1D tables (dyadic
//     tables, src/assembly.py:310-330), leaves still cut at the maximum depth
//     point by point at their Gauss points (src/assembly.py:380-423), the
//     physical and fictitious parts kept apart, then K_o = sk (K_in + alpha
//     K_out), M_o = sm (M_in + alpha M_out) and the cut-cell lumping
//     (src/assembly.py:575-592, HRZ src/stabilization.py:117-131).
// Sums are factorised axis by axis and grouped by the leaf's first-axis
// interval, so a p = 3 cut cell costs ~1e6 flops instead of ~2e7.
#include "wcb_internal.cuh"

#include <atomic>
#include <cmath>
#include <cstring>
#include <thread>

namespace wcb {
namespace {

struct Balls {
    int dim;
    std::vector<double> c, r2;   // centres (dim each), squared radii
    int64_t n() const { return (int64_t)r2.size(); }
};

enum { OUT = 0, IN = 1, CUTC = 2 };

// BallVoids.classify_boxes for one box against a ball subset
int classify_box(const Balls& B, const int64_t* sel, int64_t ns, const double* lo, const double* hi) {
    const int d = B.dim;
    bool touches = false, covered = false;
    for (int64_t t = 0; t < ns; ++t) {
        const double* c = B.c.data() + sel[t] * d;
        double near = 0.0, far = 0.0;
        for (int k = 0; k < d; ++k) {
            const double cl = std::min(std::max(c[k], lo[k]), hi[k]) - c[k];
            near += cl * cl;
            const double f = std::max(std::fabs(lo[k] - c[k]), std::fabs(hi[k] - c[k]));
            far += f * f;
        }
        touches |= near < B.r2[sel[t]];
        covered |= far < B.r2[sel[t]];
    }
    return covered ? OUT : touches ? CUTC : IN;
}

bool contains(const Balls& B, const int64_t* sel, int64_t ns, const double* x) {
    for (int k = 0; k < B.dim; ++k)
        if (!(x[k] >= 0.0 && x[k] <= 1.0)) return false;
    for (int64_t t = 0; t < ns; ++t) {
        const double* c = B.c.data() + sel[t] * B.dim;
        double s = 0.0;
        for (int k = 0; k < B.dim; ++k) s += (x[k] - c[k]) * (x[k] - c[k]);
        if (!(s >= B.r2[sel[t]])) return false;
    }
    return true;
}

// 1D tables of the dyadic intervals (setup/basis.py dyadic_tables)
struct Tables {
    int N = 0, q = 0, depth = 0;
    const int64_t* offsets = nullptr;   // depth + 1
    const double* xi = nullptr;         // n_int x q   (reference coordinates)
    const double* w = nullptr;          // n_int x q
    const double* V = nullptr;          // n_int x q x N
    const double* D = nullptr;          // n_int x q x N
    const double* m1 = nullptr;         // n_int x N x N
    const double* k1 = nullptr;         // n_int x N x N
};

// One cut cell.  Accumulators: for every integral X in {M, K} and part
// {in, out}, a full N^d x N^d matrix; settled leaves enter through
// per-first-axis-interval partial sums S[id0] of the remaining axes.
struct CellWork {
    int d, N, L, Lr;                         // Lr = N^(d-1)
    std::vector<double> acc;                 // [4][L][L]: M_in, M_out, K_in, K_out
    std::vector<double> S;                   // per (id0 slot, integral term, part): Lr x Lr partials
    std::vector<double> PG;                  // per (id0 slot, term, axis-0 Gauss point): pointwise partials
    std::vector<int64_t> ids0;               // distinct first-axis intervals seen
    std::vector<int64_t> sel;                // balls near the cell
    std::vector<double> blo, bhi, nlo, nhi;  // box lists of the tree walk
    std::vector<int> bcls;
};

// term t of the stiffness is axis t differentiated; term d is the mass.
// 1D factor of axis k for term t: k == t ? k1 : m1.

void cut_cell(const Balls& B, const Tables& T, int64_t n_e, int depth, int64_t cell, CellWork& W,
              double* M_in, double* M_out, double* K_in, double* K_out) {
    const int d = B.dim, N = T.N, q = T.q;
    const int L = W.L, Lr = W.Lr;
    const double h = 1.0 / (double)n_e;
    int64_t ijk[3] = {0, 0, 0};
    {
        int64_t c = cell;
        for (int k = d - 1; k >= 0; --k) { ijk[k] = c % n_e; c /= n_e; }
    }
    double lo[3], hi[3];
    for (int k = 0; k < d; ++k) {
        lo[k] = 0.0 + (double)ijk[k] * h;
        hi[k] = lo[k] + h;
    }
    // balls that reach the cell (BallVoids.restricted)
    W.sel.clear();
    for (int64_t t = 0; t < B.n(); ++t) {
        const double* c = B.c.data() + t * d;
        double near = 0.0;
        for (int k = 0; k < d; ++k) {
            const double cl = std::min(std::max(c[k], lo[k]), hi[k]) - c[k];
            near += cl * cl;
        }
        if (near < B.r2[t]) W.sel.push_back(t);
    }
    const int64_t* sel = W.sel.data();
    const int64_t ns = (int64_t)W.sel.size();
    std::fill(W.acc.begin(), W.acc.end(), 0.0);
    // first-axis interval slots: partial sums over the other axes
    // S layout: [slot][part 0..3 (M_in, M_out, K_in, K_out) x term][Lr][Lr]
    W.ids0.clear();
    const int nterms = d + 1;   // d stiffness terms (axis differentiated) + mass
    auto slot_of = [&](int64_t id0) -> double* {
        for (size_t s = 0; s < W.ids0.size(); ++s)
            if (W.ids0[s] == id0) return W.S.data() + s * (size_t)2 * nterms * Lr * Lr;
        W.ids0.push_back(id0);
        const size_t need = W.ids0.size() * (size_t)2 * nterms * Lr * Lr;
        if (W.S.size() < need) W.S.resize(need);
        const size_t pgs = (size_t)nterms * q * Lr * Lr;
        if (W.PG.size() < W.ids0.size() * pgs) W.PG.resize(W.ids0.size() * pgs);
        std::fill(W.PG.begin() + (W.ids0.size() - 1) * pgs, W.PG.begin() + W.ids0.size() * pgs, 0.0);
        double* p = W.S.data() + (W.ids0.size() - 1) * (size_t)2 * nterms * Lr * Lr;
        std::fill(p, p + (size_t)2 * nterms * Lr * Lr, 0.0);
        return p;
    };
    auto pg_of = [&](int64_t id0) -> double* {   // after slot_of(id0)
        for (size_t s = 0; s < W.ids0.size(); ++s)
            if (W.ids0[s] == id0) return W.PG.data() + s * (size_t)nterms * q * Lr * Lr;
        return nullptr;
    };
    // S[slot][part(0 in / 1 out)][term][Lr*Lr], term < d: axis `term` differentiated, term d: mass
    auto Sidx = [&](double* base, int part, int term) { return base + ((size_t)part * nterms + term) * Lr * Lr; };

    // tensor sum over the other axes (1 or 2) of a settled leaf: partial[(b,c),(e,f)]
    auto settle = [&](const int64_t* id, int part) {
        double* base = slot_of(id[0]);
        for (int term = 0; term <= d; ++term) {
            // factor of axis 0 is applied later (grouped by id0): here axes 1..d-1
            double* S = Sidx(base, part, term);
            const double* A1 = (term == 1 ? T.k1 : T.m1) + id[1] * N * N;
            if (d == 2) {
                for (int b = 0; b < N; ++b)
                    for (int e = 0; e < N; ++e) S[b * N + e] += A1[b * N + e];
            } else {
                const double* A2 = (term == 2 ? T.k1 : T.m1) + id[2] * N * N;
                for (int b = 0; b < N; ++b)
                    for (int c = 0; c < N; ++c)
                        for (int e = 0; e < N; ++e) {
                            const double ab = A1[b * N + e];
                            double* row = S + (size_t)(b * N + c) * Lr + e * N;
                            for (int f = 0; f < N; ++f) row[f] += ab * A2[c * N + f];
                        }
            }
        }
    };
    // pointwise part of a cut leaf at the maximum depth: physical quadrature
    // (inside points) into part 0 and the full leaf minus it into part 1
    auto cut_leaf = [&](const int64_t* id) {
        // inside flags of the q^d tensor points (last axis fastest)
        const int nq = d == 2 ? q * q : q * q * q;
        double wt[16 * 16 * 16];
        double x[3];
        for (int p = 0; p < nq; ++p) {
            int ii[3] = {0, 0, 0}, r = p;
            for (int k = d - 1; k >= 0; --k) { ii[k] = r % q; r /= q; }
            double w = 1.0;
            for (int k = 0; k < d; ++k) {
                const double xr = T.xi[id[k] * q + ii[k]];
                x[k] = lo[k] + (xr + 1.0) / 2.0 * (hi[k] - lo[k]);
                w *= T.w[id[k] * q + ii[k]];
            }
            wt[p] = contains(B, sel, ns, x) ? w : 0.0;
        }
        slot_of(id[0]);
        double* PGs = pg_of(id[0]);
        // per term: G_i[(b,c),(e,f)] += sum_{j,k} wt(i,j,k) A1[j,b]A1[j,e] A2[k,c]A2[k,f]
        // (axis 0 applied once per first-axis interval, after the walk)
        for (int term = 0; term <= d; ++term) {
            const double* A1 = (term == 1 ? T.D : T.V) + id[1] * q * N;
            const double* A2 = d == 3 ? (term == 2 ? T.D : T.V) + id[2] * q * N : nullptr;
            for (int i = 0; i < q; ++i) {
                double* G = PGs + ((size_t)term * q + i) * Lr * Lr;
                if (d == 2) {
                    for (int j = 0; j < q; ++j) {
                        const double wj = wt[i * q + j];
                        if (wj == 0.0) continue;
                        for (int b = 0; b < N; ++b)
                            for (int e = 0; e < N; ++e) G[b * N + e] += wj * A1[j * N + b] * A1[j * N + e];
                    }
                } else {
                    for (int j = 0; j < q; ++j) {
                        double tz[16 * 16];
                        bool any = false;
                        for (int cf = 0; cf < N * N; ++cf) tz[cf] = 0.0;
                        for (int k = 0; k < q; ++k) {
                            const double wk = wt[(i * q + j) * q + k];
                            if (wk == 0.0) continue;
                            any = true;
                            for (int c = 0; c < N; ++c)
                                for (int f = 0; f < N; ++f) tz[c * N + f] += wk * A2[k * N + c] * A2[k * N + f];
                        }
                        if (!any) continue;
                        for (int b = 0; b < N; ++b)
                            for (int e = 0; e < N; ++e) {
                                const double ab = A1[j * N + b] * A1[j * N + e];
                                for (int c = 0; c < N; ++c) {
                                    double* row = G + (size_t)(b * N + c) * Lr + e * N;
                                    for (int f = 0; f < N; ++f) row[f] += ab * tz[c * N + f];
                                }
                            }
                    }
                }
            }
        }
        // the full leaf (table Kronecker products) into the fictitious part;
        // the physical part is moved from there to "in" with the partials
        settle(id, 1);
    };

    // tree walk (setup/geometry.py tree_partition): level by level
    W.blo.assign(lo, lo + d);
    W.bhi.assign(hi, hi + d);
    for (int lev = 0; lev <= depth; ++lev) {
        const size_t nb = W.blo.size() / d;
        W.nlo.clear();
        W.nhi.clear();
        for (size_t bi = 0; bi < nb; ++bi) {
            const double* blo = W.blo.data() + bi * d;
            const double* bhi = W.bhi.data() + bi * d;
            const int cls = classify_box(B, sel, ns, blo, bhi);
            if (cls == CUTC && lev < depth) {
                const int nc = 1 << d;
                for (int ch = 0; ch < nc; ++ch)
                    for (int k = 0; k < d; ++k) {
                        const int bit = (ch >> (d - 1 - k)) & 1;   // last axis fastest
                        const double mid = 0.5 * (blo[k] + bhi[k]);
                        W.nlo.push_back(bit ? mid : blo[k]);
                        W.nhi.push_back(bit ? bhi[k] : mid);
                    }
                continue;
            }
            int64_t id[3];
            for (int k = 0; k < d; ++k) {
                const double A = 2.0 * (blo[k] - lo[k]) / (hi[k] - lo[k]) - 1.0;
                const int64_t pos = (int64_t)std::nearbyint((A + 1.0) / 2.0 * std::ldexp(1.0, lev));
                id[k] = T.offsets[lev] + pos;
            }
            if (cls == IN) settle(id, 0);
            else if (cls == OUT) settle(id, 1);
            else cut_leaf(id);
        }
        W.blo.swap(W.nlo);
        W.bhi.swap(W.nhi);
        if (W.blo.empty()) break;
    }
    // axis 0 of the settled partial sums: acc[(a,r),(dd,s)] += A0[id0][a][dd] S[r][s]
    for (size_t sidx = 0; sidx < W.ids0.size(); ++sidx) {
        const int64_t id0 = W.ids0[sidx];
        double* base = W.S.data() + sidx * (size_t)2 * nterms * Lr * Lr;
        for (int part = 0; part < 2; ++part)
            for (int term = 0; term <= d; ++term) {
                const double* A0 = (term == 0 ? T.k1 : T.m1) + id0 * N * N;
                const double* S = Sidx(base, part, term);
                double* acc = W.acc.data() + (size_t)((term == d ? 0 : 2) + part) * L * L;
                for (int a = 0; a < N; ++a)
                    for (int dd = 0; dd < N; ++dd) {
                        const double f0 = A0[a * N + dd];
                        for (int r = 0; r < Lr; ++r) {
                            double* o = acc + (size_t)(a * Lr + r) * L + dd * Lr;
                            const double* s = S + (size_t)r * Lr;
                            for (int c = 0; c < Lr; ++c) o[c] += f0 * s[c];
                        }
                    }
            }
    }
    // axis 0 of the pointwise partials: in += G, out -= G
    for (size_t sidx = 0; sidx < W.ids0.size(); ++sidx) {
        const int64_t id0 = W.ids0[sidx];
        const double* PGs = W.PG.data() + sidx * (size_t)nterms * q * Lr * Lr;
        for (int term = 0; term <= d; ++term) {
            const double* A0 = (term == 0 ? T.D : T.V) + id0 * q * N;
            double* acc_in = W.acc.data() + (size_t)(term == d ? 0 : 2) * L * L;
            double* acc_out = W.acc.data() + (size_t)(term == d ? 1 : 3) * L * L;
            for (int i = 0; i < q; ++i) {
                const double* G = PGs + ((size_t)term * q + i) * Lr * Lr;
                for (int a = 0; a < N; ++a)
                    for (int dd = 0; dd < N; ++dd) {
                        const double f0 = A0[i * N + a] * A0[i * N + dd];
                        if (f0 == 0.0) continue;
                        for (int r = 0; r < Lr; ++r) {
                            double* oi = acc_in + (size_t)(a * Lr + r) * L + dd * Lr;
                            double* oo = acc_out + (size_t)(a * Lr + r) * L + dd * Lr;
                            const double* g = G + (size_t)r * Lr;
                            for (int c = 0; c < Lr; ++c) {
                                const double v = f0 * g[c];
                                oi[c] += v;
                                oo[c] -= v;
                            }
                        }
                    }
            }
        }
    }
    std::memcpy(M_in, W.acc.data(), sizeof(double) * L * L);
    std::memcpy(M_out, W.acc.data() + (size_t)L * L, sizeof(double) * L * L);
    std::memcpy(K_in, W.acc.data() + (size_t)2 * L * L, sizeof(double) * L * L);
    std::memcpy(K_out, W.acc.data() + (size_t)3 * L * L, sizeof(double) * L * L);
}

}  // namespace
}  // namespace wcb

using namespace wcb;

extern "C" {

int wcb_setup_ball_classify(int dim, int64_t n_e, int64_t n_balls, const double* centers, const double* radii,
                            int8_t* cls) {
    if ((dim != 2 && dim != 3) || n_e <= 0 || n_balls < 0 || !cls || (n_balls && (!centers || !radii)))
        return WCB_E_ARG;
    const int d = dim;
    const int64_t n_cells = d == 2 ? n_e * n_e : n_e * n_e * n_e;
    std::memset(cls, IN, (size_t)n_cells);
    const double h = 1.0 / (double)n_e;
    // touched / covered flags from every ball over its bounding box of cells
    std::vector<uint8_t> touch((size_t)n_cells, 0), cover((size_t)n_cells, 0);
    for (int64_t t = 0; t < n_balls; ++t) {
        const double* c = centers + t * d;
        const double r = radii[t], r2 = r * r;
        int64_t a[3] = {0, 0, 0}, b[3] = {1, 1, 1};
        for (int k = 0; k < d; ++k) {
            a[k] = std::max<int64_t>(0, (int64_t)std::floor((c[k] - r) / h) - 1);
            b[k] = std::min<int64_t>(n_e, (int64_t)std::floor((c[k] + r) / h) + 2);
        }
        const int64_t nz = d == 3 ? b[2] - a[2] : 1;
        const int64_t z0 = d == 3 ? a[2] : 0;
        for (int64_t i = a[0]; i < b[0]; ++i)
            for (int64_t j = a[1]; j < b[1]; ++j)
                for (int64_t kk = 0; kk < nz; ++kk) {
                    const int64_t ijk[3] = {i, j, z0 + kk};
                    double near = 0.0, far = 0.0;
                    for (int k = 0; k < d; ++k) {
                        const double lo = 0.0 + (double)ijk[k] * h, hi = lo + h;
                        const double cl = std::min(std::max(c[k], lo), hi) - c[k];
                        near += cl * cl;
                        const double f = std::max(std::fabs(lo - c[k]), std::fabs(hi - c[k]));
                        far += f * f;
                    }
                    const int64_t idx = d == 2 ? i * n_e + j : (i * n_e + j) * n_e + z0 + kk;
                    if (near < r2) touch[idx] = 1;
                    if (far < r2) cover[idx] = 1;
                }
    }
    for (int64_t i = 0; i < n_cells; ++i) cls[i] = cover[i] ? OUT : touch[i] ? CUTC : IN;
    return WCB_OK;
}

// Physical cut-cell stiffness K_o = sk (K_in + alpha K_out) (n_cells x L x L)
// and mass: lumping 0 = consistent sm (M_in + alpha M_out) (n_cells x L x L),
// 1 = HRZ, 2 = row sum (n_cells x L).  Tables as setup/basis.py dyadic_tables
// for the Lagrange family (one signature for every cell).
int wcb_setup_ball_cut_cells(int dim, int p, int64_t n_e, int64_t n_balls, const double* centers,
                             const double* radii, int depth, int q, const int64_t* offsets, const double* xi,
                             const double* w, const double* V, const double* D, const double* m1,
                             const double* k1, int64_t n_cells, const int64_t* cells, double alpha, double sk,
                             double sm, int lumping, int nthreads, double* K_out, double* M_out) {
    if ((dim != 2 && dim != 3) || p < 1 || p > 8 || q < 1 || q > 16 || depth < 0 || !cells || !K_out || !M_out)
        return WCB_E_ARG;
    Balls B;
    B.dim = dim;
    B.c.assign(centers, centers + n_balls * dim);
    B.r2.resize(n_balls);
    for (int64_t t = 0; t < n_balls; ++t) B.r2[t] = radii[t] * radii[t];
    Tables T;
    T.N = p + 1;
    T.q = q;
    T.depth = depth;
    T.offsets = offsets;
    T.xi = xi;
    T.w = w;
    T.V = V;
    T.D = D;
    T.m1 = m1;
    T.k1 = k1;
    const int N = p + 1;
    const int L = dim == 2 ? N * N : N * N * N;
    const int Lr = dim == 2 ? N : N * N;
    if (nthreads <= 0) nthreads = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::atomic<int> bad{0};
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(nthreads, n_cells));
    std::vector<CellWork> works(nt);
    std::atomic<int64_t> next{0};
    auto worker = [&](int tix) {
        CellWork& Wk = works[tix];
        Wk.d = dim;
        Wk.N = N;
        Wk.L = L;
        Wk.Lr = Lr;
        Wk.acc.assign((size_t)4 * L * L, 0.0);
        std::vector<double> Mi(L * L), Mo(L * L), Ki(L * L), Ko(L * L);
        for (;;) {
            const int64_t e = next.fetch_add(1);
            if (e >= n_cells) break;
            if (cells[e] < 0) { bad = 1; continue; }
            cut_cell(B, T, n_e, depth, cells[e], Wk, Mi.data(), Mo.data(), Ki.data(), Ko.data());
            double* Kd = K_out + e * (int64_t)L * L;
            for (int i = 0; i < L * L; ++i) Kd[i] = sk * (Ki[i] + alpha * Ko[i]);
            std::vector<double>& Mc = Mi;   // M_o = sm (M_in + alpha M_out), in place
            for (int i = 0; i < L * L; ++i) Mc[i] = sm * (Mi[i] + alpha * Mo[i]);
            if (lumping == 0) {
                std::memcpy(M_out + e * (int64_t)L * L, Mc.data(), sizeof(double) * L * L);
            } else if (lumping == 1) {   // HRZ: diagonal scaled to the total element mass
                double tot = 0.0, dsum = 0.0;
                for (int r = 0; r < L; ++r)
                    for (int c = 0; c < L; ++c) tot += Mc[r * L + c];
                for (int r = 0; r < L; ++r) dsum += Mc[r * L + r];
                const double scale = tot / dsum;
                for (int r = 0; r < L; ++r) M_out[e * L + r] = Mc[r * L + r] * scale;
            } else {                     // row sum
                for (int r = 0; r < L; ++r) {
                    double s = 0.0;
                    for (int c = 0; c < L; ++c) s += Mc[r * L + c];
                    M_out[e * L + r] = s;
                }
            }
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(worker, t);
    worker(0);
    for (auto& x : th) x.join();
    return bad ? WCB_E_ARG : WCB_OK;
}

// The sliver rule (src/assembly.py:187-211, threshold src/geometry.py:33) for
// the cut cells of a ball-void grid, as setup/grid.py _discard_slivers:
// cells with an interior sample (4^d points) at distance >= 0.01 h from every
// void boundary certainly keep more than the threshold; the others get their
// physical fraction by adaptive 2^d-section (settled boxes exact, cut boxes
// at the last level by their centre, early exit once the certified inside
// volume exceeds the threshold).  discard[i] = 1: demote cut cell i.
int wcb_setup_ball_slivers(int dim, int64_t n_e, int64_t n_balls, const double* centers, const double* radii,
                           int64_t n_cut, const int64_t* cut_cells, double min_fraction, int depth,
                           uint8_t* discard) {
    if ((dim != 2 && dim != 3) || n_e <= 0 || n_cut < 0 || (n_cut && (!cut_cells || !discard)))
        return WCB_E_ARG;
    Balls B;
    B.dim = dim;
    B.c.assign(centers, centers + n_balls * dim);
    B.r2.resize(n_balls);
    for (int64_t t = 0; t < n_balls; ++t) B.r2[t] = radii[t] * radii[t];
    const int d = dim;
    const double h = 1.0 / (double)n_e;
    const int nth = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::atomic<int64_t> next{0};
    auto worker = [&] {
        std::vector<int64_t> sel;
        std::vector<double> blo, bhi, nlo, nhi;
        for (;;) {
            const int64_t e = next.fetch_add(1);
            if (e >= n_cut) break;
            int64_t c0 = cut_cells[e], ijk[3] = {0, 0, 0};
            for (int k = d - 1; k >= 0; --k) { ijk[k] = c0 % n_e; c0 /= n_e; }
            double lo[3], hi[3];
            for (int k = 0; k < d; ++k) { lo[k] = 0.0 + (double)ijk[k] * h; hi[k] = lo[k] + h; }
            // candidate test (BallVoids.sliver_candidates), every ball
            double best = -INFINITY;
            const int ns1 = 4, npts = d == 2 ? 16 : 64;
            for (int pt = 0; pt < npts; ++pt) {
                int ii[3] = {0, 0, 0}, r = pt;
                for (int k = d - 1; k >= 0; --k) { ii[k] = r % ns1; r /= ns1; }
                double x[3];
                for (int k = 0; k < d; ++k) x[k] = lo[k] + ((2.0 * ii[k] + 1.0) / 8.0) * h;
                double margin = INFINITY;
                for (int64_t t = 0; t < n_balls; ++t) {
                    double s2 = 0.0;
                    for (int k = 0; k < d; ++k) s2 += (x[k] - centers[t * d + k]) * (x[k] - centers[t * d + k]);
                    margin = std::min(margin, std::sqrt(s2) - radii[t]);
                }
                best = std::max(best, margin);
            }
            discard[e] = 0;
            if (!(best < 0.01 * h)) continue;
            // restricted geometry and the fraction by subdivision
            sel.clear();
            for (int64_t t = 0; t < n_balls; ++t) {
                double near = 0.0;
                for (int k = 0; k < d; ++k) {
                    const double cl = std::min(std::max(centers[t * d + k], lo[k]), hi[k]) - centers[t * d + k];
                    near += cl * cl;
                }
                if (near < B.r2[t]) sel.push_back(t);
            }
            double vol = 1.0;
            for (int k = 0; k < d; ++k) vol *= hi[k] - lo[k];
            double acc = 0.0;
            bool stopped = false;
            blo.assign(lo, lo + d);
            bhi.assign(hi, hi + d);
            for (int lev = 0; lev <= depth && !stopped; ++lev) {
                const size_t nb = blo.size() / d;
                nlo.clear();
                nhi.clear();
                double lev_in = 0.0;
                std::vector<size_t> cuts;
                for (size_t bi = 0; bi < nb; ++bi) {
                    const int cls = classify_box(B, sel.data(), (int64_t)sel.size(), &blo[bi * d], &bhi[bi * d]);
                    double w = 1.0;
                    for (int k = 0; k < d; ++k) w *= bhi[bi * d + k] - blo[bi * d + k];
                    if (cls == IN) lev_in += w;
                    else if (cls == CUTC) cuts.push_back(bi);
                }
                acc += lev_in;
                if (acc > min_fraction * vol) { stopped = true; break; }
                if (lev == depth) {
                    for (size_t bi : cuts) {
                        double x[3], w = 1.0;
                        for (int k = 0; k < d; ++k) {
                            x[k] = 0.5 * (blo[bi * d + k] + bhi[bi * d + k]);
                            w *= bhi[bi * d + k] - blo[bi * d + k];
                        }
                        if (contains(B, sel.data(), (int64_t)sel.size(), x)) acc += w;
                    }
                    break;
                }
                if (cuts.empty()) break;
                for (size_t bi : cuts) {
                    const double* bl = &blo[bi * d];
                    const double* bh = &bhi[bi * d];
                    for (int ch = 0; ch < (1 << d); ++ch)
                        for (int k = 0; k < d; ++k) {
                            const int bit = (ch >> (d - 1 - k)) & 1;
                            const double mid = 0.5 * (bl[k] + bh[k]);
                            nlo.push_back(bit ? mid : bl[k]);
                            nhi.push_back(bit ? bh[k] : mid);
                        }
                }
                blo.swap(nlo);
                bhi.swap(nhi);
            }
            discard[e] = (!stopped && acc / vol < min_fraction) ? 1 : 0;
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nth; ++t) th.emplace_back(worker);
    worker();
    for (auto& x : th) x.join();
    return WCB_OK;
}

// Compact DOF map of a classified Lagrange grid (src/assembly.py:159-180,
// setup/grid.py Grid.dofmap): a node is a DOF when one of its cells is kept
// (inside or cut), a c DOF when one of its cells is cut; lex = (I n1 + J) [n1
// + K].  Pass lex_of_compact = NULL to count: returns n_dof (>= 0) or an
// error code (< 0); *n_c receives the c count.  Threads over node rows.
int64_t wcb_setup_dofmap(int dim, int p, int64_t n_e, const int8_t* cls, int64_t* lex_of_compact,
                         int64_t* c_idx, int64_t* n_c, int64_t* d_idx, int64_t* compact_of_lex) {
    if ((dim != 2 && dim != 3) || p < 1 || n_e <= 0 || !cls) return -WCB_E_ARG;
    const int d = dim;
    const int64_t n1 = n_e * p + 1;
    const int64_t per_row = d == 2 ? n1 : n1 * n1;
    const int nth = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<int64_t> cnt(n1 + 1, 0), ccnt(n1 + 1, 0);
    // cells incident to node coordinate I along one axis: (I-1)/p .. I/p within range
    auto cells_of = [&](int64_t I, int64_t* e, int& ne) {
        ne = 0;
        if (I % p == 0) {
            if (I / p - 1 >= 0) e[ne++] = I / p - 1;
            if (I / p < n_e) e[ne++] = I / p;
        } else {
            e[ne++] = I / p;
        }
    };
    auto node_flags = [&](int64_t I, int64_t J, int64_t K, bool& kept, bool& cut) {
        int64_t ex[2], ey[2], ez[2] = {0, 0};
        int nx, ny, nz = 1;
        cells_of(I, ex, nx);
        cells_of(J, ey, ny);
        if (d == 3) cells_of(K, ez, nz);
        kept = cut = false;
        for (int a = 0; a < nx; ++a)
            for (int b = 0; b < ny; ++b)
                for (int c = 0; c < nz; ++c) {
                    const int8_t v = d == 2 ? cls[ex[a] * n_e + ey[b]] : cls[(ex[a] * n_e + ey[b]) * n_e + ez[c]];
                    kept |= v != OUT;
                    cut |= v == CUTC;
                }
    };
    auto pass = [&](bool fill) {
        std::atomic<int64_t> next{0};
        auto worker = [&] {
            for (;;) {
                const int64_t I = next.fetch_add(1);
                if (I >= n1) break;
                int64_t k = fill ? cnt[I] : 0, kc = fill ? ccnt[I] : 0;
                int64_t kd = fill ? cnt[I] - ccnt[I] : 0;
                for (int64_t r = 0; r < per_row; ++r) {
                    const int64_t J = d == 2 ? r : r / n1, K = d == 2 ? 0 : r % n1;
                    bool kept, cut;
                    node_flags(I, J, K, kept, cut);
                    if (!kept) {
                        if (fill && compact_of_lex) compact_of_lex[I * per_row + r] = -1;
                        continue;
                    }
                    if (fill) {
                        lex_of_compact[k] = I * per_row + r;
                        if (compact_of_lex) compact_of_lex[I * per_row + r] = k;
                        if (cut) c_idx[kc++] = k;
                        else if (d_idx) d_idx[kd++] = k;
                    } else if (cut) {
                        ++kc;
                    }
                    ++k;
                }
                if (!fill) { cnt[I + 1] = k; ccnt[I + 1] = kc; }
            }
        };
        std::vector<std::thread> th;
        for (int t = 1; t < nth; ++t) th.emplace_back(worker);
        worker();
        for (auto& x : th) x.join();
    };
    pass(false);
    for (int64_t I = 0; I < n1; ++I) { cnt[I + 1] += cnt[I]; ccnt[I + 1] += ccnt[I]; }
    if (n_c) *n_c = ccnt[n1];
    if (lex_of_compact && c_idx) pass(true);
    return cnt[n1];
}

// Lumped diagonal mass of a Lagrange cut-cell grid (setup/problem.py
// _assemble_mass): sm * prod_k w[a_k] from every inside cell of a node (in
// ascending local position), then the lumped cut-cell vectors in cut-cell
// order -- the same sums in the same order as the Python assembly.
int wcb_setup_lumped_mass(int dim, int p, int64_t n_e, const int8_t* cls, const double* w, double sm,
                          int64_t n_dof, const int64_t* lex_of_compact, int64_t n_cut, const int64_t* cut_cells,
                          const double* cut_M, const int64_t* compact_of_lex, double* m) {
    if ((dim != 2 && dim != 3) || p < 1 || n_e <= 0 || !cls || !w || !lex_of_compact || !m) return WCB_E_ARG;
    const int d = dim;
    const int64_t n1 = n_e * p + 1;
    const int nth = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::atomic<int64_t> next{0};
    auto worker = [&] {
        for (;;) {
            const int64_t i0 = next.fetch_add(4096);
            if (i0 >= n_dof) break;
            for (int64_t i = i0; i < std::min<int64_t>(n_dof, i0 + 4096); ++i) {
                const int64_t lex = lex_of_compact[i];
                int64_t X[3];
                int64_t r = lex;
                for (int k = d - 1; k >= 0; --k) { X[k] = r % n1; r /= n1; }
                // local positions ascending (a before a + p), last axis fastest
                int64_t la[3][2], ec[3][2];
                int nl[3];
                for (int k = 0; k < d; ++k) {
                    nl[k] = 0;
                    if (X[k] % p == 0) {
                        if (X[k] / p < n_e) { la[k][nl[k]] = 0; ec[k][nl[k]++] = X[k] / p; }
                        if (X[k] / p - 1 >= 0) { la[k][nl[k]] = p; ec[k][nl[k]++] = X[k] / p - 1; }
                    } else {
                        la[k][nl[k]] = X[k] % p;
                        ec[k][nl[k]++] = X[k] / p;
                    }
                }
                double s = 0.0;
                const int nz = d == 3 ? nl[2] : 1;
                for (int a = 0; a < nl[0]; ++a)
                    for (int b = 0; b < nl[1]; ++b)
                        for (int c = 0; c < nz; ++c) {
                            const int64_t cell = d == 2 ? ec[0][a] * n_e + ec[1][b]
                                                        : (ec[0][a] * n_e + ec[1][b]) * n_e + ec[2][c];
                            if (cls[cell] != IN) continue;
                            // sm * prod(w): (w_a w_b) w_c first, as np.prod
                            const double pw = d == 3 ? (w[la[0][a]] * w[la[1][b]]) * w[la[2][c]]
                                                     : w[la[0][a]] * w[la[1][b]];
                            s += sm * pw;
                        }
                m[i] = s;
            }
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nth; ++t) th.emplace_back(worker);
    worker();
    for (auto& x : th) x.join();
    // cut-cell lumped vectors, in cut-cell order (np.add.at)
    const int N = p + 1;
    const int L = d == 2 ? N * N : N * N * N;
    for (int64_t e = 0; e < n_cut; ++e) {
        int64_t c = cut_cells[e], ijk[3] = {0, 0, 0};
        for (int k = d - 1; k >= 0; --k) { ijk[k] = c % n_e; c /= n_e; }
        for (int q = 0; q < L; ++q) {
            int loc[3] = {0, 0, 0}, r = q;
            for (int k = d - 1; k >= 0; --k) { loc[k] = r % N; r /= N; }
            int64_t lex = 0;
            for (int k = 0; k < d; ++k) lex = lex * n1 + ijk[k] * p + loc[k];
            const int64_t i = compact_of_lex[lex];
            if (i >= 0) m[i] += cut_M[e * L + q];
        }
    }
    return WCB_OK;
}

}  // extern "C"
