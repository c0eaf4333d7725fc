// Matrix-free spectral-cell stiffness (GLL Lagrange, SCM) on a Cartesian grid,
// fused with the explicit CDM update.
//
// Reference: the global CSR K = sum over kept cells of element matrices
// (src/assembly.py:518-612); uncut cells share sk*(k1 (x) m1 + m1 (x) k1)
// (src/assembly.py:263-295), cut cells carry dense K_o (src/assembly.py:582).
// The reference's own matrix-free precedent is TensorSystem.k_matvec
// (src/assembly.py:674-684).
//
// Device layout ("state"): the lexicographic node grid (axis 0 slowest,
// src/assembly.py:85-89) padded by P rows above/below and PADJ columns on the
// left, row pitch a multiple of 32 doubles, zeros at non-DOF slots.
//
// 2D kernel (one fused pass per step):
//   * a warp owns a strip of 32 element columns (32*P node columns, lane t
//     owns the P columns of element column t) and RP element rows; the 8 warps
//     of a CTA stack vertically;
//   * the warp streams down its rows.  Per node row it loads its P values
//     (vector loads) and gets the neighbours' values by shuffles, contracts
//     along y with m1/k1 (the "y pass", masked per cell), and accumulates the
//     x pass into registers -- sum factorisation, no shared-memory staging;
//   * the element-boundary row is shared by two element rows: its value is
//     carry (from the row above) + own, in that fixed order, within a warp in
//     registers and across warps through shared memory -- deterministic, no
//     atomics (src/harness.py:462-485 bit-identity contract);
//   * cut cells are masked out of the tensor pass; their dense K_o u_e is
//     gathered per cut node by a small kernel into Ycut (fixed pair order)
//     and added in the epilogue of the warps that own cut nodes;
//   * epilogue: psi_new = 2 psi - psi_prev + dt^2 minv (f F - K psi), block
//     max |psi_new| -> one atomicMax per CTA (src/timeint.py:179-190).
#include "wcb_internal.cuh"

#include <algorithm>
#include <cstring>
#include <memory>
#include <numeric>

namespace wcb {

constexpr int PADJ = 32;
constexpr int SCM_NW = 8;    // warps per CTA (stacked along x)
constexpr int SCM_RP = 2;    // element rows per warp

// y pass uses the unscaled 1D factors, the x pass carries sk:
//   sk (k1_x (x) m1_y + m1_x (x) k1_y) = (sk k1)_x (x) m1_y + (sk m1)_x (x) k1_y
template <int P>
struct Mats2 {
    double m1[(P + 1) * (P + 1)];   // y pass
    double k1[(P + 1) * (P + 1)];   // y pass
    double xk[(P + 1) * (P + 1)];   // sk * k1, x pass
    double xm[(P + 1) * (P + 1)];   // sk * m1, x pass
};

struct Scm2DGeo {
    int64_t n_e;       // cells per axis
    int64_t n1;        // nodes per axis
    int64_t pitch;     // row pitch (doubles)
    const uint8_t* mask;      // (n_e+2)^2, 1 = uncut kept cell, padded by one ring of 0
    const uint8_t* wflags;    // per warp tile: bit0 kept node, bit1 cut node
    int64_t n_strips;
    const double* ycut;       // cut-cell contributions (state layout)
};

enum { MODE_STEP = 0, MODE_APPLY = 1 };

template <int P>
__device__ __forceinline__ void load_row(const double* __restrict__ u, int64_t rowbase,
                                         int64_t Jl, int lane, double (&own)[P],
                                         double (&left)[P], double& right) {
    const double* p = u + rowbase + Jl + PADJ;
    if constexpr ((P % 2) == 0) {
        #pragma unroll
        for (int j = 0; j < P; j += 2) {
            double2 v = __ldg(reinterpret_cast<const double2*>(p + j));
            own[j] = v.x;
            own[j + 1] = v.y;
        }
    } else {
        #pragma unroll
        for (int j = 0; j < P; ++j) own[j] = __ldg(p + j);
    }
    #pragma unroll
    for (int j = 0; j < P; ++j) left[j] = __shfl_up_sync(0xffffffffu, own[j], 1);
    right = __shfl_down_sync(0xffffffffu, own[0], 1);
    if (lane == 0) {
        #pragma unroll
        for (int j = 0; j < P; ++j) left[j] = __ldg(p - P + j);
    }
    if (lane == 31) right = __ldg(p + P);
}

// y pass of one node row: W1[j] = sum_d m1[j][d] u_e[d] (masked per cell),
// W2 likewise with k1; column j = 0 also receives the left cell (its b = P).
template <int P>
__device__ __forceinline__ void ypass(const Mats2<P>& mt, const double (&own)[P],
                                      const double (&left)[P], double right, double chiR,
                                      double chiL, double (&W1)[P], double (&W2)[P]) {
    constexpr int N = P + 1;
    #pragma unroll
    for (int j = 0; j < P; ++j) {
        double s1 = 0.0, s2 = 0.0;
        #pragma unroll
        for (int d = 0; d < N; ++d) {
            const double ud = d < P ? own[d] : right;
            s1 = fma(mt.m1[j * N + d], ud, s1);
            s2 = fma(mt.k1[j * N + d], ud, s2);
        }
        W1[j] = chiR * s1;
        W2[j] = chiR * s2;
    }
    double l1 = 0.0, l2 = 0.0;
    #pragma unroll
    for (int d = 0; d < N; ++d) {
        const double ud = d < P ? left[d] : own[0];
        l1 = fma(mt.m1[P * N + d], ud, l1);
        l2 = fma(mt.k1[P * N + d], ud, l2);
    }
    W1[0] = fma(chiL, l1, W1[0]);
    W2[0] = fma(chiL, l2, W2[0]);
}

template <int P, int MODE>
__device__ __forceinline__ void epilogue_row(const Scm2DGeo& g, const StepArgs& a, int64_t I,
                                             int64_t Jl, bool has_cut, const double (&Ku)[P],
                                             unsigned long long& amp) {
    if (I < 0 || I >= g.n1) return;
    const int64_t base = (I + P) * g.pitch + Jl + PADJ;
    double yc[P];
    #pragma unroll
    for (int j = 0; j < P; ++j) yc[j] = 0.0;
    if (has_cut) {
        #pragma unroll
        for (int j = 0; j < P; ++j) yc[j] = __ldg(g.ycut + base + j);
    }
    if constexpr (MODE == MODE_APPLY) {
        #pragma unroll
        for (int j = 0; j < P; ++j)
            if (Jl + j < g.n1) a.out[base + j] = Ku[j] + yc[j];
    } else {
        const double f = __ldg(a.ft + a.k);
        double u[P], up[P], mi[P];
        #pragma unroll
        for (int j = 0; j < P; ++j) {
            u[j] = __ldg(a.cur + base + j);
            up[j] = a.prev[base + j];
            mi[j] = __ldg(a.minv + base + j);
        }
        #pragma unroll
        for (int j = 0; j < P; ++j) {
            if (Jl + j < g.n1) {
                const double K = Ku[j] + yc[j];
                const double v = leapfrog(u[j], up[j], K, mi[j], f * source_at(a.F, base + j),
                                          a.dt2);
                a.out[base + j] = v;
                unsigned long long b = amp_bits(v);
                amp = b > amp ? b : amp;
            }
        }
    }
}

template <int P, int MODE>
__global__ void __launch_bounds__(SCM_NW * 32) k_scm2d(Scm2DGeo g, Mats2<P> mt, StepArgs a) {
    constexpr int N = P + 1;
    constexpr int TR = SCM_RP * P;  // rows per warp
    __shared__ double carry_s[SCM_NW + 1][32][P];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int64_t strip = blockIdx.x;
    const int64_t J0 = strip * (32 * P);
    const int64_t I0 = (int64_t)blockIdx.y * (SCM_NW * TR);
    const int64_t R0 = I0 + (int64_t)w * TR;
    const int64_t ey = J0 / P + lane;
    const int64_t Jl = J0 + (int64_t)lane * P;
    const uint8_t fl = g.wflags[((int64_t)blockIdx.y * SCM_NW + w) * g.n_strips + strip];
    const bool active = fl & 1;
    const bool has_cut = fl & 2;
    const double* __restrict__ u = a.cur;
    const int64_t mstride = g.n_e + 2;
    auto chi = [&](int64_t ex, int64_t eyy) -> double {
        return (double)__ldg(g.mask + (ex + 1) * mstride + (eyy + 1));
    };

    unsigned long long amp = 0ULL;
    double Yfirst[P];
    double carry[P];
    #pragma unroll
    for (int j = 0; j < P; ++j) { Yfirst[j] = 0.0; carry[j] = 0.0; }

    const int64_t ex_begin = R0 / P;
    const int64_t ex_end = min(ex_begin + SCM_RP, g.n_e);  // exclusive
    if (active) {
        double own[P], left[P], right = 0.0;
        bool have_row = false;
        for (int64_t ex = ex_begin; ex < ex_end; ++ex) {
            const double chiR = ey <= g.n_e ? chi(ex, ey) : 0.0;
            const double chiL = ey <= g.n_e ? chi(ex, ey - 1) : 0.0;
            double Y[N][P];
            #pragma unroll
            for (int r = 0; r < N; ++r)
                #pragma unroll
                for (int j = 0; j < P; ++j) Y[r][j] = 0.0;
            #pragma unroll
            for (int c = 0; c < N; ++c) {
                const int64_t I = ex * P + c;
                if (!(c == 0 && have_row)) load_row<P>(u, (I + P) * g.pitch, Jl, lane, own, left, right);
                double W1[P], W2[P];
                ypass<P>(mt, own, left, right, chiR, chiL, W1, W2);
                #pragma unroll
                for (int r = 0; r < N; ++r)
                    #pragma unroll
                    for (int j = 0; j < P; ++j)
                        Y[r][j] = fma(mt.xk[r * N + c], W1[j], fma(mt.xm[r * N + c], W2[j], Y[r][j]));
            }
            have_row = true;  // own/left/right now hold row (ex+1)*P = next c = 0
            if (ex == ex_begin) {
                #pragma unroll
                for (int j = 0; j < P; ++j) Yfirst[j] = Y[0][j];
            } else {
                double K0[P];
                #pragma unroll
                for (int j = 0; j < P; ++j) K0[j] = carry[j] + Y[0][j];
                epilogue_row<P, MODE>(g, a, ex * P, Jl, has_cut, K0, amp);
            }
            #pragma unroll
            for (int r = 1; r < P; ++r) epilogue_row<P, MODE>(g, a, ex * P + r, Jl, has_cut, Y[r], amp);
            #pragma unroll
            for (int j = 0; j < P; ++j) carry[j] = Y[P][j];
        }
        // last node row of the grid: only the row above contributes
        if (ex_end == g.n_e && ex_end > ex_begin) {
            const int64_t I = g.n_e * P;
            if (I >= R0 && I < R0 + TR) {
                double K0[P];
                #pragma unroll
                for (int j = 0; j < P; ++j) K0[j] = carry[j] + 0.0;
                epilogue_row<P, MODE>(g, a, I, Jl, has_cut, K0, amp);
            }
        }
        if (ex_end <= ex_begin) {
            #pragma unroll
            for (int j = 0; j < P; ++j) carry[j] = 0.0;
        }
    }
    // carry-out of warp w feeds the first row of warp w+1
    #pragma unroll
    for (int j = 0; j < P; ++j) carry_s[w + 1][lane][j] = active ? carry[j] : 0.0;
    if (w == 0) {
        // carry-in of the CTA: element row ex0-1 recomputed (output row a = P only)
        const int64_t ex = I0 / P - 1;
        double cin[P];
        #pragma unroll
        for (int j = 0; j < P; ++j) cin[j] = 0.0;
        if (ex >= 0 && ex < g.n_e && active) {
            const double chiR = ey <= g.n_e ? chi(ex, ey) : 0.0;
            const double chiL = ey <= g.n_e ? chi(ex, ey - 1) : 0.0;
            double own[P], left[P], right = 0.0;
            #pragma unroll
            for (int c = 0; c < N; ++c) {
                const int64_t I = ex * P + c;
                load_row<P>(u, (I + P) * g.pitch, Jl, lane, own, left, right);
                double W1[P], W2[P];
                ypass<P>(mt, own, left, right, chiR, chiL, W1, W2);
                #pragma unroll
                for (int j = 0; j < P; ++j)
                    cin[j] = fma(mt.xk[P * N + c], W1[j], fma(mt.xm[P * N + c], W2[j], cin[j]));
            }
        }
        #pragma unroll
        for (int j = 0; j < P; ++j) carry_s[0][lane][j] = cin[j];
    }
    __syncthreads();
    if (active && R0 < g.n1) {
        double K0[P];
        #pragma unroll
        for (int j = 0; j < P; ++j) K0[j] = carry_s[w][lane][j] + Yfirst[j];
        epilogue_row<P, MODE>(g, a, R0, Jl, has_cut, K0, amp);
    }
    if constexpr (MODE == MODE_STEP) block_amp_max<SCM_NW * 32>(amp, a.amp);
}

// Cut cells: Ycut[node] = sum over (cell, local row) pairs of K_o[row] . u_cell
// (pairs in ascending cell order; each dot in local DOF order).
__global__ void k_cut_apply(int64_t n_cn, const int64_t* __restrict__ cn_state,
                            const int64_t* __restrict__ cn_ptr, const int32_t* __restrict__ pr_cell,
                            const int32_t* __restrict__ pr_row, const int64_t* __restrict__ cell_state,
                            const double* __restrict__ Kc, int L, const double* __restrict__ u,
                            double* __restrict__ ycut) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_cn) return;
    double s = 0.0;
    for (int64_t q = cn_ptr[i]; q < cn_ptr[i + 1]; ++q) {
        const int64_t e = pr_cell[q];
        const double* Kr = Kc + (e * L + pr_row[q]) * (int64_t)L;
        const int64_t* cs = cell_state + e * L;
        double t = 0.0;
        for (int m = 0; m < L; ++m) t = fma(__ldg(Kr + m), __ldg(u + cs[m]), t);
        s += t;
    }
    ycut[cn_state[i]] = s;
}

struct ScmOperator final : Operator {
    int dim = 2, p = 4;
    int64_t n_e = 0, n1 = 0, pitch = 0, rows = 0;
    std::vector<int64_t> sidx;
    DevBuf<int64_t> d_sidx;
    DevBuf<uint8_t> mask, wflags;
    int64_t n_strips = 0, n_rtiles = 0;
    std::vector<double> m1, k1;
    double sk = 1.0;
    // cut cells
    int64_t n_cut = 0, n_cn = 0;
    int L = 0;
    DevBuf<int64_t> cn_state, cn_ptr, cell_state;
    DevBuf<int32_t> pr_cell, pr_row;
    DevBuf<double> Kc, ycut;
    double bytes_step = 0.0;

    const char* name() const override { return "scm"; }
    const std::vector<int64_t>& state_index() const override { return sidx; }
    void scatter(const double* src, double* dst) override { launch_scatter(ctx, n, d_sidx.p, src, dst); }
    void gather(const double* src, double* dst) override { launch_gather(ctx, n, d_sidx.p, src, dst); }

    void cut_pass(const double* u) {
        if (!n_cn) return;
        k_cut_apply<<<(unsigned)ceil_div(n_cn, 128), 128, 0, ctx->stream>>>(
            n_cn, cn_state.p, cn_ptr.p, pr_cell.p, pr_row.p, cell_state.p, Kc.p, L, u, ycut.p);
        ctx->launches++;
    }

    template <int P, int MODE>
    void launch2d(const StepArgs& a) {
        Mats2<P> mt;
        for (int i = 0; i < (P + 1) * (P + 1); ++i) {
            mt.m1[i] = m1[i];
            mt.k1[i] = k1[i];
            mt.xk[i] = sk * k1[i];
            mt.xm[i] = sk * m1[i];
        }
        Scm2DGeo g{n_e, n1, pitch, mask.p, wflags.p, n_strips, ycut.p};
        dim3 grid((unsigned)n_strips, (unsigned)n_rtiles);
        k_scm2d<P, MODE><<<grid, SCM_NW * 32, 0, ctx->stream>>>(g, mt, a);
        ctx->launches++;
    }
    template <int MODE>
    void dispatch2d(const StepArgs& a) {
        switch (p) {
            case 1: launch2d<1, MODE>(a); break;
            case 2: launch2d<2, MODE>(a); break;
            case 3: launch2d<3, MODE>(a); break;
            case 4: launch2d<4, MODE>(a); break;
            case 5: launch2d<5, MODE>(a); break;
            case 6: launch2d<6, MODE>(a); break;
            default: throw Error{WCB_E_UNSUPPORTED, "2D SCM kernel built for p = 1..6"};
        }
    }
    void apply(const double* x, double* y) override {
        cut_pass(x);
        StepArgs a;
        a.cur = x;
        a.out = y;
        dispatch2d<MODE_APPLY>(a);
        WCB_CHECK_LAUNCH();
    }
    void cdm_step(const StepArgs& a) override {
        cut_pass(a.cur);
        dispatch2d<MODE_STEP>(a);
        WCB_CHECK_LAUNCH();
    }
    double step_bytes() const override { return bytes_step; }
};

Operator* make_scm_operator(Context* ctx, const wcb_scm_desc* d) {
    WCB_REQUIRE(d->dim == 2 || d->dim == 3, "dim must be 2 or 3");
    if (d->dim == 3) throw Error{WCB_E_UNSUPPORTED, "3D SCM kernel not built yet"};
    const int p = d->p;
    WCB_REQUIRE(p >= 1 && p <= 6, "p must be in 1..6 for the 2D kernel");
    WCB_REQUIRE(d->n_e[0] == d->n_e[1] && d->n_e[0] >= 1, "square grids only (n_e[0] == n_e[1])");
    WCB_REQUIRE(d->k1 && d->m1 && d->cell_class && (d->n_dof == 0 || d->lex_of_compact),
                "NULL array in SCM descriptor");
    auto* op = new ScmOperator();
    std::unique_ptr<ScmOperator> guard(op);
    op->ctx = ctx;
    op->dim = 2;
    op->p = p;
    const int64_t n_e = d->n_e[0];
    const int64_t n1 = n_e * p + 1;
    op->n_e = n_e;
    op->n1 = n1;
    op->n = d->n_dof;
    // columns: PADJ left pad, lanes may read up to (n_e+1)*p + p past the origin
    const int64_t need_cols = PADJ + (int64_t)ceil_div(n1, 32 * p) * 32 * p + p + 1;
    op->pitch = ceil_div(need_cols, 32) * 32;
    op->rows = n1 + 2 * p;
    op->n_state = op->rows * op->pitch;
    const int N = p + 1;
    op->m1.assign(d->m1, d->m1 + N * N);
    op->k1.assign(d->k1, d->k1 + N * N);
    op->sk = d->sk;
    const int64_t n_cells = n_e * n_e;
    std::vector<uint8_t> mask((n_e + 2) * (n_e + 2), 0);
    std::vector<uint8_t> kept_cell(n_cells), cut_cell(n_cells);
    for (int64_t i = 0; i < n_e; ++i)
        for (int64_t j = 0; j < n_e; ++j) {
            const int8_t c = d->cell_class[i * n_e + j];
            WCB_REQUIRE(c >= 0 && c <= 2, "cell_class values must be 0, 1 or 2");
            mask[(i + 1) * (n_e + 2) + (j + 1)] = (c == 1);
            kept_cell[i * n_e + j] = (c != 0);
            cut_cell[i * n_e + j] = (c == 2);
        }
    // state index of every compact DOF
    op->sidx.resize(op->n);
    for (int64_t i = 0; i < op->n; ++i) {
        const int64_t lex = d->lex_of_compact[i];
        WCB_REQUIRE(lex >= 0 && lex < n1 * n1, "lex_of_compact out of range");
        const int64_t I = lex / n1, J = lex % n1;
        op->sidx[i] = (I + p) * op->pitch + J + PADJ;
    }
    // node masks: kept nodes, cut nodes
    std::vector<uint8_t> kept_node(n1 * n1, 0), cut_node(n1 * n1, 0);
    for (int64_t i = 0; i < op->n; ++i) kept_node[d->lex_of_compact[i]] = 1;
    for (int64_t c = 0; c < n_cells; ++c)
        if (cut_cell[c]) {
            const int64_t ci = c / n_e, cj = c % n_e;
            for (int a = 0; a <= p; ++a)
                for (int b = 0; b <= p; ++b) cut_node[(ci * p + a) * n1 + cj * p + b] = 1;
        }
    // warp tiles
    const int64_t TR = (int64_t)SCM_RP * p;
    op->n_strips = ceil_div(n1, 32 * p);
    op->n_rtiles = ceil_div(n1, SCM_NW * TR);
    std::vector<uint8_t> wf(op->n_rtiles * SCM_NW * op->n_strips, 0);
    for (int64_t I = 0; I < n1; ++I) {
        const int64_t wt = I / TR;  // global warp-row index = rtile*NW + w
        for (int64_t J = 0; J < n1; ++J) {
            const int64_t s = J / (32 * p);
            uint8_t& f = wf[wt * op->n_strips + s];
            if (kept_node[I * n1 + J]) f |= 1;
            if (cut_node[I * n1 + J]) f |= 2;
        }
    }
    cudaStream_t st = ctx->stream;
    op->d_sidx.alloc(std::max<int64_t>(op->n, 1));
    op->d_sidx.upload(op->sidx.data(), op->n, st);
    op->mask.alloc(mask.size());
    op->mask.upload(mask.data(), mask.size(), st);
    op->wflags.alloc(wf.size());
    op->wflags.upload(wf.data(), wf.size(), st);
    // cut cells
    op->n_cut = d->n_cut;
    op->L = N * N;
    const int L = op->L;
    op->ycut.alloc(op->n_state);
    op->ycut.zero(st);
    if (op->n_cut) {
        WCB_REQUIRE(d->cut_cells && d->cut_K, "cut arrays NULL");
        std::vector<int64_t> cell_state(op->n_cut * L);
        std::vector<std::vector<std::pair<int32_t, int32_t>>> pairs;  // per cut node
        std::vector<int64_t> node_of(n1 * n1, -1);
        std::vector<int64_t> cn_lex;
        for (int64_t e = 0; e < op->n_cut; ++e) {
            const int64_t c = d->cut_cells[e];
            WCB_REQUIRE(c >= 0 && c < n_cells && cut_cell[c], "cut_cells must list cut cells");
            if (e) WCB_REQUIRE(d->cut_cells[e - 1] < c, "cut_cells must be ascending");
            const int64_t ci = c / n_e, cj = c % n_e;
            for (int a = 0; a <= p; ++a)
                for (int b = 0; b <= p; ++b) {
                    const int64_t I = ci * p + a, J = cj * p + b;
                    const int loc = a * N + b;
                    cell_state[e * L + loc] = (I + p) * op->pitch + J + PADJ;
                    int64_t& k = node_of[I * n1 + J];
                    if (k < 0) {
                        k = (int64_t)cn_lex.size();
                        cn_lex.push_back(I * n1 + J);
                        pairs.emplace_back();
                    }
                    pairs[k].emplace_back((int32_t)e, (int32_t)loc);
                }
        }
        // sort cut nodes by lex for locality; pairs are already in cell order
        std::vector<int64_t> order(cn_lex.size());
        std::iota(order.begin(), order.end(), 0);
        std::sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return cn_lex[x] < cn_lex[y]; });
        std::vector<int64_t> cs, cp(1, 0);
        std::vector<int32_t> pc, prr;
        for (int64_t k : order) {
            const int64_t lex = cn_lex[k];
            cs.push_back((lex / n1 + p) * op->pitch + lex % n1 + PADJ);
            for (auto& pr : pairs[k]) { pc.push_back(pr.first); prr.push_back(pr.second); }
            cp.push_back((int64_t)pc.size());
        }
        op->n_cn = (int64_t)cs.size();
        op->cn_state.alloc(cs.size()); op->cn_state.upload(cs.data(), cs.size(), st);
        op->cn_ptr.alloc(cp.size()); op->cn_ptr.upload(cp.data(), cp.size(), st);
        op->pr_cell.alloc(pc.size()); op->pr_cell.upload(pc.data(), pc.size(), st);
        op->pr_row.alloc(prr.size()); op->pr_row.upload(prr.data(), prr.size(), st);
        op->cell_state.alloc(cell_state.size()); op->cell_state.upload(cell_state.data(), cell_state.size(), st);
        op->Kc.alloc(op->n_cut * L * L); op->Kc.upload(d->cut_K, op->n_cut * L * L, st);
    }
    // algorithmic bytes per step: 32 B per DOF + packed cut K
    op->bytes_step = 32.0 * (double)op->n + 8.0 * (double)L * (L + 1) / 2.0 * (double)op->n_cut;
    WCB_CUDA(cudaStreamSynchronize(st));
    return guard.release();
}

}  // namespace wcb
