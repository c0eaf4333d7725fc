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
// 2D kernel (one fused pass per step, no atomics, deterministic):
//   * a warp owns a strip of 32 element columns (lane t owns the P node
//     columns of element column t) and RP element rows; the 8 warps of a CTA
//     stack vertically (consecutive row ranges of the same strip);
//   * the warp streams down its rows.  Per node row: one vector load of the
//     lane's P values, neighbour values by shuffles, the y contraction with
//     m1/k1 (masked per cell), and the x contraction accumulated in
//     registers (sum factorisation).  The next element row is prefetched
//     into L1 while the current one is computed;
//   * the node row shared by two element rows gets carry (row above) + own,
//     in that fixed order -- in registers inside a warp, through shared memory
//     between the warps of a CTA (warp 0 recomputes its carry-in row);
//   * a cut cell is masked out of the tensor contraction and its dense
//     K_o u_e is added by the lanes owning its columns (K_o stored
//     transposed so a lane reads its rows contiguously);
//   * epilogue: psi_new = 2 psi - psi_prev + dt^2 minv (f F - K psi) and the
//     block max |psi_new| (one atomicMax per CTA), src/timeint.py:179-190.
#include "wcb_scm.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>

namespace wcb {
__device__ __forceinline__ int smid() { int r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }

// element rows per tile; one compute warp each plus one halo warp
#ifndef WCB2D_RPE
#define WCB2D_RPE 3
#endif
#ifndef WCB2D_MINB
#define WCB2D_MINB 4
#endif
#ifndef WCB2D_EPI_TMA
#define WCB2D_EPI_TMA 1      // 1: psi_{k-1} and 1/m also staged by TMA
#endif
__host__ __device__ constexpr int rpe_for(int P) { return P <= 4 ? WCB2D_RPE : 2; }

// Tile geometry of the 2D kernel: a tile is 32p node columns x RPE*p node rows;
// only psi_k (with its halo) is staged in shared memory by TMA.
template <int P>
struct Tile2 {
    static constexpr int RPE = rpe_for(P);
    static constexpr int NWARP = RPE + 1;
    static constexpr int TJ = 32 * P;                       // owned node columns
    static constexpr int TI = RPE * P;                      // owned node rows
    // TMA boxes must start 16-byte aligned: for odd P the u tile starts one
    // column early and node columns sit at offset CO inside the tile
    static constexpr int CO = P & 1;
    static constexpr int UW = ((TJ + P + 1 + CO) + 1) / 2 * 2;  // cols J0-P-CO..J0+TJ, even
    static constexpr int UH = TI + P + 1;                   // u tile rows (I0-P..I0+TI)
    static constexpr size_t U_BYTES = (size_t)UW * UH * 8;
    static constexpr size_t E_BYTES = WCB2D_EPI_TMA ? (size_t)TJ * TI * 8 : 0;  // prev / minv tiles
    static constexpr size_t OFF_PREV = (U_BYTES + 127) / 128 * 128;
    static constexpr size_t OFF_MINV = OFF_PREV + (E_BYTES + 127) / 128 * 128;
    static constexpr size_t OFF_CARRY = OFF_MINV + (E_BYTES + 127) / 128 * 128;   // [RPE+1][P][32]
    static constexpr size_t OFF_BAR = OFF_CARRY + (size_t)(RPE + 1) * P * 32 * 8;
    static constexpr size_t SMEM = OFF_BAR + 16;   // [0] psi_k tile, [1] epilogue tiles
};

// Local geometry of a 2D operator.  x (axis 0) may be a slab of the global
// grid: local cell row 0 is the (possibly phantom) cell row above the first
// owned one, so every tile can recompute the row above it; owned node rows
// are [row_lo, row_hi) in local numbering.
struct Scm2DGeo {
    int64_t n_ex;             // local cell rows (incl. the halo row 0)
    int64_t n_ey;             // cells along y (global)
    int64_t n1y;              // nodes along y
    int64_t row_lo, row_hi;   // owned local node rows
    const uint8_t* mask;      // (n_ex+2) x (n_ey+2) cell codes with a zero ring
    const int32_t* cut_id;    // n_ex x n_ey -> cut index or -1
    const double* KT;         // n_cut * L * L, transposed physical cut stiffness / sk
    const uint8_t* cflags;    // per tile (strip-major): 1 = owns a DOF
    const int32_t* order;     // live tiles (strip-major ids), most expensive first
    int64_t n_strips;
    int64_t n_rtiles;
    int64_t pitch;            // row pitch of the state (doubles)
    // per tile (strip-major): every owned node's 1/m equals the interior
    // table (checked bitwise once per plan) -- the 1/m tile is not loaded.
    // null: every tile loads 1/m.
    const uint8_t* tclean;
    int32_t chunk_nt;         // streaming kernel (k_scm2s): row tiles per chunk
};

template <int P>
struct MinvTab2 {
    double v[P * P];   // (r, j) of the owned nodes of an interior uncut cell
};

// clean[c] for every local cell c of a plane-strain operator: both
// components of all P x P owned nodes carry minv == tab (bitwise)
template <int P>
__global__ void k_clean2e(int64_t n_ex, int64_t n_ey, int64_t row_hi, int64_t pitch, int64_t plane,
                          MinvTab2<P> tab, const double* __restrict__ minv, uint8_t* clean) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_ex * n_ey) return;
    const int64_t ex = c / n_ey, ey = c % n_ey;
    bool ok = ex >= 1;
    for (int r = 0; r < P && ok; ++r)
        for (int j = 0; j < P && ok; ++j) {
            const int64_t I = ex * P + r;
            const int64_t s = (I + P) * pitch + ey * P + j + PADJ;
            const long long t = __double_as_longlong(tab.v[r * P + j]);
            ok = I < row_hi && __double_as_longlong(minv[s]) == t && __double_as_longlong(minv[s + plane]) == t;
        }
    clean[c] = ok ? 1 : 0;
}

// tclean[t] for every tile t: 1 when all owned nodes carry minv == tab (bitwise)
template <int P>
__global__ void k_clean2d(Scm2DGeo g, int TI, int TJ, MinvTab2<P> tab, const double* __restrict__ minv,
                          uint8_t* tclean) {
    const int64_t t = blockIdx.x;
    const int64_t strip = t / g.n_rtiles, rt = t % g.n_rtiles;
    const int64_t I0 = g.row_lo + rt * TI, J0 = strip * TJ;
    bool ok = true;
    for (int q = threadIdx.x; q < TI * TJ && ok; q += blockDim.x) {
        const int64_t I = I0 + q / TJ, J = J0 + q % TJ;
        if (I >= g.row_hi || J >= g.n1y) continue;
        const double m = minv[(I + P) * g.pitch + J + PADJ];
        ok = __double_as_longlong(m) == __double_as_longlong(tab.v[(I % P) * P + J % P]);
    }
    ok = __syncthreads_and(ok);
    if (threadIdx.x == 0) tclean[t] = ok ? 1 : 0;
}

// P consecutive doubles of a lane from shared memory (16-byte loads for
// even P: the row starts are 16-byte aligned in every tile layout)
template <int P>
__device__ __forceinline__ void lds_row(const double* p, double (&v)[P]) {
    if constexpr ((P % 2) == 0) {
        #pragma unroll
        for (int j = 0; j < P; j += 2) {
            const double2 t = *reinterpret_cast<const double2*>(p + j);
            v[j] = t.x;
            v[j + 1] = t.y;
        }
    } else {
        #pragma unroll
        for (int j = 0; j < P; ++j) v[j] = p[j];
    }
}

// One node row of the smem tile: y contraction (masked) then x contraction
// accumulated into Y.  `row` points at tile column 0 of that row.
template <int P, bool MASK = true, bool HALO = false>
__device__ __forceinline__ void row_contract(const double (&mc)[orb_count(P)],
                                             const double (&kc)[orb_count(P)], const double* row,
                                             int lane, double chiR, double chiL, int c,
                                             double (&Y)[P + 1][P]) {
    constexpr int N = P + 1;
    row += Tile2<P>::CO;
    const double* own_p = row + P + lane * P;
    double own[P];
    if constexpr ((P % 2) == 0) {
        #pragma unroll
        for (int j = 0; j < P; j += 2) {
            double2 v = *reinterpret_cast<const double2*>(own_p + j);
            own[j] = v.x;
            own[j + 1] = v.y;
        }
    } else {
        #pragma unroll
        for (int j = 0; j < P; ++j) own[j] = own_p[j];
    }
    double right = __shfl_down_sync(0xffffffffu, own[0], 1);
    if (lane == 31) right = own_p[P];
    double W1[P], W2[P];
    #pragma unroll
    for (int j = 0; j < P; ++j) {
        double s1 = mc[orb(P, j, P)] * right, s2 = kc[orb(P, j, P)] * right;
        #pragma unroll
        for (int d = 0; d < P; ++d) {
            s1 = fma(mc[orb(P, j, d)], own[d], s1);
            s2 = fma(kc[orb(P, j, d)], own[d], s2);
        }
        W1[j] = MASK ? chiR * s1 : s1;
        W2[j] = MASK ? chiR * s2 : s2;
    }
    // left cell: its local column P is our column 0
    double l1 = mc[orb(P, P, P)] * own[0], l2 = kc[orb(P, P, P)] * own[0];
    #pragma unroll
    for (int d = 0; d < P; ++d) {
        double ud = __shfl_up_sync(0xffffffffu, own[d], 1);
        if (lane == 0) ud = row[d];
        l1 = fma(mc[orb(P, P, d)], ud, l1);
        l2 = fma(kc[orb(P, P, d)], ud, l2);
    }
    W1[0] = MASK ? fma(chiL, l1, W1[0]) : W1[0] + l1;
    W2[0] = MASK ? fma(chiL, l2, W2[0]) : W2[0] + l2;
    #pragma unroll
    for (int r = HALO ? P : 0; r < N; ++r)   // the halo warp only needs output row P
        #pragma unroll
        for (int j = 0; j < P; ++j)
            Y[r][j] = fma(kc[orb(P, r, c)], W1[j], fma(mc[orb(P, r, c)], W2[j], Y[r][j]));
}

// Cut cells of one element row, handled cooperatively by the warp: for each
// cut cell (ascending lane order) lane r < L computes output row r of K_o u_e
// (K_o stored transposed -> coalesced), then the results are routed by
// shuffles to the lanes owning the cell's columns (columns 0..P-1: the cell's
// lane; column P: the next lane).  `rows` points at tile column 0 of node row
// ex*P; cut_lanes = ballot of lanes whose own cell is cut; edge = lane 0's
// left neighbour (previous strip) is cut.
template <int P, int UW, int CO>
__device__ __forceinline__ void cut_cells_warp(const Scm2DGeo& g, const double* rows, int64_t ex,
                                               int64_t ey0, int lane, unsigned cut_lanes,
                                               bool edge, int32_t cid, int32_t cidL,
                                               double (&Y)[P + 1][P]) {
    constexpr int N = P + 1;
    constexpr int L = N * N;
    int src = edge ? -1 : (__ffs(cut_lanes) - 1);
    if (!edge) cut_lanes &= cut_lanes - 1;
    while (src >= -1) {
        // cut ids were fetched by their lanes in the prologue
        const int32_t id = src >= 0 ? __shfl_sync(0xffffffffu, cid, src) : __shfl_sync(0xffffffffu, cidL, 0);
        const double* KT = g.KT + (int64_t)id * L * L;
        const double* corner = rows + CO + P + src * P;
        constexpr int RR = (L + 31) / 32;   // output rows per lane
        double t[RR];
        #pragma unroll
        for (int q = 0; q < RR; ++q) {
            t[q] = 0.0;
            const int r = lane + 32 * q;
            if (r < L) {
                #pragma unroll
                for (int m = 0; m < L; ++m)
                    t[q] = fma(__ldg(KT + m * L + r), corner[(m / N) * UW + (m % N)], t[q]);
            }
        }
        #pragma unroll
        for (int r = 0; r < L; ++r) {
            const double v = __shfl_sync(0xffffffffu, t[r / 32], r % 32);
            const int a = r / N, b = r % N;
            if (b < P) {
                if (lane == src) Y[a][b % P] += v;
            } else {
                if (lane == src + 1) Y[a][0] += v;
            }
        }
        if (!cut_lanes) break;
        src = __ffs(cut_lanes) - 1;
        cut_lanes &= cut_lanes - 1;
    }
}

// One CTA per tile (grid = strips x row tiles).  The halo warp recomputes
// the element row above the tile (its output row a = P only); warp w < RPE
// computes element row ex0 + w.  psi_k arrives by one TMA box; psi_{k-1} and
// 1/m are read straight from global memory in the epilogue.
template <int P, int MODE>
__global__ void __launch_bounds__(Tile2<P>::NWARP * 32, WCB2D_MINB) k_scm2d(
    const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_prev,
    const __grid_constant__ CUtensorMap tm_minv, Scm2DGeo g, Mats2<P> mt, MinvTab2<P> mtab, double sk,
    StepArgs a) {
    using T = Tile2<P>;
    constexpr int N = P + 1;
    constexpr int RPE = T::RPE;
    extern __shared__ __align__(128) unsigned char smem[];
    const double* us = reinterpret_cast<const double*>(smem);
    double* carry = reinterpret_cast<double*>(smem + T::OFF_CARRY);   // [RPE+1][P][32]
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    // tiles are dispatched longest-first (cut-cell tiles lead) so the last
    // wave is made of cheap interior tiles
#ifdef WCB2D_EMPTY
    return;
#endif
#ifdef WCB2D_TRACE
    unsigned long long t_0, t_1, t_2, t_3, t_4;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_0));
#endif
    if (MODE == MODE_STEP) pdl_trigger();
    const int32_t tid = __ldg(g.order + blockIdx.x);
    const int64_t strip = tid / g.n_rtiles, rtile = tid % g.n_rtiles;
    const int64_t J0 = strip * T::TJ, I0 = g.row_lo + rtile * T::TI;
    const bool tcl = MODE == MODE_STEP && g.tclean && __ldg(g.tclean + tid) != 0;
    if (MODE == MODE_STEP) pdl_wait();   // the previous step's psi is complete from here on
    if (MODE == MODE_STEP && blockIdx.x == 0) record_observers(a);
    // two barriers: the contraction starts as soon as the psi_k tile lands,
    // psi_{k-1} / 1/m (epilogue only) keep streaming meanwhile
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        const bool epi = WCB2D_EPI_TMA && MODE == MODE_STEP;
        mbar_expect_tx(bar, (uint32_t)T::U_BYTES);
        tma_load_2d(smem, &tm_u, (int32_t)(J0 - P - T::CO + PADJ), (int32_t)I0, bar);
        if (epi) {
            mbar_expect_tx(bar + 1, (uint32_t)((tcl ? 1 : 2) * T::E_BYTES));
            tma_load_2d(smem + T::OFF_PREV, &tm_prev, (int32_t)(J0 + PADJ), (int32_t)(I0 + P), bar + 1);
            if (!tcl) tma_load_2d(smem + T::OFF_MINV, &tm_minv, (int32_t)(J0 + PADJ), (int32_t)(I0 + P), bar + 1);
        }
    }
    // cell codes (and the epilogue's psi_{k-1}, 1/m) while the tile is in flight
    const bool halo = (w == RPE);
    const int64_t ex = halo ? I0 / P - 1 : I0 / P + w;
    const int64_t ey = J0 / P + lane;
    uint8_t mR = 0, mL = 0;
    if (ex >= 0 && ex < g.n_ex && ey <= g.n_ey) {
        const int64_t ms_ = g.n_ey + 2;
        mR = __ldg(g.mask + (ex + 1) * ms_ + (ey + 1));
        mL = __ldg(g.mask + (ex + 1) * ms_ + ey);
    }
    const int32_t cid = mR == 2 ? __ldg(g.cut_id + ex * g.n_ey + ey) : -1;
    const int32_t cidL = (lane == 0 && mL == 2) ? __ldg(g.cut_id + ex * g.n_ey + ey - 1) : -1;
    const int64_t Jl = J0 + lane * P;
    if (MODE == MODE_STEP && !halo && !WCB2D_EPI_TMA) {
        #pragma unroll
        for (int r = 0; r < P; ++r) {
            const int64_t base = (ex * P + r + P) * g.pitch + Jl + PADJ;
            asm volatile("prefetch.global.L1 [%0];" ::"l"(a.prev + base));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(a.minv + base));
        }
    }
    __syncthreads();   // barrier init visible
#ifdef WCB2D_TRACE
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_1));
#endif
    mbar_wait(bar, 0);
#ifdef WCB2D_TRACE
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_2));
#endif

    double mc[orb_count(P)], kc[orb_count(P)];
    #pragma unroll
    for (int i = 0; i < orb_count(P); ++i) { mc[i] = mt.m[i]; kc[i] = mt.k[i]; }
    const int rbase = halo ? -P : w * P;   // tile row of node row ex*P, minus P
    double Y[N][P];
    #pragma unroll
    for (int r = 0; r < N; ++r)
        #pragma unroll
        for (int j = 0; j < P; ++j) Y[r][j] = 0.0;
    if (__any_sync(0xffffffffu, (mR | mL) != 0)) {
        const double chiR = mR == 1 ? 1.0 : 0.0;
        const double chiL = mL == 1 ? 1.0 : 0.0;
        const double* rows = us + (size_t)(rbase + P) * T::UW;
#ifndef WCB2D_NOTENSOR
        #pragma unroll
        for (int c = 0; c < N; ++c) row_contract<P>(mc, kc, rows + (size_t)c * T::UW, lane, chiR, chiL, c, Y);
#endif
        const unsigned cl = __ballot_sync(0xffffffffu, mR == 2);
        const bool ed = __shfl_sync(0xffffffffu, mL == 2, 0);
#ifndef WCB2D_NOCUT
        if ((cl || ed) && g.KT) cut_cells_warp<P, T::UW, T::CO>(g, rows, ex, J0 / P, lane, cl, ed, cid, cidL, Y);
#endif
    }
    // row a = P of element row ex is row a = 0 of element row ex+1
    #pragma unroll
    for (int j = 0; j < P; ++j) carry[((halo ? 0 : w + 1) * P + j) * 32 + lane] = Y[P][j];
#ifdef WCB2D_TRACE
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_3));
#endif
    __syncthreads();
    unsigned long long amp = 0ULL;
    if (!halo) {
        #pragma unroll
        for (int j = 0; j < P; ++j) Y[0][j] = carry[(w * P + j) * 32 + lane] + Y[0][j];
        #pragma unroll
        for (int r = 0; r < P; ++r)
            #pragma unroll
            for (int j = 0; j < P; ++j) Y[r][j] *= sk;
        const double f = (MODE == MODE_STEP) ? __ldg(a.ft + a.k) : 0.0;
        const bool edge = (J0 + T::TJ > g.n1y);
        #pragma unroll
        for (int r = 0; r < P; ++r) {
            const int64_t I = ex * P + r;
            if (I >= g.row_hi) break;
            const int64_t base = (I + P) * g.pitch + Jl + PADJ;
            const double* urow = us + (size_t)(rbase + r + P) * T::UW + T::CO + P + lane * P;
            if constexpr (MODE == MODE_APPLY) {
                #pragma unroll
                for (int j = 0; j < P; ++j)
                    if (!edge || Jl + j < g.n1y) a.out[base + j] = Y[r][j];
            } else {
                double up[P], mi[P];
                if constexpr (WCB2D_EPI_TMA != 0) {
                    if (r == 0) mbar_wait(bar + 1, 0);
                    const double* ps = reinterpret_cast<const double*>(smem + T::OFF_PREV) +
                                       (size_t)(w * P + r) * T::TJ + lane * P;
                    const double* msm = reinterpret_cast<const double*>(smem + T::OFF_MINV) +
                                        (size_t)(w * P + r) * T::TJ + lane * P;
                    lds_row<P>(ps, up);
                    if (tcl) {
                        #pragma unroll
                        for (int j = 0; j < P; ++j) mi[j] = mtab.v[r * P + j];
                    } else {
                        lds_row<P>(msm, mi);
                    }
                } else {
                    #pragma unroll
                    for (int j = 0; j < P; ++j) {
                        up[j] = a.prev[base + j];
                        mi[j] = __ldg(a.minv + base + j);
                    }
                }
                const bool src = base + P - 1 >= a.F.lo && base <= a.F.hi;
                double v[P], uu[P];
                lds_row<P>(urow, uu);
                #pragma unroll
                for (int j = 0; j < P; ++j) {
                    const double fF = src ? f * source_at(a.F, base + j) : f * 0.0;
                    v[j] = leapfrog(uu[j], up[j], Y[r][j], mi[j], fF, a.dt2);
                }
                if constexpr (P == 4) {
                    if (!edge) {
                        // one 32-byte store per lane: every sector written exactly once
                        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(a.out + base),
                                     "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]) : "memory");
                        #pragma unroll
                        for (int j = 0; j < P; ++j) {
                            unsigned long long b = mi[j] != 0.0 ? amp_bits(v[j]) : 0ULL;
                            amp = b > amp ? b : amp;
                        }
                        continue;
                    }
                }
                #pragma unroll
                for (int j = 0; j < P; ++j) {
                    if (!edge || Jl + j < g.n1y) {
                        a.out[base + j] = v[j];
                        unsigned long long b = mi[j] != 0.0 ? amp_bits(v[j]) : 0ULL;
                        amp = b > amp ? b : amp;
                    }
                }
            }
        }
    }
#ifndef WCB2D_NOAMP
    if constexpr (MODE == MODE_STEP) warp_amp_max(amp, a.amp);
#endif
#ifdef WCB2D_TRACE
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_4));
    if (MODE == MODE_STEP && a.k == 100 && threadIdx.x == 0)
        printf("TRACE blk %d w %d sm %d start %llu pre %llu tma %llu comp %llu end %llu\n", blockIdx.x, threadIdx.x >> 5,
               smid(), t_0, t_1 - t_0, t_2 - t_0, t_3 - t_0, t_4 - t_0);
#endif
}


// ---------------------------------------------------------------------------
// Streaming 2D step (default for scalar SCM operators): a CTA owns one strip
// of 32 cell columns and a chunk of NT consecutive row tiles, and walks down
// the chunk tile by tile.  Per tile every warp computes one cell row (no halo
// warp: the shared node row above a tile is carried from the previous tile's
// bottom warp; only the chunk's first tile recomputes the cell row above, in
// a prologue).  psi_k (TI+1 node rows) and psi_{k-1} (TI rows) of tile t+1
// stream into the other half of a double-buffered TMA stage while tile t is
// computed.  Same fixed-order sums as k_scm2d (carry + own), bitwise equal.
#ifndef WCB2S_MINB
#define WCB2S_MINB 3
#endif
#ifndef WCB2S_PREV_TMA
#define WCB2S_PREV_TMA 1     // psi_{k-1} staged by TMA (0: loaded in the epilogue)
#endif
__host__ __device__ constexpr int minb_2s(int P) { return P <= 4 ? WCB2S_MINB : 2; }
__host__ __device__ constexpr size_t al128(size_t b) { return (b + 127) / 128 * 128; }
template <int P>
struct Tile2S {
    static constexpr int RPE = Tile2<P>::RPE;   // same row tiles as k_scm2d (cflags, tclean)
    static constexpr int NWARP = RPE;
    static constexpr int TJ = 32 * P;
    static constexpr int TI = RPE * P;
    static constexpr int CO = P & 1;
    static constexpr int UW = Tile2<P>::UW;
    static constexpr int UH = TI + 1;       // node rows I0 .. I0+TI
    static constexpr int HH = P + 1;        // chunk halo rows I0-P .. I0
    static constexpr size_t U_BYTES = (size_t)UW * UH * 8;
    static constexpr size_t H_BYTES = (size_t)UW * HH * 8;
    static constexpr size_t E_BYTES = WCB2S_PREV_TMA ? (size_t)TJ * TI * 8 : 0;
    static constexpr size_t STAGE = al128(U_BYTES) + al128(E_BYTES);
    static constexpr int NS = 2;
    static constexpr size_t OFF_HALO = NS * STAGE;
    static constexpr size_t OFF_CARRY = OFF_HALO + al128(H_BYTES);               // [2][RPE+1][P][32]
    static constexpr size_t OFF_BAR = OFF_CARRY + (size_t)2 * (RPE + 1) * P * 32 * 8;
    static constexpr size_t SMEM = OFF_BAR + 8 * (NS + 1);
};

// the cell row whose node rows start at `rows` (stride UW): y/x contraction
// (unmasked fast path when the warp's cells are all uncut) and cut cells
template <int P, int UW, int CO>
__device__ __forceinline__ void cell_row2(const Scm2DGeo& g, const double (&mc)[orb_count(P)],
                                          const double (&kc)[orb_count(P)], const double* rows, int64_t ex,
                                          int64_t ey, int lane, double (&Y)[P + 1][P]) {
    constexpr int N = P + 1;
    uint8_t mR = 0, mL = 0;
    if (ex >= 0 && ex < g.n_ex && ey <= g.n_ey) {
        const int64_t ms_ = g.n_ey + 2;
        mR = __ldg(g.mask + (ex + 1) * ms_ + (ey + 1));
        mL = __ldg(g.mask + (ex + 1) * ms_ + ey);
    }
    const int32_t cid = mR == 2 ? __ldg(g.cut_id + ex * g.n_ey + ey) : -1;
    const int32_t cidL = (lane == 0 && mL == 2) ? __ldg(g.cut_id + ex * g.n_ey + ey - 1) : -1;
    #pragma unroll
    for (int r = 0; r < N; ++r)
        #pragma unroll
        for (int j = 0; j < P; ++j) Y[r][j] = 0.0;
    if (!__any_sync(0xffffffffu, (mR | mL) != 0)) return;
    if (__all_sync(0xffffffffu, mR == 1 && mL == 1)) {
        #pragma unroll
        for (int c = 0; c < N; ++c) row_contract<P, false>(mc, kc, rows + (size_t)c * UW, lane, 1.0, 1.0, c, Y);
        return;
    }
    const double chiR = mR == 1 ? 1.0 : 0.0;
    const double chiL = mL == 1 ? 1.0 : 0.0;
    #pragma unroll
    for (int c = 0; c < N; ++c) row_contract<P, true>(mc, kc, rows + (size_t)c * UW, lane, chiR, chiL, c, Y);
    const unsigned cl = __ballot_sync(0xffffffffu, mR == 2);
    const bool ed = __shfl_sync(0xffffffffu, mL == 2, 0);
    if (cl || ed) cut_cells_warp<P, UW, CO>(g, rows, ex, ey - lane, lane, cl, ed, cid, cidL, Y);
}

template <int P, int MODE>
__global__ void __launch_bounds__(Tile2S<P>::NWARP * 32, minb_2s(P)) k_scm2s(
    const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_h,
    const __grid_constant__ CUtensorMap tm_prev, Scm2DGeo g, Mats2<P> mt, MinvTab2<P> mtab, double sk,
    StepArgs a) {
    using T = Tile2S<P>;
    constexpr int N = P + 1;
    constexpr int RPE = T::RPE;
    extern __shared__ __align__(128) unsigned char smem[];
    double* carry = reinterpret_cast<double*>(smem + T::OFF_CARRY);   // [2][RPE+1][P][32]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);  // [NS] stages, [NS] halo
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    if (MODE == MODE_STEP) pdl_trigger();
    const int32_t chunk = __ldg(g.order + blockIdx.x);
    const int64_t strip = chunk / g.n_rtiles, rt0 = chunk % g.n_rtiles;
    const int nt = (int)min((int64_t)g.chunk_nt, g.n_rtiles - rt0);
    const int64_t J0 = strip * T::TJ;
    const int64_t I00 = g.row_lo + rt0 * T::TI;
    if (MODE == MODE_STEP) pdl_wait();
    if (MODE == MODE_STEP && blockIdx.x == 0) record_observers(a);
    auto issue = [&](int t) {   // tile t of the chunk into stage t % NS
        const int b = t % T::NS;
        unsigned char* st = smem + (size_t)b * T::STAGE;
        const int64_t I0 = I00 + (int64_t)t * T::TI;
        mbar_expect_tx(&full[b], (uint32_t)(T::U_BYTES + (MODE == MODE_STEP ? T::E_BYTES : 0)));
        tma_load_2d(st, &tm_u, (int32_t)(J0 - P - T::CO + PADJ), (int32_t)(I0 + P), &full[b]);
        if (MODE == MODE_STEP && WCB2S_PREV_TMA)
            tma_load_2d(st + al128(T::U_BYTES), &tm_prev, (int32_t)(J0 + PADJ), (int32_t)(I0 + P), &full[b]);
    };
    if (threadIdx.x == 0) {
        #pragma unroll
        for (int q = 0; q < T::NS + 1; ++q) mbar_init(&full[q], 1);
        mbar_expect_tx(&full[T::NS], (uint32_t)T::H_BYTES);
        tma_load_2d(smem + T::OFF_HALO, &tm_h, (int32_t)(J0 - P - T::CO + PADJ), (int32_t)I00, &full[T::NS]);
        issue(0);
    }
    double mc[orb_count(P)], kc[orb_count(P)];
    #pragma unroll
    for (int i = 0; i < orb_count(P); ++i) { mc[i] = mt.m[i]; kc[i] = mt.k[i]; }
    const int64_t ey = J0 / P + lane;
    const int64_t Jl = J0 + lane * P;
    const bool edge = (J0 + T::TJ > g.n1y);
    const double f = (MODE == MODE_STEP) ? __ldg(a.ft + a.k) : 0.0;
    __syncthreads();   // barrier init visible
    double Y[N][P];
    if (w == 0) {      // the cell row above the chunk: its bottom row feeds tile 0's top row
        mbar_wait(&full[T::NS], 0);
        cell_row2<P, T::UW, T::CO>(g, mc, kc, reinterpret_cast<const double*>(smem + T::OFF_HALO),
                                   I00 / P - 1, ey, lane, Y);
        #pragma unroll
        for (int j = 0; j < P; ++j) carry[((1 * (RPE + 1) + RPE) * P + j) * 32 + lane] = Y[P][j];
    }
    unsigned long long amp = 0ULL;
    for (int t = 0; t < nt; ++t) {
        const int b = t % T::NS, par = t & 1;
        if (threadIdx.x == 0 && t + 1 < nt) issue(t + 1);
        const unsigned char* st = smem + (size_t)b * T::STAGE;
        const double* us = reinterpret_cast<const double*>(st);
        const int64_t I0 = I00 + (int64_t)t * T::TI;
        const int64_t rt = rt0 + t;
        const bool tcl = MODE == MODE_STEP && g.tclean && __ldg(g.tclean + strip * g.n_rtiles + rt) != 0;
        mbar_wait(&full[b], (uint32_t)((t / T::NS) & 1));
        const int64_t ex = I0 / P + w;
        cell_row2<P, T::UW, T::CO>(g, mc, kc, us + (size_t)(w * P) * T::UW, ex, ey, lane, Y);
        #pragma unroll
        for (int j = 0; j < P; ++j) carry[((par * (RPE + 1) + w + 1) * P + j) * 32 + lane] = Y[P][j];
        __syncthreads();
        {
            const double* cin = carry + (size_t)(w == 0 ? ((par ^ 1) * (RPE + 1) + RPE) : (par * (RPE + 1) + w)) * P * 32;
            #pragma unroll
            for (int j = 0; j < P; ++j) Y[0][j] = cin[j * 32 + lane] + Y[0][j];
        }
        #pragma unroll
        for (int r = 0; r < P; ++r)
            #pragma unroll
            for (int j = 0; j < P; ++j) Y[r][j] *= sk;
        #pragma unroll
        for (int r = 0; r < P; ++r) {
            const int64_t I = ex * P + r;
            if (I >= g.row_hi) break;
            const int64_t base = (I + P) * g.pitch + Jl + PADJ;
            const double* urow = us + (size_t)(w * P + r) * T::UW + T::CO + P + lane * P;
            if constexpr (MODE == MODE_APPLY) {
                #pragma unroll
                for (int j = 0; j < P; ++j)
                    if (!edge || Jl + j < g.n1y) a.out[base + j] = Y[r][j];
            } else {
                double up[P], mi[P], uu[P], v[P];
                if constexpr (WCB2S_PREV_TMA != 0) {
                    lds_row<P>(reinterpret_cast<const double*>(st + al128(T::U_BYTES)) +
                                   (size_t)(w * P + r) * T::TJ + lane * P, up);
                } else {
                    #pragma unroll
                    for (int j = 0; j < P; ++j) up[j] = (!edge || Jl + j < g.n1y) ? a.prev[base + j] : 0.0;
                }
                if (tcl) {
                    #pragma unroll
                    for (int j = 0; j < P; ++j) mi[j] = mtab.v[r * P + j];
                } else {
                    #pragma unroll
                    for (int j = 0; j < P; ++j) mi[j] = (!edge || Jl + j < g.n1y) ? __ldg(a.minv + base + j) : 0.0;
                }
                lds_row<P>(urow, uu);
                const bool src = base + P - 1 >= a.F.lo && base <= a.F.hi;
                #pragma unroll
                for (int j = 0; j < P; ++j) {
                    const double fF = src ? f * source_at(a.F, base + j) : f * 0.0;
                    v[j] = leapfrog(uu[j], up[j], Y[r][j], mi[j], fF, a.dt2);
                }
                if constexpr (P == 4) {
                    if (!edge) {
                        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(a.out + base),
                                     "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]) : "memory");
                        #pragma unroll
                        for (int j = 0; j < P; ++j) {
                            const unsigned long long bb = mi[j] != 0.0 ? amp_bits(v[j]) : 0ULL;
                            amp = bb > amp ? bb : amp;
                        }
                        continue;
                    }
                }
                #pragma unroll
                for (int j = 0; j < P; ++j) {
                    if (!edge || Jl + j < g.n1y) {
                        a.out[base + j] = v[j];
                        const unsigned long long bb = mi[j] != 0.0 ? amp_bits(v[j]) : 0ULL;
                        amp = bb > amp ? bb : amp;
                    }
                }
            }
        }
        __syncthreads();   // stage b and this parity's carry are free again
    }
    if constexpr (MODE == MODE_STEP) warp_amp_max(amp, a.amp);
}

// ---------------------------------------------------------------------------
// K x at a set of DOF rows (IMEX c rows) from the cells touching them only:
// one warp per cell computes the dense element product y_e = K_e u_e (the
// shared uncut element matrix in shared memory, or the cell's cut matrix),
// then every row sums its cells' contributions in ascending cell order.
template <int L>
__global__ void __launch_bounds__(256) k_rc_cells(int64_t n_cells, const int64_t* __restrict__ base,
                                                  const int32_t* __restrict__ cutid, const double* __restrict__ Kref,
                                                  const double* __restrict__ KT, int64_t pitch, int64_t plane,
                                                  int P, int ncomp, double sk, const double* __restrict__ x,
                                                  double* __restrict__ out) {
    __shared__ double Ks[L * L];
    __shared__ double us[8][L];
    for (int i = threadIdx.x; i < L * L; i += blockDim.x) Ks[i] = Kref[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int N = P + 1;
    for (int64_t c = (int64_t)blockIdx.x * 8 + w; c < n_cells; c += (int64_t)gridDim.x * 8) {
        const int64_t b0 = base[c];
        for (int m = lane; m < L; m += 32) {
            const int comp = m / (N * N), a = (m / N) % N, bb = m % N;
            us[w][m] = x[b0 + comp * plane + a * pitch + bb];
        }
        __syncwarp();
        const int32_t id = cutid[c];
        for (int r = lane; r < L; r += 32) {
            double t = 0.0;
            if (id < 0) {
                for (int m = 0; m < L; ++m) t = fma(Ks[r * L + m], us[w][m], t);
            } else {
                const double* K = KT + (int64_t)id * L * L;
                for (int m = 0; m < L; ++m) t = fma(__ldg(K + m * L + r), us[w][m], t);
            }
            out[c * L + r] = sk * t;
        }
        __syncwarp();
    }
}
__global__ void k_rc_rows(int64_t n_rows, const int32_t* __restrict__ ptr, const int64_t* __restrict__ src,
                          const double* __restrict__ cell_out, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int j = ptr[i]; j < ptr[i + 1]; ++j) s += cell_out[src[j]];
        y[i] = s;
    }
}


#include "wcb_ela2d.cuh"

struct ScmOperator final : Operator {
    int dim = 2, p = 4;
    int64_t n_e = 0, n1 = 0, pitch = 0, rows = 0;
    int64_t pplane = 0, n_zs = 0, n_yb = 0, n_xc = 0, xc3 = 0, ex_last = 0;   // 3D streaming grid
    int64_t probe_base = -1;          // 3D: state index of an interior uncut cell's node (0,0,0)
    std::vector<double> minv_tab;     // its P^3 owned 1/m values (bind_minv)
    DevBuf<uint8_t> clean;            // 3D: per local cell: 1/m class (1: owned 1/m == minv_tab, 2: no DOF)
    DevBuf<uint8_t> cinfo;            // 3D: mask with the class in bits 2-3
    DevBuf<uint8_t> tclean;           // 2D: per tile
    DevBuf<uint8_t> sflags;           // elastic streaming step: per (x chunk, strip) owns a DOF
    int64_t n_xs = 0, xs_len = 0;     // elastic streaming step: x chunks, cell rows per chunk
    const double* minv_bound = nullptr;
    // x slab (local numbering): cell rows 0..n_ex-1 (0 = halo row above),
    // node rows 0..n1x-1, owned node rows [row_lo, row_hi)
    int64_t n_ex = 0, n1x = 0, row_lo = 0, row_hi = 0, xstride = 0;
    bool has_top = false, owns_last = true;
    std::vector<int64_t> sidx;
    DevBuf<int64_t> d_sidx;
    DevBuf<uint8_t> mask, cflags;
    DevBuf<int32_t> cut_id;
    MapCache maps;
    DevBuf<double> KT;
    DevBuf<double> KP, cut_out;      // 3D: packed cut matrices, per-step products
    DevBuf<int64_t> cut_base;        // 3D: state index of each cut cell's first node
    DevBuf<double2> zline;           // 3D, n_e % 32 == 0: z-lines of the last cell column
    DevBuf<int32_t> order;        // 2D tile kernel: live tiles, most expensive first
    int64_t n_order = 0;
    std::vector<double> tile_cost;           // 2D: per tile (strip-major), for the chunk order
    DevBuf<int32_t> chunks;                  // streaming kernel: live chunks, most expensive first
    int64_t n_chunks = 0, chunk_nt = 0;
    // apply restricted to the tiles owning a given DOF subset (IMEX c rows)
    DevBuf<int32_t> order_sub;
    int64_t n_order_sub = 0;
    bool sub_ready = false, sub_active = false;
    std::vector<int32_t> order_h;            // host copy of the dispatch order
    std::vector<uint8_t> mask_h;             // 2D: host copy of the cell codes (zero ring)
    // step split (IMEX): every node of every cut cell is an implicit row, whose
    // explicit K psi is multiplied by 1/m = 0 -- the part steps skip the dense
    // cut-cell products
    bool part_skip_cut = false;
    DevBuf<int32_t> order_part[2];           // step split: far / near tiles (dispatch order kept)
    int64_t n_order_part[2] = {0, 0};
    int part_active = -1;
    int64_t n_strips = 0, n_rtiles = 0;
    std::vector<double> m1, k1;
    double sk = 1.0;
    // plane-strain elasticity (ncomp = 2): component planes `plane` apart
    int ncomp = 1;
    std::vector<double> g1;
    double lam = 0.0, mu = 0.0;
    int64_t plane = 0;
    int64_t n_cut = 0;
    int L = 0;
    double bytes_step = 0.0;

    const char* name() const override { return "scm"; }
    std::string step_kernel() const override {
        const std::string P = std::to_string(p);
        if (dim == 3)
            return std::string("k_scm3d<") + P + ",STEP> + k_cut_pre<" + P + ">" +
                   (n_e % 32 == 0 ? " + k_scm3d_zline/zcol" : "");
        if (ncomp == 2) return "k_ela2d<" + P + ",STEP> (plane strain, fused CDM update)";
        return (stream2d_off ? "k_scm2d<" : "k_scm2s<") + P + ",STEP> (fused CDM update)";
    }
    const std::vector<int64_t>& state_index() const override { return sidx; }
    void scatter(const double* src, double* dst) override { launch_scatter(ctx, n, d_sidx.p, src, dst); }
    void gather(const double* src, double* dst) override { launch_gather(ctx, n, d_sidx.p, src, dst); }

    template <int P>
    const CUtensorMap& state_map(const double* ptr, int kind = 0) {
        using T = Tile2<P>;
        return maps.get(ptr, kind, [&] {
            const uint64_t dims[2] = {(uint64_t)pitch, (uint64_t)rows};
            const uint64_t strides[1] = {(uint64_t)pitch};
            const uint32_t box_u[2] = {(uint32_t)T::UW, (uint32_t)T::UH};
            const uint32_t box_e[2] = {(uint32_t)T::TJ, (uint32_t)T::TI};
            return make_map_f64(ptr, 2, dims, strides, kind == 0 ? box_u : box_e);
        });
    }
    // streaming step / apply of scalar 2D operators (k_scm2s): chunks of
    // chunk_nt row tiles per CTA; WAVECELL_B200_TILE2D=1 keeps the tile kernel
    // measured slower than the tile kernel on config 2 (41-44 vs 25.5 us per
    // step): opt-in with WAVECELL_B200_STREAM2D=1
    bool stream2d_off = !(getenv("WAVECELL_B200_STREAM2D") && getenv("WAVECELL_B200_STREAM2D")[0] == '1');
    bool use_stream2d() const {
        return !stream2d_off && ncomp == 1 && part_active < 0 && !sub_active && !tile_cost.empty();
    }
    template <int P>
    void build_chunks() {
        using T = Tile2S<P>;
        int per_sm = 0;
        ensure_smem_attr((const void*)k_scm2s<P, MODE_STEP>, ctx->device, (size_t)T::SMEM);
        WCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_scm2s<P, MODE_STEP>, T::NWARP * 32,
                                                               T::SMEM));
        const int64_t slots = std::max(1, per_sm) * (int64_t)ctx->sm_count;
        int64_t live = 0;
        for (double c : tile_cost) live += c > 0.0;
        // about WAVES waves of chunks (load balance) unless overridden
        const char* e = getenv("WAVECELL_B200_CHUNK_NT");
        const double waves = getenv("WAVECELL_B200_CHUNK_WAVES") ? atof(getenv("WAVECELL_B200_CHUNK_WAVES")) : 2.0;
        chunk_nt = e ? std::max(1, atoi(e)) : std::max<int64_t>(1, (int64_t)std::llround(live / (waves * slots)));
        std::vector<std::pair<double, int32_t>> w;
        for (int64_t st = 0; st < n_strips; ++st)
            for (int64_t rt = 0; rt < n_rtiles; rt += chunk_nt) {
                double c = 0.0;
                for (int64_t q = rt; q < std::min<int64_t>(rt + chunk_nt, n_rtiles); ++q) c += tile_cost[st * n_rtiles + q];
                if (c > 0.0) w.emplace_back(-c, (int32_t)(st * n_rtiles + rt));
            }
        std::stable_sort(w.begin(), w.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
        std::vector<int32_t> ord(w.size());
        for (size_t i = 0; i < w.size(); ++i) ord[i] = w[i].second;
        n_chunks = (int64_t)ord.size();
        chunks.alloc(std::max<int64_t>(n_chunks, 1));
        if (n_chunks) chunks.upload(ord.data(), ord.size(), ctx->stream);
        WCB_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    template <int P>
    const CUtensorMap& stream_map2(const double* ptr, int kind) {
        using T = Tile2S<P>;
        return maps.get(ptr, 40 + kind, [&] {
            const uint64_t dims[2] = {(uint64_t)pitch, (uint64_t)rows};
            const uint64_t strides[1] = {(uint64_t)pitch};
            const uint32_t box_u[2] = {(uint32_t)T::UW, (uint32_t)T::UH};
            const uint32_t box_h[2] = {(uint32_t)T::UW, (uint32_t)T::HH};
            const uint32_t box_e[2] = {(uint32_t)T::TJ, (uint32_t)T::TI};
            return make_map_f64(ptr, 2, dims, strides, kind == 0 ? box_u : kind == 1 ? box_h : box_e);
        });
    }
    template <int P, int MODE>
    void launch2st(const StepArgs& a, const Mats2<P>& mt) {
        using T = Tile2S<P>;
        if (!chunk_nt) build_chunks<P>();
        if (!n_chunks) return;
        ensure_smem_attr((const void*)k_scm2s<P, MODE>, ctx->device, (size_t)T::SMEM);
        Scm2DGeo g{n_ex, n_e, n1, row_lo, row_hi, mask.p, cut_id.p, KT.p, cflags.p, chunks.p, n_strips, n_rtiles,
                   pitch, nullptr, (int32_t)chunk_nt};
        MinvTab2<P> tab{};
        if (MODE == MODE_STEP && a.minv && a.minv == minv_bound && tclean.p) {
            g.tclean = tclean.p;
            for (int i = 0; i < P * P; ++i) tab.v[i] = minv_tab[i];
        }
        const CUtensorMap& mu = stream_map2<P>(a.cur, 0);
        const CUtensorMap& mh = stream_map2<P>(a.cur, 1);
        const CUtensorMap& mp = MODE == MODE_STEP ? stream_map2<P>(a.prev, 2) : mu;
        dim3 grid((unsigned)n_chunks);
        if (MODE == MODE_STEP && pdl_enabled()) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = grid;
            cfg.blockDim = dim3(T::NWARP * 32);
            cfg.dynamicSmemBytes = T::SMEM;
            cfg.stream = ctx->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            WCB_CUDA(cudaLaunchKernelEx(&cfg, k_scm2s<P, MODE>, mu, mh, mp, g, mt, tab, sk, a));
        } else {
            k_scm2s<P, MODE><<<grid, T::NWARP * 32, T::SMEM, ctx->stream>>>(mu, mh, mp, g, mt, tab, sk, a);
        }
        ctx->launches++;
    }
    template <int P, int MODE>
    void launch2d(const StepArgs& a) {
        using T = Tile2<P>;
        ensure_smem_attr((const void*)k_scm2d<P, MODE>, ctx->device, (size_t)T::SMEM);
        Mats2<P> mt;
        for (int i = 0; i <= P; ++i)
            for (int j = 0; j <= P; ++j)
                if (orb_key(P, i, j) == i * 16 + j) {
                    mt.m[orb(P, i, j)] = m1[i * (P + 1) + j];
                    mt.k[orb(P, i, j)] = k1[i * (P + 1) + j];
                }
        if (use_stream2d() && halo_part < 0) {
            launch2st<P, MODE>(a, mt);
            return;
        }
        const int32_t* ord = part_active >= 0 ? order_part[part_active].p : sub_active ? order_sub.p : order.p;
        int64_t n_ord = part_active >= 0 ? n_order_part[part_active] : sub_active ? n_order_sub : n_order;
        StepArgs a2 = a;
        if (MODE == MODE_STEP && halo_part >= 0) {   // slab step split around the halo exchange
            ord = order_halo[halo_part].p;
            n_ord = n_order_halo[halo_part];
            if (halo_part == 1) a2.obs_out = nullptr;   // observers recorded once, by part 0
        }
        if (!n_ord) return;
        Scm2DGeo g{n_ex, n_e, n1, row_lo, row_hi, mask.p, cut_id.p, KT.p, cflags.p, ord, n_strips, n_rtiles, pitch};
        if (MODE == MODE_STEP && part_active >= 0 && part_skip_cut) g.KT = nullptr;   // cut cells act on implicit rows only
        dim3 grid((unsigned)n_ord);
        const CUtensorMap& mu = state_map<P>(a.cur);
        const bool epi = WCB2D_EPI_TMA && MODE == MODE_STEP;
        const CUtensorMap& mp = epi ? state_map<P>(a.prev, 1) : mu;
        const CUtensorMap& mm = epi ? state_map<P>(a.minv, 1) : mu;
        MinvTab2<P> tab{};
        if (MODE == MODE_STEP && a.minv && a.minv == minv_bound && tclean.p) {
            g.tclean = tclean.p;
            for (int i = 0; i < P * P; ++i) tab.v[i] = minv_tab[i];
        }
        if (MODE == MODE_STEP && pdl_enabled() && part_active < 0) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = grid;
            cfg.blockDim = dim3(T::NWARP * 32);
            cfg.dynamicSmemBytes = T::SMEM;
            cfg.stream = ctx->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            WCB_CUDA(cudaLaunchKernelEx(&cfg, k_scm2d<P, MODE>, mu, mp, mm, g, mt, tab, sk, a2));
        } else {
            k_scm2d<P, MODE><<<grid, T::NWARP * 32, T::SMEM, ctx->stream>>>(mu, mp, mm, g, mt, tab, sk, a2);
        }
        ctx->launches++;
    }
    template <int P>
    const CUtensorMap& state_map_e(const double* ptr, int kind) {
        using T = Tile2E<P>;
        return maps.get(ptr, 20 + kind, [&] {
            const uint64_t dims[2] = {(uint64_t)pitch, (uint64_t)(2 * rows)};
            const uint64_t strides[1] = {(uint64_t)pitch};
            const uint32_t box[2] = {(uint32_t)(kind ? T::TJ : T::UW), (uint32_t)(kind ? T::TI : T::UH)};
            return make_map_f64(ptr, 2, dims, strides, box);
        });
    }
    template <int P>
    EMats<P> emats() const {
        constexpr int N = P + 1;
        EMats<P> mt;
        const double l2m = lam + 2.0 * mu;
        for (int r = 0; r < N; ++r)
            for (int c = 0; c < N; ++c) {
                const int rc = r * N + c, cr = c * N + r;
                mt.ym[rc] = m1[rc];
                mt.yk[rc] = k1[rc];
                mt.yg[rc] = g1[rc];
                mt.xa[0][0][rc] = l2m * k1[rc];
                mt.xa[0][1][rc] = mu * m1[rc];
                mt.xa[0][2][rc] = lam * g1[rc];
                mt.xa[0][3][rc] = mu * g1[cr];
                mt.xa[1][0][rc] = mu * k1[rc];
                mt.xa[1][1][rc] = l2m * m1[rc];
                mt.xa[1][2][rc] = lam * g1[cr];
                mt.xa[1][3][rc] = mu * g1[rc];
            }
        return mt;
    }
    // streaming elastic step (k_ela2s): maps with boxes (UW, P) and (TJ, P)
    template <int P>
    const CUtensorMap& stream_map_e(const double* ptr, int kind) {
        using T = Str2E<P>;
        return maps.get(ptr, 30 + kind, [&] {
            const uint64_t dims[2] = {(uint64_t)pitch, (uint64_t)(2 * rows)};
            const uint64_t strides[1] = {(uint64_t)pitch};
            const uint32_t box[2] = {(uint32_t)(kind ? T::TJ : T::UW), (uint32_t)P};
            return make_map_f64(ptr, 2, dims, strides, box);
        });
    }
    template <int P>
    void launch2s(const StepArgs& a) {
        using T = Str2E<P>;
        ensure_smem_attr((const void*)k_ela2s<P>, ctx->device, (size_t)T::SMEM);
        Scm2DGeo g{n_ex, n_e, n1, row_lo, row_hi, mask.p, cut_id.p, KT.p, sflags.p, nullptr, n_strips, n_rtiles,
                   pitch, nullptr};
        MinvTabE<P> tab{};
        const uint8_t* cl = nullptr;
        if (a.minv && a.minv == minv_bound && clean.p) {
            cl = clean.p;
            for (int i = 0; i < P * P; ++i) tab.v[i] = minv_tab[i];
        }
        const EMats<P> mt = emats<P>();
        dim3 grid((unsigned)n_strips, (unsigned)n_xs);
        k_ela2s<P><<<grid, 64, T::SMEM, ctx->stream>>>(stream_map_e<P>(a.cur, 0), stream_map_e<P>(a.prev, 1), g, mt,
                                                      plane, (int32_t)rows, xs_len, ex_last, cl, tab, a);
        ctx->launches++;
    }
    template <int P, int MODE>
    void launch2e(const StepArgs& a) {
        using T = Tile2E<P>;
        if (MODE == MODE_STEP && n_xs > 0 && getenv("WAVECELL_B200_STREAM_ELASTIC")) {   // experimental
            launch2s<P>(a);
            return;
        }
        ensure_smem_attr((const void*)k_ela2d<P, MODE>, ctx->device, (size_t)T::SMEM);
        const int32_t* ord = part_active >= 0 ? order_part[part_active].p : sub_active ? order_sub.p : order.p;
        const int64_t n_ord = part_active >= 0 ? n_order_part[part_active] : sub_active ? n_order_sub : n_order;
        if (!n_ord) return;
        const EMats<P> mt = emats<P>();
        Scm2DGeo g{n_ex, n_e, n1, row_lo, row_hi, mask.p, cut_id.p, KT.p, cflags.p, ord, n_strips, n_rtiles, pitch};
        if (MODE == MODE_STEP && part_active >= 0 && part_skip_cut) g.KT = nullptr;   // cut cells act on implicit rows only
        const CUtensorMap& mu_ = state_map_e<P>(a.cur, 0);
        const bool epi = MODE == MODE_STEP;
        const CUtensorMap& mp = epi ? state_map_e<P>(a.prev, 1) : mu_;
        const CUtensorMap& mm = epi ? state_map_e<P>(a.minv, 1) : mu_;
        MinvTabE<P> tab{};
        if (MODE == MODE_STEP && a.minv && a.minv == minv_bound && tclean.p) {
            g.tclean = tclean.p;
            for (int i = 0; i < P * P; ++i) tab.v[i] = minv_tab[i];
        }
        k_ela2d<P, MODE><<<(unsigned)n_ord, T::NWARP * 32, T::SMEM, ctx->stream>>>(
            mu_, mp, mm, g, mt, plane, (int32_t)rows, tab, a);
        ctx->launches++;
    }
    template <int MODE>
    void dispatch2e(const StepArgs& a) {
        switch (p) {
            case 1: launch2e<1, MODE>(a); break;
            case 2: launch2e<2, MODE>(a); break;
            case 3: launch2e<3, MODE>(a); break;
            case 4: launch2e<4, MODE>(a); break;
            case 5: launch2e<5, MODE>(a); break;
            default: throw Error{WCB_E_UNSUPPORTED, "2D elastic kernel built for p = 1..5"};
        }
    }
    template <int MODE>
    void dispatch2d(const StepArgs& a) {
        if (ncomp == 2) {
            dispatch2e<MODE>(a);
            return;
        }
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
    template <int P>
    const CUtensorMap& state_map3(const double* ptr) {
        using T = Str3<P>;
        return maps.get(ptr, 3, [&] {
            const uint64_t dims[3] = {(uint64_t)pitch, (uint64_t)rows, (uint64_t)(n1x + 2 * p)};
            const uint64_t strides[2] = {(uint64_t)pitch, (uint64_t)pplane};
            const uint32_t box[3] = {(uint32_t)T::UW, (uint32_t)T::UR, 1u};
            return make_map_f64(ptr, 3, dims, strides, box);
        });
    }
    template <int P>
    const CUtensorMap& prev_map3(const double* ptr) {   // owned box of one cell row
        using T = Str3<P>;
        return maps.get(ptr, 4, [&] {
            const uint64_t dims[3] = {(uint64_t)pitch, (uint64_t)rows, (uint64_t)(n1x + 2 * p)};
            const uint64_t strides[2] = {(uint64_t)pitch, (uint64_t)pplane};
            const uint32_t box[3] = {(uint32_t)T::TZ, (uint32_t)(T::WY * P), (uint32_t)P};
            return make_map_f64(ptr, 3, dims, strides, box);
        });
    }
    template <int P, int MODE>
    void launch3d(const StepArgs& a) {
        Mats2<P> mt;
        for (int i = 0; i <= P; ++i)
            for (int j = 0; j <= P; ++j)
                if (orb_key(P, i, j) == i * 16 + j) {
                    mt.m[orb(P, i, j)] = m1[i * (P + 1) + j];
                    mt.k[orb(P, i, j)] = k1[i * (P + 1) + j];
                }
        if (halo_part != 1) launch_cut_pre<P>(ctx, n_cut, KP.p, cut_base.p, pplane, pitch, a.cur, cut_out.p);
        Scm3DGeo g = geo3();
        MinvTab<P> tab{};
        if (MODE == MODE_STEP && a.minv && a.minv == minv_bound && clean.p) {
            g.clean = clean.p;
            g.mask = cinfo.p;   // codes + 1/m classes
            for (int i = 0; i < P * P * P; ++i) tab.v[i] = minv_tab[i];
        }
        const CUtensorMap& mu = state_map3<P>(a.cur);
        launch_scm3d<P, MODE>(ctx, mu, MODE == MODE_STEP ? prev_map3<P>(a.prev) : mu, g, mt, tab, sk, a,
                              MODE == MODE_STEP ? halo_part : -1);
    }
    Scm3DGeo geo3() const {
        return Scm3DGeo{n_ex, row_lo, row_hi, n_e, n1, pitch, pplane, mask.p, cut_id.p, cut_out.p, cflags.p,
                        n_zs, n_yb, n_xc, xc3, ex_last, nullptr, zline.p};
    }
    template <int P>
    void bind3(const double* d_minv) {
        MinvTab<P> tab{};
        std::vector<double> h(P * P * P);
        for (int q = 0; q < P; ++q)
            for (int r = 0; r < P; ++r)
                WCB_CUDA(cudaMemcpyAsync(h.data() + (q * P + r) * P, d_minv + probe_base + q * pplane + r * pitch,
                                         P * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        WCB_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int i = 0; i < P * P * P; ++i) {
            if (!(h[i] > 0.0)) return;   // probe is not a DOF cell: keep loading 1/m everywhere
            tab.v[i] = h[i];
        }
        if (!clean.p) clean.alloc((size_t)n_ex * n_e * n_e);
        if (!cinfo.p) cinfo.alloc(mask.n);
        WCB_CUDA(cudaMemcpyAsync(cinfo.p, mask.p, mask.n, cudaMemcpyDeviceToDevice, ctx->stream));
        launch_clean3d<P>(ctx, geo3(), tab, d_minv, clean.p, cinfo.p, zero_dead);
        WCB_CHECK_LAUNCH();
        std::vector<uint8_t> hc(clean.n);
        WCB_CUDA(cudaMemcpyAsync(hc.data(), clean.p, hc.size(), cudaMemcpyDeviceToHost, ctx->stream));
        WCB_CUDA(cudaStreamSynchronize(ctx->stream));
        int64_t nclean = 0;
        for (uint8_t v : hc) nclean += v == 1;
        minv_skipped = (double)nclean * P * P * P;
        minv_tab = h;
        minv_bound = d_minv;
    }
    template <int P>
    void bind2(const double* d_minv) {
        using T = Tile2<P>;
        MinvTab2<P> tab{};
        std::vector<double> h(P * P);
        for (int r = 0; r < P; ++r)
            WCB_CUDA(cudaMemcpyAsync(h.data() + r * P, d_minv + probe_base + r * pitch, P * sizeof(double),
                                     cudaMemcpyDeviceToHost, ctx->stream));
        WCB_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int i = 0; i < P * P; ++i) {
            if (!(h[i] > 0.0)) return;
            tab.v[i] = h[i];
        }
        const int64_t nt = n_strips * n_rtiles;
        if (!tclean.p) tclean.alloc((size_t)nt);
        Scm2DGeo g{n_ex, n_e, n1, row_lo, row_hi, mask.p, cut_id.p, KT.p, cflags.p, order.p, n_strips, n_rtiles,
                   pitch, nullptr};
        k_clean2d<P><<<(unsigned)nt, 128, 0, ctx->stream>>>(g, T::TI, T::TJ, tab, d_minv, tclean.p);
        ctx->launches++;
        WCB_CHECK_LAUNCH();
        std::vector<uint8_t> hc(nt);
        WCB_CUDA(cudaMemcpyAsync(hc.data(), tclean.p, nt, cudaMemcpyDeviceToHost, ctx->stream));
        WCB_CUDA(cudaStreamSynchronize(ctx->stream));
        minv_skipped = 0.0;
        for (int64_t t = 0; t < nt; ++t)
            if (hc[t]) {
                const int64_t I0 = row_lo + (t % n_rtiles) * T::TI, J0 = (t / n_rtiles) * T::TJ;
                minv_skipped += (double)(std::min<int64_t>(T::TI, row_hi - I0) * std::min<int64_t>(T::TJ, n1 - J0));
            }
        minv_tab = h;
        minv_bound = d_minv;
    }
    template <int P>
    void bind2e(const double* d_minv) {
        MinvTab2<P> tab{};
        std::vector<double> h(P * P);
        for (int r = 0; r < P; ++r)
            WCB_CUDA(cudaMemcpyAsync(h.data() + r * P, d_minv + probe_base + r * pitch, P * sizeof(double),
                                     cudaMemcpyDeviceToHost, ctx->stream));
        WCB_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int i = 0; i < P * P; ++i) {
            if (!(h[i] > 0.0)) return;
            tab.v[i] = h[i];
        }
        const int64_t nc = n_ex * n_e;
        if (!clean.p) clean.alloc((size_t)nc);
        k_clean2e<P><<<(unsigned)ceil_div(nc, 256), 256, 0, ctx->stream>>>(n_ex, n_e, row_hi, pitch, plane, tab,
                                                                          d_minv, clean.p);
        ctx->launches++;
        WCB_CHECK_LAUNCH();
        std::vector<uint8_t> hc(nc);
        WCB_CUDA(cudaMemcpyAsync(hc.data(), clean.p, nc, cudaMemcpyDeviceToHost, ctx->stream));
        WCB_CUDA(cudaStreamSynchronize(ctx->stream));
        int64_t ncl = 0;
        for (uint8_t v : hc) ncl += v;
        minv_skipped = 2.0 * (double)ncl * P * P;   // both components (streaming kernel)
        // tile kernel: a tile is clean when all its cells are
        {
            using TE = Tile2E<P>;
            const int64_t nt = n_strips * n_rtiles;
            std::vector<uint8_t> tc(nt, 0);
            double skipped_tiles = 0.0;
            for (int64_t t = 0; t < nt; ++t) {
                const int64_t strip = t / n_rtiles, rt = t % n_rtiles;
                const int64_t ex0 = (row_lo + rt * TE::TI) / P, ey0 = strip * 32;
                bool ok = ey0 + 32 <= n_e && ex0 + TE::RPE <= n_ex;
                for (int64_t ex = ex0; ok && ex < ex0 + TE::RPE; ++ex)
                    for (int64_t ey = ey0; ok && ey < ey0 + 32; ++ey) ok = hc[ex * n_e + ey] != 0;
                if (ok) {
                    tc[t] = 1;
                    skipped_tiles += 2.0 * (double)(std::min<int64_t>(TE::TI, row_hi - (row_lo + rt * TE::TI)) * TE::TJ);
                }
            }
            if (!tclean.p) tclean.alloc((size_t)nt);
            tclean.upload(tc.data(), nt, ctx->stream);
            WCB_CUDA(cudaStreamSynchronize(ctx->stream));
            if (!n_xs || !getenv("WAVECELL_B200_STREAM_ELASTIC")) minv_skipped = skipped_tiles;
        }
        minv_tab = h;
        minv_bound = d_minv;
    }
    bool zero_dead = false;
    void bind_minv(const double* d_minv, bool zero_is_dead) override {
        zero_dead = zero_is_dead;
        minv_bound = nullptr;
        minv_skipped = 0.0;
        if (probe_base < 0 || !d_minv || getenv("WAVECELL_B200_NO_MINV_TAB")) return;
        if (dim == 2 && ncomp == 2) {
            switch (p) {
                case 1: bind2e<1>(d_minv); break;
                case 2: bind2e<2>(d_minv); break;
                case 3: bind2e<3>(d_minv); break;
                case 4: bind2e<4>(d_minv); break;
                case 5: bind2e<5>(d_minv); break;
            }
            return;
        }
        if (dim == 2) {
            if (ncomp != 1 || !WCB2D_EPI_TMA) return;
            switch (p) {
                case 1: bind2<1>(d_minv); break;
                case 2: bind2<2>(d_minv); break;
                case 3: bind2<3>(d_minv); break;
                case 4: bind2<4>(d_minv); break;
                case 5: bind2<5>(d_minv); break;
                case 6: bind2<6>(d_minv); break;
            }
            return;
        }
        switch (p) {
            case 1: bind3<1>(d_minv); break;
            case 2: bind3<2>(d_minv); break;
            case 3: bind3<3>(d_minv); break;
            case 4: bind3<4>(d_minv); break;
        }
    }
    template <int MODE>
    void dispatch3d(const StepArgs& a) {
        switch (p) {
            case 1: launch3d<1, MODE>(a); break;
            case 2: launch3d<2, MODE>(a); break;
            case 3: launch3d<3, MODE>(a); break;
            case 4: launch3d<4, MODE>(a); break;
            default: throw Error{WCB_E_UNSUPPORTED, "3D SCM kernel built for p = 1..4"};
        }
    }
    void apply(const double* x, double* y) override {
        StepArgs a;
        a.cur = x;
        a.out = y;
        if (dim == 3) dispatch3d<MODE_APPLY>(a); else dispatch2d<MODE_APPLY>(a);
        WCB_CHECK_LAUNCH();
    }
    void cdm_step(const StepArgs& a) override {
        if (dim == 3) dispatch3d<MODE_STEP>(a); else dispatch2d<MODE_STEP>(a);
        WCB_CHECK_LAUNCH();
    }
    bool set_apply_subset(const int64_t* ids, int64_t n_ids) override {
        if (dim != 2) return false;
        const int RX = ncomp == 2 ? rpe_e(p) : rpe_for(p);
        const int64_t TI = (int64_t)RX * p, TJ = 32 * (int64_t)p;
        std::vector<uint8_t> mark(n_strips * n_rtiles, 0);
        for (int64_t k = 0; k < n_ids; ++k) {
            const int64_t sidx_k = sidx[ids[k]] % plane;   // same tile in both planes
            const int64_t row = sidx_k / pitch - p, col = sidx_k % pitch - PADJ;
            mark[(col / TJ) * n_rtiles + (row - row_lo) / TI] = 1;
        }
        std::vector<int32_t> ord;
        for (int64_t t = 0; t < (int64_t)mark.size(); ++t)
            if (mark[t]) ord.push_back((int32_t)t);
        n_order_sub = (int64_t)ord.size();
        order_sub.alloc(std::max<int64_t>(n_order_sub, 1));
        if (n_order_sub) order_sub.upload(ord.data(), ord.size(), ctx->stream);
        WCB_CUDA(cudaStreamSynchronize(ctx->stream));
        sub_ready = true;
        return true;
    }
    bool set_step_split(const int64_t* ids, int64_t n_ids) override {
        if (dim != 2 || order_h.empty()) return false;
        const int RX = ncomp == 2 ? rpe_e(p) : rpe_for(p);
        const int64_t TI = (int64_t)RX * p, TJ = 32 * (int64_t)p;
        std::vector<uint8_t> near(n_strips * n_rtiles, 0);
        for (int64_t k = 0; k < n_ids; ++k) {
            const int64_t sk_ = sidx[ids[k]] % plane;
            const int64_t row = sk_ / pitch - p, col = sk_ % pitch - PADJ;   // local node coordinates
            // tiles whose input footprint [I0-p, I0+TI] x [J0-p-1, J0+TJ+1] holds the node
            const int64_t rt_lo = std::max<int64_t>(0, (row - TI - row_lo) / TI - 1);
            const int64_t rt_hi = std::min<int64_t>(n_rtiles - 1, (row + p - row_lo) / TI + 1);
            const int64_t st_lo = std::max<int64_t>(0, (col - TJ - 1) / TJ - 1);
            const int64_t st_hi = std::min<int64_t>(n_strips - 1, (col + p + 1) / TJ + 1);
            for (int64_t rt = rt_lo; rt <= rt_hi; ++rt)
                for (int64_t st = st_lo; st <= st_hi; ++st) {
                    const int64_t I0 = row_lo + rt * TI, J0 = st * TJ;
                    if (row >= I0 - p && row <= I0 + TI && col >= J0 - p - 1 && col <= J0 + TJ + 1)
                        near[st * n_rtiles + rt] = 1;
                }
        }
        // are all nodes of all cut cells implicit rows?
        part_skip_cut = false;
        if (!mask_h.empty() && !getenv("WAVECELL_B200_IMEX_KEEP_CUT")) {
            std::vector<uint8_t> is_c((size_t)plane * ncomp, 0);
            for (int64_t k = 0; k < n_ids; ++k) is_c[sidx[ids[k]]] = 1;
            bool all = true;
            const int64_t ms_ = n_e + 2;
            for (int64_t ex = 0; ex < n_ex && all; ++ex)
                for (int64_t ey = 0; ey < n_e && all; ++ey) {
                    if (mask_h[(ex + 1) * ms_ + ey + 1] != 2) continue;
                    for (int a = 0; a <= p && all; ++a)
                        for (int b = 0; b <= p && all; ++b)
                            for (int cc = 0; cc < ncomp && all; ++cc)
                                all = is_c[cc * plane + (ex * p + a + p) * pitch + ey * p + b + PADJ] != 0;
                }
            part_skip_cut = all;
        }
        std::vector<int32_t> part[2];
        for (int32_t t : order_h) part[near[t] ? 1 : 0].push_back(t);
        for (int q = 0; q < 2; ++q) {
            n_order_part[q] = (int64_t)part[q].size();
            order_part[q].alloc(std::max<int64_t>(n_order_part[q], 1));
            if (n_order_part[q]) order_part[q].upload(part[q].data(), part[q].size(), ctx->stream);
        }
        WCB_CUDA(cudaStreamSynchronize(ctx->stream));
        return true;
    }
    void cdm_step_part(const StepArgs& a, int part) override {
        if (dim != 2 || n_order_part[0] + n_order_part[1] == 0) {
            if (part == 1) cdm_step(a);
            return;
        }
        part_active = part;
        dispatch2d<MODE_STEP>(a);
        part_active = -1;
        WCB_CHECK_LAUNCH();
    }
    void apply_subset(const double* x, double* y) override {
        if (!sub_ready) { apply(x, y); return; }
        sub_active = true;
        StepArgs a;
        a.cur = x;
        a.out = y;
        dispatch2d<MODE_APPLY>(a);
        sub_active = false;
        WCB_CHECK_LAUNCH();
    }
    // slab step split around the halo exchange (cdm_step_halo_part)
    int halo_part = -1;
    bool halo_split_built = false;
    DevBuf<int32_t> order_halo[2];           // 2D: tiles writing exchanged rows / the rest
    int64_t n_order_halo[2] = {0, 0};
    bool halo_split_ready() override {
        int64_t h[8];
        if (!halo(h) || ncomp != 1) return false;
        if (dim == 3) return n_xc >= 3;
        if (!halo_split_built) {
            // tiles holding an owned node row sent to a neighbour: the first
            // owned row (-> previous slab) and the last p owned rows (-> next)
            const int64_t TI = (int64_t)rpe_for(p) * p;
            std::vector<int32_t> part[2];
            for (int32_t t : order_h) {
                const int64_t rt = t % n_rtiles;
                const int64_t I0 = row_lo + rt * TI, I1 = std::min<int64_t>(I0 + TI, row_hi);
                const bool sends = (has_top && I0 <= row_lo && row_lo < I1) ||
                                   (!owns_last && I1 > row_hi - p);
                part[sends ? 0 : 1].push_back(t);
            }
            for (int q = 0; q < 2; ++q) {
                n_order_halo[q] = (int64_t)part[q].size();
                order_halo[q].alloc(std::max<int64_t>(n_order_halo[q], 1));
                if (n_order_halo[q]) order_halo[q].upload(part[q].data(), part[q].size(), ctx->stream);
            }
            WCB_CUDA(cudaStreamSynchronize(ctx->stream));
            halo_split_built = true;
        }
        return n_order_halo[0] > 0 && n_order_halo[1] > 0;
    }
    void cdm_step_halo_part(const StepArgs& a, int part) override {
        halo_part = part;
        try {
            if (dim == 3) dispatch3d<MODE_STEP>(a); else dispatch2d<MODE_STEP>(a);
        } catch (...) {
            halo_part = -1;
            throw;
        }
        halo_part = -1;
        WCB_CHECK_LAUNCH();
    }
    // IMEX c rows by cells (set_row_subset / apply_rows)
    int64_t rc_n_cells = 0, rc_n_rows = 0;
    DevBuf<int64_t> rc_base, rc_src;
    DevBuf<int32_t> rc_cutid, rc_ptr;
    DevBuf<double> rc_Kref, rc_out;
    bool set_row_subset(const int64_t* ids, int64_t n_ids) override {
        if (dim != 2) return false;
        const int P = p, N = p + 1;
        const int Lr = ncomp * N * N;
        if (Lr != 25 && Lr != 72 && Lr != 16 && Lr != 9 && Lr != 4 && Lr != 36 && Lr != 49 && Lr != 8 &&
            Lr != 18 && Lr != 32 && Lr != 50)
            return false;
        // cells touching each row's node: local (ex, ey) with ex*P <= I <= ex*P+P
        std::vector<std::pair<int64_t, int>> contrib;   // (cell key, local row) per row, flattened
        std::vector<int32_t> ptr(n_ids + 1, 0);
        std::vector<int64_t> cells;
        std::vector<std::vector<std::pair<int64_t, int>>> per(n_ids);
        const int64_t ms_ = n_e + 2;
        std::vector<uint8_t> hmask;
        {
            hmask.resize(mask.n);
            WCB_CUDA(cudaMemcpy(hmask.data(), mask.p, mask.n, cudaMemcpyDeviceToHost));
        }
        for (int64_t k = 0; k < n_ids; ++k) {
            const int64_t st = sidx[ids[k]];
            const int comp = (int)(st / (plane ? plane : INT64_MAX));
            const int64_t s0 = st - comp * plane;
            const int64_t I = s0 / pitch - P, J = s0 % pitch - PADJ;   // local node coordinates
            for (int64_t ex = I / P - 1; ex <= I / P; ++ex) {
                if (ex < 0 || ex >= n_ex || I < ex * P || I > ex * P + P) continue;
                for (int64_t ey = J / P - 1; ey <= J / P; ++ey) {
                    if (ey < 0 || ey >= n_e || J < ey * P || J > ey * P + P) continue;
                    if (hmask[(ex + 1) * ms_ + ey + 1] == 0) continue;
                    const int a = (int)(I - ex * P), b = (int)(J - ey * P);
                    per[k].emplace_back(ex * n_e + ey, comp * N * N + a * N + b);
                    cells.push_back(ex * n_e + ey);
                }
            }
        }
        std::sort(cells.begin(), cells.end());
        cells.erase(std::unique(cells.begin(), cells.end()), cells.end());
        std::vector<int64_t> src, cbase(cells.size());
        std::vector<int32_t> cid(cells.size(), -1);
        std::vector<int32_t> hcid(cut_id.n);
        WCB_CUDA(cudaMemcpy(hcid.data(), cut_id.p, cut_id.n * sizeof(int32_t), cudaMemcpyDeviceToHost));
        for (size_t q = 0; q < cells.size(); ++q) {
            const int64_t ex = cells[q] / n_e, ey = cells[q] % n_e;
            cbase[q] = (ex * P + P) * pitch + ey * P + PADJ;
            cid[q] = hcid[cells[q]];
        }
        for (int64_t k = 0; k < n_ids; ++k) {
            std::sort(per[k].begin(), per[k].end());
            for (auto& e : per[k]) {
                const int64_t q = std::lower_bound(cells.begin(), cells.end(), e.first) - cells.begin();
                src.push_back(q * Lr + e.second);
            }
            ptr[k + 1] = (int32_t)src.size();
        }
        // uncut element matrix / sk (the kernels scale by sk, as the cut KT)
        std::vector<double> Kr((size_t)Lr * Lr, 0.0);
        const double l2m = lam + 2.0 * mu;
        for (int r = 0; r < Lr; ++r)
            for (int m = 0; m < Lr; ++m) {
                const int cr = r / (N * N), ar = (r / N) % N, br = r % N;
                const int cm = m / (N * N), am = (m / N) % N, bm = m % N;
                const double Kxx = k1[ar * N + am] * m1[br * N + bm];   // x derivatives
                const double Kyy = m1[ar * N + am] * k1[br * N + bm];
                double v;
                if (ncomp == 1) {
                    v = Kxx + Kyy;
                } else {
                    // Kxy[(a,b),(c,d)] = g1[a][c] g1[d][b]; Kuv = lam Kxy + mu Kxy^T
                    const double Kxy = g1[ar * N + am] * g1[bm * N + br];
                    const double KxyT = g1[am * N + ar] * g1[br * N + bm];
                    if (cr == 0 && cm == 0) v = l2m * Kxx + mu * Kyy;
                    else if (cr == 1 && cm == 1) v = mu * Kxx + l2m * Kyy;
                    else if (cr == 0) v = lam * Kxy + mu * KxyT;
                    else v = lam * KxyT + mu * Kxy;   // (Kuv)^T
                }
                Kr[(size_t)r * Lr + m] = v;
            }
        cudaStream_t st = ctx->stream;
        rc_n_cells = (int64_t)cells.size();
        rc_n_rows = n_ids;
        rc_base.alloc(std::max<int64_t>(rc_n_cells, 1), st); rc_base.upload(cbase.data(), cbase.size(), st);
        rc_cutid.alloc(std::max<int64_t>(rc_n_cells, 1), st); rc_cutid.upload(cid.data(), cid.size(), st);
        rc_ptr.alloc(ptr.size(), st); rc_ptr.upload(ptr.data(), ptr.size(), st);
        rc_src.alloc(std::max<size_t>(src.size(), 1), st); rc_src.upload(src.data(), src.size(), st);
        rc_Kref.alloc(Kr.size(), st); rc_Kref.upload(Kr.data(), Kr.size(), st);
        rc_out.alloc(std::max<int64_t>(rc_n_cells, 1) * Lr, st);
        WCB_CUDA(cudaStreamSynchronize(st));
        return true;
    }
    template <int L>
    void launch_rc(const double* x, double* out) {
        const int64_t blocks = std::min<int64_t>(ceil_div(rc_n_cells, 8), (int64_t)ctx->sm_count * 8);
        if (rc_n_cells)
            k_rc_cells<L><<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, ctx->stream>>>(
                rc_n_cells, rc_base.p, rc_cutid.p, rc_Kref.p, KT.p, pitch, plane, p, ncomp, ncomp == 1 ? sk : 1.0, x,
                rc_out.p);
        k_rc_rows<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rc_n_rows, 256), (int64_t)ctx->sm_count * 8)),
                    256, 0, ctx->stream>>>(rc_n_rows, rc_ptr.p, rc_src.p, rc_out.p, out);
        ctx->launches += 2;
    }
    bool apply_rows(const double* x, double* out) override {
        if (!rc_n_rows) return false;
        switch (ncomp * (p + 1) * (p + 1)) {
            case 4: launch_rc<4>(x, out); break;
            case 8: launch_rc<8>(x, out); break;
            case 9: launch_rc<9>(x, out); break;
            case 16: launch_rc<16>(x, out); break;
            case 18: launch_rc<18>(x, out); break;
            case 25: launch_rc<25>(x, out); break;
            case 32: launch_rc<32>(x, out); break;
            case 36: launch_rc<36>(x, out); break;
            case 49: launch_rc<49>(x, out); break;
            case 50: launch_rc<50>(x, out); break;
            case 72: launch_rc<72>(x, out); break;
            default: return false;
        }
        WCB_CHECK_LAUNCH();
        return true;
    }
    double step_bytes() const override { return bytes_step; }
    bool halo(int64_t* h) const override {
        // state row = local node row + p
        h[0] = xstride;
        h[1] = has_top ? p : 0;                 // top halo: local rows 0..p-1
        h[2] = has_top ? p : 0;
        h[3] = owns_last ? 0 : row_hi + p;      // bottom halo: local row row_hi
        h[4] = owns_last ? 0 : 1;
        h[5] = row_hi;                          // last p owned rows (state rows) -> next slab
        h[6] = owns_last ? 0 : p;
        h[7] = row_lo + p;                      // first owned row -> previous slab's bottom halo
        return has_top || !owns_last;
    }
};

template <int P>
static int ela2s_occ() {
    int nb = 0;
    WCB_CUDA(cudaFuncSetAttribute(k_ela2s<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Str2E<P>::SMEM));
    WCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_ela2s<P>, 64, Str2E<P>::SMEM));
    return nb;
}
static int ela2s_ctas_per_sm(int p) {
    switch (p) {
        case 1: return ela2s_occ<1>();
        case 2: return ela2s_occ<2>();
        case 3: return ela2s_occ<3>();
        case 4: return ela2s_occ<4>();
        default: return ela2s_occ<5>();
    }
}

// Both dimensions: slab preprocessing (cell rows [x_cell_lo-1, x_cell_hi) of
// the global grid along x, one halo cell row above), state layout, tile flags,
// cut-cell tables.
static Operator* build_scm_operator(Context* ctx, const wcb_scm_desc* d, int ncomp, double lam,
                                    double mu, const double* g1);

Operator* make_scm_operator(Context* ctx, const wcb_scm_desc* d) {
    return build_scm_operator(ctx, d, 1, 0.0, 0.0, nullptr);
}

// Plane strain: the node grid of the scalar descriptor carries two
// displacement components (compact DOF = comp * n_node + node).
Operator* make_elastic_operator(Context* ctx, const wcb_elastic_desc* e) {
    WCB_REQUIRE(e && e->m1 && e->k1 && e->g1, "NULL array in elastic descriptor");
    WCB_REQUIRE(e->p >= 1 && e->p <= 5, "p must be in 1..5 for the elastic kernel");
    WCB_REQUIRE(e->lam + 2.0 * e->mu > 0.0 && e->mu > 0.0, "Lame parameters must give a positive operator");
    wcb_scm_desc d{};
    d.dim = 2;
    d.p = e->p;
    d.n_e[0] = e->n_e[0];
    d.n_e[1] = e->n_e[1];
    d.n_e[2] = 1;
    d.k1 = e->k1;
    d.m1 = e->m1;
    d.sk = 1.0;
    d.cell_class = e->cell_class;
    d.n_dof = e->n_node;
    d.lex_of_compact = e->lex_of_compact;
    d.n_cut = e->n_cut;
    d.cut_cells = e->cut_cells;
    d.cut_K = e->cut_K;
    d.x_cell_lo = e->x_cell_lo;
    d.x_cell_hi = e->x_cell_hi;
    d.x_owns_last = e->x_owns_last;
    return build_scm_operator(ctx, &d, 2, e->lam, e->mu, e->g1);
}

static Operator* build_scm_operator(Context* ctx, const wcb_scm_desc* d, int ncomp, double lam,
                                    double mu, const double* g1) {
    WCB_REQUIRE(d->dim == 2 || d->dim == 3, "dim must be 2 or 3");
    const int dim = d->dim;
    const int p = d->p;
    if (dim == 2) WCB_REQUIRE(p >= 1 && p <= 6, "p must be in 1..6 for the 2D kernel");
    else WCB_REQUIRE(p >= 1 && p <= 4, "p must be in 1..4 for the 3D kernel");
    WCB_REQUIRE(ncomp == 1 || dim == 2, "elastic operator: 2D");
    for (int k = 1; k < dim; ++k)
        WCB_REQUIRE(d->n_e[k] == d->n_e[0], "cubic grids only (n_e equal on all axes)");
    WCB_REQUIRE(d->n_e[0] >= 1, "n_e must be >= 1");
    WCB_REQUIRE(d->k1 && d->m1 && d->cell_class && (d->n_dof == 0 || d->lex_of_compact),
                "NULL array in SCM descriptor");
    auto* op = new ScmOperator();
    std::unique_ptr<ScmOperator> guard(op);
    op->ctx = ctx;
    op->dim = dim;
    op->p = p;
    const int64_t n_e = d->n_e[0];
    const int64_t n1 = n_e * p + 1;
    op->n_e = n_e;
    op->n1 = n1;
    op->n = ncomp * d->n_dof;
    op->ncomp = ncomp;
    op->lam = lam;
    op->mu = mu;
    if (ncomp == 2) op->g1.assign(g1, g1 + (p + 1) * (p + 1));
    // slab
    const int64_t lo = d->x_cell_lo;
    const int64_t hi = d->x_cell_hi > 0 ? d->x_cell_hi : n_e;
    const bool last = d->x_cell_hi > 0 ? (d->x_owns_last != 0) : true;
    WCB_REQUIRE(lo >= 0 && lo < hi && hi <= n_e, "slab cell range must satisfy 0 <= lo < hi <= n_e");
    WCB_REQUIRE(!last || hi == n_e, "only the slab ending at n_e can own the last node row");
    op->has_top = lo > 0;
    op->owns_last = last;
    op->n_ex = hi - lo + 1;
    op->n1x = op->n_ex * p + 1;
    op->row_lo = p;
    op->row_hi = last ? op->n1x : op->n1x - 1;
    const int64_t TJ = 32 * (int64_t)p;
    const int64_t need_cols = PADJ + ceil_div(n1, TJ) * TJ + p + 2;
    op->pitch = ceil_div(need_cols, 32) * 32;
    const int64_t cells_row = dim == 2 ? n_e : n_e * n_e;    // cells per x cell row
    const int64_t nodes_row = dim == 2 ? n1 : n1 * n1;       // nodes per x node row
    if (dim == 2) {
        op->rows = op->n1x + 2 * p;
        op->xstride = op->pitch;
    } else {
        op->rows = n1 + 2 * p;                                // y rows of a plane
        op->pplane = op->rows * op->pitch;
        op->xstride = op->pplane;
    }
    const int64_t xrows = op->n1x + 2 * p;
    op->plane = xrows * op->xstride;
    op->n_state = ncomp * op->plane;
    op->halo_nplanes = ncomp;
    op->halo_pstride = op->plane;
    const int N = p + 1;
    op->m1.assign(d->m1, d->m1 + N * N);
    op->k1.assign(d->k1, d->k1 + N * N);
    op->sk = d->sk;
    // local cell classes: row 0 = global cell row lo-1 (zeros if lo == 0)
    const int64_t first_given = op->has_top ? lo - 1 : lo;        // first row present in desc
    std::vector<int8_t> cls(op->n_ex * cells_row, 0);
    for (int64_t gx = first_given; gx < hi; ++gx)
        for (int64_t c = 0; c < cells_row; ++c) {
            const int8_t v = d->cell_class[(gx - first_given) * cells_row + c];
            WCB_REQUIRE(v >= 0 && v <= 2, "cell_class values must be 0, 1 or 2");
            cls[(gx - lo + 1) * cells_row + c] = v;
        }
    // 3D probe for the interior 1/m table: a cell (local row >= 2) whose 8
    // cells sharing its owned corner block are all uncut
    if (dim == 3) {
        auto C = [&](int64_t x, int64_t y, int64_t z) { return cls[(x * n_e + y) * n_e + z]; };
        for (int64_t x = std::max<int64_t>(2, op->n_ex / 2); x < op->n_ex && op->probe_base < 0; ++x)
            for (int64_t y = std::max<int64_t>(1, n_e / 2); y < n_e && op->probe_base < 0; ++y)
                for (int64_t z = std::max<int64_t>(1, n_e / 2); z < n_e && op->probe_base < 0; ++z) {
                    bool ok = (x * p + p - 1) < op->row_hi;
                    for (int d = 0; d < 8 && ok; ++d) ok = C(x - (d >> 2), y - ((d >> 1) & 1), z - (d & 1)) == 1;
                    if (ok) op->probe_base = (x * p + p) * op->xstride + (y * p + p) * op->pitch + z * p + PADJ;
                }
    }
    if (dim == 2) {
        auto C = [&](int64_t x, int64_t y) { return cls[x * n_e + y]; };
        for (int64_t x = std::max<int64_t>(2, op->n_ex / 2); x < op->n_ex && op->probe_base < 0; ++x)
            for (int64_t y = std::max<int64_t>(1, n_e / 2); y < n_e && op->probe_base < 0; ++y) {
                bool ok = (x * p + p - 1) < op->row_hi;
                for (int d = 0; d < 4 && ok; ++d) ok = C(x - (d >> 1), y - (d & 1)) == 1;
                if (ok) op->probe_base = (x * p + p) * op->xstride + y * p + PADJ;
            }
    }
    // mask with a zero ring
    std::vector<uint8_t> mask;
    if (dim == 2) {
        const int64_t s_ = n_e + 2;
        mask.assign((op->n_ex + 2) * s_, 0);
        for (int64_t i = 0; i < op->n_ex; ++i)
            for (int64_t j = 0; j < n_e; ++j) mask[(i + 1) * s_ + (j + 1)] = (uint8_t)cls[i * n_e + j];
        op->mask_h = mask;
    } else {
        const int64_t s_ = n_e + 2;
        mask.assign((op->n_ex + 2) * s_ * s_, 0);
        for (int64_t i = 0; i < op->n_ex; ++i)
            for (int64_t j = 0; j < n_e; ++j)
                for (int64_t k = 0; k < n_e; ++k)
                    mask[((i + 1) * s_ + (j + 1)) * s_ + (k + 1)] = (uint8_t)cls[(i * n_e + j) * n_e + k];
    }
    // owned DOFs -> state index; tile flags
    const int RX = ncomp == 2 ? rpe_e(p) : dim == 2 ? rpe_for(p) : 1;
    const int64_t TI = (int64_t)RX * p;
    const int64_t n_tiles_x = ceil_div(op->row_hi - op->row_lo, TI);
    std::vector<uint8_t> cf;
    int64_t WY3 = 1;
    if (dim == 2) {
        op->n_strips = ceil_div(n1, TJ);
        op->n_rtiles = n_tiles_x;
        cf.assign(op->n_rtiles * op->n_strips, 0);
    } else {
        // streaming 3D grid: z strips of 32 cells (the node column z = n1-1 of
        // a grid with n_e % 32 == 0 goes to k_scm3d_zcol), y blocks of WY cell
        // rows, x chunks sized so the grid fills the resident CTA slots
        WY3 = p == 1 ? wy_for3(1) : p == 2 ? wy_for3(2) : p == 3 ? wy_for3(3) : wy_for3(4);
        op->n_zs = ceil_div(n_e, 32);
        op->n_yb = ceil_div(n_e + 1, WY3);   // cell rows 0..n_e (row n_e: the last node row)
        op->ex_last = (op->row_hi - 1) / p;
        const int64_t rows_out = op->ex_last;                  // cell rows 1..ex_last
        const int64_t slots = (int64_t)ctx->sm_count * (p == 1 ? cpsm_for3(1) : p == 2 ? cpsm_for3(2) : p == 3 ? cpsm_for3(3) : cpsm_for3(4));
        const int64_t per_chunk = op->n_zs * op->n_yb;
        // waves x (rows per chunk + its halo row), minimised over the chunk count
        int64_t nxc = 1;
        double best = 1e300;
        for (int64_t c = 1; c <= std::min<int64_t>(rows_out, 32); ++c) {
            const double cost = (double)ceil_div(per_chunk * c, slots) * (double)(ceil_div(rows_out, c) + 1);
            if (cost < best - 1e-9) { best = cost; nxc = c; }
        }
        if (const char* e = getenv("WAVECELL_B200_XCHUNKS")) nxc = std::max<int64_t>(1, std::min<int64_t>(atoll(e), rows_out));
        op->xc3 = ceil_div(rows_out, nxc);
        op->n_xc = ceil_div(rows_out, op->xc3);
        cf.assign(op->n_xc * op->n_yb * op->n_zs, 0);
    }
    op->sidx.resize(op->n);
    // elastic streaming step: x chunks of cell rows x strips, sized so the
    // grid fills the resident CTA slots (waves x (rows + halo row) minimal)
    std::vector<uint8_t> sf;
    if (ncomp == 2) {
        op->ex_last = (op->row_hi - 1) / p;
        const int64_t rows_out = op->ex_last;
        const int64_t slots = (int64_t)ctx->sm_count * std::max(1, ela2s_ctas_per_sm(p));
        const int64_t per_chunk = ceil_div(n1, TJ);
        int64_t nxc = 1;
        double best = 1e300;
        for (int64_t c = 1; c <= std::min<int64_t>(rows_out, 256); ++c) {
            const double cost = (double)ceil_div(per_chunk * c, slots) * (double)(ceil_div(rows_out, c) + 1);
            if (cost < best - 1e-9) { best = cost; nxc = c; }
        }
        op->xs_len = ceil_div(rows_out, nxc);
        op->n_xs = ceil_div(rows_out, op->xs_len);
        sf.assign(op->n_xs * per_chunk, 0);
    }
    const int64_t x0 = lo * p - p;   // global node row of local row 0
    for (int64_t i = 0; i < d->n_dof; ++i) {
        const int64_t lex = d->lex_of_compact[i];
        if (i) WCB_REQUIRE(d->lex_of_compact[i - 1] < lex, "lex_of_compact must be ascending");
        const int64_t I = lex / nodes_row, rest = lex % nodes_row;
        const int64_t Il = I - x0;
        WCB_REQUIRE(lex >= 0 && Il >= op->row_lo && Il < op->row_hi, "a DOF lies outside the slab");
        const int64_t t = (Il - op->row_lo) / TI;
        if (dim == 2) {
            op->sidx[i] = (Il + p) * op->xstride + rest + PADJ;
            cf[(rest / TJ) * op->n_rtiles + t] = 1;
            if (ncomp == 2) sf[((Il / p - 1) / op->xs_len) * op->n_strips + rest / TJ] = 1;
        } else {
            const int64_t J = rest / n1, K = rest % n1;
            op->sidx[i] = (Il + p) * op->xstride + (J + p) * op->pitch + K + PADJ;
            // owner: x cell row (Il-1)/p+1 ... plane Il belongs to cell row Il/p (local a = Il%p)
            const int64_t exo = Il / p, eyo = J / p, ezo = std::min<int64_t>(K / p, n_e - 1);
            const int64_t xcx = (exo - 1) / op->xc3;
            cf[(xcx * op->n_yb + eyo / WY3) * op->n_zs + ezo / 32] = 1;
        }
    }
    for (int64_t i = 0; i < (ncomp - 1) * d->n_dof; ++i) op->sidx[d->n_dof + i] = op->plane + op->sidx[i];
    // cut cells (global cell lex) within the local cell rows
    op->n_cut = d->n_cut;
    op->L = ncomp * (dim == 2 ? N * N : N * N * N);
    const int L = op->L;
    std::vector<int32_t> cid(op->n_ex * cells_row, -1);
    // 2D: full transposed matrices; 3D: packed lower triangles (k_cut_pre)
    const int64_t LP = dim == 3 ? (int64_t)cut_lp_stride(p) : (int64_t)L * (L + 1) / 2;   // packed stride
    std::vector<double> KT(dim == 2 ? (size_t)std::max<int64_t>(op->n_cut, 1) * L * L : 1, 0.0);
    std::vector<double> KP(dim == 3 ? (size_t)std::max<int64_t>(op->n_cut, 1) * LP : 1, 0.0);
    std::vector<int64_t> cbase(std::max<int64_t>(op->n_cut, 1), 0);
    for (int64_t e = 0; e < op->n_cut; ++e) {
        WCB_REQUIRE(d->cut_cells && d->cut_K, "cut arrays NULL");
        const int64_t c = d->cut_cells[e];
        if (e) WCB_REQUIRE(d->cut_cells[e - 1] < c, "cut_cells must be ascending");
        const int64_t cx = c / cells_row, crest = c % cells_row;
        const int64_t lx = cx - lo + 1;
        WCB_REQUIRE(c >= 0 && lx >= 0 && lx < op->n_ex && cls[lx * cells_row + crest] == 2,
                    "cut_cells must list cut cells of the slab");
        cid[lx * cells_row + crest] = (int32_t)e;
        const double* K = d->cut_K + e * L * L;
        // divided by sk: the kernels scale every output node by sk once
        // (tensor and cut parts alike)
        if (dim == 2) {
            double* T = KT.data() + e * L * L;   // transposed: lane r reads column r
            for (int r = 0; r < L; ++r)
                for (int m = 0; m < L; ++m) T[m * L + r] = K[r * L + m] / d->sk;
        } else {
            double* T = KP.data() + e * LP;      // row r, columns m <= r
            for (int r = 0; r < L; ++r)
                for (int m = 0; m <= r; ++m) T[(int64_t)r * (r + 1) / 2 + m] = K[r * L + m] / d->sk;
            const int64_t cy = crest / n_e, cz = crest % n_e;
            cbase[e] = (lx * p + p) * op->xstride + (cy * p + p) * op->pitch + cz * p + PADJ;
        }
    }
    for (size_t c = 0; c < cls.size(); ++c)
        WCB_REQUIRE(cls[c] != 2 || cid[c] >= 0, "a cut cell is missing from cut_cells");
    if (dim == 2) {
        // dispatch order of the tile kernel: live tiles by decreasing cost
        // (one unit per tile + CUT_COST per cut cell it integrates, the halo
        // row above included), ties in strip-major order
        constexpr double CUT_COST = 0.15;
        const int64_t TI_cells = RX;
        std::vector<std::pair<double, int32_t>> w;
        for (int64_t t = 0; t < (int64_t)cf.size(); ++t) {
            if (!cf[t]) continue;
            const int64_t strip = t / op->n_rtiles, rt = t % op->n_rtiles;
            const int64_t ex0 = (op->row_lo + rt * TI) / p - 1, ey0 = strip * (TJ / p) - 1;
            int n_c = 0;
            for (int64_t ex = std::max<int64_t>(ex0, 0); ex < std::min<int64_t>(ex0 + 1 + TI_cells, op->n_ex); ++ex)
                for (int64_t ey = std::max<int64_t>(ey0, 0); ey < std::min<int64_t>(ey0 + 1 + TJ / p, n_e); ++ey)
                    n_c += cid[ex * cells_row + ey] >= 0;
            w.emplace_back(-(1.0 + CUT_COST * n_c), (int32_t)t);
        }
        op->tile_cost.assign(cf.size(), 0.0);
        for (const auto& x : w) op->tile_cost[x.second] = -x.first;
        std::stable_sort(w.begin(), w.end(),
                         [](const auto& a, const auto& b) { return a.first < b.first; });
        std::vector<int32_t> ord(w.size());
        for (size_t i = 0; i < w.size(); ++i) ord[i] = w[i].second;
        op->n_order = (int64_t)ord.size();
        op->order.alloc(std::max<int64_t>(op->n_order, 1));
        op->order.upload(ord.data(), ord.size(), ctx->stream);
        op->order_h = ord;
    }
    cudaStream_t st = ctx->stream;
    op->d_sidx.alloc(std::max<int64_t>(op->n, 1));
    op->d_sidx.upload(op->sidx.data(), op->n, st);
    op->mask.alloc(mask.size());
    op->mask.upload(mask.data(), mask.size(), st);
    op->cflags.alloc(cf.size());
    op->cflags.upload(cf.data(), cf.size(), st);
    if (!sf.empty()) {
        op->sflags.alloc(sf.size());
        op->sflags.upload(sf.data(), sf.size(), st);
    }
    op->cut_id.alloc(cid.size());
    op->cut_id.upload(cid.data(), cid.size(), st);
    op->KT.alloc(KT.size());
    op->KT.upload(KT.data(), KT.size(), st);
    if (dim == 3) {
        op->KP.alloc(KP.size());
        op->KP.upload(KP.data(), KP.size(), st);
        op->cut_base.alloc(cbase.size());
        op->cut_base.upload(cbase.data(), cbase.size(), st);
        op->cut_out.alloc((size_t)std::max<int64_t>(op->n_cut, 1) * L);
        if (n_e % 32 == 0) op->zline.alloc((size_t)(op->n_ex * p + 1) * n1);
    }
    // algorithmic bytes per step: 32 B per DOF + packed cut K
    op->bytes_step = 32.0 * (double)op->n + 8.0 * (double)L * (L + 1) / 2.0 * (double)op->n_cut;
    WCB_CUDA(cudaStreamSynchronize(st));
    return guard.release();
}

}  // namespace wcb
