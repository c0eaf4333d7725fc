// 2D plane-strain elastic operator: fused CDM step / apply (BASELINE config 4).
//
// Two displacement components live in two planes of the state (plane 1 starts
// `plane` doubles after plane 0, same padded lex layout as the scalar 2D
// kernel).  A tile is TI = RPE*p node rows x 32p node columns; warps come in
// two groups, one per output component, each with RPE element-row warps and
// one halo warp (the cell row above the tile, output row p only -> carry).
//
// Per cell, output component o, with s = o and t = 1 - o (setup/elastic.py):
//   out_o = X_a1(Y_m1 u_s) + X_a2(Y_k1 u_s) + X_a3(Y_Cy u_t) + X_a4(Y_Dy u_t)
// where Y_A contracts the y (fast) index and X_A the x (slow) index, and
//   o = 0: a1 = (l+2m) k1, a2 = m m1, a3 = l G, a4 = m G^T, Cy = G^T, Dy = G
//   o = 1: a1 = m k1, a2 = (l+2m) m1, a3 = l G^T, a4 = m G, Cy = G, Dy = G^T
// with G[a][b] = int phi_a' phi_b.  Cut cells add their dense 2L x 2L matrix
// (stored transposed) exactly as the scalar kernel does, rows of the warp's
// component only.  Bitwise deterministic: fixed accumulation order, carry
// rows added as (row above) + (own).
#pragma once
// (included inside namespace wcb by wcb_scm.cu)

// p = 5: five cell rows per tile, one CTA of 12 warps per SM (227 KB of shared
// memory).  Since the IMEX part steps skip the dense cut-cell products the
// halo warps' redundant row is the dominant overhead: measured on config 4,
// IMEX step 1315 (RPE 2, two CTAs per SM) / 1238 (3) / 1206 (4) / 1135 us (5).
#ifndef WCB_ELA_RPE5
#define WCB_ELA_RPE5 5
#endif
#ifndef WCB_ELA_MINB
#define WCB_ELA_MINB 1
#endif
__host__ __device__ constexpr int rpe_e(int P) { return P <= 3 ? 3 : P == 5 ? WCB_ELA_RPE5 : 2; }

template <int P>
struct Tile2E {
    static constexpr int RPE = rpe_e(P);
    static constexpr int NWB = RPE + 1;            // warps per component group
    static constexpr int NWARP = 2 * NWB;
    static constexpr int TJ = 32 * P;
    static constexpr int TI = RPE * P;
    static constexpr int CO = P & 1;
    static constexpr int UW = ((TJ + P + 1 + CO) + 1) / 2 * 2;
    static constexpr int UH = TI + P + 1;
    static constexpr size_t U_BYTES = (size_t)UW * UH * 8;
    static constexpr size_t E_BYTES = (size_t)TJ * TI * 8;
    static constexpr size_t U_R = (U_BYTES + 127) / 128 * 128;
    static constexpr size_t E_R = (E_BYTES + 127) / 128 * 128;
    static constexpr size_t OFF_U1 = U_R;
    static constexpr size_t OFF_PREV = 2 * U_R;               // [comp]
    static constexpr size_t OFF_MINV = OFF_PREV + 2 * E_R;    // [comp]
    static constexpr size_t OFF_CARRY = OFF_MINV + 2 * E_R;   // [comp][RPE+1][P][32]
    static constexpr size_t OFF_BAR = OFF_CARRY + (size_t)2 * (RPE + 1) * P * 32 * 8;
    static constexpr size_t SMEM = OFF_BAR + 16;   // [0] u tiles, [1] epilogue tiles
};

// 1D factors: y pass uses m1, k1, G; x pass uses per-component scaled
// matrices xa[o][term][r * N + c]
template <int P>
struct EMats {
    double ym[(P + 1) * (P + 1)];
    double yk[(P + 1) * (P + 1)];
    double yg[(P + 1) * (P + 1)];
    double xa[2][4][(P + 1) * (P + 1)];
};

// y-pass matrix element A[j][l] for the four y contractions of component O:
// term 0 = m1, 1 = k1, 2 = Cy, 3 = Dy
template <int P, int O, int TERM>
__device__ __forceinline__ double ycoef(const EMats<P>& mt, int j, int l) {
    constexpr int N = P + 1;
    if constexpr (TERM == 0) return mt.ym[j * N + l];
    else if constexpr (TERM == 1) return mt.yk[j * N + l];
    else if constexpr ((TERM == 2) == (O == 0)) return mt.yg[l * N + j];   // G^T
    else return mt.yg[j * N + l];                                          // G
}

template <int P, int O, int TERM>
__device__ __forceinline__ void ypass_one(const EMats<P>& mt, const double (&own)[P], double right,
                                          const double (&left)[P], double own0, double chiR,
                                          double chiL, double (&W)[P]) {
    #pragma unroll
    for (int j = 0; j < P; ++j) {
        double s = ycoef<P, O, TERM>(mt, j, P) * right;
        #pragma unroll
        for (int l = 0; l < P; ++l) s = fma(ycoef<P, O, TERM>(mt, j, l), own[l], s);
        W[j] = chiR * s;
    }
    // left cell: its local column P is our column 0
    double s = ycoef<P, O, TERM>(mt, P, P) * own0;
    #pragma unroll
    for (int l = 0; l < P; ++l) s = fma(ycoef<P, O, TERM>(mt, P, l), left[l], s);
    W[0] = fma(chiL, s, W[0]);
}

// One node row (input row c of the element) of both component tiles.
template <int P, int O, int UW, int CO, bool NBS = false>
__device__ __forceinline__ void row_contract_e(const EMats<P>& mt, const double* row_s,
                                               const double* row_t, int lane, double chiR,
                                               double chiL, int c, double (&Y)[P + 1][P]) {
    constexpr int N = P + 1;
    double own_s[P], own_t[P], left_s[P], left_t[P];
    lds_row<P>(row_s + CO + P + lane * P, own_s);
    lds_row<P>(row_t + CO + P + lane * P, own_t);
    double right_s, right_t;
    if constexpr (NBS) {   // neighbours straight from shared memory (streaming kernel)
        right_s = row_s[CO + P + lane * P + P];
        right_t = row_t[CO + P + lane * P + P];
        #pragma unroll
        for (int l = 0; l < P; ++l) {
            left_s[l] = row_s[CO + lane * P + l];
            left_t[l] = row_t[CO + lane * P + l];
        }
    } else {               // by shuffles (tile kernel: fewer live registers)
        right_s = __shfl_down_sync(0xffffffffu, own_s[0], 1);
        right_t = __shfl_down_sync(0xffffffffu, own_t[0], 1);
        if (lane == 31) {
            right_s = row_s[CO + P + 32 * P];
            right_t = row_t[CO + P + 32 * P];
        }
        #pragma unroll
        for (int l = 0; l < P; ++l) {
            double a = __shfl_up_sync(0xffffffffu, own_s[l], 1);
            double b = __shfl_up_sync(0xffffffffu, own_t[l], 1);
            if (lane == 0) {
                a = row_s[CO + l];
                b = row_t[CO + l];
            }
            left_s[l] = a;
            left_t[l] = b;
        }
    }
    double W[P];
    ypass_one<P, O, 0>(mt, own_s, right_s, left_s, own_s[0], chiR, chiL, W);
    #pragma unroll
    for (int r = 0; r < N; ++r)
        #pragma unroll
        for (int j = 0; j < P; ++j) Y[r][j] = fma(mt.xa[O][0][r * N + c], W[j], Y[r][j]);
    ypass_one<P, O, 1>(mt, own_s, right_s, left_s, own_s[0], chiR, chiL, W);
    #pragma unroll
    for (int r = 0; r < N; ++r)
        #pragma unroll
        for (int j = 0; j < P; ++j) Y[r][j] = fma(mt.xa[O][1][r * N + c], W[j], Y[r][j]);
    ypass_one<P, O, 2>(mt, own_t, right_t, left_t, own_t[0], chiR, chiL, W);
    #pragma unroll
    for (int r = 0; r < N; ++r)
        #pragma unroll
        for (int j = 0; j < P; ++j) Y[r][j] = fma(mt.xa[O][2][r * N + c], W[j], Y[r][j]);
    ypass_one<P, O, 3>(mt, own_t, right_t, left_t, own_t[0], chiR, chiL, W);
    #pragma unroll
    for (int r = 0; r < N; ++r)
        #pragma unroll
        for (int j = 0; j < P; ++j) Y[r][j] = fma(mt.xa[O][3][r * N + c], W[j], Y[r][j]);
}

// Cut cells of one element row for output component O (rows O*LN .. O*LN+LN-1
// of the cell's 2LN x 2LN matrix), cooperatively by the warp.
template <int P, int O, int UW, int CO>
__device__ __forceinline__ void cut_cells_warp_e(const Scm2DGeo& g, const double* rows0,
                                                 const double* rows1, int lane, unsigned cut_lanes,
                                                 bool edge, int32_t cid, int32_t cidL,
                                                 double (&Y)[P + 1][P],
                                                 const double* rowP0 = nullptr, const double* rowP1 = nullptr) {
    if (!rowP0) {
        rowP0 = rows0 + P * UW;
        rowP1 = rows1 + P * UW;
    }
    constexpr int N = P + 1;
    constexpr int LN = N * N;
    constexpr int L = 2 * LN;
    constexpr int RR = (LN + 31) / 32;
    int src = edge ? -1 : (__ffs(cut_lanes) - 1);
    if (!edge) cut_lanes &= cut_lanes - 1;
    while (src >= -1) {
        const int32_t id = src >= 0 ? __shfl_sync(0xffffffffu, cid, src) : __shfl_sync(0xffffffffu, cidL, 0);
        const double* KT = g.KT + (int64_t)id * L * L;
        const double* c0 = rows0 + CO + P + src * P;
        const double* c1 = rows1 + CO + P + src * P;
        const double* c0P = rowP0 + CO + P + src * P - P * UW;   // row P at c0P[P * UW + b]
        const double* c1P = rowP1 + CO + P + src * P - P * UW;
        double t[RR];
        #pragma unroll
        for (int q = 0; q < RR; ++q) {
            t[q] = 0.0;
            const int r = lane + 32 * q;
            if (r < LN) {
                const double* kt = KT + O * LN + r;
                // bounded unroll: at most N loads in flight per lane (registers)
                #pragma unroll 1
                for (int a0 = 0; a0 < N; ++a0) {
                    const double* ra = a0 < P ? c0 : c0P;
                    #pragma unroll
                    for (int b0 = 0; b0 < N; ++b0)
                        t[q] = fma(__ldg(kt + (int64_t)(a0 * N + b0) * L), ra[a0 * UW + b0], t[q]);
                }
                #pragma unroll 1
                for (int a0 = 0; a0 < N; ++a0) {
                    const double* ra = a0 < P ? c1 : c1P;
                    #pragma unroll
                    for (int b0 = 0; b0 < N; ++b0)
                        t[q] = fma(__ldg(kt + (int64_t)(LN + a0 * N + b0) * L), ra[a0 * UW + b0], t[q]);
                }
            }
        }
        #pragma unroll
        for (int r = 0; r < LN; ++r) {
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

template <int P>
struct MinvTabE {
    double v[P * P];
};

template <int P, int MODE, int O>
__device__ __forceinline__ void ela2d_warp(const Scm2DGeo& g, const EMats<P>& mt, const StepArgs& a,
                                           int64_t plane, unsigned char* smem, int wi, int lane,
                                           int64_t J0, int64_t I0, unsigned long long& amp, bool tcl,
                                           const MinvTabE<P>& mtab) {
    using T = Tile2E<P>;
    constexpr int N = P + 1;
    constexpr int RPE = T::RPE;
    const bool halo = (wi == RPE);
    const int64_t ex = halo ? I0 / P - 1 : I0 / P + wi;
    const int64_t ey = J0 / P + lane;
    uint8_t mR = 0, mL = 0;
    if (ex >= 0 && ex < g.n_ex && ey <= g.n_ey) {
        const int64_t ms_ = g.n_ey + 2;
        mR = __ldg(g.mask + (ex + 1) * ms_ + (ey + 1));
        mL = __ldg(g.mask + (ex + 1) * ms_ + ey);
    }
    const int32_t cid = mR == 2 ? __ldg(g.cut_id + ex * g.n_ey + ey) : -1;
    const int32_t cidL = (lane == 0 && mL == 2) ? __ldg(g.cut_id + ex * g.n_ey + ey - 1) : -1;
    const double* u0 = reinterpret_cast<const double*>(smem);
    const double* u1 = reinterpret_cast<const double*>(smem + T::OFF_U1);
    const double* us = O == 0 ? u0 : u1;
    const double* ut = O == 0 ? u1 : u0;
    double* carry = reinterpret_cast<double*>(smem + T::OFF_CARRY) + (size_t)O * (RPE + 1) * P * 32;
    const int rbase = halo ? -P : wi * P;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
    mbar_wait(bar, 0);
    double Y[N][P];
    #pragma unroll
    for (int r = 0; r < N; ++r)
        #pragma unroll
        for (int j = 0; j < P; ++j) Y[r][j] = 0.0;
    if (__any_sync(0xffffffffu, (mR | mL) != 0)) {
        const double chiR = mR == 1 ? 1.0 : 0.0;
        const double chiL = mL == 1 ? 1.0 : 0.0;
        const size_t r0 = (size_t)(rbase + P) * T::UW;
        #pragma unroll 1
        for (int c = 0; c < N; ++c)
            row_contract_e<P, O, T::UW, T::CO>(mt, us + r0 + (size_t)c * T::UW, ut + r0 + (size_t)c * T::UW,
                                               lane, chiR, chiL, c, Y);
        const unsigned cl = __ballot_sync(0xffffffffu, mR == 2);
        const bool ed = __shfl_sync(0xffffffffu, mL == 2, 0);
        if ((cl || ed) && g.KT) cut_cells_warp_e<P, O, T::UW, T::CO>(g, u0 + r0, u1 + r0, lane, cl, ed, cid, cidL, Y);
    }
    #pragma unroll
    for (int j = 0; j < P; ++j) carry[((halo ? 0 : wi + 1) * P + j) * 32 + lane] = Y[P][j];
    __syncthreads();
    if (halo) return;
    #pragma unroll
    for (int j = 0; j < P; ++j) Y[0][j] = carry[(wi * P + j) * 32 + lane] + Y[0][j];
    const double f = (MODE == MODE_STEP) ? __ldg(a.ft + a.k) : 0.0;
    const bool edge = (J0 + T::TJ > g.n1y);
    const int64_t Jl = J0 + lane * P;
    #pragma unroll
    for (int r = 0; r < P; ++r) {
        const int64_t I = ex * P + r;
        if (I >= g.row_hi) break;
        const int64_t base = O * plane + (I + P) * g.pitch + Jl + PADJ;
        if constexpr (MODE == MODE_APPLY) {
            #pragma unroll
            for (int j = 0; j < P; ++j)
                if (!edge || Jl + j < g.n1y) a.out[base + j] = Y[r][j];
        } else {
            if (r == 0) mbar_wait(bar + 1, 0);
            const double* urow = us + (size_t)(rbase + r + P) * T::UW + T::CO + P + lane * P;
            const double* ps = reinterpret_cast<const double*>(smem + T::OFF_PREV + O * T::E_R) +
                               (size_t)(wi * P + r) * T::TJ + lane * P;
            const double* msm = reinterpret_cast<const double*>(smem + T::OFF_MINV + O * T::E_R) +
                                (size_t)(wi * P + r) * T::TJ + lane * P;
            double up[P], mi[P], uu[P];
            lds_row<P>(ps, up);
            if (tcl) {
                #pragma unroll
                for (int j = 0; j < P; ++j) mi[j] = mtab.v[r * P + j];
            } else {
                lds_row<P>(msm, mi);
            }
            lds_row<P>(urow, uu);
            const bool src = base + P - 1 >= a.F.lo && base <= a.F.hi;
            #pragma unroll
            for (int j = 0; j < P; ++j) {
                if (!edge || Jl + j < g.n1y) {
                    const double fF = src ? f * source_at(a.F, base + j) : f * 0.0;
                    const double v = leapfrog(uu[j], up[j], Y[r][j], mi[j], fF, a.dt2);
                    a.out[base + j] = v;
                    const unsigned long long b = mi[j] != 0.0 ? amp_bits(v) : 0ULL;
                    amp = b > amp ? b : amp;
                }
            }
        }
    }
}

// One CTA per tile (order[] = live tiles, most expensive first).  The state
// tensor maps cover both component planes: plane 1 is `rows` TMA rows below.
template <int P, int MODE>
__global__ void __launch_bounds__(Tile2E<P>::NWARP * 32, WCB_ELA_MINB) k_ela2d(
    const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_prev,
    const __grid_constant__ CUtensorMap tm_minv, Scm2DGeo g, const __grid_constant__ EMats<P> mt,
    int64_t plane, int32_t rows, const __grid_constant__ MinvTabE<P> mtab, StepArgs a) {
    using T = Tile2E<P>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int32_t tid = __ldg(g.order + blockIdx.x);
    const int64_t strip = tid / g.n_rtiles, rtile = tid % g.n_rtiles;
    if (MODE == MODE_STEP && blockIdx.x == 0) record_observers(a);
    const int64_t J0 = strip * T::TJ, I0 = g.row_lo + rtile * T::TI;
    const bool tcl = MODE == MODE_STEP && g.tclean && __ldg(g.tclean + tid) != 0;
    // the contraction waits for the u tiles only ([0]); psi_{k-1} / 1/m ([1])
    // keep streaming until the epilogue
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        const bool epi = MODE == MODE_STEP;
        mbar_expect_tx(bar, (uint32_t)(2 * T::U_BYTES));
        const int32_t xu = (int32_t)(J0 - P - T::CO + PADJ), xe = (int32_t)(J0 + PADJ);
        tma_load_2d(smem, &tm_u, xu, (int32_t)I0, bar);
        tma_load_2d(smem + T::OFF_U1, &tm_u, xu, (int32_t)I0 + rows, bar);
        if (epi) {
            mbar_expect_tx(bar + 1, (uint32_t)((tcl ? 2 : 4) * T::E_BYTES));
            for (int o = 0; o < 2; ++o) {
                tma_load_2d(smem + T::OFF_PREV + o * T::E_R, &tm_prev, xe, (int32_t)(I0 + P) + o * rows, bar + 1);
                if (!tcl)
                    tma_load_2d(smem + T::OFF_MINV + o * T::E_R, &tm_minv, xe, (int32_t)(I0 + P) + o * rows,
                                bar + 1);
            }
        }
    }
    __syncthreads();
    unsigned long long amp = 0ULL;
    if (w < T::NWB) ela2d_warp<P, MODE, 0>(g, mt, a, plane, smem, w, lane, J0, I0, amp, tcl, mtab);
    else ela2d_warp<P, MODE, 1>(g, mt, a, plane, smem, w - T::NWB, lane, J0, I0, amp, tcl, mtab);
    if constexpr (MODE == MODE_STEP) warp_amp_max(amp, a.amp);
}


// ---------------------------------------------------------------------------
// Streaming variant of the fused step (MODE_STEP): one CTA = one y strip of 32
// cells x one chunk of x cell rows, two warps (output component 0 / 1).  Node
// rows stream through a two-slot TMA ring (slot = the P node rows ex*P ..
// ex*P+P-1 of both components; row P of cell row ex is row 0 of the next
// slot); the x pass accumulates in registers and plane P of a cell row is
// carried in registers into the next one, so the only redundant work is one
// cell row per chunk (vs one halo row per tile in k_ela2d).  psi_{k-1} of the
// owned rows arrives by TMA during the row; 1/m comes from the interior table
// on clean cells.
#ifndef WCB_ELA2S_MINB
#define WCB_ELA2S_MINB 4
#endif
template <int P>
struct Str2E {
    static constexpr int TJ = 32 * P;
    static constexpr int CO = P & 1;
    static constexpr int UW = ((TJ + P + 1 + CO) + 1) / 2 * 2;
    // TMA destinations are 128-byte aligned
    static constexpr size_t COMP = ((size_t)UW * P * 8 + 127) / 128 * 128;   // one component of a slot
    static constexpr size_t SLOT = 2 * COMP;
    static constexpr size_t PCOMP = ((size_t)TJ * P * 8 + 127) / 128 * 128;  // psi_{k-1}, one component
    static constexpr size_t OFF_PREV = 2 * SLOT;
    static constexpr size_t OFF_BAR = OFF_PREV + 2 * PCOMP;
    static constexpr size_t SMEM = OFF_BAR + 8 * 3;
};

template <int P>
__global__ void __launch_bounds__(64, WCB_ELA2S_MINB) k_ela2s(const __grid_constant__ CUtensorMap tm_u,
                                             const __grid_constant__ CUtensorMap tm_prev, Scm2DGeo g,
                                             const __grid_constant__ EMats<P> mt, int64_t plane, int32_t rows,
                                             int64_t xc_len, int64_t ex_last, const uint8_t* __restrict__ clean,
                                             const __grid_constant__ MinvTabE<P> mtab, StepArgs a) {
    using T = Str2E<P>;
    constexpr int N = P + 1;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);   // [2] ring, [2] = prev
    const int lane = threadIdx.x & 31;
    const int O = threadIdx.x >> 5;
    const int64_t strip = blockIdx.x, xc = blockIdx.y;
    if (blockIdx.x == 0 && blockIdx.y == 0) record_observers(a);
    if (!g.cflags[xc * g.n_strips + strip]) return;
    const int64_t J0 = strip * T::TJ;
    const int64_t exA = 1 + xc * xc_len;
    const int64_t exE = exA + xc_len < ex_last + 1 ? exA + xc_len : ex_last + 1;
    const int32_t xu = (int32_t)(J0 - P - T::CO + PADJ);
    auto issue = [&](int64_t ex) {   // node rows ex*P .. ex*P+P-1 of both components
        const int s = (int)(ex & 1);
        unsigned char* dst = smem + s * T::SLOT;
        mbar_expect_tx(&full[s], (uint32_t)(2 * T::UW * P * 8));
        tma_load_2d(dst, &tm_u, xu, (int32_t)(ex * P + P), &full[s]);
        tma_load_2d(dst + T::COMP, &tm_u, xu, (int32_t)(ex * P + P) + rows, &full[s]);
    };
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_init(&full[2], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        issue(exA - 1);
        issue(exA);
    }
    const int64_t ey = J0 / P + lane;
    const int64_t Jl = J0 + lane * P;
    const bool edge = (J0 + T::TJ > g.n1y);
    const double f = __ldg(a.ft + a.k);
    const int64_t ms_ = g.n_ey + 2;
    double Y[N][P];
    #pragma unroll
    for (int r = 0; r < N; ++r)
        #pragma unroll
        for (int j = 0; j < P; ++j) Y[r][j] = 0.0;
    unsigned long long amp = 0ULL;
    for (int64_t ex = exA - 1; ex < exE; ++ex) {
        const bool epi = ex >= exA;
        if (epi && threadIdx.x == 0) {   // psi_{k-1} of this row's owned nodes (buffer free: last epilogue done)
            mbar_expect_tx(&full[2], (uint32_t)(2 * T::TJ * P * 8));
            const int32_t xe = (int32_t)(J0 + PADJ), ye = (int32_t)(ex * P + P);
            tma_load_2d(smem + T::OFF_PREV, &tm_prev, xe, ye, &full[2]);
            tma_load_2d(smem + T::OFF_PREV + T::PCOMP, &tm_prev, xe, ye + rows, &full[2]);
        }
        uint8_t mR = 0, mL = 0;
        if (ex >= 0 && ex < g.n_ex && ey <= g.n_ey) {
            mR = __ldg(g.mask + (ex + 1) * ms_ + (ey + 1));
            mL = __ldg(g.mask + (ex + 1) * ms_ + ey);
        }
        const int32_t cid = mR == 2 ? __ldg(g.cut_id + ex * g.n_ey + ey) : -1;
        const int32_t cidL = (lane == 0 && mL == 2) ? __ldg(g.cut_id + ex * g.n_ey + ey - 1) : -1;
        const bool cln = clean && mR == 1 && ey < g.n_ey && __ldg(clean + ex * g.n_ey + ey) != 0;
        const unsigned char* sA = smem + (ex & 1) * T::SLOT;        // rows ex*P + 0..P-1
        const unsigned char* sB = smem + ((ex + 1) & 1) * T::SLOT;  // row (ex+1)*P
        const double* a0 = reinterpret_cast<const double*>(sA);
        const double* a1 = reinterpret_cast<const double*>(sA + T::COMP);
        const double* b0 = reinterpret_cast<const double*>(sB);
        const double* b1 = reinterpret_cast<const double*>(sB + T::COMP);
        const double* us = O == 0 ? a0 : a1;
        const double* ut = O == 0 ? a1 : a0;
        const double* usP = O == 0 ? b0 : b1;
        const double* utP = O == 0 ? b1 : b0;
        const uint32_t par = (uint32_t)(((ex - (exA - 1)) >> 1) & 1);   // uses of this slot so far
        mbar_wait(&full[ex & 1], par);
        const bool any = __any_sync(0xffffffffu, (mR | mL) != 0);
        const double chiR = mR == 1 ? 1.0 : 0.0;
        const double chiL = mL == 1 ? 1.0 : 0.0;
        if (any) {
            #pragma unroll 1
            for (int c = 0; c < P; ++c) {
                if (O == 0)
                    row_contract_e<P, 0, T::UW, T::CO, true>(mt, us + (size_t)c * T::UW, ut + (size_t)c * T::UW, lane,
                                                       chiR, chiL, c, Y);
                else
                    row_contract_e<P, 1, T::UW, T::CO, true>(mt, us + (size_t)c * T::UW, ut + (size_t)c * T::UW, lane,
                                                       chiR, chiL, c, Y);
            }
        }
        mbar_wait(&full[(ex + 1) & 1], (uint32_t)(((ex + 1 - (exA - 1)) >> 1) & 1));
        if (any) {
            if (O == 0) row_contract_e<P, 0, T::UW, T::CO, true>(mt, usP, utP, lane, chiR, chiL, P, Y);
            else row_contract_e<P, 1, T::UW, T::CO, true>(mt, usP, utP, lane, chiR, chiL, P, Y);
            const unsigned cl = __ballot_sync(0xffffffffu, mR == 2);
            const bool ed = __shfl_sync(0xffffffffu, mL == 2, 0);
            if (cl || ed) {
                if (O == 0) cut_cells_warp_e<P, 0, T::UW, T::CO>(g, a0, a1, lane, cl, ed, cid, cidL, Y, b0, b1);
                else cut_cells_warp_e<P, 1, T::UW, T::CO>(g, a0, a1, lane, cl, ed, cid, cidL, Y, b0, b1);
            }
        }
        if (epi) {
            mbar_wait(&full[2], (uint32_t)((ex - exA) & 1));
            const double* ps = reinterpret_cast<const double*>(smem + T::OFF_PREV + O * T::PCOMP);
            #pragma unroll
            for (int r = 0; r < P; ++r) {
                const int64_t I = ex * P + r;
                if (I >= g.row_hi) break;
                const int64_t base = O * plane + (I + P) * g.pitch + Jl + PADJ;
                double up[P], uu[P];
                lds_row<P>(ps + (size_t)r * T::TJ + lane * P, up);
                lds_row<P>(us + (size_t)r * T::UW + T::CO + P + lane * P, uu);
                const bool src = base + P - 1 >= a.F.lo && base <= a.F.hi;
                #pragma unroll
                for (int j = 0; j < P; ++j) {
                    if (!edge || Jl + j < g.n1y) {
                        const double mi = cln ? mtab.v[r * P + j] : __ldg(a.minv + base + j);
                        const double fF = src ? f * source_at(a.F, base + j) : f * 0.0;
                        const double v = leapfrog(uu[j], up[j], Y[r][j], mi, fF, a.dt2);
                        a.out[base + j] = v;
                        const unsigned long long bb = mi != 0.0 ? amp_bits(v) : 0ULL;
                        amp = bb > amp ? bb : amp;
                    }
                }
            }
        }
        #pragma unroll
        for (int j = 0; j < P; ++j) {
            Y[0][j] = Y[P][j];
            #pragma unroll
            for (int r = 1; r < N; ++r) Y[r][j] = 0.0;
        }
        __syncthreads();   // both warps done with slot ex and the prev buffer
        if (threadIdx.x == 0 && ex + 2 <= exE) issue(ex + 2);
    }
    block_amp_max<64>(amp, a.amp);
}
