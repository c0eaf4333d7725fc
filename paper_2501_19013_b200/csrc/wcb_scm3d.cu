// 3D matrix-free spectral-cell stiffness fused with the CDM update.
//
// Reference operator: K = sum over kept cells of element matrices; uncut cells
// share sk (k1 (x) m1 (x) m1 + m1 (x) k1 (x) m1 + m1 (x) m1 (x) k1)
// (src/assembly.py:285-288, local order z fastest, src/assembly.py:426-429),
// cut cells carry dense K_o (src/assembly.py:582).
//
// Factorisation used here, per element row in x (fixed ex) and x-plane c:
//   Au = (m1_y (x) m1_z) u_c,   Bu = (k1_y (x) m1_z + m1_y (x) k1_z) u_c
//   Y[a] += k1_x[a][c] Au + m1_x[a][c] Bu          (x pass, registers)
// computed for the P x P (y, z) nodes each thread owns.  A CTA is one z strip
// (32 cells, lane = z cell) x one y cell row x RX x cell rows (one warp each)
// plus a halo warp recomputing the x cell row above.  Contributions from the
// z-left cell come by shuffles (as in 2D); the y-up cell's contribution to
// the thread's first y row is computed from the same smem tile (rows above).
// The x-shared node plane gets carry (x row above) + own in a fixed order.
#include "wcb_scm.cuh"

namespace wcb {

// z pass of one y row of the tile: m/k contractions for the right cell
// (outputs j = 0..P-1) and the left cell's column P (feeds j = 0).
template <int P>
__device__ __forceinline__ void zpass_row(const double (&mc)[orb_count(P)],
                                          const double (&kc)[orb_count(P)], const double* row,
                                          int lane, double (&zmR)[P], double (&zkR)[P],
                                          double& zmL, double& zkL) {
    row += Tile3<P>::CO;
    const double* own_p = row + P + lane * P;
    double own[P];
    #pragma unroll
    for (int j = 0; j < P; ++j) own[j] = own_p[j];
    double right = __shfl_down_sync(0xffffffffu, own[0], 1);
    if (lane == 31) right = own_p[P];
    #pragma unroll
    for (int j = 0; j < P; ++j) {
        double s1 = mc[orb(P, j, P)] * right, s2 = kc[orb(P, j, P)] * right;
        #pragma unroll
        for (int d = 0; d < P; ++d) {
            s1 = fma(mc[orb(P, j, d)], own[d], s1);
            s2 = fma(kc[orb(P, j, d)], own[d], s2);
        }
        zmR[j] = s1;
        zkR[j] = s2;
    }
    double l1 = mc[orb(P, P, P)] * own[0], l2 = kc[orb(P, P, P)] * own[0];
    #pragma unroll
    for (int d = 0; d < P; ++d) {
        double ud = __shfl_up_sync(0xffffffffu, own[d], 1);
        if (lane == 0) ud = row[d];
        l1 = fma(mc[orb(P, P, d)], ud, l1);
        l2 = fma(kc[orb(P, P, d)], ud, l2);
    }
    zmL = l1;
    zkL = l2;
}

// Cut cells of one x cell row: the products K_o u_e / sk were computed by
// k_cut_pre; the lanes owning the outputs add them in ascending cell order.
// `up` selects the y-up cell row (only its y-local row P is routed, to our y
// row 0); z routing as in 2D: z-local j < P -> the cell's lane, j = P -> the
// next lane.
template <int P>
__device__ __forceinline__ void cut_cells_warp3(const Scm3DGeo& g, int64_t ex, int64_t eyc,
                                                int64_t ez0, int lane, unsigned cut_lanes,
                                                bool edge, bool up, double (&Y)[P + 1][P][P]) {
    constexpr int N = P + 1;
    constexpr int L = N * N * N;
    int src = edge ? -1 : (__ffs(cut_lanes) - 1);
    if (!edge) cut_lanes &= cut_lanes - 1;
    while (true) {
        const int64_t ecol = ez0 + src;
        const bool mine = lane == src || lane == src + 1;
        if (mine) {
            const int32_t id = __ldg(g.cut_id + (ex * g.n_e + eyc) * g.n_e + ecol);   // ex local
            const double* o = g.cut_out + (int64_t)id * L;
            #pragma unroll
            for (int r = 0; r < L; ++r) {
                const int a = r / (N * N), b = (r / N) % N, j = r % N;
                const bool yok = up ? (b == P) : (b < P);
                if (yok) {
                    const int bb = up ? 0 : (b % P);
                    if (j < P) {
                        if (lane == src) Y[a][bb][j % P] += __ldcg(o + r);
                    } else {
                        if (lane == src + 1) Y[a][bb][0] += __ldcg(o + r);
                    }
                }
            }
        }
        if (!cut_lanes) break;
        src = __ffs(cut_lanes) - 1;
        cut_lanes &= cut_lanes - 1;
    }
}

// One warp per cut cell: gather u_e (64 nodes for p = 3) from the state, stage
// the packed lower triangle of K_o / sk in shared memory (one coalesced read
// of L(L+1)/2 doubles -- half the full matrix), lane r forms row r in
// ascending column order.
template <int P>
__host__ __device__ constexpr int cut_pre_warps() {
    return (int)(200 * 1024 / (((P + 1) * (P + 1) * (P + 1)) * (((P + 1) * (P + 1) * (P + 1)) + 3) / 2 * 8)) > 4
               ? 4
               : (int)(200 * 1024 / (((P + 1) * (P + 1) * (P + 1)) * (((P + 1) * (P + 1) * (P + 1)) + 3) / 2 * 8));
}

template <int P>
__global__ void __launch_bounds__(128) k_cut_pre(int64_t n_cut, const double* __restrict__ KP,
                                                 const int64_t* __restrict__ cut_base, int64_t pplane,
                                                 int64_t prow, const double* __restrict__ u,
                                                 double* __restrict__ out) {
    constexpr int N = P + 1;
    constexpr int L = N * N * N;
    constexpr int LP = L * (L + 1) / 2;
    extern __shared__ double smc[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* kp = smc + (size_t)w * (LP + L);
    double* uu = kp + LP;
    const int64_t e = (int64_t)blockIdx.x * cut_pre_warps<P>() + w;
    if (e >= n_cut) return;
    const double* src = KP + e * LP;
    for (int i = lane; i < LP; i += 32) kp[i] = __ldg(src + i);
    const int64_t base = cut_base[e];
    for (int m = lane; m < L; m += 32) {
        const int a = m / (N * N), b = (m / N) % N, j = m % N;
        uu[m] = u[base + a * pplane + b * prow + j];
    }
    __syncwarp();
    for (int r = lane; r < L; r += 32) {
        double t = 0.0;
        #pragma unroll 8
        for (int m = 0; m < L; ++m) {
            const int hi = r >= m ? r : m, lo = r >= m ? m : r;
            t = fma(kp[hi * (hi + 1) / 2 + lo], uu[m], t);
        }
        out[e * L + r] = t;
    }
}

template <int P>
void launch_cut_pre(Context* ctx, int64_t n_cut, const double* KP, const int64_t* cut_base,
                    int64_t pplane, int64_t prow, const double* u, double* out) {
    if (!n_cut) return;
    constexpr int L = (P + 1) * (P + 1) * (P + 1);
    constexpr int W = cut_pre_warps<P>();
    const size_t smem = (size_t)W * (L * (L + 1) / 2 + L) * 8;
    static bool attr_set = false;
    if (!attr_set) {
        WCB_CUDA(cudaFuncSetAttribute(k_cut_pre<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set = true;
    }
    k_cut_pre<P><<<(unsigned)ceil_div(n_cut, W), 32 * W, smem, ctx->stream>>>(n_cut, KP, cut_base, pplane, prow,
                                                                         u, out);
    ctx->launches++;
}

template <int P, int MODE>
__global__ void __launch_bounds__(Tile3<P>::NWARP * 32) k_scm3d(const __grid_constant__ CUtensorMap tm_u,
                                                               Scm3DGeo g, Mats2<P> mt, double sk,
                                                               StepArgs a) {
    using T = Tile3<P>;
    constexpr int N = P + 1;
    constexpr int RX = T::RX;
    extern __shared__ __align__(128) unsigned char smem[];
    const double* us = reinterpret_cast<const double*>(smem);
    double* carry = reinterpret_cast<double*>(smem + T::OFF_CARRY);   // [RX+1][P*P][32]
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int64_t zs = blockIdx.x, ey = blockIdx.y, xt = blockIdx.z;
    if (MODE == MODE_STEP && zs == 0 && ey == 0 && xt == 0) record_observers(a);
    if (!g.cflags[(xt * (g.n_e + 1) + ey) * g.n_zs + zs]) return;
    const int64_t K0 = zs * T::TZ;
    const int64_t ex0 = g.row_lo / P + xt * RX;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_expect_tx(bar, (uint32_t)T::U_BYTES);
        tma_load_3d(smem, &tm_u, (int32_t)(K0 - P - T::CO + PADJ), (int32_t)(ey * P),
                    (int32_t)(ex0 * P), bar);
    }
    const bool halo = (w == RX);
    const int64_t ex = halo ? ex0 - 1 : ex0 + w;
    const int64_t ez = K0 / P + lane;
    // cell codes of the 4 (y, z) neighbours in this x cell row
    uint8_t cRR = 0, cRL = 0, cUR = 0, cUL = 0;   // (ey, ez), (ey, ez-1), (ey-1, ez), (ey-1, ez-1)
    if (ex >= 0 && ex < g.n_ex && ez <= g.n_e) {
        const int64_t s_ = g.n_e + 2;
        const uint8_t* mrow = g.mask + ((ex + 1) * s_ + (ey + 1)) * s_;
        if (ey < g.n_e) { cRR = __ldg(mrow + ez + 1); cRL = __ldg(mrow + ez); }
        const uint8_t* urow = mrow - s_;
        if (ey >= 1) { cUR = __ldg(urow + ez + 1); cUL = __ldg(urow + ez); }
    }
    double mc[orb_count(P)], kc[orb_count(P)];
    #pragma unroll
    for (int i = 0; i < orb_count(P); ++i) { mc[i] = mt.m[i]; kc[i] = mt.k[i]; }
    __syncthreads();
    mbar_wait(bar, 0);

    const int po = halo ? 0 : (w + 1) * P;   // tile plane of node plane ex*P
    double Y[N][P][P];
    #pragma unroll
    for (int r = 0; r < N; ++r)
        #pragma unroll
        for (int b = 0; b < P; ++b)
            #pragma unroll
            for (int j = 0; j < P; ++j) Y[r][b][j] = 0.0;
    if (__any_sync(0xffffffffu, (cRR | cRL | cUR | cUL) != 0)) {
        const double xRR = cRR == 1, xRL = cRL == 1, xUR = cUR == 1, xUL = cUL == 1;
        #pragma unroll
        for (int c = 0; c < N; ++c) {
            const double* plane = us + (size_t)(po + c) * T::UR * T::UW;
            double Au[P][P], Bu[P][P];
            #pragma unroll
            for (int b = 0; b < P; ++b)
                #pragma unroll
                for (int j = 0; j < P; ++j) { Au[b][j] = 0.0; Bu[b][j] = 0.0; }
            #pragma unroll
            for (int e = -P; e <= P; ++e) {
                double zmR[P], zkR[P], zmL, zkL;
                zpass_row<P>(mc, kc, plane + (size_t)(e + P) * T::UW, lane, zmR, zkR, zmL, zkL);
                if (e >= 0) {   // local row e of cell row ey
                    double am[P], ak[P];
                    #pragma unroll
                    for (int j = 0; j < P; ++j) { am[j] = xRR * zmR[j]; ak[j] = xRR * zkR[j]; }
                    am[0] = fma(xRL, zmL, am[0]);
                    ak[0] = fma(xRL, zkL, ak[0]);
                    #pragma unroll
                    for (int b = 0; b < P; ++b)
                        #pragma unroll
                        for (int j = 0; j < P; ++j) {
                            Au[b][j] = fma(mc[orb(P, b, e)], am[j], Au[b][j]);
                            Bu[b][j] = fma(kc[orb(P, b, e)], am[j], fma(mc[orb(P, b, e)], ak[j], Bu[b][j]));
                        }
                }
                if (e <= 0) {   // local row e+P of cell row ey-1 -> our y row 0
                    double am[P], ak[P];
                    #pragma unroll
                    for (int j = 0; j < P; ++j) { am[j] = xUR * zmR[j]; ak[j] = xUR * zkR[j]; }
                    am[0] = fma(xUL, zmL, am[0]);
                    ak[0] = fma(xUL, zkL, ak[0]);
                    #pragma unroll
                    for (int j = 0; j < P; ++j) {
                        Au[0][j] = fma(mc[orb(P, P, e + P)], am[j], Au[0][j]);
                        Bu[0][j] = fma(kc[orb(P, P, e + P)], am[j], fma(mc[orb(P, P, e + P)], ak[j], Bu[0][j]));
                    }
                }
            }
            #pragma unroll
            for (int r = 0; r < N; ++r)
                #pragma unroll
                for (int b = 0; b < P; ++b)
                    #pragma unroll
                    for (int j = 0; j < P; ++j)
                        Y[r][b][j] = fma(kc[orb(P, r, c)], Au[b][j], fma(mc[orb(P, r, c)], Bu[b][j], Y[r][b][j]));
        }
        // dense cut cells: own y row (ey) and the y-up row (ey-1)
        const unsigned clR = __ballot_sync(0xffffffffu, cRR == 2);
        const bool edR = __shfl_sync(0xffffffffu, cRL == 2, 0);
#ifndef WCB3D_NOCUT
        if (clR || edR) cut_cells_warp3<P>(g, ex, ey, K0 / P, lane, clR, edR, false, Y);
#endif
        const unsigned clU = __ballot_sync(0xffffffffu, cUR == 2);
        const bool edU = __shfl_sync(0xffffffffu, cUL == 2, 0);
#ifndef WCB3D_NOCUT
        if (clU || edU) cut_cells_warp3<P>(g, ex, ey - 1, K0 / P, lane, clU, edU, true, Y);
#endif
    }
    // x plane a = P of cell row ex is plane a = 0 of cell row ex+1
    #pragma unroll
    for (int b = 0; b < P; ++b)
        #pragma unroll
        for (int j = 0; j < P; ++j)
            carry[((halo ? 0 : w + 1) * P * P + b * P + j) * 32 + lane] = Y[P][b][j];
    __syncthreads();
    unsigned long long amp = 0ULL;
    if (!halo) {
        #pragma unroll
        for (int b = 0; b < P; ++b)
            #pragma unroll
            for (int j = 0; j < P; ++j)
                Y[0][b][j] = carry[(w * P * P + b * P + j) * 32 + lane] + Y[0][b][j];
        const double f = (MODE == MODE_STEP) ? __ldg(a.ft + a.k) : 0.0;
        const int64_t Kl = K0 + lane * P;
        #pragma unroll
        for (int r = 0; r < P; ++r) {
            const int64_t I = ex * P + r;
            if (I >= g.row_hi) break;
            #pragma unroll
            for (int b = 0; b < P; ++b) {
                const int64_t J = ey * P + b;
                if (J >= g.n1) break;
                const int64_t base = (I + P) * g.pplane + (J + P) * g.prow + Kl + PADJ;
                const double* urow = us + ((size_t)(po + r) * T::UR + P + b) * T::UW + T::CO + P + lane * P;
                if constexpr (MODE == MODE_APPLY) {
                    #pragma unroll
                    for (int j = 0; j < P; ++j)
                        if (Kl + j < g.n1) a.out[base + j] = sk * Y[r][b][j];
                } else {
                    const bool src = base + P - 1 >= a.F.lo && base <= a.F.hi;
                    #pragma unroll
                    for (int j = 0; j < P; ++j) {
                        if (Kl + j < g.n1) {
                            const double fF = src ? f * source_at(a.F, base + j) : f * 0.0;
                            const double mi = __ldg(a.minv + base + j);
                            const double v = leapfrog(urow[j], a.prev[base + j], sk * Y[r][b][j], mi,
                                                      fF, a.dt2);
                            a.out[base + j] = v;
                            unsigned long long bits = mi != 0.0 ? amp_bits(v) : 0ULL;
                            amp = bits > amp ? bits : amp;
                        }
                    }
                }
            }
        }
    }
    if constexpr (MODE == MODE_STEP) block_amp_max<T::NWARP * 32>(amp, a.amp);
}

template <int P, int MODE>
void launch_scm3d(Context* ctx, const CUtensorMap& map_u, const Scm3DGeo& g, const Mats2<P>& mt,
                  double sk, const StepArgs& a) {
    using T = Tile3<P>;
    static bool attr_set = false;
    if (!attr_set) {
        WCB_CUDA(cudaFuncSetAttribute(k_scm3d<P, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)T::SMEM));
        attr_set = true;
    }
    dim3 grid((unsigned)g.n_zs, (unsigned)(g.n_e + 1), (unsigned)g.n_xt);
    k_scm3d<P, MODE><<<grid, T::NWARP * 32, T::SMEM, ctx->stream>>>(map_u, g, mt, sk, a);
    ctx->launches++;
}

#define WCB_INST3(P)                                                                            \
    template void launch_scm3d<P, MODE_STEP>(Context*, const CUtensorMap&, const Scm3DGeo&,    \
                                             const Mats2<P>&, double, const StepArgs&);        \
    template void launch_scm3d<P, MODE_APPLY>(Context*, const CUtensorMap&, const Scm3DGeo&,   \
                                              const Mats2<P>&, double, const StepArgs&);
#define WCB_INSTC(P) \
    template void launch_cut_pre<P>(Context*, int64_t, const double*, const int64_t*, int64_t, int64_t, \
                                    const double*, double*);
WCB_INSTC(1)
WCB_INSTC(2)
WCB_INSTC(3)
WCB_INSTC(4)
WCB_INST3(1)
WCB_INST3(2)
WCB_INST3(3)
WCB_INST3(4)

}  // namespace wcb
