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
    row += Str3<P>::CO;
    const double* own_p = row + P + lane * P;
    // own nodes, the right neighbour's first node and the left cell's nodes
    // straight from shared memory (no shuffles: uniform, no warp collectives)
    double own[P];
    #pragma unroll
    for (int j = 0; j < P; ++j) own[j] = own_p[j];
    const double right = own_p[P];
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
        const double ud = own_p[d - P];
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

// Cut-cell products u_e -> K_o u_e / sk.  Persistent warps walk the cut
// cells with a two-deep pipeline: the packed lower triangle of the next
// cell's K_o / sk (L(L+1)/2 doubles, one 1D bulk copy) and its u_e (cp.async
// gather from the state) land in shared memory while the current cell is
// multiplied.  Lane r forms row r in ascending column order (running packed
// indices: m <= r along row r, m > r down column r) -- the same sums as a
// dense symmetric row.
template <int P>
struct CutPre {
    static constexpr int N = P + 1;
    static constexpr int L = N * N * N;
    static constexpr int LP = L * (L + 1) / 2;
    static constexpr int LPS = cut_lp_stride(P);                        // 16-byte multiple
    static constexpr int W = P <= 2 ? 8 : P == 3 ? 6 : 1;               // warps per CTA
    static constexpr int NS = 2;                                        // pipeline stages per warp (6 warps x 2 beat 4 x 3)
    static constexpr size_t KB = ((size_t)LPS * 8 + 127) / 128 * 128;   // packed matrix buffer
    static constexpr size_t UB = ((size_t)L * 8 + 127) / 128 * 128;     // u_e buffer
    static constexpr size_t PER_WARP = NS * (KB + UB);
    static constexpr size_t OFF_BAR = W * PER_WARP;
    static constexpr size_t SMEM = OFF_BAR + W * NS * 8;
};

__device__ __forceinline__ void cp_async8_g(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int P>
__global__ void __launch_bounds__(256) k_cut_pre(int64_t n_cut, const double* __restrict__ KP,
                                                 const int64_t* __restrict__ cut_base, int64_t pplane,
                                                 int64_t prow, const double* __restrict__ u,
                                                 double* __restrict__ out) {
    using C = CutPre<P>;
    constexpr int N = C::N, L = C::L;
    extern __shared__ __align__(128) unsigned char smc[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned char* mine = smc + (size_t)w * C::PER_WARP;
    constexpr int NS = C::NS;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smc + C::OFF_BAR) + NS * w;
    const int64_t stride = (int64_t)gridDim.x * C::W;
    const int64_t e0 = (int64_t)blockIdx.x * C::W + w;
    if (lane == 0) {
        #pragma unroll
        for (int q = 0; q < NS; ++q) mbar_init(&bar[q], 1);
    }
    __syncwarp();
    auto fetch = [&](int64_t e, int buf) {   // K_o by bulk copy, u_e by cp.async
        double* kp = reinterpret_cast<double*>(mine + buf * (C::KB + C::UB));
        double* uu = reinterpret_cast<double*>(mine + buf * (C::KB + C::UB) + C::KB);
        if (lane == 0) {
            mbar_expect_tx(&bar[buf], (uint32_t)(C::LPS * 8));
            bulk_load(kp, KP + e * C::LPS, (uint32_t)(C::LPS * 8), &bar[buf]);
        }
        const int64_t base = cut_base[e];
        for (int m = lane; m < L; m += 32) {
            const int a = m / (N * N), b = (m / N) % N, j = m % N;
            cp_async8_g(uu + m, u + base + a * pplane + b * prow + j);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // NS-1 cells in flight ahead of the one being multiplied (one cp.async
    // group per fetch slot, empty groups past the end keep the count uniform)
    #pragma unroll
    for (int q = 0; q < NS - 1; ++q) {
        const int64_t eq = e0 + q * stride;
        if (eq < n_cut) fetch(eq, q);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    int it = 0;
    for (int64_t e = e0; e < n_cut; e += stride, ++it) {
        const int buf = it % NS;
        const int64_t en = e + (NS - 1) * stride;
        if (en < n_cut) fetch(en, (it + NS - 1) % NS);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(NS - 1) : "memory");
        __syncwarp();   // every lane's u_e gather of this cell is visible
        mbar_wait(&bar[buf], (uint32_t)((it / NS) & 1));
        const double* kp = reinterpret_cast<const double*>(mine + buf * (C::KB + C::UB));
        const double* uu = reinterpret_cast<const double*>(mine + buf * (C::KB + C::UB) + C::KB);
        for (int r = lane; r < L; r += 32) {
            double t = 0.0;
            int idx = r * (r + 1) / 2;   // (r, 0)
            #pragma unroll 8
            for (int m = 0; m <= r; ++m) t = fma(kp[idx + m], uu[m], t);
            idx = (r + 1) * (r + 2) / 2 + r;   // (r+1, r)
            #pragma unroll 8
            for (int m = r + 1; m < L; ++m) {
                t = fma(kp[idx], uu[m], t);
                idx += m + 1;
            }
            out[e * L + r] = t;
        }
        __syncwarp();   // buffer reused NS cells later
    }
}

template <int P>
void launch_cut_pre(Context* ctx, int64_t n_cut, const double* KP, const int64_t* cut_base,
                    int64_t pplane, int64_t prow, const double* u, double* out) {
    if (!n_cut) return;
    using C = CutPre<P>;
    ensure_smem_attr((const void*)k_cut_pre<P>, ctx->device, (size_t)C::SMEM);
    const int64_t blocks = std::min<int64_t>(ceil_div(n_cut, C::W), (int64_t)ctx->sm_count * std::max<int64_t>(1, (int64_t)(220 * 1024 / C::SMEM)));
    k_cut_pre<P><<<(unsigned)blocks, 32 * C::W, C::SMEM, ctx->stream>>>(n_cut, KP, cut_base, pplane, prow, u, out);
    ctx->launches++;
}

// Streaming stencil + fused CDM epilogue.  Per node plane c of x cell row ex
// (planes ex*P .. ex*P+P, TMA ring): each warp z-contracts the P+1 y rows of
// its cell row and y-contracts them into Au/Bu for its P+1 output rows; row P
// (shared with the next cell row) goes to the next warp through shared memory
// and is added to that warp's row 0 (the halo warp supplies it for the first
// row); the x pass accumulates Y[a] += k1[a][c] Au + m1[a][c] Bu in registers.
// After plane c = P the cut-cell products are added, planes a < P are final
// (epilogue), and Y[P] becomes Y[0] of the next cell row.  Each chunk of x
// cell rows starts one row early (no epilogue) to build that carry, so every
// node value is the same fixed-order sum whatever the chunking (slabs too).
template <int P, int MODE>
__global__ void __launch_bounds__(Str3<P>::NWARP * 32, cpsm_for3(P))
    k_scm3d_v1(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_p, Scm3DGeo g,
            Mats2<P> mt, MinvTab<P> mtab, double sk, StepArgs a) {
    using T = Str3<P>;
    constexpr int N = P + 1;
    constexpr int WY = T::WY;
    constexpr int S = T::S;
    extern __shared__ __align__(128) unsigned char smem[];
    const double* ring = reinterpret_cast<const double*>(smem);
    double* xch = reinterpret_cast<double*>(smem + T::OFF_XCH);   // [2][NWARP][2P][32]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
    uint64_t* pbar = full + S;                                           // psi_{k-1} of a cell row
    const double* prv = reinterpret_cast<const double*>(smem + T::OFF_PREV);   // [P][WY*P][TZ]
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int64_t zs = blockIdx.x, yb = blockIdx.y, xc = blockIdx.z + g.xc0;
    if (MODE == MODE_STEP && zs == 0 && yb == 0 && blockIdx.z == 0) record_observers(a);
    if (!g.cflags[(xc * g.n_yb + yb) * g.n_zs + zs]) return;
    const int64_t K0 = zs * T::TZ;
    const int64_t ey0 = yb * WY;
    const int64_t exA = 1 + xc * g.xc;                                   // first row with an epilogue
    const int64_t exE = exA + g.xc < g.ex_last + 1 ? exA + g.xc : g.ex_last + 1;
    const int64_t G0 = (exA - 1) * P, G1 = (exE - 1) * P + P;           // node planes streamed
    const bool halo = (w == WY);
    const int64_t ey = halo ? ey0 - 1 : ey0 + w;                         // this warp's cell row
    const int64_t ez = K0 / P + lane;
    const int trow = (halo ? 0 : w + 1) * P;                             // tile row of node row ey*P
    const bool producer = halo && lane == 0;
    auto issue = [&](int64_t gp) {   // plane gp -> its ring slot
        const int s = (int)((gp - G0) % S);
        mbar_expect_tx(&full[s], (uint32_t)(T::PLANE * 8));
        tma_load_3d(smem + (size_t)s * T::SLOT * 8, &tm_u, (int32_t)(K0 - P - T::CO + PADJ),
                    (int32_t)(ey0 * P), (int32_t)(gp + P), &full[s]);
    };
    if (threadIdx.x == 0) {
        #pragma unroll
        for (int s = 0; s < S + 1; ++s) mbar_init(&full[s], 1);
    }
    __syncthreads();
    if (producer)
        for (int64_t gp = G0; gp <= G1 && gp < G0 + S; ++gp) issue(gp);
    double mc[orb_count(P)], kc[orb_count(P)];
    #pragma unroll
    for (int i = 0; i < orb_count(P); ++i) { mc[i] = mt.m[i]; kc[i] = mt.k[i]; }
    const double f = (MODE == MODE_STEP) ? __ldg(a.ft + a.k) : 0.0;
    const int64_t s_ = g.n_e + 2;
    const int up = halo ? WY : (w == 0 ? WY : w - 1);   // exchange source warp
    double Y[N][P][P];
    #pragma unroll
    for (int r = 0; r < N; ++r)
        #pragma unroll
        for (int b = 0; b < P; ++b)
            #pragma unroll
            for (int j = 0; j < P; ++j) Y[r][b][j] = 0.0;
    unsigned long long amp = 0ULL;
    // Au/Bu persist across cell rows: plane P of row ex is plane 0 of row
    // ex+1, so when no uncut flag of the CTA changes between the rows its
    // y/z contraction is reused instead of recomputed.  YP accumulates this
    // warp's contribution to the next warp's node row 0 (y-local row P) for
    // every x plane of the row; it is exchanged once per cell row.
    double Au[N][P], Bu[N][P];
    double YP[N][P];
    bool pxRR = false, pxRL = false;
    for (int64_t ex = exA - 1; ex < exE; ++ex) {
        // codes of (ex, ey, ez), (ex, ey, ez-1), (ex, ey-1, ez), (ex, ey-1, ez-1)
        uint8_t cRR = 0, cRL = 0, cUR = 0, cUL = 0;
        if (ex >= 0 && ex < g.n_ex && ez <= g.n_e && ey >= -1 && ey <= g.n_e) {
            const uint8_t* mrow = g.mask + ((ex + 1) * s_ + (ey + 1)) * s_;
            if (ey < g.n_e && ey >= 0) { cRR = __ldg(mrow + ez + 1); cRL = __ldg(mrow + ez); }
            if (!halo && ey >= 1) { cUR = __ldg(mrow - s_ + ez + 1); cUL = __ldg(mrow - s_ + ez); }
        }
        const double xRR = cRR == 1, xRL = cRL == 1;
        const bool cln = g.clean && cRR == 1 && ex >= 1 && __ldg(g.clean + (ex * g.n_e + ey) * g.n_e + ez) != 0;
        // row-start barrier: every warp is past row ex-1's epilogue
        const bool live = __syncthreads_or((cRR | cRL) != 0);   // any uncut/cut work in this CTA row
#if WCB3D_REUSE
        const bool reuse = ex > exA - 1 && !__syncthreads_or((cRR == 1) != pxRR || (cRL == 1) != pxRL);
#else
        const bool reuse = false;
#endif
        pxRR = cRR == 1;
        pxRL = cRL == 1;
        if (producer && ex >= exA) {   // refill row ex-1's planes (a full row of look-ahead)
            #pragma unroll 1
            for (int q = 0; q < P; ++q) {
                const int64_t np = (ex - 1) * P + q + S;
                if (np <= G1) issue(np);
            }
            if (MODE == MODE_STEP) {   // psi_{k-1} of row ex's owned nodes for its epilogue
                mbar_expect_tx(pbar, (uint32_t)T::PREV_BYTES);
                tma_load_3d(smem + T::OFF_PREV, &tm_p, (int32_t)(K0 + PADJ), (int32_t)(ey0 * P + P),
                            (int32_t)(ex * P + P), pbar);
            }
        }
        #pragma unroll
        for (int a2 = 0; a2 < N; ++a2)
            #pragma unroll
            for (int j = 0; j < P; ++j) YP[a2][j] = 0.0;
        #pragma unroll
        for (int c = 0; c < N; ++c) {
          if (!(c == 0 && reuse)) {   // CTA-uniform
            const int64_t gp = ex * P + c;
            const int slot = (int)((gp - G0) % S);
            const double* plane = ring + (size_t)slot * T::SLOT;
            #pragma unroll
            for (int b = 0; b < N; ++b)
                #pragma unroll
                for (int j = 0; j < P; ++j) { Au[b][j] = 0.0; Bu[b][j] = 0.0; }
            mbar_wait(&full[slot], (uint32_t)(((gp - G0) / S) & 1));
            if (live) {
                #pragma unroll
                for (int e = 0; e < N; ++e) {
                    double zmR[P], zkR[P], zmL, zkL;
                    zpass_row<P>(mc, kc, plane + (size_t)(trow + e) * T::UW, lane, zmR, zkR, zmL, zkL);
                    double am[P], ak[P];
                    #pragma unroll
                    for (int j = 0; j < P; ++j) { am[j] = xRR * zmR[j]; ak[j] = xRR * zkR[j]; }
                    am[0] = fma(xRL, zmL, am[0]);
                    ak[0] = fma(xRL, zkL, ak[0]);
                    #pragma unroll
                    for (int b = 0; b < N; ++b) {
                        if (halo && b < P) continue;
                        #pragma unroll
                        for (int j = 0; j < P; ++j) {
                            Au[b][j] = fma(mc[orb(P, b, e)], am[j], Au[b][j]);
                            Bu[b][j] = fma(kc[orb(P, b, e)], am[j], fma(mc[orb(P, b, e)], ak[j], Bu[b][j]));
                        }
                    }
                }
            }
          }
            // x pass (plane 0 of a reused row takes the previous row's plane-P Au/Bu)
            #pragma unroll
            for (int r = 0; r < N; ++r) {
                #pragma unroll
                for (int j = 0; j < P; ++j)
                    YP[r][j] = fma(kc[orb(P, r, c)], Au[P][j], fma(mc[orb(P, r, c)], Bu[P][j], YP[r][j]));
                if (!halo) {
                    #pragma unroll
                    for (int b = 0; b < P; ++b)
                        #pragma unroll
                        for (int j = 0; j < P; ++j)
                            Y[r][b][j] = fma(kc[orb(P, r, c)], Au[b][j], fma(mc[orb(P, r, c)], Bu[b][j], Y[r][b][j]));
                }
            }
        }
        // y exchange of the shared node row: own + row above's contribution
        {
            double* xw = xch + (size_t)w * N * P * 32 + lane;
            #pragma unroll
            for (int r = 0; r < N; ++r)
                #pragma unroll
                for (int j = 0; j < P; ++j) xw[(r * P + j) * 32] = YP[r][j];
        }
        __syncthreads();
        if (!halo) {
            const double* xr = xch + (size_t)up * N * P * 32 + lane;
            #pragma unroll
            for (int r = 0; r < N; ++r)
                #pragma unroll
                for (int j = 0; j < P; ++j) Y[r][0][j] += xr[(r * P + j) * 32];
            // dense cut cells: own y row (ey) and the y-up row (ey-1)
            const unsigned clR = __ballot_sync(0xffffffffu, cRR == 2);
            const bool edR = __shfl_sync(0xffffffffu, cRL == 2, 0);
            if (clR || edR) cut_cells_warp3<P>(g, ex, ey, K0 / P, lane, clR, edR, false, Y);
            const unsigned clU = __ballot_sync(0xffffffffu, cUR == 2);
            const bool edU = __shfl_sync(0xffffffffu, cUL == 2, 0);
            if (clU || edU) cut_cells_warp3<P>(g, ex, ey - 1, K0 / P, lane, clU, edU, true, Y);
            if (ex >= exA) {
                if (MODE == MODE_STEP) mbar_wait(pbar, (uint32_t)((ex - exA) & 1));
                const int64_t Kl = K0 + lane * P;
                #pragma unroll
                for (int r = 0; r < P; ++r) {
                    const int64_t I = ex * P + r;
                    if (I >= g.row_hi) break;
                    const double* pl = ring + (size_t)((I - G0) % S) * T::SLOT;
                    #pragma unroll
                    for (int b = 0; b < P; ++b) {
                        const int64_t J = ey * P + b;
                        if (J >= g.n1) break;
                        const int64_t base = (I + P) * g.pplane + (J + P) * g.prow + Kl + PADJ;
                        if constexpr (MODE == MODE_APPLY) {
                            #pragma unroll
                            for (int j = 0; j < P; ++j)
                                if (Kl + j < g.n1) a.out[base + j] = sk * Y[r][b][j];
                        } else {
                            const double* urow = pl + (size_t)(trow + b) * T::UW + T::CO + P + lane * P;
                            const bool src = base + P - 1 >= a.F.lo && base <= a.F.hi;
                            #pragma unroll
                            for (int j = 0; j < P; ++j) {
                                if (Kl + j < g.n1) {
                                    const double fF = src ? f * source_at(a.F, base + j) : f * 0.0;
                                    const double mi = cln ? mtab.v[(r * P + b) * P + j] : __ldg(a.minv + base + j);
                                    const double up = prv[((size_t)r * WY * P + w * P + b) * T::TZ + lane * P + j];
                                    const double v = leapfrog(urow[j], up, sk * Y[r][b][j], mi, fF, a.dt2);
                                    a.out[base + j] = v;
                                    const unsigned long long bits = mi != 0.0 ? amp_bits(v) : 0ULL;
                                    amp = bits > amp ? bits : amp;
                                }
                            }
                        }
                    }
                }
            }
            // x plane P of cell row ex is plane 0 of cell row ex+1
            #pragma unroll
            for (int b = 0; b < P; ++b)
                #pragma unroll
                for (int j = 0; j < P; ++j) {
                    Y[0][b][j] = Y[P][b][j];
                    #pragma unroll
                    for (int r = 1; r < N; ++r) Y[r][b][j] = 0.0;
                }
        }
    }
    if constexpr (MODE == MODE_STEP) block_amp_max<T::NWARP * 32>(amp, a.amp);
}

// Dataflow version of the streaming stencil (default).  Same sums in the same
// order as k_scm3d_v1 (bitwise equal fields), but no block barrier inside the
// x loop: warps run loosely coupled through mbarriers --
//   full[s]    TMA ring slot s landed (as before)
//   rowdone    every compute warp is past cell row t (its epilogue included):
//              the halo/producer warp waits on it before refilling row t's ring
//              slots and the psi_{k-1} buffer
//   xfull[w] / xempty[w]   the shared y node row of warp w (YP) handed to the
//              warp below it, single buffer with a full/empty handshake
// so a warp delayed by cut cells or a non-table 1/m row no longer stalls the
// other seven (ncu on v1: 17 % barrier stalls).  `live` and `reuse` are
// warp-level votes (both only skip work whose result is identical).  The cell
// codes of row t+1 are loaded during row t.  Accumulators start from their
// first product instead of being zeroed (v1: 11 % of all instructions were
// CS2R zeroing).  Epilogue: lanes whose cell takes 1/m from the interior
// table and whose rows hold no source node run a branch-free path with the
// table as immediate constants and all loads of a node row issued before its
// arithmetic (v1: a dependent constant/global load per node, 20 % long
// scoreboard stalls); other lanes keep the general path.
template <int P, int MODE>
__global__ void __launch_bounds__(Str3<P>::NWARP * 32, cpsm_for3(P))
    k_scm3d(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_p, Scm3DGeo g,
            Mats2<P> mt, MinvTab<P> mtab, double sk, StepArgs a) {
    using T = Str3<P>;
    constexpr int N = P + 1;
    constexpr int WY = T::WY;
    constexpr int S = T::S;
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(128) unsigned char smem[];
    const double* ring = reinterpret_cast<const double*>(smem);
    double* xch = reinterpret_cast<double*>(smem + T::OFF_XCH);   // [NWARP][N*P][32]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
    uint64_t* pbar = full + S;                                           // psi_{k-1} of a cell row
    uint64_t* rowdone = pbar + 1;
    uint64_t* xfull = rowdone + 1;
    uint64_t* xempty = xfull + T::NWARP;
    const double* prv = reinterpret_cast<const double*>(smem + T::OFF_PREV);   // [P][WY*P][TZ]
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int64_t zs = blockIdx.x, yb = blockIdx.y, xc = blockIdx.z + g.xc0;
    if (MODE == MODE_STEP && zs == 0 && yb == 0 && blockIdx.z == 0) record_observers(a);
    if (!g.cflags[(xc * g.n_yb + yb) * g.n_zs + zs]) return;
    const int64_t K0 = zs * T::TZ;
    const int64_t ey0 = yb * WY;
    const int64_t exA = 1 + xc * g.xc;                                   // first row with an epilogue
    const int64_t exE = exA + g.xc < g.ex_last + 1 ? exA + g.xc : g.ex_last + 1;
    const int64_t G0 = (exA - 1) * P;
    const int nplanes = (int)(exE - exA + 1) * P + 1;                    // node planes streamed (G0 ..)
    const bool halo = (w == WY);
    const int64_t ey = halo ? ey0 - 1 : ey0 + w;                         // this warp's cell row
    const int64_t ez = K0 / P + lane;
    const int trow = (halo ? 0 : w + 1) * P;                             // tile row of node row ey*P
    auto issue = [&](int lp) {   // streamed plane lp (global plane G0 + lp) -> its ring slot
        const int s = lp % S;
        mbar_expect_tx(&full[s], (uint32_t)(T::PLANE * 8));
        tma_load_3d(smem + (size_t)s * T::SLOT * 8, &tm_u, (int32_t)(K0 - P - T::CO + PADJ),
                    (int32_t)(ey0 * P), (int32_t)(G0 + lp + P), &full[s]);
    };
    if (threadIdx.x == 0) {
        #pragma unroll
        for (int s = 0; s < S + 1; ++s) mbar_init(&full[s], 1);
        mbar_init(rowdone, WY * 32);
        for (int q = 0; q < T::NWARP; ++q) {
            mbar_init(&xfull[q], 32);
            mbar_init(&xempty[q], 32);
        }
    }
    __syncthreads();
    if (halo && lane == 0)
        for (int lp = 0; lp < nplanes && lp < S; ++lp) issue(lp);
    double mc[orb_count(P)], kc[orb_count(P)];
    #pragma unroll
    for (int i = 0; i < orb_count(P); ++i) { mc[i] = mt.m[i]; kc[i] = mt.k[i]; }
    const double f = (MODE == MODE_STEP) ? __ldg(a.ft + a.k) : 0.0;
    const double f0 = f * 0.0;
    const int64_t s_ = g.n_e + 2;
    const int up = w == 0 ? WY : w - 1;              // exchange source warp (compute warps)
    const bool sends = halo || w < WY - 1;           // the last compute warp's row P belongs to the next block
    double* const xw = xch + (size_t)w * N * P * 32 + lane;
    const double* const xr = xch + (size_t)up * N * P * 32 + lane;
    // cell codes of (ex, ey, ez), (ex, ey, ez-1), (ex, ey-1, ez), (ex, ey-1, ez-1), packed
    auto codes = [&](int64_t ex) -> uint32_t {
        uint32_t cRR = 0, cRL = 0, cUR = 0, cUL = 0;
        if (ex >= 0 && ex < g.n_ex && ez <= g.n_e && ey >= -1 && ey <= g.n_e) {
            const uint8_t* mrow = g.mask + ((ex + 1) * s_ + (ey + 1)) * s_;
            if (ey < g.n_e && ey >= 0) { cRR = __ldg(mrow + ez + 1); cRL = __ldg(mrow + ez); }
            if (!halo && ey >= 1) { cUR = __ldg(mrow - s_ + ez + 1); cUL = __ldg(mrow - s_ + ez); }
        }
        return cRR | (cRL << 8) | (cUR << 16) | (cUL << 24);
    };
    auto clean_of = [&](int64_t ex) -> uint32_t {
        if (halo || !g.clean || ex < 1 || ex >= g.n_ex || ey >= g.n_e || ez >= g.n_e) return 0u;
        return __ldg(g.clean + (ex * g.n_e + ey) * g.n_e + ez);
    };
    double Y[N][P][P];
    #pragma unroll
    for (int b = 0; b < P; ++b)
        #pragma unroll
        for (int j = 0; j < P; ++j) Y[0][b][j] = 0.0;
    unsigned long long amp = 0ULL;
    // Au/Bu persist across cell rows: plane P of row ex is plane 0 of row
    // ex+1, so when none of this warp's uncut flags changes between the rows
    // its y/z contraction is reused instead of recomputed.  YP accumulates this
    // warp's contribution to the next warp's node row 0 (y-local row P) for
    // every x plane of the row; it is handed over once per cell row.
    double Au[N][P], Bu[N][P];
    double YP[N][P];
    #pragma unroll
    for (int b = 0; b < N; ++b)
        #pragma unroll
        for (int j = 0; j < P; ++j) { Au[b][j] = 0.0; Bu[b][j] = 0.0; }
    bool pxRR = false, pxRL = false;
    uint32_t ncode = codes(exA - 1), nclean = clean_of(exA - 1);
    int t = 0;                                        // row index within the chunk
    for (int64_t ex = exA - 1; ex < exE; ++ex, ++t) {
        const uint32_t code = ncode;
        const uint32_t cRR = code & 0xff, cRL = (code >> 8) & 0xff;
        const bool cln = cRR == 1 && nclean != 0;
        if (ex + 1 < exE) { ncode = codes(ex + 1); nclean = clean_of(ex + 1); }
        const double xRR = cRR == 1, xRL = cRL == 1;
        const bool live = __any_sync(FULL, (cRR | cRL) != 0);
#if WCB3D_REUSE
        const bool reuse = t > 0 && !__any_sync(FULL, (cRR == 1) != pxRR || (cRL == 1) != pxRL);
#else
        const bool reuse = false;
#endif
        pxRR = cRR == 1;
        pxRL = cRL == 1;
        if (halo && t > 0) {   // refill row t-1's planes (a full row of look-ahead), psi_{k-1} of row t
            mbar_wait(rowdone, (uint32_t)((t - 1) & 1));
            if (lane == 0) {
                #pragma unroll 1
                for (int q = 0; q < P; ++q) {
                    const int lp = (t - 1) * P + q + S;
                    if (lp < nplanes) issue(lp);
                }
                if (MODE == MODE_STEP) {
                    mbar_expect_tx(pbar, (uint32_t)T::PREV_BYTES);
                    tma_load_3d(smem + T::OFF_PREV, &tm_p, (int32_t)(K0 + PADJ), (int32_t)(ey0 * P + P),
                                (int32_t)(ex * P + P), pbar);
                }
            }
            __syncwarp();
        }
        #pragma unroll
        for (int c = 0; c < N; ++c) {
            if (!(c == 0 && reuse)) {   // warp-uniform
                const int lp = t * P + c;
                const int slot = lp % S;
                const double* plane = ring + (size_t)slot * T::SLOT;
                mbar_wait(&full[slot], (uint32_t)((lp / S) & 1));
                if (live) {
                    #pragma unroll
                    for (int e = 0; e < N; ++e) {
                        double zmR[P], zkR[P], zmL, zkL;
                        zpass_row<P>(mc, kc, plane + (size_t)(trow + e) * T::UW, lane, zmR, zkR, zmL, zkL);
                        double am[P], ak[P];
                        #pragma unroll
                        for (int j = 0; j < P; ++j) { am[j] = xRR * zmR[j]; ak[j] = xRR * zkR[j]; }
                        am[0] = fma(xRL, zmL, am[0]);
                        ak[0] = fma(xRL, zkL, ak[0]);
                        #pragma unroll
                        for (int b = 0; b < N; ++b) {
                            if (halo && b < P) continue;
                            #pragma unroll
                            for (int j = 0; j < P; ++j) {
                                if (e == 0) {   // first product starts the sum (== fma onto 0)
                                    Au[b][j] = mc[orb(P, b, e)] * am[j];
                                    Bu[b][j] = fma(kc[orb(P, b, e)], am[j], mc[orb(P, b, e)] * ak[j]);
                                } else {
                                    Au[b][j] = fma(mc[orb(P, b, e)], am[j], Au[b][j]);
                                    Bu[b][j] = fma(kc[orb(P, b, e)], am[j], fma(mc[orb(P, b, e)], ak[j], Bu[b][j]));
                                }
                            }
                        }
                    }
                } else {
                    #pragma unroll
                    for (int b = 0; b < N; ++b)
                        #pragma unroll
                        for (int j = 0; j < P; ++j) { Au[b][j] = 0.0; Bu[b][j] = 0.0; }
                }
            }
            // x pass (plane 0 of a reused row takes the previous row's plane-P Au/Bu)
            #pragma unroll
            for (int r = 0; r < N; ++r) {
                #pragma unroll
                for (int j = 0; j < P; ++j) {
                    if (c == 0) YP[r][j] = fma(kc[orb(P, r, c)], Au[P][j], mc[orb(P, r, c)] * Bu[P][j]);
                    else YP[r][j] = fma(kc[orb(P, r, c)], Au[P][j], fma(mc[orb(P, r, c)], Bu[P][j], YP[r][j]));
                }
                if (!halo) {
                    #pragma unroll
                    for (int b = 0; b < P; ++b)
                        #pragma unroll
                        for (int j = 0; j < P; ++j) {
                            if (c == 0 && r > 0)
                                Y[r][b][j] = fma(kc[orb(P, r, c)], Au[b][j], mc[orb(P, r, c)] * Bu[b][j]);
                            else
                                Y[r][b][j] = fma(kc[orb(P, r, c)], Au[b][j], fma(mc[orb(P, r, c)], Bu[b][j], Y[r][b][j]));
                        }
                }
            }
        }
        // hand the shared y node row to the warp below (single buffer, full/empty)
        if (sends) {
            if (t > 0) mbar_wait(&xempty[w], (uint32_t)((t - 1) & 1));
            #pragma unroll
            for (int r = 0; r < N; ++r)
                #pragma unroll
                for (int j = 0; j < P; ++j) xw[(r * P + j) * 32] = YP[r][j];
            mbar_arrive(&xfull[w]);
        }
        if (!halo) {
            mbar_wait(&xfull[up], (uint32_t)(t & 1));
            #pragma unroll
            for (int r = 0; r < N; ++r)
                #pragma unroll
                for (int j = 0; j < P; ++j) Y[r][0][j] += xr[(r * P + j) * 32];
            mbar_arrive(&xempty[up]);
            // dense cut cells: own y row (ey) and the y-up row (ey-1)
            const uint32_t cUR = (code >> 16) & 0xff, cUL = code >> 24;
            const unsigned clR = __ballot_sync(FULL, cRR == 2);
            const bool edR = __shfl_sync(FULL, cRL == 2, 0);
            if (clR || edR) cut_cells_warp3<P>(g, ex, ey, K0 / P, lane, clR, edR, false, Y);
            const unsigned clU = __ballot_sync(FULL, cUR == 2);
            const bool edU = __shfl_sync(FULL, cUL == 2, 0);
            if (clU || edU) cut_cells_warp3<P>(g, ex, ey - 1, K0 / P, lane, clU, edU, true, Y);
            if (t > 0) {
                if (MODE == MODE_STEP) mbar_wait(pbar, (uint32_t)((t - 1) & 1));
                const int64_t Kl = K0 + lane * P;
                const int64_t base0 = (ex * P + P) * g.pplane + (ey * P + P) * g.prow + Kl + PADJ;
                const int64_t baseL = base0 + (P - 1) * (g.pplane + g.prow) + (P - 1);
                bool fast = false;
                if constexpr (MODE == MODE_STEP) fast = cln && (baseL < a.F.lo || base0 > a.F.hi);
                if (fast) {
                    // every node of the cell is an owned DOF with the table's 1/m, no source node
                    const double* up0 = prv + (size_t)(w * P) * T::TZ + lane * P;
                    const int u0 = trow * T::UW + T::CO + P + lane * P;
                    #pragma unroll
                    for (int r = 0; r < P; ++r) {
                        const double* pl = ring + (size_t)((t * P + r) % S) * T::SLOT + u0;
                        double* orow = a.out + base0 + r * g.pplane;
                        #pragma unroll
                        for (int b = 0; b < P; ++b) {
                            double uu[P], pp[P], v[P];
                            #pragma unroll
                            for (int j = 0; j < P; ++j) {
                                uu[j] = pl[b * T::UW + j];
                                pp[j] = up0[((size_t)r * WY * P + b) * T::TZ + j];
                            }
                            #pragma unroll
                            for (int j = 0; j < P; ++j)
                                v[j] = leapfrog(uu[j], pp[j], sk * Y[r][b][j], mtab.v[(r * P + b) * P + j], f0, a.dt2);
                            #pragma unroll
                            for (int j = 0; j < P; ++j) {
                                orow[b * g.prow + j] = v[j];
                                const unsigned long long bits = amp_bits(v[j]);
                                amp = bits > amp ? bits : amp;
                            }
                        }
                    }
                } else {
                    #pragma unroll
                    for (int r = 0; r < P; ++r) {
                        const int64_t I = ex * P + r;
                        if (I >= g.row_hi) break;
                        const double* pl = ring + (size_t)((t * P + r) % S) * T::SLOT;
                        #pragma unroll
                        for (int b = 0; b < P; ++b) {
                            const int64_t J = ey * P + b;
                            if (J >= g.n1) break;
                            const int64_t base = (I + P) * g.pplane + (J + P) * g.prow + Kl + PADJ;
                            if constexpr (MODE == MODE_APPLY) {
                                #pragma unroll
                                for (int j = 0; j < P; ++j)
                                    if (Kl + j < g.n1) a.out[base + j] = sk * Y[r][b][j];
                            } else {
                                const double* urow = pl + (size_t)(trow + b) * T::UW + T::CO + P + lane * P;
                                const bool src = base + P - 1 >= a.F.lo && base <= a.F.hi;
                                #pragma unroll
                                for (int j = 0; j < P; ++j) {
                                    if (Kl + j < g.n1) {
                                        const double fF = src ? f * source_at(a.F, base + j) : f0;
                                        const double mi = cln ? mtab.v[(r * P + b) * P + j] : __ldg(a.minv + base + j);
                                        const double upv = prv[((size_t)r * WY * P + w * P + b) * T::TZ + lane * P + j];
                                        const double v = leapfrog(urow[j], upv, sk * Y[r][b][j], mi, fF, a.dt2);
                                        a.out[base + j] = v;
                                        const unsigned long long bits = mi != 0.0 ? amp_bits(v) : 0ULL;
                                        amp = bits > amp ? bits : amp;
                                    }
                                }
                            }
                        }
                    }
                }
            }
            // x plane P of cell row ex is plane 0 of cell row ex+1
            #pragma unroll
            for (int b = 0; b < P; ++b)
                #pragma unroll
                for (int j = 0; j < P; ++j) Y[0][b][j] = Y[P][b][j];
            mbar_arrive(rowdone);
        }
    }
    if constexpr (MODE == MODE_STEP) block_amp_max<T::NWARP * 32>(amp, a.amp);
}

// The node column z = n1-1 when n_e is a multiple of 32 (no strip lane owns
// it).  Stage 1: the z contraction of the last cell column onto its node
// z = n1-1 for every (x plane, y row): zline = (m1[P] . u, k1[P] . u).
// Stage 2: one thread per (x plane, y row) sums its <= 4 cells (ex, ey, n_e-1)
// in ascending (ex, ey) order from those lines (coalesced in y).
template <int P>
__global__ void __launch_bounds__(256) k_scm3d_zline(Scm3DGeo g, Mats2<P> mt, const double* __restrict__ u,
                                                    double2* __restrict__ zl) {
    constexpr int N = P + 1;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t npl = g.n_ex * P + 1;
    if (t >= npl * g.n1) return;
    const int64_t I = t / g.n1, J = t % g.n1;
    const double* row = u + (I + P) * g.pplane + (J + P) * g.prow + (g.n1 - 1 - P) + PADJ;
    double zm = 0.0, zk = 0.0;
    #pragma unroll
    for (int j = 0; j < N; ++j) {
        const double v = row[j];
        zm = fma(mt.m[orb(P, P, j)], v, zm);
        zk = fma(mt.k[orb(P, P, j)], v, zk);
    }
    zl[t] = make_double2(zm, zk);
}

template <int P, int MODE>
__global__ void __launch_bounds__(128) k_scm3d_zcol(Scm3DGeo g, Mats2<P> mt, double sk, const double2* __restrict__ zl,
                                                   StepArgs a) {
    constexpr int N = P + 1;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n_pl = g.row_hi - g.row_lo;
    unsigned long long amp = 0ULL;
    if (t < n_pl * g.n1) {
        const int64_t I = g.row_lo + t / g.n1, J = t % g.n1, K = g.n1 - 1;
        const int64_t s_ = g.n_e + 2;
        double acc = 0.0;
        for (int dx = 1; dx >= 0; --dx) {
            const int64_t ex = I / P - dx;
            const int ia = (int)(I - ex * P);
            if (ex < 0 || ex >= g.n_ex || ia > P) continue;
            for (int dy = 1; dy >= 0; --dy) {
                const int64_t ey = J / P - dy;
                const int ib = (int)(J - ey * P);
                if (ey < 0 || ey >= g.n_e || ib > P) continue;
                const int64_t ez = g.n_e - 1;
                const uint8_t code = g.mask[((ex + 1) * s_ + (ey + 1)) * s_ + ez + 1];
                if (code == 1) {
                    double s = 0.0;
                    #pragma unroll
                    for (int q = 0; q < N; ++q)
                        #pragma unroll
                        for (int r = 0; r < N; ++r) {
                            const double2 z = zl[(ex * P + q) * g.n1 + ey * P + r];
                            const double mq = mt.m[orb(P, ia, q)], kq = mt.k[orb(P, ia, q)];
                            const double mr = mt.m[orb(P, ib, r)], kr = mt.k[orb(P, ib, r)];
                            s = fma(kq * mr + mq * kr, z.x, fma(mq * mr, z.y, s));
                        }
                    acc += s;
                } else if (code == 2) {
                    const int32_t id = g.cut_id[(ex * g.n_e + ey) * g.n_e + ez];
                    acc += g.cut_out[(int64_t)id * N * N * N + (ia * N + ib) * N + P];
                }
            }
        }
        const int64_t base = (I + P) * g.pplane + (J + P) * g.prow + K + PADJ;
        if constexpr (MODE == MODE_APPLY) {
            a.out[base] = sk * acc;
        } else {
            const double f = __ldg(a.ft + a.k);
            const double mi = a.minv[base];
            const double v = leapfrog(a.cur[base], a.prev[base], sk * acc, mi, f * source_at(a.F, base), a.dt2);
            a.out[base] = v;
            amp = mi != 0.0 ? amp_bits(v) : 0ULL;
        }
    }
    if constexpr (MODE == MODE_STEP) block_amp_max<128>(amp, a.amp);
}

template <int P>
__global__ void k_clean3d(Scm3DGeo g, MinvTab<P> tab, const double* __restrict__ minv, uint8_t* clean) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nc = g.n_ex * g.n_e * g.n_e;
    if (c >= nc) return;
    const int64_t ex = c / (g.n_e * g.n_e), ey = (c / g.n_e) % g.n_e, ez = c % g.n_e;
    bool ok = ex >= 1;
    for (int q = 0; q < P && ok; ++q)
        for (int r = 0; r < P && ok; ++r)
            for (int j = 0; j < P && ok; ++j) {
                const int64_t I = ex * P + q;
                const int64_t s = (I + P) * g.pplane + (ey * P + r + P) * g.prow + ez * P + j + PADJ;
                ok = I < g.row_hi && __double_as_longlong(minv[s]) == __double_as_longlong(tab.v[(q * P + r) * P + j]);
            }
    clean[c] = ok ? 1 : 0;
}

template <int P>
void launch_clean3d(Context* ctx, const Scm3DGeo& g, const MinvTab<P>& tab, const double* minv, uint8_t* clean) {
    const int64_t nc = g.n_ex * g.n_e * g.n_e;
    k_clean3d<P><<<(unsigned)ceil_div(nc, 256), 256, 0, ctx->stream>>>(g, tab, minv, clean);
    ctx->launches++;
}

template <int P, int MODE>
void launch_scm3d(Context* ctx, const CUtensorMap& map_u, const CUtensorMap& map_p, const Scm3DGeo& g0,
                  const Mats2<P>& mt, const MinvTab<P>& mtab, double sk, const StepArgs& a0, int part) {
    using T = Str3<P>;
    auto launch = [&](int64_t xc0, int64_t nz, bool obs) {
        if (nz <= 0) return;
        Scm3DGeo g = g0;
        g.xc0 = xc0;
        StepArgs a = a0;
        if (!obs) a.obs_out = nullptr;
        dim3 grid((unsigned)g.n_zs, (unsigned)g.n_yb, (unsigned)nz);
        static const bool v1 = [] { const char* e = getenv("WCB3D_V1"); return e && e[0] == '1'; }();
        if (v1) {
            ensure_smem_attr((const void*)k_scm3d_v1<P, MODE>, ctx->device, (size_t)T::SMEM);
            k_scm3d_v1<P, MODE><<<grid, T::NWARP * 32, T::SMEM, ctx->stream>>>(map_u, map_p, g, mt, mtab, sk, a);
        } else {
            ensure_smem_attr((const void*)k_scm3d<P, MODE>, ctx->device, (size_t)T::SMEM);
            k_scm3d<P, MODE><<<grid, T::NWARP * 32, T::SMEM, ctx->stream>>>(map_u, map_p, g, mt, mtab, sk, a);
        }
        ctx->launches++;
    };
    const int64_t n = g0.n_xc;
    if (part < 0) {
        launch(0, n, true);
    } else if (part == 0) {   // chunks holding the rows exchanged with the neighbours
        launch(0, 1, true);
        if (n > 1) launch(n - 1, 1, false);
    } else {
        launch(1, n - 2, false);
    }
    if (part != 1 && g0.n_e % 32 == 0) {
        const Scm3DGeo& g = g0;
        WCB_REQUIRE(g.zline, "z-line buffer missing");
        const int64_t nl = (g.n_ex * P + 1) * g.n1;
        k_scm3d_zline<P><<<(unsigned)ceil_div(nl, 256), 256, 0, ctx->stream>>>(g, mt, a0.cur, g.zline);
        const int64_t nn = (g.row_hi - g.row_lo) * g.n1;
        k_scm3d_zcol<P, MODE><<<(unsigned)ceil_div(nn, 128), 128, 0, ctx->stream>>>(g, mt, sk, g.zline, a0);
        ctx->launches += 2;
    }
}

#define WCB_INST3(P)                                                                            \
    template void launch_scm3d<P, MODE_STEP>(Context*, const CUtensorMap&, const CUtensorMap&, const Scm3DGeo&, \
                                             const Mats2<P>&, const MinvTab<P>&, double,        \
                                             const StepArgs&, int);                             \
    template void launch_scm3d<P, MODE_APPLY>(Context*, const CUtensorMap&, const CUtensorMap&, const Scm3DGeo&, \
                                              const Mats2<P>&, const MinvTab<P>&, double,       \
                                              const StepArgs&, int);                            \
    template void launch_clean3d<P>(Context*, const Scm3DGeo&, const MinvTab<P>&, const double*, uint8_t*);
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
