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

// Cut-cell products u_e -> K_o u_e / sk.  Persistent warp groups walk the cut
// cells with a two-deep pipeline: the packed lower triangle of the next
// cell's K_o / sk (L(L+1)/2 doubles, one 1D bulk copy) and its u_e (cp.async
// gather from the state) land in shared memory while the current cell is
// multiplied.  A group is G = ceil(L/32) warps (two for P = 3), one row per
// lane: lane r forms row r in ascending column order (m <= r along row r,
// m > r down column r of the packed triangle) -- the same sums as a dense
// symmetric row.  (One warp per cell with two rows per lane left the
// SM at 6 warps, stalled on shared-memory latency: ncu, 312 us on config 5.)
template <int P>
struct CutPre {
    static constexpr int N = P + 1;
    static constexpr int L = N * N * N;
    static constexpr int LP = L * (L + 1) / 2;
    static constexpr int LPS = cut_lp_stride(P);                        // 16-byte multiple
    static constexpr int G = (L + 31) / 32 > 4 ? 4 : (L + 31) / 32;     // warps per cell
    static constexpr int NG = P <= 2 ? 8 : P == 3 ? 6 : 1;              // groups per CTA
    static constexpr int W = NG * G;                                    // warps per CTA
    static constexpr int NS = 2;                                        // pipeline stages per group
    static constexpr size_t KB = ((size_t)LPS * 8 + 127) / 128 * 128;   // packed matrix buffer
    static constexpr size_t UB = ((size_t)L * 8 + 127) / 128 * 128;     // u_e buffer
    static constexpr size_t PER_GROUP = NS * (KB + UB);
    static constexpr size_t OFF_BAR = NG * PER_GROUP;
    static constexpr size_t SMEM = OFF_BAR + NG * NS * 8;
};

__device__ __forceinline__ void cp_async8_g(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int P>
__global__ void __launch_bounds__(CutPre<P>::W * 32) k_cut_pre(int64_t n_cut, const double* __restrict__ KP,
                                                               const int64_t* __restrict__ cut_base, int64_t pplane,
                                                               int64_t prow, const double* __restrict__ u,
                                                               double* __restrict__ out) {
    using C = CutPre<P>;
    constexpr int N = C::N, L = C::L, G = C::G, NS = C::NS;
    extern __shared__ __align__(128) unsigned char smc[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int grp = w / G, sub = w % G;           // group and warp within the group
    const int gt = sub * 32 + lane;               // thread within the group
    unsigned char* mine = smc + (size_t)grp * C::PER_GROUP;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smc + C::OFF_BAR) + NS * grp;
    const int64_t stride = (int64_t)gridDim.x * C::NG;
    const int64_t e0 = (int64_t)blockIdx.x * C::NG + grp;
    auto gsync = [&]() {   // the group's warps
        if (G == 1) __syncwarp();
        else asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(G * 32) : "memory");
    };
    if (gt == 0) {
        #pragma unroll
        for (int q = 0; q < NS; ++q) mbar_init(&bar[q], 1);
    }
    gsync();
    auto fetch = [&](int64_t e, int buf) {   // K_o by bulk copy, u_e by cp.async
        double* kp = reinterpret_cast<double*>(mine + buf * (C::KB + C::UB));
        double* uu = reinterpret_cast<double*>(mine + buf * (C::KB + C::UB) + C::KB);
        if (gt == 0) {
            mbar_expect_tx(&bar[buf], (uint32_t)(C::LPS * 8));
            bulk_load(kp, KP + e * C::LPS, (uint32_t)(C::LPS * 8), &bar[buf]);
        }
        const int64_t base = cut_base[e];
        for (int m = gt; m < L; m += G * 32) {
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
        gsync();   // every thread's u_e gather of this cell is visible
        mbar_wait(&bar[buf], (uint32_t)((it / NS) & 1));
        const double* kp = reinterpret_cast<const double*>(mine + buf * (C::KB + C::UB));
        const double* uu = reinterpret_cast<const double*>(mine + buf * (C::KB + C::UB) + C::KB);
        for (int r = gt; r < L; r += G * 32) {
            // row r in ascending column order from the packed lower triangle:
            // (r, m) for m <= r, (m, r) below the diagonal.  One loop for both
            // parts (the lanes of a warp switch at different m: two loops
            // diverged for half of the columns); column indices are constants.
            double t = 0.0;
            const int tr = r * (r + 1) / 2;
            #pragma unroll
            for (int m = 0; m < L; ++m) {
                const int idx = m <= r ? tr + m : m * (m + 1) / 2 + r;
                t = fma(kp[idx], uu[m], t);
            }
            out[e * L + r] = t;
        }
        gsync();   // buffer reused NS cells later
    }
}

template <int P>
void launch_cut_pre(Context* ctx, int64_t n_cut, const double* KP, const int64_t* cut_base,
                    int64_t pplane, int64_t prow, const double* u, double* out) {
    if (!n_cut) return;
    using C = CutPre<P>;
    ensure_smem_attr((const void*)k_cut_pre<P>, ctx->device, (size_t)C::SMEM);
    const int64_t blocks = std::min<int64_t>(ceil_div(n_cut, C::NG), (int64_t)ctx->sm_count * std::max<int64_t>(1, (int64_t)(220 * 1024 / C::SMEM)));
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
//
// No block barrier inside the x loop: the warps run loosely coupled through
// mbarriers (ncu on the barrier version: 17 % barrier stalls, every warp
// waiting for the slowest three times per row) --
//   full[s]    TMA ring slot s landed
//   rowdone    every compute warp is past cell row t (epilogue included)
//   pbar       the halo/producer warp's per-row post: after rowdone(t-1) it
//              stores the cell codes of row t+1 (loaded during its row t) into
//              the shared code buffer, refills row t-1's ring slots and fetches
//              psi_{k-1} of row t; compute warps wait on it before their epilogue
//   xfull[w] / xempty[w]   the shared y node row of warp w (YP) handed to the
//              warp below it, single buffer with a full/empty handshake
// `live` and `reuse` are warp-level votes (both only skip work whose result
// is identical).  The P+1 planes of a row run through one rolled loop (x pass
// factors from shared memory): unrolled, the kernel was 83 KB of code and
// ncu showed 11 % instruction-fetch stalls.  Epilogue, one x plane (P x P nodes per thread) at a time:
// every load of the plane is issued before its arithmetic; 1/m comes from the
// interior table (class 1 cells), is 0 without a load (1/m == 0 on every owned
// node: class 2, slots that are no DOFs under a diagonal-mass CDM plan and are
// left untouched; class 3, the implicit rows of an IMEX / consistent-mass plan,
// whose slots still receive 2 psi_k - psi_{k-1}) or is loaded (class 0,
// prefetched into L2 at row start).
template <int P, int MODE>
__global__ void __launch_bounds__(Str3<P>::NWARP * 32, cpsm_for3(P))
    k_scm3d(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_p, Scm3DGeo g,
            Mats2<P> mt, MinvTab<P> mtab, double sk, StepArgs a) {
    using T = Str3<P>;
    constexpr int N = P + 1;
    constexpr int WY = T::WY;
    constexpr int S = T::S;
    constexpr int CW = T::CODE_W;
    constexpr unsigned FULL = 0xffffffffu;
    constexpr bool LATE_REFILL = S >= 2 * P + 1;   // the ring holds two full cell rows
    constexpr int EB = P <= 3 ? P : 1;             // node rows per batch of epilogue loads
    extern __shared__ __align__(128) unsigned char smem[];
    const double* ring = reinterpret_cast<const double*>(smem);
    double* xch = reinterpret_cast<double*>(smem + T::OFF_XCH);   // [NWARP][N*P][32]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
    uint64_t* pbar = full + S;
    uint64_t* rowdone = pbar + 1;
    uint64_t* xfull = rowdone + 1;
    uint64_t* xempty = xfull + T::NWARP;
    const double* prv = reinterpret_cast<const double*>(smem + T::OFF_PREV);   // [P][WY*P][TZ]
    double* stab = reinterpret_cast<double*>(smem + T::OFF_TAB);
    uint8_t* cbuf = smem + T::OFF_CODE;                                    // [2][WY+1][CW]
    double* xtab = reinterpret_cast<double*>(smem + T::OFF_XTAB);          // [c][k1[.][c] | m1[.][c]]
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
    const int trow = (halo ? 0 : w + 1) * P;                             // tile row of node row ey*P
    const int64_t s_ = g.n_e + 2;
    auto issue = [&](int lp) {   // streamed plane lp (global plane G0 + lp) -> its ring slot
        const int s = lp % S;
        mbar_expect_tx(&full[s], (uint32_t)(T::PLANE * 8));
        tma_load_3d(smem + (size_t)s * T::SLOT * 8, &tm_u, (int32_t)(K0 - P - T::CO + PADJ),
                    (int32_t)(ey0 * P), (int32_t)(G0 + lp + P), &full[s]);
    };
    // Cell codes of one x cell row for the whole CTA: rows ey0-1 .. ey0+WY-1,
    // cells ez0-1 .. ez0+31 (ring coordinates: +1), one byte each (bits 0-1:
    // 0 out, 1 uncut, 2 cut; bits 2-3: 1/m class).  Loaded by the halo warp:
    // lane l takes column l of every row, lanes 0..WY the last column.
    uint32_t hc[WY + 2];
    const int64_t ez0 = K0 / P;
    auto load_codes = [&](int64_t ex) {
        const bool in = ex >= 0 && ex < g.n_ex;
        const uint8_t* base = g.mask + ((ex + 1) * s_ + ey0) * s_ + ez0;    // (ex, ey0-1, ez0-1)
        #pragma unroll
        for (int q = 0; q <= WY; ++q) {
            hc[q] = 0;
            if (in && ey0 + q < s_ && ez0 + lane < s_) hc[q] = __ldg(base + q * s_ + lane);
        }
        hc[WY + 1] = 0;
        if (in && lane <= WY && ey0 + lane < s_ && ez0 + 32 < s_) hc[WY + 1] = __ldg(base + lane * s_ + 32);
    };
    auto store_codes = [&](int buf) {
        uint8_t* c = cbuf + buf * (WY + 1) * CW;
        #pragma unroll
        for (int q = 0; q <= WY; ++q) c[q * CW + lane] = (uint8_t)hc[q];
        if (lane <= WY) c[lane * CW + 32] = (uint8_t)hc[WY + 1];
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
    if (threadIdx.x < P * P * P) stab[threadIdx.x] = mtab.v[threadIdx.x];
    if (threadIdx.x == 32) {
        #pragma unroll
        for (int c = 0; c < N; ++c)
            #pragma unroll
            for (int r = 0; r < N; ++r) {
                xtab[(c * 2 + 0) * N + r] = mt.k[orb(P, r, c)];
                xtab[(c * 2 + 1) * N + r] = mt.m[orb(P, r, c)];
            }
    }
    if (halo) {
        load_codes(exA - 1);
        store_codes(0);
    }
    __syncthreads();
    if (halo && lane == 0)
        for (int lp = 0; lp < nplanes && lp < S; ++lp) issue(lp);
    double mc[orb_count(P)], kc[orb_count(P)];
    #pragma unroll
    for (int i = 0; i < orb_count(P); ++i) { mc[i] = mt.m[i]; kc[i] = mt.k[i]; }
    const double f = (MODE == MODE_STEP) ? __ldg(a.ft + a.k) : 0.0;
    const double f0 = f * 0.0;
    const int up = w == 0 ? WY : w - 1;              // exchange source warp (compute warps)
    const bool sends = halo || w < WY - 1;           // the last compute warp's row P belongs to the next block
    double* const xw = xch + (size_t)w * N * P * 32 + lane;
    const double* const xr = xch + (size_t)up * N * P * 32 + lane;
    const int crow = halo ? 0 : w + 1;               // this warp's row of the code buffer
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
    int t = 0;                                        // row index within the chunk
    // halo warp, once per row: codes of row t+1 -> shared, ring refill, psi_{k-1}
    auto post = [&](int64_t ex) {
        if (t > 0) mbar_wait(rowdone, (uint32_t)((t - 1) & 1));
        store_codes((t + 1) & 1);
        __syncwarp();
        if (lane == 0) {
            if (t > 0) {
                #pragma unroll 1
                for (int q = 0; q < P; ++q) {
                    const int lp = (t - 1) * P + q + S;
                    if (lp < nplanes) issue(lp);
                }
            }
            if (MODE == MODE_STEP && t > 0) {
                mbar_expect_tx(pbar, (uint32_t)T::PREV_BYTES);
                tma_load_3d(smem + T::OFF_PREV, &tm_p, (int32_t)(K0 + PADJ), (int32_t)(ey0 * P + P),
                            (int32_t)(ex * P + P), pbar);
            } else {
                mbar_arrive(pbar);
            }
        }
        __syncwarp();
    };
    for (int64_t ex = exA - 1; ex < exE; ++ex, ++t) {
        const uint8_t* crw = cbuf + ((t & 1) * (WY + 1) + crow) * CW + lane;
        const uint32_t bRR = crw[1];
        const uint32_t cRR = bRR & 3, cRL = crw[0] & 3;
        const uint32_t cUR = halo ? 0u : (crw[1 - CW] & 3u), cUL = halo ? 0u : (crw[-CW] & 3u);
        const uint32_t cls = (MODE == MODE_STEP) ? (bRR >> 2) : 0u;
        if (halo) {
            load_codes(ex + 1 < exE ? ex + 1 : -1);
            if (!LATE_REFILL) post(ex);
        }
        const int64_t Kl = K0 + lane * P;
        const int64_t base0 = (ex * P + P) * g.pplane + (ey * P + P) * g.prow + Kl + PADJ;
        if (MODE == MODE_STEP && !halo && t > 0 && cls == 0) {
            // 1/m of this cell is loaded in the epilogue: start it towards L2 now
            #pragma unroll
            for (int r = 0; r < P; ++r)
                #pragma unroll
                for (int b = 0; b < P; ++b) {
                    const double* q = a.minv + base0 + r * g.pplane + b * g.prow;
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(q + P - 1));
                }
        }
        const double xRR = cRR == 1, xRL = cRL == 1;
        const bool live = __any_sync(FULL, (cRR | cRL) != 0);
#if WCB3D_REUSE
        const bool reuse = t > 0 && !__any_sync(FULL, (cRR == 1) != pxRR || (cRL == 1) != pxRL);
#else
        const bool reuse = false;
#endif
        pxRR = cRR == 1;
        pxRL = cRL == 1;
        // the planes of the row in a rolled loop (one copy of the y/z
        // contraction in the instruction cache); x pass factors of plane c
        // from shared memory
        #pragma unroll
        for (int r = 0; r < N; ++r)
            #pragma unroll
            for (int j = 0; j < P; ++j) YP[r][j] = 0.0;
        if (!halo) {
            #pragma unroll
            for (int r = 1; r < N; ++r)
                #pragma unroll
                for (int b = 0; b < P; ++b)
                    #pragma unroll
                    for (int j = 0; j < P; ++j) Y[r][b][j] = 0.0;
        }
        #pragma unroll 1
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
            const double* xt = xtab + c * 2 * N;
            #pragma unroll
            for (int r = 0; r < N; ++r) {
                const double xk = xt[r], xm = xt[N + r];
                #pragma unroll
                for (int j = 0; j < P; ++j) YP[r][j] = fma(xk, Au[P][j], fma(xm, Bu[P][j], YP[r][j]));
                if (!halo) {
                    #pragma unroll
                    for (int b = 0; b < P; ++b)
                        #pragma unroll
                        for (int j = 0; j < P; ++j) Y[r][b][j] = fma(xk, Au[b][j], fma(xm, Bu[b][j], Y[r][b][j]));
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
        // with a two-row ring the halo warp posts after its own row, so that warp 0
        // never waits for the shared node row behind the row-done wait
        if (LATE_REFILL && halo) post(ex);
        if (!halo) {
            mbar_wait(&xfull[up], (uint32_t)(t & 1));
            #pragma unroll
            for (int r = 0; r < N; ++r)
                #pragma unroll
                for (int j = 0; j < P; ++j) Y[r][0][j] += xr[(r * P + j) * 32];
            mbar_arrive(&xempty[up]);
            // dense cut cells: own y row (ey) and the y-up row (ey-1)
            const unsigned clR = __ballot_sync(FULL, cRR == 2);
            const bool edR = __shfl_sync(FULL, cRL == 2, 0);
            if (clR || edR) cut_cells_warp3<P>(g, ex, ey, K0 / P, lane, clR, edR, false, Y);
            const unsigned clU = __ballot_sync(FULL, cUR == 2);
            const bool edU = __shfl_sync(FULL, cUL == 2, 0);
            if (clU || edU) cut_cells_warp3<P>(g, ex, ey - 1, K0 / P, lane, clU, edU, true, Y);
            mbar_wait(pbar, (uint32_t)(t & 1));   // codes of row t+1 visible, psi_{k-1} of row t landed
            if (t > 0) {
                if constexpr (MODE == MODE_APPLY) {
                    #pragma unroll
                    for (int r = 0; r < P; ++r) {
                        if (ex * P + r >= g.row_hi) break;
                        #pragma unroll
                        for (int b = 0; b < P; ++b) {
                            if (ey * P + b >= g.n1) break;
                            #pragma unroll
                            for (int j = 0; j < P; ++j)
                                if (Kl + j < g.n1) a.out[base0 + r * g.pplane + b * g.prow + j] = sk * Y[r][b][j];
                        }
                    }
                } else if (!__all_sync(FULL, cls == 2)) {
                    const int64_t baseL = base0 + (P - 1) * (g.pplane + g.prow) + (P - 1);
                    const bool anysrc = !(baseL < a.F.lo || base0 > a.F.hi);
                    const double* up0 = prv + (size_t)(w * P) * T::TZ + lane * P;
                    const int u0 = trow * T::UW + T::CO + P + lane * P;
                    bool kin[P];
                    #pragma unroll
                    for (int j = 0; j < P; ++j) kin[j] = Kl + j < g.n1;
                    #pragma unroll
                    for (int r = 0; r < P; ++r) {
                        const bool okr = ex * P + r < g.row_hi && cls != 2;
                        const double* pl = ring + (size_t)((t * P + r) % S) * T::SLOT + u0;
                        const int64_t baser = base0 + r * g.pplane;
                        #pragma unroll
                        for (int b0 = 0; b0 < P; b0 += EB) {   // EB node rows per batch of loads
                            double mi[EB][P], uu[EB][P], pp[EB][P], fF[EB][P];
                            #pragma unroll
                            for (int bb = 0; bb < EB; ++bb) {
                                const int b = b0 + bb;
                                const bool okb = okr && ey * P + b < g.n1;
                                #pragma unroll
                                for (int j = 0; j < P; ++j) {
                                    mi[bb][j] = cls == 1 ? stab[(r * P + b) * P + j] : 0.0;
                                    if (cls == 0 && okb && kin[j]) mi[bb][j] = __ldg(a.minv + baser + b * g.prow + j);
                                    uu[bb][j] = pl[b * T::UW + j];
                                    pp[bb][j] = up0[((size_t)r * WY * P + b) * T::TZ + j];
                                    fF[bb][j] = f0;
                                }
                            }
                            if (anysrc) {   // rare: a source node in this cell's index range
                                #pragma unroll
                                for (int bb = 0; bb < EB; ++bb)
                                    #pragma unroll
                                    for (int j = 0; j < P; ++j)
                                        fF[bb][j] = f * source_at(a.F, baser + (b0 + bb) * g.prow + j);
                            }
                            #pragma unroll
                            for (int bb = 0; bb < EB; ++bb) {
                                const int b = b0 + bb;
                                const bool okb = okr && ey * P + b < g.n1;
                                #pragma unroll
                                for (int j = 0; j < P; ++j) {
                                    const double v = leapfrog(uu[bb][j], pp[bb][j], sk * Y[r][b][j], mi[bb][j], fF[bb][j], a.dt2);
                                    if (okb && kin[j]) a.out[baser + b * g.prow + j] = v;
                                    const unsigned long long bits = mi[bb][j] != 0.0 ? amp_bits(v) : 0ULL;
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
                for (int j = 0; j < P; ++j) Y[0][b][j] = Y[P][b][j];
            // one arrival per warp and phase: the ring holds two cell rows, so
            // a warp could otherwise finish row t+1 (and arrive twice) before
            // a slower warp has arrived for row t
            if (t > 0) mbar_wait(rowdone, (uint32_t)((t - 1) & 1));
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

// four threads per node, one per adjacent cell (ex, ey, n_e-1); lane 0 of the
// quad adds the contributions in the fixed order (ex-1, ey-1), (ex-1, ey),
// (ex, ey-1), (ex, ey) and runs the epilogue
template <int P, int MODE>
__global__ void __launch_bounds__(128) k_scm3d_zcol(Scm3DGeo g, Mats2<P> mt, double sk, const double2* __restrict__ zl,
                                                   StepArgs a) {
    constexpr int N = P + 1;
    const int64_t t4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t t = t4 >> 2;
    const int q4 = (int)(t4 & 3);
    const int64_t n_pl = g.row_hi - g.row_lo;
    const bool node = t < n_pl * g.n1;
    const int64_t I = g.row_lo + (node ? t / g.n1 : 0), J = node ? t % g.n1 : 0, K = g.n1 - 1;
    const int64_t s_ = g.n_e + 2;
    double s = 0.0;
    bool has = false;
    if (node) {
        const int dx = 1 - (q4 >> 1), dy = 1 - (q4 & 1);
        const int64_t ex = I / P - dx, ey = J / P - dy;
        const int ia = (int)(I - ex * P), ib = (int)(J - ey * P);
        if (ex >= 0 && ex < g.n_ex && ia <= P && ey >= 0 && ey < g.n_e && ib <= P) {
            const int64_t ez = g.n_e - 1;
            const uint8_t code = g.mask[((ex + 1) * s_ + (ey + 1)) * s_ + ez + 1] & 3;
            if (code == 1) {
                has = true;
                double2 z[N][N];
                #pragma unroll
                for (int q = 0; q < N; ++q)
                    #pragma unroll
                    for (int r = 0; r < N; ++r) z[q][r] = zl[(ex * P + q) * g.n1 + ey * P + r];
                double mq[N], kq[N], mr[N], kr[N];
                #pragma unroll
                for (int q = 0; q < N; ++q) {   // ia, ib are runtime: select the factor rows
                    mq[q] = kq[q] = mr[q] = kr[q] = 0.0;
                    #pragma unroll
                    for (int i = 0; i < N; ++i) {
                        if (i == ia) { mq[q] = mt.m[orb(P, i, q)]; kq[q] = mt.k[orb(P, i, q)]; }
                        if (i == ib) { mr[q] = mt.m[orb(P, i, q)]; kr[q] = mt.k[orb(P, i, q)]; }
                    }
                }
                #pragma unroll
                for (int q = 0; q < N; ++q)
                    #pragma unroll
                    for (int r = 0; r < N; ++r)
                        s = fma(kq[q] * mr[r] + mq[q] * kr[r], z[q][r].x, fma(mq[q] * mr[r], z[q][r].y, s));
            } else if (code == 2) {
                has = true;
                const int32_t id = g.cut_id[(ex * g.n_e + ey) * g.n_e + ez];
                s = g.cut_out[(int64_t)id * N * N * N + (ia * N + ib) * N + P];
            }
        }
    }
    double acc = 0.0;
    const int qb = (threadIdx.x & 31) & ~3;
    #pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
        const double v = __shfl_sync(0xffffffffu, s, qb + qq);
        const bool h = __shfl_sync(0xffffffffu, has ? 1 : 0, qb + qq) != 0;
        if (h) acc += v;
    }
    unsigned long long amp = 0ULL;
    if (node && q4 == 0) {
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

// 1/m class of every local cell c: 1 when every owned node carries the
// interior table's 1/m (bitwise), 2 or 3 when 1/m == +0 on all of them (the step
// does not load 1/m there; 2: it does not store either), else 0.  The
// class goes into bits 2-3 of the cell's code byte (cinfo = mask | cls << 2).
template <int P>
__global__ void k_clean3d(Scm3DGeo g, MinvTab<P> tab, const double* __restrict__ minv, uint8_t* clean,
                          uint8_t* cinfo, bool zero_is_dead) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nc = g.n_ex * g.n_e * g.n_e;
    if (c >= nc) return;
    const int64_t ex = c / (g.n_e * g.n_e), ey = (c / g.n_e) % g.n_e, ez = c % g.n_e;
    bool ok = ex >= 1, zero = true;
    for (int q = 0; q < P; ++q)
        for (int r = 0; r < P; ++r)
            for (int j = 0; j < P; ++j) {
                const int64_t I = ex * P + q;
                const int64_t s = (I + P) * g.pplane + (ey * P + r + P) * g.prow + ez * P + j + PADJ;
                const long long bits = __double_as_longlong(minv[s]);
                ok = ok && I < g.row_hi && bits == __double_as_longlong(tab.v[(q * P + r) * P + j]);
                zero = zero && bits == 0LL;
            }
    const uint8_t cls = ok ? 1 : zero ? (zero_is_dead ? 2 : 3) : 0;
    clean[c] = cls;
    const int64_t s_ = g.n_e + 2;
    const int64_t m = ((ex + 1) * s_ + (ey + 1)) * s_ + ez + 1;
    cinfo[m] = (uint8_t)((g.mask[m] & 3) | (cls << 2));
}

template <int P>
void launch_clean3d(Context* ctx, const Scm3DGeo& g, const MinvTab<P>& tab, const double* minv, uint8_t* clean,
                    uint8_t* cinfo, bool zero_is_dead) {
    const int64_t nc = g.n_ex * g.n_e * g.n_e;
    k_clean3d<P><<<(unsigned)ceil_div(nc, 256), 256, 0, ctx->stream>>>(g, tab, minv, clean, cinfo, zero_is_dead);
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
        ensure_smem_attr((const void*)k_scm3d<P, MODE>, ctx->device, (size_t)T::SMEM);
        k_scm3d<P, MODE><<<grid, T::NWARP * 32, T::SMEM, ctx->stream>>>(map_u, map_p, g, mt, mtab, sk, a);
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
        k_scm3d_zcol<P, MODE><<<(unsigned)ceil_div(4 * nn, 128), 128, 0, ctx->stream>>>(g, mt, sk, g.zline, a0);
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
    template void launch_clean3d<P>(Context*, const Scm3DGeo&, const MinvTab<P>&, const double*, uint8_t*, uint8_t*, bool);
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
