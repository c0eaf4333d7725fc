// Implicit-explicit split integration on the device: imex_run,
// src/timeint.py:196-292 (Algorithm 2).
//
// Per step k (all on the device, stream-ordered):
//   1. fused explicit step of the operator on every node (d rows get
//      psi_d^{k+1} = 2 psi - psi_prev + dt^2 (f(t_k) F - K psi)/m_d, src :261-269;
//      c slots carry 1/m = 0 and are overwritten next);
//   2. c predictor psi_c^pred = psi_c + dt v_c + dt^2/2 (1-2beta) a_c, written
//      into the new state (src :271-274);
//   3. rhs_c = f(t_k + dt) F_c - (K psi_mixed)_c (src :275) -- K applied to the
//      c rows only where the operator supports it;
//   4. a_c = S_cc^-1 rhs_c with S_cc = M_cc + beta dt^2 K_cc prefactorised on
//      the host (SuperLU, the reference's factorize(), src/linalg.py:70-80):
//      row permutation, forward solve with L, backward solve with U, column
//      permutation (src :278);
//   5. corrector psi_c = pred + beta dt^2 a_c, v_c = v_pred + gamma dt a_c,
//      and max|psi_c| into the divergence slot (src :279-282).
// The triangular solves are synchronisation-free: warps take rows in
// elimination order from an atomic counter, wait (acquire) for the rows they
// depend on, sum in a fixed lane order and publish (release) their row -- one
// launch per solve, deterministic results.
#include "wcb_internal.cuh"
#include "wcb_tma.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>

namespace wcb {

// Level schedule of a triangular factor split by connected component: the
// c-set of an immersed grid is a union of independent patches (one ring of cut
// cells per void), and SuperLU keeps them independent, so every component is
// solved by one CTA with its unknowns in shared memory and one barrier per
// elimination level -- instead of a device-wide chain of global-memory
// handshakes.  Entries of a row are visited in the same lane-strided order and
// reduced by the same shuffle tree as the sync-free kernel (bitwise equal).
#ifndef WCB_TRSV_GW
#define WCB_TRSV_GW 16
#endif
#ifndef WCB_TRSV_STAGE_LATE
#define WCB_TRSV_STAGE_LATE 1
#endif
constexpr int TRSV_DMAX = 12;
static __host__ __device__ inline size_t trsv_slot_bytes(int e, int r);             // max ring depth (levels in flight)
constexpr int TRSV_SMEM = 220 * 1024;     // dynamic shared memory budget
constexpr int TRSV_THREADS = 1024;     // launch bound
constexpr int TRSV_THREADS_DEF = 768;  // measured: 256 2770, 384 2485, 512 2329, 768 2253, 1024 2295 us per config-4 step

struct TriSched {
    bool ok = false;
    int64_t n_comp = 0, max_size = 0, n_levels = 0, max_levels = 0;
    int64_t max_lvl_rows = 0, max_lvl_ent = 0;   // widest level
    int slot_e = 0, slot_r = 0;                  // ring slot capacities (entries, rows)
    int depth = 3;                               // ring depth (levels in flight)
    bool recip = false;                          // sdiag holds 1/diag
    bool pf_ok = false;                          // k_trsv_pf fits (unknowns + level offsets in smem)
    // k_trsv_ring: every level (split into pieces of <= PIECE_BYTES) packed as
    // one 16-byte aligned segment [hdr | row ptrs | pivots | values | column
    // slots], streamed by one producer warp into a shared-memory ring
    bool ring_ok = false;
    int ring_depth = 0;
    int64_t max_pieces = 0;
    DevBuf<unsigned char> blob;
    DevBuf<int64_t> piece_off;   // byte offset of each piece's segment
    DevBuf<int32_t> piece_bytes;
    DevBuf<int32_t> comp_piece;  // n_comp + 1: offsets into the pieces
    DevBuf<int32_t> comp_order;  // launch order: components by decreasing level count
    DevBuf<int32_t> ring_order;  // launch order of k_trsv_ring: by decreasing streamed bytes
    DevBuf<int32_t> comp_rows;   // n_comp + 1: offsets into rows
    DevBuf<int32_t> comp_lvl;    // n_comp + 1: offsets into lvl_off
    DevBuf<int32_t> lvl_off;     // n_levels + 1: offsets into rows
    DevBuf<int32_t> lvl_ent;     // n_levels + 1: offsets into the packed entries
    DevBuf<int32_t> rows;        // n: row ids grouped by component, then level
    DevBuf<int32_t> pos;         // n: local slot of each row in its component
    // off-diagonal entries packed in schedule order (a level's rows are
    // contiguous, so the next level can be prefetched with coalesced loads)
    DevBuf<int32_t> sptr;        // n + 1
    DevBuf<int32_t> slcol;       // local slot of the column
    DevBuf<double> sval;
    DevBuf<double> sdiag;        // n, schedule order
    size_t smem_bytes() const;
};

__device__ __forceinline__ uint32_t smem_u32_imex(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

static int64_t uf_find(std::vector<int64_t>& p, int64_t a) {
    while (p[a] != a) { p[a] = p[p[a]]; a = p[a]; }
    return a;
}

// components of the union of both factors' patterns
static std::vector<int64_t> factor_components(int64_t n, const wcb_lu* lu, int64_t* n_comp) {
    std::vector<int64_t> par(n);
    for (int64_t i = 0; i < n; ++i) par[i] = i;
    for (int f = 0; f < 2; ++f) {
        const int64_t* ptr = f ? lu->U_indptr : lu->L_indptr;
        const int32_t* idx = f ? lu->U_indices : lu->L_indices;
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = ptr[i]; j < ptr[i + 1]; ++j) {
                const int64_t a = uf_find(par, i), b = uf_find(par, idx[j]);
                if (a != b) par[std::max(a, b)] = std::min(a, b);
            }
    }
    std::vector<int64_t> comp(n), label(n, -1);
    int64_t nc = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t r = uf_find(par, i);
        if (label[r] < 0) label[r] = nc++;
        comp[i] = label[r];
    }
    *n_comp = nc;
    return comp;
}

// Segment layout of one piece (every offset a multiple of 16 bytes):
// int32 hdr[8] = {nrow, k0, ne, bytes, kind, gbase, 0, 0}, then
//   kind 0 (rows [k0, k0+nrow) of one level): int32 rptr[nrow+1] (entry offsets
//     within the piece); double pivot[nrow]; double val[ne]; int32 col[ne]:
//     x_k = (x_k - sum val x_col) * pivot
//   kind 1 (rows of a group of narrow levels, entries outside the group only):
//     same arrays; t[k0 + k - gbase] = x_k - sum val x_col (scratch, no pivot)
//   kind 2 (the group's dense part): double W[nrow (nrow+1) / 2], the packed
//     rows of inv(T), T the group's triangular block with its diagonal:
//     x_k = sum_{j <= k} W[k][j] t[j]
// The whole piece is one bulk copy.
//
// Groups: the factors' dependency chains end in long runs of levels holding
// one or two rows (the dense trailing triangle of a patch: on config 4 the
// longest patch has 454 levels, the last 230 of one row each, 130-250 entries
// per row), where the level-scheduled solve pays one consumer barrier and one
// serial dot product per row.  A run of consecutive levels of at most
// TRSV_NARROW rows each (up to TRSV_GMAX rows in total) is solved in two
// parallel steps instead: the entries outside the run for all its rows at
// once (kind 1), then the multiplication by the host-inverted triangular block
// (kind 2).  Mathematically the same solve; the rounding differs (bounded by
// the parity tests).  WAVECELL_B200_TRSV_GROUPS=0 keeps one piece per level.
// largest piece (bulk copy); WAVECELL_B200_TRSV_PIECE_KB overrides (measured on
// config 4: 40 KB pieces in a 160 KB ring beat 24-32 KB pieces in 48-64 KB)
static int64_t trsv_piece_bytes() {
    static const int64_t v = [] {
        const char* e = getenv("WAVECELL_B200_TRSV_PIECE_KB");
        const int64_t kb = e ? atoll(e) : 40;
        return std::max<int64_t>(20, std::min<int64_t>(kb, 64)) * 1024;   // >= the dense part of a group
    }();
    return v;
}
#define TRSV_PIECE_BYTES trsv_piece_bytes()
static int64_t trsv_ring_cap() {   // cap of the circular piece buffer (WAVECELL_B200_TRSV_RING_KB)
    static const int64_t v = [] {
        const char* e = getenv("WAVECELL_B200_TRSV_RING_KB");
        const int64_t kb = e ? atoll(e) : 160;
        return std::max<int64_t>(40, std::min<int64_t>(kb, 160)) * 1024;
    }();
    return v;
}
constexpr int TRSV_GMAX = 64;      // rows per group (dense part: 16.6 KB)
constexpr int TRSV_NARROW = 16;    // a level joins a group when it has at most this many rows
constexpr int TRSV_HDR = 32;
static inline int64_t pad16(int64_t b) { return (b + 15) / 16 * 16; }
static inline int64_t piece_size(int64_t nrow, int64_t ne) {
    return TRSV_HDR + pad16(4 * (nrow + 1)) + pad16(8 * nrow) + pad16(8 * ne) + pad16(4 * ne);
}
static void pack_pieces(TriSched& T, int64_t n, const std::vector<int32_t>& comp_rows,
                        const std::vector<int32_t>& comp_lvl, const std::vector<int32_t>& lvl_off,
                        const std::vector<int32_t>& sptr, const std::vector<double>& sdiag,
                        const std::vector<double>& tdiag, const std::vector<double>& sval,
                        const std::vector<int32_t>& slcol, cudaStream_t s) {
    std::vector<int64_t> off;
    std::vector<int32_t> bytes, cpiece(T.n_comp + 1, 0);
    std::vector<unsigned char> blob;
    int64_t maxp = 0;
    bool ok = true;
    const bool groups = !(getenv("WAVECELL_B200_TRSV_GROUPS") && getenv("WAVECELL_B200_TRSV_GROUPS")[0] == '0');
    // rows [k, e) (schedule order) as pieces of `kind`; entries with a column
    // slot >= slot_lo are skipped (kind 1: they are in the dense part)
    // consumer warps of k_trsv_ring (rows of a piece get a whole warp when there are few)
    const int ncw = [] { const char* e2 = getenv("WAVECELL_B200_TRSV_NC"); return e2 && atoi(e2) > 0 ? atoi(e2) : 16; }();
    // lanes per row of a piece: fewest (passes over the row groups) x (latency
    // of one pass), a pass costing a fixed part, the row's multiply-add steps
    // (two per lane in flight) and the shuffle tree
    auto lanes_for = [&](int64_t nrow, int64_t ne) {
        const double per_row = nrow > 0 ? (double)ne / (double)nrow : 0.0;
        int best = 16;
        double best_cost = 1e300;
        for (int gw : {2, 4, 8, 16, 32}) {
            const int64_t groups = (int64_t)ncw * 32 / gw;
            const double passes = (double)((nrow + groups - 1) / groups);
            int lg = 0;
            while ((1 << lg) < gw) ++lg;
            const double iters = std::ceil(per_row / (2.0 * gw));
            const double cost = passes * (300.0 + 80.0 * iters + 30.0 * lg);
            if (cost < best_cost) { best_cost = cost; best = gw; }
        }
        return best;
    };
    auto emit_rows = [&](int64_t k, int64_t e, int kind, int64_t gbase, int64_t slot_lo) {
        std::vector<int32_t> cnt;   // kept entries per row
        cnt.reserve(e - k);
        for (int64_t r = k; r < e; ++r) {
            int32_t c = 0;
            for (int32_t j = sptr[r]; j < sptr[r + 1]; ++j) c += slcol[j] < slot_lo;
            cnt.push_back(c);
        }
        int64_t r0 = k;
        while (r0 < e && ok) {
            int64_t r1 = r0, ne = 0;
            if (piece_size(1, cnt[r0 - k]) > TRSV_PIECE_BYTES) { ok = false; break; }
            while (r1 < e && piece_size(r1 + 1 - r0, ne + cnt[r1 - k]) <= TRSV_PIECE_BYTES) { ne += cnt[r1 - k]; ++r1; }
            const int64_t nrow = r1 - r0;
            const int64_t sz = piece_size(nrow, ne);
            const int64_t base = (int64_t)blob.size();
            blob.resize(base + sz, 0);
            unsigned char* p = blob.data() + base;
            int32_t* hdr = reinterpret_cast<int32_t*>(p);
            hdr[0] = (int32_t)nrow;
            hdr[1] = (int32_t)r0;
            hdr[2] = (int32_t)ne;
            hdr[3] = (int32_t)sz;
            hdr[4] = kind;
            hdr[5] = (int32_t)gbase;
            hdr[6] = lanes_for(nrow, ne);        // lanes per row
            hdr[7] = r1 == e ? 1 : 0;            // last piece of its level / outside part: consumers meet
            int32_t* rp = reinterpret_cast<int32_t*>(p + TRSV_HDR);
            double* dg = reinterpret_cast<double*>(p + TRSV_HDR + pad16(4 * (nrow + 1)));
            double* vv = dg + pad16(8 * nrow) / 8;
            int32_t* cc = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(vv) + pad16(8 * ne));
            int32_t at = 0;
            for (int64_t q = 0; q < nrow; ++q) {
                rp[q] = at;
                dg[q] = sdiag[r0 + q];
                for (int32_t j = sptr[r0 + q]; j < sptr[r0 + q + 1]; ++j)
                    if (slcol[j] < slot_lo) { vv[at] = sval[j]; cc[at] = slcol[j]; ++at; }
            }
            rp[nrow] = at;
            off.push_back(base);
            bytes.push_back((int32_t)sz);
            r0 = r1;
        }
    };
    for (int64_t c = 0; c < T.n_comp && ok; ++c) {
        cpiece[c] = (int32_t)off.size();
        const int64_t start = comp_rows[c];
        int32_t l = comp_lvl[c];
        const int32_t lend = comp_lvl[c + 1];
        while (l < lend && ok) {
            // a run of narrow levels?
            int32_t l2 = l;
            int64_t tot = 0;
            while (groups && l2 < lend && lvl_off[l2 + 1] - lvl_off[l2] <= TRSV_NARROW &&
                   tot + (lvl_off[l2 + 1] - lvl_off[l2]) <= TRSV_GMAX) {
                tot += lvl_off[l2 + 1] - lvl_off[l2];
                ++l2;
            }
            if (l2 - l >= 2) {
                const int64_t ka = lvl_off[l], kb = lvl_off[l2], nr = kb - ka;
                const int64_t slot_lo = ka - start;   // first local slot of the group
                emit_rows(ka, kb, 1, ka, slot_lo);
                // T = the group's triangular block (schedule order), W = inv(T)
                std::vector<double> Tm((size_t)nr * nr, 0.0), W((size_t)nr * nr, 0.0);
                for (int64_t r = 0; r < nr; ++r) {
                    Tm[r * nr + r] = tdiag[ka + r];
                    for (int32_t j = sptr[ka + r]; j < sptr[ka + r + 1]; ++j)
                        if (slcol[j] >= slot_lo) Tm[r * nr + (slcol[j] - slot_lo)] = sval[j];
                }
                for (int64_t col = 0; col < nr; ++col) {   // forward substitution on unit vectors
                    for (int64_t r = col; r < nr; ++r) {
                        double acc = r == col ? 1.0 : 0.0;
                        for (int64_t j = col; j < r; ++j) acc -= Tm[r * nr + j] * W[j * nr + col];
                        W[r * nr + col] = acc / Tm[r * nr + r];
                    }
                }
                const int64_t sz = TRSV_HDR + pad16(8 * nr * (nr + 1) / 2);
                const int64_t base = (int64_t)blob.size();
                blob.resize(base + sz, 0);
                unsigned char* p = blob.data() + base;
                int32_t* hdr = reinterpret_cast<int32_t*>(p);
                hdr[0] = (int32_t)nr;
                hdr[1] = (int32_t)ka;
                hdr[2] = 0;
                hdr[3] = (int32_t)sz;
                hdr[4] = 2;
                hdr[5] = (int32_t)ka;
                hdr[6] = 16;
                hdr[7] = 1;
                double* wp = reinterpret_cast<double*>(p + TRSV_HDR);
                for (int64_t r = 0; r < nr; ++r)
                    for (int64_t j = 0; j <= r; ++j) wp[r * (r + 1) / 2 + j] = W[r * nr + j];
                off.push_back(base);
                bytes.push_back((int32_t)sz);
                l = l2;
            } else {
                emit_rows(lvl_off[l], lvl_off[l + 1], 0, 0, INT64_MAX);
                ++l;
            }
        }
        maxp = std::max<int64_t>(maxp, (int64_t)off.size() - cpiece[c]);
    }
    T.ring_ok = false;
    if (!ok || off.empty()) return;
    cpiece[T.n_comp] = (int32_t)off.size();
    const int64_t avail = (int64_t)TRSV_SMEM - T.max_size * 8 - 1024 - TRSV_GMAX * 8;
    T.ring_depth = (int)std::min<int64_t>(4, avail / TRSV_PIECE_BYTES);
    if (avail < 2 * TRSV_PIECE_BYTES) return;   // the circular buffer holds >= 2 of the largest pieces
    T.max_pieces = maxp;
    T.blob.alloc(blob.size(), s); T.blob.upload(blob.data(), blob.size(), s);
    T.piece_off.alloc(off.size(), s); T.piece_off.upload(off.data(), off.size(), s);
    T.piece_bytes.alloc(bytes.size(), s); T.piece_bytes.upload(bytes.data(), bytes.size(), s);
    T.comp_piece.alloc(cpiece.size(), s); T.comp_piece.upload(cpiece.data(), cpiece.size(), s);
    // launch order of the ring kernel: most streamed bytes first (a patch's time
    // follows its pieces, not its level count, once narrow levels are grouped)
    {
        std::vector<int64_t> cb(T.n_comp, 0);
        for (int64_t c = 0; c < T.n_comp; ++c)
            for (int32_t q = cpiece[c]; q < cpiece[c + 1]; ++q) cb[c] += bytes[q];
        std::vector<int32_t> co(T.n_comp);
        for (int64_t c = 0; c < T.n_comp; ++c) co[c] = (int32_t)c;
        std::stable_sort(co.begin(), co.end(), [&](int32_t a, int32_t b) { return cb[a] > cb[b]; });
        T.ring_order.alloc(std::max<int64_t>(T.n_comp, 1), s);
        T.ring_order.upload(co.data(), T.n_comp, s);
    }
    WCB_CUDA(cudaStreamSynchronize(s));
    T.ring_ok = true;
    (void)n;
}

static void build_sched(TriSched& T, int64_t n, const int64_t* ptr, const int32_t* idx,
                        const double* val, bool upper,
                        const std::vector<int64_t>& comp, int64_t n_comp, cudaStream_t s) {
    std::vector<int32_t> lev(n, 0);
    auto visit = [&](int64_t i) {
        int32_t l = 0;
        for (int64_t j = ptr[i]; j < ptr[i + 1]; ++j)
            if (idx[j] != i) l = std::max(l, lev[idx[j]] + 1);
        lev[i] = l;
    };
    if (upper) for (int64_t i = n - 1; i >= 0; --i) visit(i);
    else for (int64_t i = 0; i < n; ++i) visit(i);
    // order rows by (component, level, row)
    std::vector<int32_t> order(n);
    for (int64_t i = 0; i < n; ++i) order[i] = (int32_t)i;
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
        return comp[a] != comp[b] ? comp[a] < comp[b] : lev[a] < lev[b];
    });
    std::vector<int32_t> comp_rows(n_comp + 1, 0), comp_lvl(n_comp + 1, 0), lvl_off, pos(n);
    int64_t k = 0;
    T.max_size = 0;
    for (int64_t c = 0; c < n_comp; ++c) {
        comp_rows[c] = (int32_t)k;
        comp_lvl[c] = (int32_t)lvl_off.size();
        const int64_t start = k;
        int32_t cur = -1;
        while (k < n && comp[order[k]] == c) {
            if (lev[order[k]] != cur) {
                cur = lev[order[k]];
                lvl_off.push_back((int32_t)k);
            }
            pos[order[k]] = (int32_t)(k - start);
            ++k;
        }
        T.max_size = std::max<int64_t>(T.max_size, k - start);
    }
    comp_rows[n_comp] = (int32_t)k;
    comp_lvl[n_comp] = (int32_t)lvl_off.size();
    T.max_levels = 0;
    for (int64_t c = 0; c < n_comp; ++c)
        T.max_levels = std::max<int64_t>(T.max_levels, comp_lvl[c + 1] - comp_lvl[c]);
    lvl_off.push_back((int32_t)n);
    // the level kernel multiplies by 1/diag (one correctly rounded reciprocal
    // per row, host-side) instead of dividing on the critical path of every
    // level; WAVECELL_B200_TRSV_DIV=1 restores the division
    const bool recip = !(getenv("WAVECELL_B200_TRSV_DIV") && getenv("WAVECELL_B200_TRSV_DIV")[0] == '1');
    T.recip = recip;
    std::vector<int32_t> sptr(n + 1, 0), slcol;
    std::vector<double> sval, sdiag(n, 0.0), tdiag(n, 0.0);
    slcol.reserve(ptr[n]);
    sval.reserve(ptr[n]);
    for (int64_t k2 = 0; k2 < n; ++k2) {
        const int64_t i = order[k2];
        sptr[k2] = (int32_t)slcol.size();
        for (int64_t j = ptr[i]; j < ptr[i + 1]; ++j) {
            if (idx[j] == i) {
                sdiag[k2] = recip ? 1.0 / val[j] : val[j];
                tdiag[k2] = val[j];
            } else {
                slcol.push_back(pos[idx[j]]);
                sval.push_back(val[j]);
            }
        }
    }
    sptr[n] = (int32_t)slcol.size();
    if (slcol.empty()) { slcol.push_back(0); sval.push_back(0.0); }
    T.n_comp = n_comp;
    T.n_levels = (int64_t)lvl_off.size() - 1;
    T.comp_rows.alloc(comp_rows.size(), s); T.comp_rows.upload(comp_rows.data(), comp_rows.size(), s);
    T.comp_lvl.alloc(comp_lvl.size(), s); T.comp_lvl.upload(comp_lvl.data(), comp_lvl.size(), s);
    T.lvl_off.alloc(lvl_off.size(), s); T.lvl_off.upload(lvl_off.data(), lvl_off.size(), s);
    T.rows.alloc(n, s); T.rows.upload(order.data(), n, s);
    T.pos.alloc(n, s); T.pos.upload(pos.data(), n, s);
    std::vector<int32_t> lvl_ent(lvl_off.size());
    for (size_t l = 0; l < lvl_off.size(); ++l) lvl_ent[l] = sptr[lvl_off[l]];
    T.max_lvl_rows = T.max_lvl_ent = 0;
    for (size_t l = 0; l + 1 < lvl_off.size(); ++l) {
        T.max_lvl_rows = std::max<int64_t>(T.max_lvl_rows, lvl_off[l + 1] - lvl_off[l]);
        T.max_lvl_ent = std::max<int64_t>(T.max_lvl_ent, lvl_ent[l + 1] - lvl_ent[l]);
    }
    T.lvl_ent.alloc(lvl_ent.size(), s); T.lvl_ent.upload(lvl_ent.data(), lvl_ent.size(), s);
    T.sptr.alloc(sptr.size(), s); T.sptr.upload(sptr.data(), sptr.size(), s);
    T.slcol.alloc(slcol.size(), s); T.slcol.upload(slcol.data(), slcol.size(), s);
    T.sval.alloc(sval.size(), s); T.sval.upload(sval.data(), sval.size(), s);
    T.sdiag.alloc(n, s); T.sdiag.upload(sdiag.data(), n, s);
    WCB_CUDA(cudaStreamSynchronize(s));   // host vectors die here
    const int64_t fixed = T.max_size * 8 + (T.max_levels + 1) * 8 + 64;
    const int64_t avail = (int64_t)TRSV_SMEM - fixed;
    // ring slots: as deep as the budget allows with every level fitting a
    // slot (cap TRSV_DMAX); if fewer than 3 such slots fit, 3 slots as large
    // as the budget allows (wider levels read global memory directly)
    const int64_t full_r = std::min<int64_t>(std::max<int64_t>(T.max_lvl_rows, 1), 1024);
    const int64_t full_e = std::max<int64_t>(T.max_lvl_ent, 1);
    const int64_t sb_full = (int64_t)trsv_slot_bytes((int)full_e, (int)full_r);
    const int64_t d_full = avail > 0 ? avail / sb_full : 0;
    if (d_full >= 3) {
        T.slot_r = (int)full_r;
        T.slot_e = (int)full_e;
        T.depth = (int)std::min<int64_t>(TRSV_DMAX, d_full);
    } else {
        T.slot_r = (int)full_r;
        const int64_t per = avail / 3 - full_r * 12 - 32;
        T.slot_e = (int)std::max<int64_t>(0, std::min<int64_t>(full_e, per / 12));
        T.depth = 3;
    }
    T.depth = T.depth >= 12 ? 12 : T.depth >= 8 ? 8 : T.depth >= 6 ? 6 : T.depth >= 4 ? 4 : 3;
    T.ok = avail > 0 && T.slot_e >= 256;
    T.pf_ok = T.max_size * 8 + (T.max_levels + 1) * 8 <= (int64_t)TRSV_SMEM;
    // launch order: longest dependency chains first (2 waves when components > SMs)
    std::vector<int32_t> co(n_comp);
    for (int64_t c = 0; c < n_comp; ++c) co[c] = (int32_t)c;
    std::stable_sort(co.begin(), co.end(), [&](int32_t a, int32_t b) {
        const int64_t la = comp_lvl[a + 1] - comp_lvl[a], lb = comp_lvl[b + 1] - comp_lvl[b];
        if (la != lb) return la > lb;
        return comp_rows[a + 1] - comp_rows[a] > comp_rows[b + 1] - comp_rows[b];
    });
    T.comp_order.alloc(std::max<int64_t>(n_comp, 1), s);
    T.comp_order.upload(co.data(), n_comp, s);
    WCB_CUDA(cudaStreamSynchronize(s));
    pack_pieces(T, n, comp_rows, comp_lvl, lvl_off, sptr, sdiag, tdiag, sval, slcol, s);
}

struct DevLU {
    int64_t n = 0;
    DevBuf<int64_t> perm_r, perm_c;
    DevBuf<int64_t> Lp, Up;
    DevBuf<int32_t> Li, Ui;
    DevBuf<double> Lx, Ux;
    TriSched Ls, Us;
    void load(const wcb_lu* lu, cudaStream_t s) {
        n = lu->n;
        perm_r.alloc(std::max<int64_t>(n, 1), s);
        perm_c.alloc(std::max<int64_t>(n, 1), s);
        perm_r.upload(lu->perm_r, n, s);
        perm_c.upload(lu->perm_c, n, s);
        const int64_t nl = lu->L_indptr[n], nu = lu->U_indptr[n];
        Lp.alloc(n + 1, s); Lp.upload(lu->L_indptr, n + 1, s);
        Up.alloc(n + 1, s); Up.upload(lu->U_indptr, n + 1, s);
        Li.alloc(std::max<int64_t>(nl, 1), s); Li.upload(lu->L_indices, nl, s);
        Ui.alloc(std::max<int64_t>(nu, 1), s); Ui.upload(lu->U_indices, nu, s);
        Lx.alloc(std::max<int64_t>(nl, 1), s); Lx.upload(lu->L_data, nl, s);
        Ux.alloc(std::max<int64_t>(nu, 1), s); Ux.upload(lu->U_data, nu, s);
        if (n > 0 && !getenv("WAVECELL_B200_SYNCFREE_TRSV")) {
            int64_t nc = 0;
            const std::vector<int64_t> comp = factor_components(n, lu, &nc);
            build_sched(Ls, n, lu->L_indptr, lu->L_indices, lu->L_data, false, comp, nc, s);
            build_sched(Us, n, lu->U_indptr, lu->U_indices, lu->U_data, true, comp, nc, s);
        }
    }
};

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Sync-free sparse triangular solve (CSR), x = T^-1 b.  `upper` processes rows
// n-1 .. 0.  done[] must be zero on entry; counter[0] = 0.
__global__ void k_sptrsv(int64_t n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                         const double* __restrict__ val, const double* __restrict__ b,
                         double* x, int* done, unsigned long long* counter, int upper) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned long long slot = 0;
        if (lane == 0) slot = atomicAdd(counter, 1ULL);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (slot >= (unsigned long long)n) break;
        const int64_t i = upper ? (n - 1 - (int64_t)slot) : (int64_t)slot;
        double s = 0.0, diag = 0.0;
        for (int64_t j = ptr[i] + lane; j < ptr[i + 1]; j += 32) {
            const int64_t c = idx[j];
            const double a = val[j];
            if (c == i) {
                diag = a;
            } else {
                while (ld_acquire(done + c) == 0) {
                }
                s = fma(a, *((volatile const double*)(x + c)), s);
            }
        }
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s += __shfl_down_sync(0xffffffffu, s, o);
            diag += __shfl_down_sync(0xffffffffu, diag, o);
        }
        if (lane == 0) {
            x[i] = (b[i] - s) / diag;
            st_release(done + i, 1);
        }
        __syncwarp();
    }
}

// Component-local level-scheduled solve (see TriSched): one CTA per
// component, unknowns in shared memory (b read in place of x).  While a level
// is solved, every warp already holds its row of the next level in registers
// (values and column slots do not depend on x), so a level costs one barrier
// plus shared-memory FMAs.  Fixed lane order and shuffle tree: deterministic.
// Level data staged into a shared-memory ring by cp.async, TRSV_D levels
// ahead: a level's rows are contiguous in schedule order, so its packed
// entries (values, column slots), row starts and diagonals are four
// contiguous ranges.  Levels too large for a ring slot read global memory.

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32_imex(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32_imex(dst)), "l"(src) : "memory");
}

static __host__ __device__ inline size_t trsv_slot_bytes(int e, int r);

template <int TRSV_D>
__global__ void __launch_bounds__(TRSV_THREADS) k_trsv_comp(
    const int32_t* __restrict__ comp_order,
    const int32_t* __restrict__ comp_rows, const int32_t* __restrict__ comp_lvl,
    const int32_t* __restrict__ lvl_off, const int32_t* __restrict__ lvl_ent, const int32_t* __restrict__ rows,
    const int32_t* __restrict__ sptr, const int32_t* __restrict__ slcol,
    const double* __restrict__ sval, const double* __restrict__ sdiag, const double* __restrict__ b,
    double* __restrict__ x, int max_size, int max_levels, int slot_e, int slot_r, int recip) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const size_t sb = trsv_slot_bytes(slot_e, slot_r);
    double* xl = reinterpret_cast<double*>(smraw + sb * TRSV_D);
    int* lo = reinterpret_cast<int*>(xl + max_size);   // this component's level offsets
    int* le = lo + max_levels + 1;                     // and entry offsets
    auto sv = [&](int l) { return reinterpret_cast<double*>(smraw + sb * (l % TRSV_D)); };
    auto sd = [&](int l) { return sv(l) + slot_e; };
    auto sc = [&](int l) { return reinterpret_cast<int*>(sd(l) + slot_r); };
    auto sp = [&](int l) { return sc(l) + slot_e; };
    const int c = comp_order[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    constexpr int GW = WCB_TRSV_GW;                 // lanes per row
    const int hw = lane / GW, l16 = lane % GW;      // row slot in the warp, lane in the row group
    const unsigned hmask = (GW == 32 ? 0xffffffffu : ((1u << GW) - 1u)) << (hw * GW);
    const int r0 = comp_rows[c], r1 = comp_rows[c + 1];
    const int l0 = comp_lvl[c], nl = comp_lvl[c + 1] - l0;
    for (int k = r0 + threadIdx.x; k < r1; k += blockDim.x) xl[k - r0] = b[rows[k]];
    for (int l = threadIdx.x; l <= nl; l += blockDim.x) {
        lo[l] = lvl_off[l0 + l];
        le[l] = lvl_ent[l0 + l];
    }
    __syncthreads();
    auto fits = [&](int l) { return lo[l + 1] - lo[l] <= slot_r && le[l + 1] - le[l] <= slot_e; };
    auto stage = [&](int l) {
        if (l < nl && fits(l)) {
            const int a = lo[l], e = lo[l + 1];
            const int pa = le[l], pe = le[l + 1];
            int* P = sp(l);
            double* D = sd(l);
            double* V = sv(l);
            int* C = sc(l);
            for (int k = threadIdx.x; k <= e - a; k += blockDim.x) cp_async4(P + k, sptr + a + k);
            for (int k = threadIdx.x; k < e - a; k += blockDim.x) cp_async8(D + k, sdiag + a + k);
            for (int j = threadIdx.x; j < pe - pa; j += blockDim.x) {
                cp_async8(V + j, sval + pa + j);
                cp_async4(C + j, slcol + pa + j);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // prologue: levels 0..D-2 in flight.  Iteration l: wait for level l,
    // one barrier (level l-1's x and level l's data visible; ring slot of
    // level l-1 free), refill that slot with level l+D-1, solve level l.
    #pragma unroll
    for (int l = 0; l < TRSV_D - 1; ++l) stage(l);
    for (int l = 0; l < nl; ++l) {
        asm volatile("cp.async.wait_group %0;" ::"n"(TRSV_D - 2) : "memory");
        __syncthreads();
#if !WCB_TRSV_STAGE_LATE
        stage(l + TRSV_D - 1);
#endif
        const int a = lo[l], e = lo[l + 1];
        if (fits(l)) {
            const int* P = sp(l);
            const double* D = sd(l);
            const double* V = sv(l);
            const int* C = sc(l);
            // GW lanes per row (levels are narrow: median 3 rows of ~47
            // entries): GW-strided entries, log2(GW)-step shuffle tree
            const int base = P[0];
            for (int k = (32 / GW) * warp + hw; k < e - a; k += (32 / GW) * nw) {
                const int p0 = P[k] - base, p1 = P[k + 1] - base;
                double sacc = 0.0;
                for (int j = p0 + l16; j < p1; j += GW) sacc = fma(V[j], xl[C[j]], sacc);
                #pragma unroll
                for (int o = GW / 2; o > 0; o >>= 1) sacc += __shfl_down_sync(hmask, sacc, o, GW);
                if (l16 == 0) xl[a + k - r0] = recip ? (xl[a + k - r0] - sacc) * D[k] : (xl[a + k - r0] - sacc) / D[k];
            }
        } else {
            for (int k = a + (32 / GW) * warp + hw; k < e; k += (32 / GW) * nw) {
                double sacc = 0.0;
                for (int j = sptr[k] + l16; j < sptr[k + 1]; j += GW) sacc = fma(sval[j], xl[slcol[j]], sacc);
                #pragma unroll
                for (int o = GW / 2; o > 0; o >>= 1) sacc += __shfl_down_sync(hmask, sacc, o, GW);
                if (l16 == 0) xl[k - r0] = recip ? (xl[k - r0] - sacc) * sdiag[k] : (xl[k - r0] - sacc) / sdiag[k];
            }
        }
#if WCB_TRSV_STAGE_LATE
        stage(l + TRSV_D - 1);   // after the level's rows: off the critical path
#endif
    }
    __syncthreads();
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    for (int k = r0 + threadIdx.x; k < r1; k += blockDim.x) x[rows[k]] = xl[k - r0];
}

static __host__ __device__ inline size_t trsv_slot_bytes(int e, int r) {
    return (((size_t)e * 12 + (size_t)r * 8 + (size_t)(r + 1) * 4) + 15) / 16 * 16;
}
size_t TriSched::smem_bytes() const {
    return trsv_slot_bytes(slot_e, slot_r) * depth + (size_t)max_size * 8 + (size_t)(max_levels + 1) * 8;
}

template <int D>
static void launch_trsv_d(Context* ctx, const TriSched& T, const double* b, double* x) {
    const size_t sm = T.smem_bytes();
    ensure_smem_attr((const void*)k_trsv_comp<D>, ctx->device, sm);
    static const int threads = [] {
        const char* e = getenv("WAVECELL_B200_TRSV_THREADS");
        const int t = e ? atoi(e) : TRSV_THREADS_DEF;
        return t >= 32 && t <= TRSV_THREADS && t % 32 == 0 ? t : TRSV_THREADS_DEF;
    }();
    k_trsv_comp<D><<<(unsigned)T.n_comp, threads, sm, ctx->stream>>>(
        T.comp_order.p, T.comp_rows.p, T.comp_lvl.p, T.lvl_off.p, T.lvl_ent.p, T.rows.p, T.sptr.p, T.slcol.p,
        T.sval.p, T.sdiag.p, b, x, (int)T.max_size, (int)T.max_levels, T.slot_e, T.slot_r, T.recip ? 1 : 0);
}

// Level-scheduled component solve with register prefetch (default):
// one CTA per component (unknowns in shared memory), NW warps in row groups
// of GW lanes.  A level costs one barrier plus its rows: every group loads
// the values / column slots / pivot of its next row while the current
// level is solved (they do not depend on x), so after the barrier only the
// shared-memory gathers of x, the FMAs and the shuffle tree remain on the
// critical path; levels further ahead are prefetched into L2 by bulk
// prefetches.  Entries are visited in the same lane-strided order and reduced
// by the same tree as k_trsv_comp / k_sptrsv (bitwise equal).
constexpr int TRSV_KPF = 4;     // entries per lane held in registers
constexpr int TRSV_PFD = 8;     // L2 prefetch distance (levels)

__device__ __forceinline__ void l2_prefetch(const void* p, size_t bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
    const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~(uintptr_t)15;
    if (e > a)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a)) : "memory");
}

template <int NW>
__global__ void __launch_bounds__(NW * 32) k_trsv_pf(
    const int32_t* __restrict__ comp_order, const int32_t* __restrict__ comp_rows,
    const int32_t* __restrict__ comp_lvl, const int32_t* __restrict__ lvl_off, const int32_t* __restrict__ lvl_ent,
    const int32_t* __restrict__ rows, const int32_t* __restrict__ sptr, const int32_t* __restrict__ slcol,
    const double* __restrict__ sval, const double* __restrict__ sdiag, const double* __restrict__ b,
    double* __restrict__ x, int max_size, int max_levels, int recip) {
    constexpr int GW = WCB_TRSV_GW;
    constexpr int G = NW * 32 / GW;                 // row groups
    extern __shared__ __align__(16) unsigned char smraw[];
    double* xl = reinterpret_cast<double*>(smraw);
    int* lo = reinterpret_cast<int*>(xl + max_size);
    int* le = lo + max_levels + 1;
    const int c = comp_order[blockIdx.x];
    const int lane = threadIdx.x & 31;
    const int grp = threadIdx.x / GW, l16 = lane % GW;
    const unsigned hmask = (GW == 32 ? 0xffffffffu : ((1u << GW) - 1u)) << ((lane / GW) * GW);
    const int r0 = comp_rows[c], r1 = comp_rows[c + 1];
    const int l0 = comp_lvl[c], nl = comp_lvl[c + 1] - l0;
    for (int k = r0 + threadIdx.x; k < r1; k += blockDim.x) xl[k - r0] = b[rows[k]];
    for (int l = threadIdx.x; l <= nl; l += blockDim.x) {
        lo[l] = lvl_off[l0 + l];
        le[l] = lvl_ent[l0 + l];
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int l = 0; l < TRSV_PFD && l < nl; ++l) {
            l2_prefetch(sval + le[l], (size_t)(le[l + 1] - le[l]) * 8);
            l2_prefetch(slcol + le[l], (size_t)(le[l + 1] - le[l]) * 4);
        }
    // this group's first row of a level: (row, entry range, pivot, first entries)
    int rk = -1, p0 = 0, p1 = 0;
    double dg = 0.0, pv[TRSV_KPF];
    int pc[TRSV_KPF];
    auto preload = [&](int l) {
        rk = -1;
        if (l >= nl) return;
        const int k = lo[l] + grp;
        if (k >= lo[l + 1]) return;
        rk = k;
        p0 = sptr[k];
        p1 = sptr[k + 1];
        dg = sdiag[k];
        #pragma unroll
        for (int q = 0; q < TRSV_KPF; ++q) {
            const int j = p0 + l16 + q * GW;
            pv[q] = j < p1 ? sval[j] : 0.0;
            pc[q] = j < p1 ? slcol[j] : 0;
        }
    };
    auto finish = [&](int k, double sacc) {
        #pragma unroll
        for (int o = GW / 2; o > 0; o >>= 1) sacc += __shfl_down_sync(hmask, sacc, o, GW);
        if (l16 == 0) {
            const int i = k - r0;
            xl[i] = recip ? (xl[i] - sacc) * sdiag[k] : (xl[i] - sacc) / sdiag[k];
        }
    };
    preload(0);
    for (int l = 0; l < nl; ++l) {
        __syncthreads();   // level l-1 solved
        if (threadIdx.x == 0 && l + TRSV_PFD < nl) {
            const int lp = l + TRSV_PFD;
            l2_prefetch(sval + le[lp], (size_t)(le[lp + 1] - le[lp]) * 8);
            l2_prefetch(slcol + le[lp], (size_t)(le[lp + 1] - le[lp]) * 4);
            l2_prefetch(sptr + lo[lp], (size_t)(lo[lp + 1] - lo[lp] + 1) * 4);
            l2_prefetch(sdiag + lo[lp], (size_t)(lo[lp + 1] - lo[lp]) * 8);
        }
        if (rk >= 0) {
            double sacc = 0.0;
            #pragma unroll
            for (int q = 0; q < TRSV_KPF; ++q)
                if (p0 + l16 + q * GW < p1) sacc = fma(pv[q], xl[pc[q]], sacc);
            for (int j = p0 + l16 + TRSV_KPF * GW; j < p1; j += GW) sacc = fma(sval[j], xl[slcol[j]], sacc);
            (void)dg;
            finish(rk, sacc);
        }
        // further rows of a wide level
        for (int k = lo[l] + grp + G; k < lo[l + 1]; k += G) {
            double sacc = 0.0;
            for (int j = sptr[k] + l16; j < sptr[k + 1]; j += GW) sacc = fma(sval[j], xl[slcol[j]], sacc);
            finish(k, sacc);
        }
        preload(l + 1);
    }
    __syncthreads();
    for (int k = r0 + threadIdx.x; k < r1; k += blockDim.x) x[rows[k]] = xl[k - r0];
}

// Producer / consumer level solve (default): one CTA per component, the
// unknowns in shared memory.  One producer thread streams the component's
// level pieces (one bulk copy each, mbarrier complete_tx) into a circular
// byte buffer -- pieces are packed back to back, so a run of narrow levels
// (median 2-3 rows, ~1.5 KB) keeps dozens of pieces in flight -- and never
// overtakes the release counters the consumers publish.  NC consumer warps
// solve a piece (row groups of GW lanes, rows strided over the groups), meet
// at a named barrier (x of the piece visible) and release it.  A level costs
// one consumer barrier plus its rows; the staging never occupies the
// consumers.  Same lane order and shuffle tree as k_trsv_comp (bitwise equal).
constexpr int TRSV_QK = 64;                       // pieces in flight (mbarrier ring)
constexpr int64_t TRSV_RING_HEAD = ((TRSV_QK * 24 + 127) / 128) * 128;   // full[QK], empty[QK], poff[QK], pneed[QK]

__device__ __forceinline__ void mbar_arrive_imex(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32_imex(bar)) : "memory");
}

// the rows of one piece with GW lanes per row (see the piece kinds above)
template <int GW, int NC>
__device__ __forceinline__ void trsv_piece(const unsigned char* pc, const int32_t* hdr, int ct, int lane, int q,
                                           double* xl, double* ts, int r0, int recip) {
    constexpr int G = NC * 32 / GW;
    const int nrow = hdr[0], k0 = hdr[1], ne = hdr[2], kind = hdr[4], gbase = hdr[5];
    const int l = ct % GW;
    // rows are dealt to the row groups starting at a per-piece offset, so
    // consecutive independent pieces of few rows land on different warps
    const int grp = (ct / GW + G - (q * 5) % G) % G;   // group grp takes rows grp, grp + G, ...
    const unsigned hmask = GW == 32 ? 0xffffffffu : (((1u << GW) - 1u) << (lane & ~(GW - 1)));
    if (kind == 2) {   // dense part of a group: x = W t
        const double* W = reinterpret_cast<const double*>(pc + TRSV_HDR);
        for (int k = grp; k < nrow; k += G) {
            double sacc = 0.0;
            const double* wr = W + k * (k + 1) / 2;
            for (int j = l; j <= k; j += GW) sacc = fma(wr[j], ts[j], sacc);
            #pragma unroll
            for (int o = GW / 2; o > 0; o >>= 1) sacc += __shfl_down_sync(hmask, sacc, o, GW);
            if (l == 0) xl[k0 + k - r0] = sacc;
        }
        return;
    }
    const int32_t* rp = reinterpret_cast<const int32_t*>(pc + TRSV_HDR);
    const double* dg = reinterpret_cast<const double*>(pc + TRSV_HDR + ((4 * (nrow + 1) + 15) / 16) * 16);
    const double* vv = dg + ((8 * nrow + 15) / 16) * 2;
    const int32_t* cc = reinterpret_cast<const int32_t*>(reinterpret_cast<const unsigned char*>(vv) +
                                                         ((8 * (int64_t)ne + 15) / 16) * 16);
    for (int k = grp; k < nrow; k += G) {
        // two interleaved partial sums per lane (independent load chains)
        double s0 = 0.0, s1 = 0.0;
        const int p1 = rp[k + 1];
        int j = rp[k] + l;
        for (; j + GW < p1; j += 2 * GW) {
            const double v0 = vv[j], v1 = vv[j + GW];
            const int c0 = cc[j], c1 = cc[j + GW];
            s0 = fma(v0, xl[c0], s0);
            s1 = fma(v1, xl[c1], s1);
        }
        if (j < p1) s0 = fma(vv[j], xl[cc[j]], s0);
        double sacc = s0 + s1;
        #pragma unroll
        for (int o = GW / 2; o > 0; o >>= 1) sacc += __shfl_down_sync(hmask, sacc, o, GW);
        if (l == 0) {
            const int i = k0 + k - r0;
            if (kind == 1) ts[k0 + k - gbase] = xl[i] - sacc;
            else xl[i] = recip ? (xl[i] - sacc) * dg[k] : (xl[i] - sacc) / dg[k];
        }
    }
}

template <int NC>
__global__ void __launch_bounds__((NC + 1) * 32) k_trsv_ring(
    const int32_t* __restrict__ comp_order, const int32_t* __restrict__ comp_rows,
    const int32_t* __restrict__ comp_piece, const int64_t* __restrict__ piece_off,
    const int32_t* __restrict__ piece_bytes, const unsigned char* __restrict__ blob,
    const int32_t* __restrict__ rows, const double* __restrict__ b, double* __restrict__ x, int max_size,
    int ring_bytes, int recip) {
    extern __shared__ __align__(128) unsigned char smraw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smraw);                 // [QK] piece landed
    uint64_t* empty = full + TRSV_QK;                                    // [QK] piece consumed by every consumer warp
    int* poff = reinterpret_cast<int*>(smraw + TRSV_QK * 16);            // [QK] ring offset of piece q
    int* pneed = poff + TRSV_QK;                                         // [QK] ring bytes the piece took (tail skip included)
    unsigned char* ring = smraw + TRSV_RING_HEAD;
    double* xl = reinterpret_cast<double*>(ring + ring_bytes);
    double* ts = xl + max_size;   // group scratch [TRSV_GMAX]
    const int c = comp_order[blockIdx.x];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = comp_rows[c], r1 = comp_rows[c + 1];
    const int q0 = comp_piece[c], nq = comp_piece[c + 1] - q0;
    if (threadIdx.x == 0) {
        for (int d = 0; d < TRSV_QK; ++d) {
            mbar_init(&full[d], 1);
            mbar_init(&empty[d], NC);
        }
    }
    for (int k = r0 + threadIdx.x; k < r1; k += blockDim.x) xl[k - r0] = b[rows[k]];
    __syncthreads();
    if (warp == 0) {   // producer warp: piece sizes / offsets fetched 32 at a time
        long long pos = 0, freed = 0;   // cumulative ring bytes placed / released
        int ro = 0;                     // oldest piece not yet known to be released
        for (int qb = 0; qb < nq; qb += 32) {
            const int qq = qb + lane;
            const uint32_t nb_l = qq < nq ? (uint32_t)piece_bytes[q0 + qq] : 0u;
            const int64_t off_l = qq < nq ? piece_off[q0 + qq] : 0;
            const int nbat = min(32, nq - qb);
            for (int i = 0; i < nbat; ++i) {
                const uint32_t nb = __shfl_sync(0xffffffffu, nb_l, i);
                const int64_t off = __shfl_sync(0xffffffffu, off_l, i);
                if (lane == 0) {
                    const int q = qb + i;
                    long long at = pos % ring_bytes;
                    long long need = nb;
                    if (at + nb > ring_bytes) { need += ring_bytes - at; at = 0; }   // wrap: skip the tail
                    // ring space and a free mbarrier slot: wait for the oldest pieces' release
                    while (pos + need - freed > ring_bytes || q - ro >= TRSV_QK) {
                        const int d0 = ro % TRSV_QK;
                        mbar_wait(&empty[d0], (uint32_t)((ro / TRSV_QK) & 1));
                        freed += pneed[d0];
                        ++ro;
                    }
                    pos += need;
                    const int d = q % TRSV_QK;
                    poff[d] = (int)at;
                    pneed[d] = (int)need;
                    mbar_expect_tx(&full[d], nb);
                    bulk_load(ring + at, blob + off, nb, &full[d]);
                }
                __syncwarp();
            }
        }
    } else {
        const int ct = threadIdx.x - 32;
        for (int q = 0; q < nq; ++q) {
            const int d = q % TRSV_QK;
            mbar_wait(&full[d], (uint32_t)((q / TRSV_QK) & 1));
            const unsigned char* pc = ring + poff[d];
            const int32_t* hdr = reinterpret_cast<const int32_t*>(pc);
            switch (hdr[6]) {   // lanes per row, chosen per piece on the host
                case 32: trsv_piece<32, NC>(pc, hdr, ct, lane, q, xl, ts, r0, recip); break;
                case 8: trsv_piece<8, NC>(pc, hdr, ct, lane, q, xl, ts, r0, recip); break;
                case 4: trsv_piece<4, NC>(pc, hdr, ct, lane, q, xl, ts, r0, recip); break;
                case 2: trsv_piece<2, NC>(pc, hdr, ct, lane, q, xl, ts, r0, recip); break;
                default: trsv_piece<16, NC>(pc, hdr, ct, lane, q, xl, ts, r0, recip); break;
            }
            // the next piece depends on this one (end of a level / of a group's
            // outside part / dense part): every consumer's rows must be visible
            if (hdr[7]) asm volatile("bar.sync 1, %0;" ::"r"(NC * 32) : "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_imex(&empty[d]);   // this warp is done with the piece's bytes
        }
    }
    __syncthreads();
    for (int k = r0 + threadIdx.x; k < r1; k += blockDim.x) x[rows[k]] = xl[k - r0];
}

static int trsv_ring_bytes(const TriSched& T) {
    const int64_t head = TRSV_RING_HEAD;
    int64_t avail = (int64_t)TRSV_SMEM - head - T.max_size * 8 - TRSV_GMAX * 8;
    avail = avail / 128 * 128;
    return (int)std::min<int64_t>(avail, trsv_ring_cap());
}

template <int NC>
static void launch_trsv_ring(Context* ctx, const TriSched& T, const double* b, double* x) {
    const int rb = trsv_ring_bytes(T);
    const size_t sm = (size_t)TRSV_RING_HEAD + (size_t)rb + (size_t)T.max_size * 8 + TRSV_GMAX * 8;
    ensure_smem_attr((const void*)k_trsv_ring<NC>, ctx->device, sm);
    k_trsv_ring<NC><<<(unsigned)T.n_comp, (NC + 1) * 32, sm, ctx->stream>>>(
        T.ring_order.p, T.comp_rows.p, T.comp_piece.p, T.piece_off.p, T.piece_bytes.p, T.blob.p, T.rows.p, b, x,
        (int)T.max_size, rb, T.recip ? 1 : 0);
}
template <int NC>
static void launch_trsv_ring_d(Context* ctx, const TriSched& T, const double* b, double* x) {
    launch_trsv_ring<NC>(ctx, T, b, x);
}

template <int NW>
static void launch_trsv_pf(Context* ctx, const TriSched& T, const double* b, double* x) {
    const size_t sm = (size_t)T.max_size * 8 + (size_t)(T.max_levels + 1) * 8;
    ensure_smem_attr((const void*)k_trsv_pf<NW>, ctx->device, sm);
    k_trsv_pf<NW><<<(unsigned)T.n_comp, NW * 32, sm, ctx->stream>>>(
        T.comp_order.p, T.comp_rows.p, T.comp_lvl.p, T.lvl_off.p, T.lvl_ent.p, T.rows.p, T.sptr.p, T.slcol.p,
        T.sval.p, T.sdiag.p, b, x, (int)T.max_size, (int)T.max_levels, T.recip ? 1 : 0);
}

static void launch_trsv(Context* ctx, const TriSched& T, const double* b, double* x) {
    static const int nw = [] {   // > 0: k_trsv_pf with nw warps (experimental)
        const char* e = getenv("WAVECELL_B200_TRSV_NW");
        return e ? atoi(e) : 0;
    }();
    static const int nc = [] {   // consumer warps of k_trsv_ring; 0: level kernel k_trsv_comp
        const char* e = getenv("WAVECELL_B200_TRSV_NC");
        return e ? atoi(e) : 16;
    }();
    if (nw <= 0 && nc > 0 && T.ring_ok) {
        switch (nc) {
            case 4: launch_trsv_ring_d<4>(ctx, T, b, x); return;
            case 8: launch_trsv_ring_d<8>(ctx, T, b, x); return;
            case 24: launch_trsv_ring_d<24>(ctx, T, b, x); return;
            default: launch_trsv_ring_d<16>(ctx, T, b, x); return;
        }
    }
    if (T.pf_ok && (nw > 0 || !T.ok)) {
        switch (nw) {
            case 4: launch_trsv_pf<4>(ctx, T, b, x); return;
            case 8: launch_trsv_pf<8>(ctx, T, b, x); return;
            case 32: launch_trsv_pf<32>(ctx, T, b, x); return;
            default: launch_trsv_pf<16>(ctx, T, b, x); return;
        }
    }
    switch (T.depth) {
        case 3: launch_trsv_d<3>(ctx, T, b, x); break;
        case 4: launch_trsv_d<4>(ctx, T, b, x); break;
        case 6: launch_trsv_d<6>(ctx, T, b, x); break;
        case 8: launch_trsv_d<8>(ctx, T, b, x); break;
        default: launch_trsv_d<12>(ctx, T, b, x); break;
    }
}

// y[perm_r[i]] = b[i]   (row permutation of SuperLU: Pr A Pc = L U)
__global__ void k_perm_rows(int64_t n, const int64_t* __restrict__ perm_r, const double* __restrict__ b,
                            double* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[perm_r[i]] = b[i];
}

// c predictor (src/timeint.py:271-274) into the state slots of c, and keep v_pred
__global__ void k_c_predict(int64_t nc, const int64_t* __restrict__ cs, const double* __restrict__ psi_c,
                            const double* __restrict__ v_c, const double* __restrict__ a_c, double dt,
                            double c1, double c2, double* __restrict__ state, double* __restrict__ pred,
                            double* __restrict__ vpred) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x) {
        // src/timeint.py:271-272, each operation rounded on its own (no FMA)
        const double p = __dadd_rn(__dadd_rn(psi_c[i], __dmul_rn(dt, v_c[i])), __dmul_rn(c1, a_c[i]));
        pred[i] = p;
        vpred[i] = __dadd_rn(v_c[i], __dmul_rn(c2, a_c[i]));
        state[cs[i]] = p;
    }
}

// rhs_c = f F_c - Kc
__global__ void k_c_rhs(int64_t nc, const double* __restrict__ Fc, const double* __restrict__ ft,
                        int64_t k, const double* __restrict__ Kc, double* __restrict__ rhs) {
    const double f = ft[k];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x)
        rhs[i] = __dsub_rn(__dmul_rn(f, Fc[i]), Kc[i]);
}

// corrector (src/timeint.py:279-282); a_c = z[perm_c[i]]; amp over c nodes
__global__ void k_c_correct(int64_t nc, const int64_t* __restrict__ cs, const int64_t* __restrict__ perm_c,
                            const double* __restrict__ z, const double* __restrict__ pred,
                            const double* __restrict__ vpred, double bdt2, double gdt,
                            double* __restrict__ a_c, double* __restrict__ psi_c, double* __restrict__ v_c,
                            double* __restrict__ state, unsigned long long* amp_slot) {
    unsigned long long amp = 0ULL;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x) {
        const double a = z[perm_c[i]];
        a_c[i] = a;
        const double p = __dadd_rn(pred[i], __dmul_rn(bdt2, a));
        psi_c[i] = p;
        v_c[i] = __dadd_rn(vpred[i], __dmul_rn(gdt, a));
        state[cs[i]] = p;
        unsigned long long b = amp_bits(p);
        amp = b > amp ? b : amp;
    }
    block_amp_max<256>(amp, amp_slot);
}

__global__ void k_gather_rows(int64_t n, const int64_t* __restrict__ map, const double* __restrict__ src,
                              double* __restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[map[i]];
}

// bootstrap (src/timeint.py:246-256): prev_d = psi - dt v + dt^2/2 a_d for d slots
__global__ void k_imex_boot(int64_t ns, const double* __restrict__ psi, const double* __restrict__ v,
                            const double* __restrict__ Kpsi, const double* __restrict__ m_d_state,
                            Source F, const double* __restrict__ ft, double dt, double* __restrict__ prev) {
    const double f0 = ft[0];
    const double c = 0.5 * dt * dt;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x) {
        const double md = m_d_state[i];
        const double a = md > 0.0 ? __ddiv_rn(__dsub_rn(__dmul_rn(f0, source_at(F, i)), Kpsi[i]), md) : 0.0;
        prev[i] = __dadd_rn(__dsub_rn(psi[i], __dmul_rn(dt, v[i])), __dmul_rn(c, a));
    }
}

// consistent-mass CDM bootstrap of the c rows (src/timeint.py:175-176):
// psi_prev_c = psi_c - dt v_c + (dt^2/2) a_c
__global__ void k_c_boot_prev(int64_t nc, const int64_t* __restrict__ cs, const double* __restrict__ psi_c,
                              const double* __restrict__ v_c, const double* __restrict__ a_c, double dt,
                              double c, double* __restrict__ prev) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x)
        prev[cs[i]] = __dadd_rn(__dsub_rn(psi_c[i], __dmul_rn(dt, v_c[i])), __dmul_rn(c, a_c[i]));
}

// consistent-mass CDM update of the c rows (src/timeint.py:185): the fused
// step left 2 psi - psi_prev in the c slots (1/m = 0 there); add dt^2 a_c
// with a_c = z[perm_c] = (M_cc^-1 rhs_c)
__global__ void k_c_cdm_update(int64_t nc, const int64_t* __restrict__ cs, const int64_t* __restrict__ perm_c,
                               const double* __restrict__ z, double dt2, double* __restrict__ state) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = cs[i];
        state[j] = __dadd_rn(state[j], __dmul_rn(dt2, z[perm_c[i]]));
    }
}

// max |psi| over a whole state vector (non-DOF slots hold 0) -- the
// divergence amplitude of src/timeint.py:91-94 once every row is final
__global__ void k_state_amp(int64_t ns, const double* __restrict__ state, unsigned long long* amp_slot) {
    unsigned long long amp = 0ULL;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long b = amp_bits(state[i]);
        amp = b > amp ? b : amp;
    }
    block_amp_max<256>(amp, amp_slot);
}

// dst[cs[i]] = src[perm[i]]  (perm may be NULL: identity)
__global__ void k_scatter_rows(int64_t n, const int64_t* __restrict__ cs, const int64_t* __restrict__ perm,
                               const double* __restrict__ src, double* __restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[cs[i]] = src[perm ? perm[i] : i];
}

// y = A x (CSR, stored order per row, as scipy's csr_matvec)
__global__ void k_csr_rows(int64_t n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                           const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int64_t j = ptr[i]; j < ptr[i + 1]; ++j) acc = __dadd_rn(acc, __dmul_rn(val[j], x[idx[j]]));
        y[i] = acc;
    }
}

}  // namespace wcb

using namespace wcb;

struct wcb_imex_plan {
    Operator* op = nullptr;
    Context* ctx = nullptr;   // retained
    int64_t n_c = 0, n_d = 0;
    // overlap of step k+1's far tiles (second stream) with step k's c solve
    bool split = false;
    cudaStream_t s2 = nullptr;
    cudaEvent_t e_near = nullptr, e_far = nullptr, e_boot = nullptr;
    ~wcb_imex_plan() {
        if (s2) { cudaStreamSynchronize(s2); cudaStreamDestroy(s2); }
        if (e_near) cudaEventDestroy(e_near);
        if (e_far) cudaEventDestroy(e_far);
        if (e_boot) cudaEventDestroy(e_boot);
    }
    DevBuf<int64_t> c_state;          // state index of each c DOF (c order)
    DevBuf<int64_t> c_compact;
    DevBuf<double> minv, m_d_state;   // 1/m_d at d slots (0 at c / non-DOF), m_d at d slots
    DevBuf<double> Fc;
    DevBuf<double> F_win;
    Source src;
    DevLU S, Mcc;
    bool has_S = false;
    // M_cc in CSR (c order), for x'Mx of the consistent-mass power iteration
    DevBuf<int64_t> mcc_ptr;
    DevBuf<int32_t> mcc_idx;
    DevBuf<double> mcc_val;
    bool has_mcc_csr = false;
    int64_t n_obs = 0;
    DevBuf<int64_t> obs_indptr, obs_idx;
    DevBuf<double> obs_val;
    // work
    DevBuf<double> A, B, T, V;
    DevBuf<double> psi_c, v_c, a_c, pred, vpred, Kc, rhs, y, z;
    DevBuf<int> done;
    DevBuf<unsigned long long> counter;
    DevBuf<unsigned long long> amp, amp_scratch;
    DevBuf<double> ft_k, ft_new;
};

namespace wcb {
static int grid1(Context* ctx, int64_t n) {
    return (int)std::min<int64_t>(std::max<int64_t>(ceil_div(n, 256), 1), (int64_t)ctx->sm_count * 8);
}

static void lu_solve(Context* ctx, wcb_imex_plan* P, DevLU& F, const double* b, double* x) {
    cudaStream_t s = ctx->stream;
    const int64_t n = F.n;
    if (!n) return;
    k_perm_rows<<<grid1(ctx, n), 256, 0, s>>>(n, F.perm_r.p, b, P->y.p);
    // forward: L w = y  (into z), backward: U v = w (into y)
    if ((F.Ls.ok || F.Ls.pf_ok || F.Ls.ring_ok) && (F.Us.ok || F.Us.pf_ok || F.Us.ring_ok)) {
        launch_trsv(ctx, F.Ls, P->y.p, P->z.p);
        launch_trsv(ctx, F.Us, P->z.p, x);
        ctx->launches += 3;
        WCB_CHECK_LAUNCH();
        return;
    }
    WCB_CUDA(cudaMemsetAsync(P->done.p, 0, n * sizeof(int), s));
    WCB_CUDA(cudaMemsetAsync(P->counter.p, 0, 2 * sizeof(unsigned long long), s));
    const int blocks = (int)std::min<int64_t>(ceil_div(n, 8), (int64_t)ctx->sm_count * 16);
    k_sptrsv<<<blocks, 256, 0, s>>>(n, F.Lp.p, F.Li.p, F.Lx.p, P->y.p, P->z.p, P->done.p, P->counter.p, 0);
    WCB_CUDA(cudaMemsetAsync(P->done.p, 0, n * sizeof(int), s));
    k_sptrsv<<<blocks, 256, 0, s>>>(n, F.Up.p, F.Ui.p, F.Ux.p, P->z.p, x, P->done.p, P->counter.p + 1, 1);
    ctx->launches += 3;
    WCB_CHECK_LAUNCH();
}
}  // namespace wcb

extern "C" {

int wcb_imex_plan_create(wcb_operator* o, int64_t n_c, const int64_t* c_idx, int64_t n_d,
                         const int64_t* d_idx, const double* m_d, const wcb_lu* S_cc,
                         const wcb_lu* M_cc, const double* F_s, const wcb_observer* obs,
                         wcb_imex_plan** out) {
    try {
        WCB_REQUIRE(o && out && F_s, "NULL argument");
        Operator* op = o->op;
        Context* ctx = op->ctx;
        WCB_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        const int64_t n = op->n, ns = op->n_state;
        WCB_REQUIRE(n_c + n_d == n, "c and d index sets must partition the DOFs");
        std::unique_ptr<wcb_imex_plan> P(new wcb_imex_plan());
        P->op = op;
        P->ctx = ctx;
        P->n_c = n_c;
        P->n_d = n_d;
        const std::vector<int64_t>& si = op->state_index();
        std::vector<uint8_t> seen(n, 0);
        std::vector<double> minv(ns, 0.0), md(ns, 0.0);
        for (int64_t i = 0; i < n_d; ++i) {
            const int64_t r = d_idx[i];
            WCB_REQUIRE(r >= 0 && r < n && !seen[r], "c and d index sets must partition the DOFs");
            seen[r] = 1;
            WCB_REQUIRE(m_d[i] > 0.0, "d mass block has non-positive diagonal entries");
            minv[si[r]] = 1.0 / m_d[i];
            md[si[r]] = m_d[i];
        }
        std::vector<int64_t> cs(std::max<int64_t>(n_c, 1));
        std::vector<double> Fc(std::max<int64_t>(n_c, 1));
        for (int64_t i = 0; i < n_c; ++i) {
            const int64_t r = c_idx[i];
            WCB_REQUIRE(r >= 0 && r < n && !seen[r], "c and d index sets must partition the DOFs");
            seen[r] = 1;
            cs[i] = si[r];
            Fc[i] = F_s[r];
        }
        P->minv.alloc(ns, s); P->minv.upload(minv.data(), ns, s);
        P->m_d_state.alloc(ns, s); P->m_d_state.upload(md.data(), ns, s);
        P->c_state.alloc(cs.size(), s); P->c_state.upload(cs.data(), n_c, s);
        P->Fc.alloc(Fc.size(), s); P->Fc.upload(Fc.data(), n_c, s);
        if (n_c) op->set_apply_subset(c_idx, n_c);   // K rows of c only, per step
        if (n_c && !getenv("WAVECELL_B200_NO_ROW_APPLY")) op->set_row_subset(c_idx, n_c);
        if (n_c && n_d && !getenv("WAVECELL_B200_NO_IMEX_OVERLAP") && op->set_step_split(c_idx, n_c)) {
            int lo_prio = 0, hi_prio = 0;
            WCB_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
            WCB_CUDA(cudaStreamCreateWithPriority(&P->s2, cudaStreamNonBlocking, lo_prio));   // lowest
            WCB_CUDA(cudaEventCreateWithFlags(&P->e_near, cudaEventDisableTiming));
            WCB_CUDA(cudaEventCreateWithFlags(&P->e_far, cudaEventDisableTiming));
            WCB_CUDA(cudaEventCreateWithFlags(&P->e_boot, cudaEventDisableTiming));
            P->split = true;
        }
        op->bind_minv(P->minv.p);                      // interior 1/m table for the d step
        // force vector for the d rows: dense window over its nonzeros
        {
            std::vector<std::pair<int64_t, double>> nz;
            for (int64_t i = 0; i < n; ++i)
                if (F_s[i] != 0.0) nz.emplace_back(si[i], F_s[i]);
            P->src = make_source(std::move(nz), P->F_win, s);
        }
        if (n_c) {
            WCB_REQUIRE(M_cc && M_cc->n == n_c && (!S_cc || S_cc->n == n_c), "LU factors of size n_c required");
            if (S_cc) {
                P->S.load(S_cc, s);
                P->has_S = true;
            }
            P->Mcc.load(M_cc, s);
        }
        if (obs && obs->n_obs > 0) {
            P->n_obs = obs->n_obs;
            const int64_t nnz = obs->indptr[obs->n_obs];
            std::vector<int64_t> sidx(std::max<int64_t>(nnz, 1));
            for (int64_t j = 0; j < nnz; ++j) {
                WCB_REQUIRE(obs->indices[j] >= 0 && obs->indices[j] < n, "observer column out of range");
                sidx[j] = si[obs->indices[j]];
            }
            P->obs_indptr.alloc(obs->n_obs + 1, s); P->obs_indptr.upload(obs->indptr, obs->n_obs + 1, s);
            P->obs_idx.alloc(sidx.size(), s); P->obs_idx.upload(sidx.data(), nnz, s);
            P->obs_val.alloc(std::max<int64_t>(nnz, 1), s); P->obs_val.upload(obs->data, nnz, s);
        }
        const int64_t m = std::max<int64_t>(n_c, 1);
        P->A.alloc(ns, s); P->B.alloc(ns, s); P->T.alloc(ns, s); P->V.alloc(ns, s);
        P->psi_c.alloc(m, s); P->v_c.alloc(m, s); P->a_c.alloc(m, s); P->pred.alloc(m, s); P->vpred.alloc(m, s);
        P->Kc.alloc(m, s); P->rhs.alloc(m, s); P->y.alloc(m, s); P->z.alloc(m, s);
        P->done.alloc(m, s);
        P->counter.alloc(2, s);
        P->amp_scratch.alloc(1, s);
        WCB_CUDA(cudaStreamSynchronize(s));
        ctx_retain(ctx);
        *out = P.release();
        return WCB_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    }
}

int wcb_imex_plan_destroy(wcb_imex_plan* plan) {
    if (!plan) return WCB_OK;
    Context* cx = plan->ctx;
    cudaSetDevice(cx->device);
    cudaStreamSynchronize(cx->stream);
    delete plan;
    ctx_release(cx);
    return WCB_OK;
}

}  // extern "C"

namespace wcb {

// The IMEX loop (src/timeint.py:196-292) for one plan, or for consecutive x
// slabs of one grid: plans sharing one context (emulated ranks, halos by
// device copies) or one plan per process with an NCCL communicator on its
// context.  The slab cuts leave every c patch and the cells around it inside
// one slab, so only the explicit d rows need the neighbours' halo rows: one
// exchange per step, after the corrector, exactly as in the CDM loop.
static void imex_run_group(std::vector<wcb_imex_plan*>& Ps, double f0, const double* ft_k,
                           const double* ft_new, double dt, int64_t n_t, double beta, double gamma,
                           const std::vector<const double*>& psi0, const std::vector<const double*>& v0,
                           const std::vector<double*>& psi_out, const std::vector<double*>& psi_dot_out,
                           const std::vector<double*>& obs_out, wcb_divergence* div, wcb_timings* tm,
                           bool cdm = false) {
    // cdm: cdm_run with the consistent mass blockdiag(diag(m_d), M_cc)
    // (src/timeint.py:159-193 through factorize()'s SuperLU path): the d rows
    // by the fused step, the c rows by rhs_c = f F_c - (K psi_k)_c and the M_cc
    // triangular solves; ft_k[k] = f(k dt) as in the IMEX d rows
    const size_t G = Ps.size();
    Context* ctx = Ps[0]->op->ctx;
    for (auto* P : Ps) WCB_REQUIRE(P->op->ctx == ctx, "group plans must share one context");
    WCB_REQUIRE(n_t >= 0, "negative n_t");
    if (!cdm)
        for (auto* P : Ps) WCB_REQUIRE(P->n_c == 0 || P->has_S, "plan has no S_cc factors (mass-only plan)");
    WCB_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    if (div) { div->step = -1; div->amplitude = 0.0; }
    if (tm) { tm->factorization = 0.0; tm->rhs = 0.0; tm->backward_insertion = 0.0; }
    std::vector<Operator*> ops;
    for (auto* P : Ps) ops.push_back(P->op);
    auto exchange = [&](const std::vector<double*>& st) {
        if (G == 1) {
            int64_t h[8];
            if (dist_slab(ops[0]) && ops[0]->halo(h))
                nccl_exchange_halo(ctx, st[0], h, ops[0]->halo_nplanes, ops[0]->halo_pstride);
        } else {
            copy_exchange_halo(ops, st, s);
        }
    };
    // force tables: index 0 = f(0) for the bootstrap; ft_k[k], ft_new[k] per step
    std::vector<double> hk(n_t + 1), hn(std::max<int64_t>(n_t, 1));
    hk[0] = f0;
    for (int64_t k = 0; k < n_t; ++k) { hk[k + 1] = ft_k[k]; hn[k] = ft_new[k]; }
    std::vector<DevBuf<double>> tmp(G), dobs(G);
    const int64_t stride = n_t + 1;
    std::vector<double*> cur(G), prev(G);
    for (size_t r = 0; r < G; ++r) {
        wcb_imex_plan* P = Ps[r];
        Operator* op = P->op;
        P->ft_k.alloc(hk.size(), s); P->ft_k.upload(hk.data(), hk.size(), s);
        P->ft_new.alloc(hn.size(), s); P->ft_new.upload(hn.data(), hn.size(), s);
        P->amp.alloc(n_t + 1, s);
        P->amp.zero(s);
        tmp[r].alloc(std::max<int64_t>(op->n, 1));
        P->A.zero(s); P->V.zero(s); P->B.zero(s); P->T.zero(s);
        if (psi0[r]) { tmp[r].upload(psi0[r], op->n, s); op->scatter(tmp[r].p, P->A.p); }
        if (v0[r]) { tmp[r].upload(v0[r], op->n, s); op->scatter(tmp[r].p, P->V.p); }
        if (P->n_obs && obs_out[r]) dobs[r].alloc(P->n_obs * stride, s);
        cur[r] = P->A.p;
        prev[r] = P->B.p;
    }
    // fault the outputs in while the loop runs (inputs are uploaded above)
    std::vector<std::unique_ptr<Prefault>> pfs;
    for (size_t r = 0; r < G; ++r)
        pfs.emplace_back(new Prefault(psi_out[r], Ps[r]->op->n * sizeof(double)));
    exchange(cur);   // psi_0 halos for the bootstrap apply
    for (size_t r = 0; r < G; ++r) {
        wcb_imex_plan* P = Ps[r];
        Operator* op = P->op;
        const int64_t ns = op->n_state, nc = P->n_c;
        // bootstrap (src/timeint.py:246-256)
        op->apply(P->A.p, P->T.p);
        k_imex_boot<<<grid1(ctx, ns), 256, 0, s>>>(ns, P->A.p, P->V.p, P->T.p, P->m_d_state.p, P->src,
                                                   P->ft_k.p, dt, P->B.p);
        ctx->launches++;
        if (nc > 0) {
            // r0_c = f0 F_c - (K psi)_c ; a_c = M_cc^-1 r0_c
            k_gather_rows<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->c_state.p, P->T.p, P->Kc.p);
            k_c_rhs<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->Fc.p, P->ft_k.p, 0, P->Kc.p, P->rhs.p);
            ctx->launches += 2;
            DevBuf<double> w(nc);
            lu_solve(ctx, P, P->Mcc, P->rhs.p, w.p);
            // a_c = w[perm_c]
            k_gather_rows<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->Mcc.perm_c.p, w.p, P->a_c.p);
            k_gather_rows<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->c_state.p, P->A.p, P->psi_c.p);
            k_gather_rows<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->c_state.p, P->V.p, P->v_c.p);
            ctx->launches += 3;
            if (cdm) {
                k_c_boot_prev<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->c_state.p, P->psi_c.p, P->v_c.p, P->a_c.p, dt,
                                                             0.5 * dt * dt, P->B.p);
                ctx->launches++;
            }
            WCB_CUDA(cudaStreamSynchronize(s));
        }
    }
    WCB_CHECK_LAUNCH();
    auto record = [&](size_t r, int64_t k, const double* psi) {
        wcb_imex_plan* P = Ps[r];
        if (!(P->n_obs && obs_out[r])) return;
        StepArgs o;
        o.cur = psi;
        o.k = k;
        o.n_obs = P->n_obs;
        o.obs_ptr = P->obs_indptr.p;
        o.obs_idx = P->obs_idx.p;
        o.obs_val = P->obs_val.p;
        o.obs_out = dobs[r].p;
        o.obs_stride = stride;
        launch_record_observers(ctx, o);
    };
    for (size_t r = 0; r < G; ++r) record(r, 0, Ps[r]->A.p);
    const double c1 = 0.5 * dt * dt * (1.0 - 2.0 * beta);
    const double c2 = dt * (1.0 - gamma);
    const double bdt2 = beta * dt * dt;
    const double gdt = gamma * dt;
    WCB_CUDA(cudaEventRecord(ctx->ev0, s));
    std::vector<unsigned long long> h_amp(G * (n_t + 1), 0ULL);
    int64_t checked = 0;
    bool diverged = false;
    auto inspect = [&](int64_t upto) -> bool {
        if (upto <= checked) return false;
        const int64_t cnt = upto - checked;
        for (size_t r = 0; r < G; ++r) {
            if (G == 1 && dist_slab(Ps[r]->op)) nccl_allreduce_max_u64(ctx, Ps[r]->amp.p + checked + 1, cnt);
            WCB_CUDA(cudaMemcpyAsync(h_amp.data() + r * (n_t + 1) + checked + 1, Ps[r]->amp.p + checked + 1,
                                     cnt * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        }
        WCB_CUDA(cudaStreamSynchronize(s));
        for (int64_t k = checked + 1; k <= upto; ++k) {
            unsigned long long bb = 0ULL;
            for (size_t r = 0; r < G; ++r) bb = std::max(bb, h_amp[r * (n_t + 1) + k]);
            double v;
            std::memcpy(&v, &bb, sizeof(v));
            if (!std::isfinite(v) || v > 1.0e12) {
                if (div) { div->step = k; div->amplitude = v; }
                return true;
            }
        }
        checked = upto;
        return false;
    };
    // Single plan, no NCCL: the explicit step is split into far tiles (input
    // footprint free of c DOFs) on a second stream and near tiles on the main
    // one; far(k+1) only needs step k's d values, so it runs while the c
    // chain of step k (c-row apply, triangular solves, corrector) runs:
    //   S0: near(k) -> [rec e_near] -> [wait e_far = far(k)] -> c chain(k)
    //   S1: [wait e_near(k)] -> far(k+1) -> [rec e_far]
    // far(k+1) writes psi_{k+2} over psi_k, read only by step k's explicit
    // tiles (done: e_near) -- the c chain reads and writes the other buffer.
    const bool overlap = !cdm && G == 1 && !dist_slab(Ps[0]->op) && Ps[0]->split;
    auto d_args = [&](wcb_imex_plan* P, int64_t k, double* c_, double* p_) {
        StepArgs a;
        a.minv = P->minv.p;
        a.F = P->src;
        a.dt2 = dt * dt;
        a.cur = c_;
        a.prev = p_;
        a.out = p_;
        a.ft = P->ft_k.p + 1;   // ft_k[k]
        a.k = k;
        a.amp = P->amp.p + (k + 1);
        return a;
    };
    auto launch_far = [&](wcb_imex_plan* P, const StepArgs& a) {
        cudaStream_t save = ctx->stream;
        ctx->stream = P->s2;
        try {
            P->op->cdm_step_part(a, 0);
        } catch (...) {
            ctx->stream = save;
            throw;
        }
        ctx->stream = save;
    };
    if (overlap && n_t > 0) {
        wcb_imex_plan* P = Ps[0];
        WCB_CUDA(cudaEventRecord(P->e_boot, s));
        WCB_CUDA(cudaStreamWaitEvent(P->s2, P->e_boot, 0));
        launch_far(P, d_args(P, 0, cur[0], prev[0]));
        WCB_CUDA(cudaEventRecord(P->e_far, P->s2));
    }
    for (int64_t k = 0; k < n_t; ++k) {
        for (size_t r = 0; r < G; ++r) {
            wcb_imex_plan* P = Ps[r];
            Operator* op = P->op;
            const int64_t ns = op->n_state, nc = P->n_c;
            if (cdm) {
                // d rows (and 2 psi - psi_prev in the c slots, 1/m = 0 there)
                StepArgs a = d_args(P, k, cur[r], prev[r]);
                if (nc > 0) a.amp = P->amp_scratch.p;   // amplitude taken below
                op->cdm_step(a);
                if (nc > 0) {
                    if (!op->apply_rows(cur[r], P->Kc.p)) {   // (K psi_k)_c
                        op->apply_subset(cur[r], P->T.p);
                        k_gather_rows<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->c_state.p, P->T.p, P->Kc.p);
                    }
                    k_c_rhs<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->Fc.p, P->ft_k.p + 1, k, P->Kc.p, P->rhs.p);
                    lu_solve(ctx, P, P->Mcc, P->rhs.p, P->y.p);
                    k_c_cdm_update<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->c_state.p, P->Mcc.perm_c.p, P->y.p,
                                                                  dt * dt, prev[r]);
                    // the fused step's amplitude saw the c slots before their
                    // update: take the step's amplitude over the final state
                    k_state_amp<<<grid1(ctx, ns), 256, 0, s>>>(ns, prev[r], P->amp.p + (k + 1));
                    ctx->launches += 4;
                }
                std::swap(cur[r], prev[r]);
                continue;
            }
            // 1. explicit d step into prev (c slots overwritten below)
            if (overlap) {
                op->cdm_step_part(d_args(P, k, cur[r], prev[r]), 1);
                WCB_CUDA(cudaEventRecord(P->e_near, s));
                WCB_CUDA(cudaStreamWaitEvent(s, P->e_far, 0));   // far(k) complete
            } else if (P->n_d > 0) {
                op->cdm_step(d_args(P, k, cur[r], prev[r]));
            } else {
                WCB_CUDA(cudaMemcpyAsync(prev[r], cur[r], ns * sizeof(double), cudaMemcpyDeviceToDevice, s));
            }
            if (nc > 0) {
                // 2. c predictor into the new state
                k_c_predict<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->c_state.p, P->psi_c.p, P->v_c.p, P->a_c.p,
                                                           dt, c1, c2, prev[r], P->pred.p, P->vpred.p);
                // 3. rhs_c with updated d and predicted c
                if (!op->apply_rows(prev[r], P->Kc.p)) {   // cells touching c rows only
                    op->apply_subset(prev[r], P->T.p);   // tiles owning c rows
                    k_gather_rows<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->c_state.p, P->T.p, P->Kc.p);
                }
                k_c_rhs<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->Fc.p, P->ft_new.p, k, P->Kc.p, P->rhs.p);
                ctx->launches += 3;
                // 4. a_c = S^-1 rhs_c (z permuted) ; 5. corrector
                lu_solve(ctx, P, P->S, P->rhs.p, P->y.p);   // result in y (column-permuted space)
                if (overlap && k + 1 < n_t) {
                    // far(k+1) enqueued behind the solves (their CTAs claim the
                    // SMs first; far tiles fill SMs the short patches free)
                    WCB_CUDA(cudaStreamWaitEvent(P->s2, P->e_near, 0));
                    launch_far(P, d_args(P, k + 1, prev[r], cur[r]));
                    WCB_CUDA(cudaEventRecord(P->e_far, P->s2));
                }
                k_c_correct<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->c_state.p, P->S.perm_c.p, P->y.p, P->pred.p,
                                                           P->vpred.p, bdt2, gdt, P->a_c.p, P->psi_c.p, P->v_c.p,
                                                           prev[r], P->amp.p + (k + 1));
                ctx->launches++;
            }
            std::swap(cur[r], prev[r]);
        }
        exchange(cur);
        for (size_t r = 0; r < G; ++r) record(r, k + 1, cur[r]);
        if ((k + 1) % 256 == 0) {
            WCB_CHECK_LAUNCH();
            if (inspect(k + 1)) { diverged = true; break; }
        }
    }
    if (overlap) WCB_CUDA(cudaStreamSynchronize(Ps[0]->s2));   // no far step left in flight
    WCB_CUDA(cudaEventRecord(ctx->ev1, s));
    WCB_CHECK_LAUNCH();
    if (!diverged) diverged = inspect(n_t);
    WCB_CUDA(cudaEventSynchronize(ctx->ev1));
    float ms = 0.f;
    WCB_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    if (tm) tm->rhs = ms * 1e-3;
    if (diverged) throw Error{WCB_E_DIVERGED, "solution diverged"};
    for (auto& pf : pfs) pf->join();
    for (size_t r = 0; r < G; ++r) {
        wcb_imex_plan* P = Ps[r];
        Operator* op = P->op;
        op->gather(cur[r], tmp[r].p);
        copy_d2h(psi_out[r], tmp[r].p, op->n * sizeof(double), s);
        // v_c in c order (the caller scatters it when d is empty, src/timeint.py:285-288)
        if (psi_dot_out[r] && P->n_c > 0 && !cdm)
            WCB_CUDA(cudaMemcpyAsync(psi_dot_out[r], P->v_c.p, P->n_c * sizeof(double), cudaMemcpyDeviceToHost, s));
        if (P->n_obs && obs_out[r]) {
            if (G == 1 && dist_slab(op)) nccl_allreduce_sum_f64(ctx, dobs[r].p, P->n_obs * stride);
            WCB_CUDA(cudaMemcpyAsync(obs_out[r], dobs[r].p, P->n_obs * stride * sizeof(double),
                                     cudaMemcpyDeviceToHost, s));
        }
    }
    WCB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace wcb

extern "C" {

int wcb_imex_plan_run(wcb_imex_plan* P, double f0, const double* ft_k, const double* ft_new,
                      double dt, int64_t n_t, double beta, double gamma, const double* psi0,
                      const double* v0, double* psi_out, double* psi_dot_out, double* obs_out,
                      wcb_divergence* div, wcb_timings* tm) {
    try {
        WCB_REQUIRE(P && psi_out, "NULL argument");
        std::vector<wcb_imex_plan*> Ps{P};
        imex_run_group(Ps, f0, ft_k, ft_new, dt, n_t, beta, gamma, {psi0}, {v0}, {psi_out}, {psi_dot_out},
                       {obs_out}, div, tm);
        return WCB_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    }
}

int wcb_imex_group_run(int n_plans, wcb_imex_plan** plans, double f0, const double* ft_k,
                       const double* ft_new, double dt, int64_t n_t, double beta, double gamma,
                       double** psi_out, double** psi_dot_out, double** obs_out,
                       wcb_divergence* div, wcb_timings* tm) {
    try {
        WCB_REQUIRE(n_plans >= 1 && plans && psi_out, "NULL argument");
        std::vector<wcb_imex_plan*> Ps(plans, plans + n_plans);
        for (auto* P : Ps) WCB_REQUIRE(P, "NULL plan");
        std::vector<const double*> none(n_plans, nullptr);
        std::vector<double*> po(psi_out, psi_out + n_plans), pd(n_plans, nullptr), ob(n_plans, nullptr);
        if (psi_dot_out) pd.assign(psi_dot_out, psi_dot_out + n_plans);
        if (obs_out) ob.assign(obs_out, obs_out + n_plans);
        imex_run_group(Ps, f0, ft_k, ft_new, dt, n_t, beta, gamma, none, none, po, pd, ob, div, tm);
        return WCB_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    }
}


int wcb_mass_plan_create(wcb_operator* K, int64_t n_c, const int64_t* c_idx, int64_t n_d,
                         const int64_t* d_idx, const double* m_d, const wcb_lu* M_cc,
                         const int64_t* Mcc_indptr, const int32_t* Mcc_indices, const double* Mcc_data,
                         const double* F_s, const wcb_observer* obs, wcb_imex_plan** out) {
    try {
        WCB_REQUIRE(out && (n_c == 0 || (M_cc && Mcc_indptr && Mcc_indices && Mcc_data)), "NULL argument");
        wcb_imex_plan* P = nullptr;
        const int rc = wcb_imex_plan_create(K, n_c, c_idx, n_d, d_idx, m_d, nullptr, M_cc, F_s, obs, &P);
        if (rc != WCB_OK) return rc;
        std::unique_ptr<wcb_imex_plan, int (*)(wcb_imex_plan*)> guard(P, wcb_imex_plan_destroy);
        if (n_c > 0) {
            cudaStream_t s = P->ctx->stream;
            const int64_t nnz = Mcc_indptr[n_c];
            for (int64_t j = 0; j < nnz; ++j)
                WCB_REQUIRE(Mcc_indices[j] >= 0 && Mcc_indices[j] < n_c, "M_cc column out of range");
            P->mcc_ptr.alloc(n_c + 1, s); P->mcc_ptr.upload(Mcc_indptr, n_c + 1, s);
            P->mcc_idx.alloc(std::max<int64_t>(nnz, 1), s); P->mcc_idx.upload(Mcc_indices, nnz, s);
            P->mcc_val.alloc(std::max<int64_t>(nnz, 1), s); P->mcc_val.upload(Mcc_data, nnz, s);
            P->has_mcc_csr = true;
            WCB_CUDA(cudaStreamSynchronize(s));
        }
        *out = guard.release();
        return WCB_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    }
}

int wcb_imex_plan_cdm_run(wcb_imex_plan* P, const double* ft, double dt, int64_t n_t, const double* psi0,
                          const double* v0, double* psi_out, double* obs_out, wcb_divergence* div,
                          wcb_timings* tm) {
    try {
        WCB_REQUIRE(P && psi_out && (ft || n_t == 0), "NULL argument");
        std::vector<double> f(std::max<int64_t>(n_t, 1), 0.0);
        if (n_t > 0) std::memcpy(f.data(), ft, n_t * sizeof(double));
        const double f0 = f[0];
        std::vector<wcb_imex_plan*> Ps{P};
        imex_run_group(Ps, f0, f.data(), f.data(), dt, n_t, 0.0, 0.5, {psi0}, {v0}, {psi_out}, {nullptr},
                       {obs_out}, div, tm, true);
        return WCB_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    }
}

int wcb_imex_plan_max_gen_eig(wcb_imex_plan* P, const double* x0, double tol, int64_t max_iter,
                              double* lam, int64_t* n_iter) {
    try {
        WCB_REQUIRE(P && x0 && lam && n_iter, "NULL argument");
        WCB_REQUIRE(P->n_c == 0 || P->has_mcc_csr, "plan has no M_cc matrix (use wcb_mass_plan_create)");
        Operator* op = P->op;
        Context* ctx = P->ctx;
        WCB_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        const int64_t n = op->n, nc = P->n_c;
        // m_diag in compact order: m_d at the d rows, 1 at the c rows
        std::vector<double> md_state(op->n_state), m(n, 1.0);
        WCB_CUDA(cudaMemcpyAsync(md_state.data(), P->m_d_state.p, op->n_state * sizeof(double),
                                 cudaMemcpyDeviceToHost, s));
        WCB_CUDA(cudaStreamSynchronize(s));
        const std::vector<int64_t>& si = op->state_index();
        for (int64_t i = 0; i < n; ++i)
            if (md_state[si[i]] > 0.0) m[i] = md_state[si[i]];
        MassHooks hooks;
        if (nc > 0) {
            hooks.solve_c = [&](const double* t, double* y) {
                k_gather_rows<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->c_state.p, t, P->rhs.p);
                lu_solve(ctx, P, P->Mcc, P->rhs.p, P->a_c.p);
                k_scatter_rows<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->c_state.p, P->Mcc.perm_c.p, P->a_c.p, y);
                ctx->launches += 2;
            };
            hooks.apply_c = [&](const double* x, double* mx) {
                k_gather_rows<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->c_state.p, x, P->rhs.p);
                k_csr_rows<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->mcc_ptr.p, P->mcc_idx.p, P->mcc_val.p, P->rhs.p,
                                                          P->Kc.p);
                k_scatter_rows<<<grid1(ctx, nc), 256, 0, s>>>(nc, P->c_state.p, nullptr, P->Kc.p, mx);
                ctx->launches += 3;
            };
        } else {
            hooks.solve_c = [](const double*, double*) {};
            hooks.apply_c = [](const double*, double*) {};
        }
        max_gen_eig_core(op, m.data(), x0, tol, max_iter, lam, n_iter, &hooks);
        return WCB_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    }
}

}  // extern "C"
