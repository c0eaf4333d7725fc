// Shared pieces of the matrix-free spectral-cell kernels (2D and 3D).
#pragma once

#include "wcb_internal.cuh"
#include "wcb_tma.cuh"

namespace wcb {

constexpr int PADJ = 32;   // left padding (doubles) of the fastest axis in the state layout

enum { MODE_STEP = 0, MODE_APPLY = 1 };

// The 1D GLL-Lagrange factors m1, k1 are symmetric and centro-symmetric
// (A[i][j] = A[j][i] = A[P-i][P-j]); only one value per orbit is kept, so all
// coefficients of the sum factorisation fit in registers.  sk is applied once
// per output node: sk (k1 (x) m1 + m1 (x) k1) u = sk * [k1 (x) m1 + m1 (x) k1] u.
__host__ __device__ constexpr int orb_key(int P, int i, int j) {
    // canonical representative: lexicographically smallest of the 4 images
    int a0 = i * 16 + j, a1 = j * 16 + i, a2 = (P - i) * 16 + (P - j), a3 = (P - j) * 16 + (P - i);
    int m = a0 < a1 ? a0 : a1;
    m = m < a2 ? m : a2;
    return m < a3 ? m : a3;
}
__host__ __device__ constexpr int orb_count(int P) {
    int n = 0;
    for (int i = 0; i <= P; ++i)
        for (int j = 0; j <= P; ++j)
            if (orb_key(P, i, j) == i * 16 + j) ++n;
    return n;
}
__host__ __device__ constexpr int orb(int P, int i, int j) {
    const int key = orb_key(P, i, j);
    int n = 0;
    for (int a = 0; a <= P; ++a)
        for (int b = 0; b <= P; ++b)
            if (orb_key(P, a, b) == a * 16 + b) {
                if (a * 16 + b == key) return n;
                ++n;
            }
    return -1;
}

template <int P>
struct Mats2 {
    double m[orb_count(P)];   // m1 orbit representatives
    double k[orb_count(P)];   // k1 orbit representatives
};


// 3D launch description (wcb_scm3d.cu).  A CTA owns one z strip (32 cells,
// lane = z cell) x WY y cell rows (one warp each) x one chunk of x cell rows,
// and streams node planes along x through a TMA ring.
struct Scm3DGeo {
    int64_t n_ex;             // local x cell rows (incl. the halo row 0)
    int64_t row_lo, row_hi;   // owned local x node planes
    int64_t n_e;              // cells along y and z
    int64_t n1;               // nodes along y and z
    int64_t prow;             // row pitch (doubles, z fastest)
    int64_t pplane;           // plane pitch (doubles)
    const uint8_t* mask;      // (n_ex+2)(n_e+2)^2 cell codes with a ring of 0: 0 out, 1 uncut, 2 cut
    const int32_t* cut_id;    // n_ex n_e^2 -> cut index or -1
    const double* cut_out;    // n_cut * L: K_o u_e / sk of every cut cell (k_cut_pre)
    const uint8_t* cflags;    // per CTA (x chunk, y block, z strip): owns a DOF
    int64_t n_zs;             // z strips
    int64_t n_yb;             // y blocks
    int64_t n_xc;             // x chunks
    int64_t xc;               // x cell rows per chunk
    int64_t ex_last;          // last local x cell row holding an owned node plane
    // non-null: `mask` carries the 1/m class of every cell in bits 2-3
    // (k_clean3d, once per plan: 1 = the P^3 owned nodes all carry the interior
    // 1/m of minv_tab, bitwise -- the epilogue skips the 1/m stream there;
    // 2 / 3 = 1/m is +0 on every owned node -- 2: the slots are not DOFs and are
    // left untouched, 3: they are stored (implicit rows of an IMEX plan)).
    // null: every node loads 1/m.
    const uint8_t* clean;
    double2* zline;           // (n_ex P + 1) x n1 z-lines of the last cell column (n_e % 32 == 0)
    int64_t xc0 = 0;          // first x chunk of this launch (blockIdx.z + xc0)
};

template <int P>
struct MinvTab {
    double v[P * P * P];   // (a, b, j) of the owned nodes of an interior uncut cell
};

// Streaming tile shape per degree: WY compute warps + 1 (halo y row and TMA
// producer); ring of S node planes = the P+1 planes of the current cell row
// plus LA planes of look-ahead.
#ifndef WCB3D_REUSE
#define WCB3D_REUSE 1
#endif
#ifndef WCB3D_WY3
#define WCB3D_WY3 7
#endif
__host__ __device__ constexpr int wy_for3(int P) { return P <= 2 ? 7 : P == 3 ? WCB3D_WY3 : 2; }
// resident CTAs per SM the launch bounds ask for
__host__ __device__ constexpr int cpsm_for3(int P) { return P == 3 && WCB3D_WY3 >= 7 ? 1 : P <= 3 ? 2 : 1; }
__host__ __device__ constexpr int la_for3(int P) { return P <= 3 ? P : 1; }

template <int P>
struct Str3 {
    static constexpr int WY = wy_for3(P);
    static constexpr int NWARP = WY + 1;            // one warp per y cell row + the halo warp
    static constexpr int TZ = 32 * P;               // owned node columns (z)
    static constexpr int CO = P & 1;                // 16-byte TMA alignment offset
    static constexpr int UW = ((TZ + P + 1 + CO) + 1) / 2 * 2;
    static constexpr int UR = (WY + 1) * P + 1;     // y rows (ey0-1)*P .. (ey0+WY)*P
    static constexpr int PLANE = UW * UR;           // doubles per ring slot
    static constexpr int S = P + 1 + la_for3(P);    // ring slots
    static constexpr int SLOT = (PLANE * 8 + 127) / 128 * 128 / 8;   // slot stride (doubles, 128 B aligned)
    static constexpr size_t RING_BYTES = (size_t)S * SLOT * 8;
    static constexpr size_t OFF_XCH = (RING_BYTES + 127) / 128 * 128;   // [NWARP][P+1][P or 1][32]
    static constexpr size_t OFF_PREV = OFF_XCH + (size_t)NWARP * (P + 1) * P * 32 * 8;   // [P][WY*P][TZ]
    static constexpr size_t PREV_BYTES = (size_t)P * WY * P * TZ * 8;
    static constexpr size_t OFF_BAR = OFF_PREV + (PREV_BYTES + 127) / 128 * 128;
    // mbarriers: full[S], prev, rowdone, xfull[NWARP], xempty[NWARP]
    static constexpr size_t OFF_TAB = OFF_BAR + 8 * (S + 2 + 2 * NWARP);   // interior 1/m table [P][P][P]
    static constexpr int CODE_W = 36;                                      // cells ez0-1 .. ez0+31 (+ pad)
    static constexpr size_t OFF_CODE = OFF_TAB + 8 * P * P * P;            // cell codes [2][WY+1][CODE_W]
    static constexpr size_t OFF_XTAB = (OFF_CODE + 2 * (WY + 1) * CODE_W + 15) / 16 * 16;   // x pass factors [P+1][2][P+1]
    static constexpr size_t SMEM = OFF_XTAB + 8 * 2 * (P + 1) * (P + 1);
};

// part: -1 all x chunks (+ z column kernels); 0 the first and last chunk
// (+ z column kernels); 1 the chunks in between
template <int P, int MODE>
void launch_scm3d(Context* ctx, const CUtensorMap& map_u, const CUtensorMap& map_p, const Scm3DGeo& g,
                  const Mats2<P>& mt, const MinvTab<P>& mtab, double sk, const StepArgs& a, int part = -1);
// clean[c] = 1/m class of local cell c (1: minv == tab bitwise on every owned
// node, 2 / 3: 1/m == 0 on every owned node, dead / stored); cinfo = mask with the class in bits 2-3
template <int P>
void launch_clean3d(Context* ctx, const Scm3DGeo& g, const MinvTab<P>& tab, const double* minv, uint8_t* clean,
                    uint8_t* cinfo, bool zero_is_dead);
// packed lower triangle of a cut cell's K_o / sk, stride padded to 16 bytes
__host__ __device__ constexpr int cut_lp_stride(int P) {
    return (((P + 1) * (P + 1) * (P + 1)) * (((P + 1) * (P + 1) * (P + 1)) + 1) / 2 + 1) / 2 * 2;
}
// dense cut-cell products u_e -> K_o u_e / sk (packed symmetric K), before the stencil
template <int P>
void launch_cut_pre(Context* ctx, int64_t n_cut, const double* KP, const int64_t* cut_base,
                    int64_t pplane, int64_t prow, const double* u, double* out);

}  // namespace wcb
