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


// 3D launch description (wcb_scm3d.cu)
struct Scm3DGeo {
    int64_t n_ex;             // local x cell rows (incl. the halo row 0)
    int64_t row_lo, row_hi;   // owned local x node planes
    int64_t n_e;              // cells along y and z
    int64_t n1;               // nodes along y and z
    int64_t prow;             // row pitch (doubles, z fastest)
    int64_t pplane;           // plane pitch (doubles)
    const uint8_t* mask;      // (n_e+2)^3 cell codes with a ring of 0: 0 out, 1 uncut, 2 cut
    const int32_t* cut_id;    // n_e^3 -> cut index or -1
    const double* KT;         // unused in 3D (cut products come from cut_out)
    const double* cut_out;    // n_cut * L: K_o u_e / sk of every cut cell (k_cut_pre)
    const uint8_t* cflags;    // per CTA tile (z strip, y row, x tile): owns a DOF
    int64_t n_zs;             // z strips
    int64_t n_xt;             // x tiles
};

__host__ __device__ constexpr int rx_for3(int P) { return P <= 3 ? 4 : 2; }

// box of the 3D psi tile (z, y, x extents)
template <int P>
struct Tile3 {
    static constexpr int RX = rx_for3(P);          // x element rows per CTA (+1 halo warp)
    static constexpr int NWARP = RX + 1;
    static constexpr int TZ = 32 * P;               // owned node columns (z)
    static constexpr int CO = P & 1;                // 16-byte TMA alignment offset
    static constexpr int UW = ((TZ + P + 1 + CO) + 1) / 2 * 2;
    static constexpr int UR = 2 * P + 1;            // y rows (ey-1)*P .. ey*P+P
    static constexpr int UP = RX * P + P + 1;       // x planes (ex0-1)*P .. (ex0+RX)*P
    static constexpr size_t U_BYTES = (size_t)UW * UR * UP * 8;
    static constexpr size_t OFF_CARRY = (U_BYTES + 127) / 128 * 128;   // [RX+1][P*P][32]
    static constexpr size_t OFF_BAR = OFF_CARRY + (size_t)(RX + 1) * P * P * 32 * 8;
    static constexpr size_t SMEM = OFF_BAR + 8;
};

template <int P, int MODE>
void launch_scm3d(Context* ctx, const CUtensorMap& map_u, const Scm3DGeo& g, const Mats2<P>& mt,
                  double sk, const StepArgs& a);
// dense cut-cell products u_e -> K_o u_e / sk (packed symmetric K), before the stencil
template <int P>
void launch_cut_pre(Context* ctx, int64_t n_cut, const double* KP, const int64_t* cut_base,
                    int64_t pplane, int64_t prow, const double* u, double* out);

}  // namespace wcb
