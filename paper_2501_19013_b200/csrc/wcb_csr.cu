// CSR stiffness operator: the generic / IGA B-spline path (K from
// src/assembly.py:518-612, applied at src/timeint.py:175,182).
//
// One row per group of TPR lanes (TPR chosen from the mean row length).  The
// group reduces its partial sums with a fixed shuffle tree, so results are
// bitwise reproducible run to run (src/harness.py:462-485 contract).  The CDM
// variant fuses the diagonal-mass leapfrog update, the force and the
// divergence amplitude into the same pass (one HBM pass per step).
#include "wcb_internal.cuh"

#include <algorithm>
#include <numeric>

namespace wcb {

template <int TPR>
__device__ __forceinline__ double row_dot(const int64_t* __restrict__ indptr,
                                          const int32_t* __restrict__ indices,
                                          const double* __restrict__ data,
                                          const double* __restrict__ x, int64_t row, int lane,
                                          bool valid) {
    double s = 0.0;
    if (valid) {
        const int64_t b = indptr[row], e = indptr[row + 1];
        #pragma unroll 4
        for (int64_t j = b + lane; j < e; j += TPR) s = fma(__ldg(data + j), __ldg(x + __ldg(indices + j)), s);
    }
    #pragma unroll
    for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, TPR);
    return s;
}

template <int TPR, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_csr_apply(int64_t n, const int64_t* __restrict__ indptr,
                                                     const int32_t* __restrict__ indices,
                                                     const double* __restrict__ data,
                                                     const double* __restrict__ x,
                                                     double* __restrict__ y) {
    const int64_t row = (blockIdx.x * (int64_t)BLOCK + threadIdx.x) / TPR;
    const int lane = threadIdx.x % TPR;
    const bool valid = row < n;
    double s = row_dot<TPR>(indptr, indices, data, x, row, lane, valid);
    if (valid && lane == 0) y[row] = s;
}

template <int TPR, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_csr_cdm(int64_t n, const int64_t* __restrict__ indptr,
                                                   const int32_t* __restrict__ indices,
                                                   const double* __restrict__ data, StepArgs a) {
    if (blockIdx.x == 0) record_observers(a);
    const int64_t row = (blockIdx.x * (int64_t)BLOCK + threadIdx.x) / TPR;
    const int lane = threadIdx.x % TPR;
    const bool valid = row < n;
    // epilogue operands first: their latency overlaps the row's dot product
    double u = 0.0, up = 0.0, mi = 0.0;
    if (valid && lane == 0) {
        u = __ldg(a.cur + row);
        up = a.prev[row];
        mi = __ldg(a.minv + row);
    }
    double Ku = row_dot<TPR>(indptr, indices, data, a.cur, row, lane, valid);
    unsigned long long amp = 0ULL;
    if (valid && lane == 0) {
        const double f = a.ft[a.k];
        const double v = leapfrog(u, up, Ku, mi, f * source_at(a.F, row), a.dt2);
        a.out[row] = v;
        amp = mi != 0.0 ? amp_bits(v) : 0ULL;
    }
    block_amp_max<BLOCK>(amp, a.amp);
}

// SELL-32: slices of 32 consecutive rows stored column-major (entry k of row
// r in slice s at sptr[s] + 32 k + r), one row per thread: every load of a
// warp is one contiguous 256 B (values) / 128 B (indices) segment.  Padding
// entries point at the row itself with value 0.  Row sums run in stored
// order (the CSR order), so results equal the CSR-vector kernel's up to
// summation order and are bitwise reproducible.
template <bool STEP>
__global__ void __launch_bounds__(256) k_sell(int64_t n, const int64_t* __restrict__ sptr,
                                              const int32_t* __restrict__ swid,
                                              const int32_t* __restrict__ sidx,
                                              const double* __restrict__ sval,
                                              const double* __restrict__ x, double* __restrict__ y,
                                              StepArgs a) {
    if (STEP && blockIdx.x == 0) record_observers(a);
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid = row < n;
    const int64_t s = row >> 5;
    const int r = (int)(row & 31);
    double u = 0.0, up = 0.0, mi = 0.0;
    if (STEP && valid) {
        u = __ldg(a.cur + row);
        up = a.prev[row];
        mi = __ldg(a.minv + row);
    }
    double acc = 0.0;
    if (valid) {
        const int w = __ldg(swid + s);
        const int64_t base = __ldg(sptr + s) + r;
        #pragma unroll 8
        for (int k = 0; k < w; ++k) {
            const int64_t j = base + 32 * (int64_t)k;
            acc = fma(__ldg(sval + j), __ldg(x + __ldg(sidx + j)), acc);
        }
    }
    if constexpr (STEP) {
        unsigned long long amp = 0ULL;
        if (valid) {
            const double f = a.ft[a.k];
            const double v = leapfrog(u, up, acc, mi, f * source_at(a.F, row), a.dt2);
            a.out[row] = v;
            amp = mi != 0.0 ? amp_bits(v) : 0ULL;
        }
        block_amp_max<256>(amp, a.amp);
    } else {
        if (valid) y[row] = acc;
    }
}

struct CsrOperator final : Operator {
    DevBuf<int64_t> indptr;
    DevBuf<int32_t> indices;
    DevBuf<double> data;
    DevBuf<int64_t> ident;  // identity map (state == compact)
    std::vector<int64_t> sidx;
    int64_t nnz = 0;
    int tpr = 8;
    bool sell = false;
    DevBuf<int64_t> s_ptr;
    DevBuf<int32_t> s_wid, s_idx;
    DevBuf<double> s_val;

    const char* name() const override { return "csr"; }
    const std::vector<int64_t>& state_index() const override { return sidx; }

    void scatter(const double* src, double* dst) override {
        if (n) WCB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice,
                                        ctx->stream));
    }
    void gather(const double* src, double* dst) override { scatter(src, dst); }

    template <int TPR>
    void apply_t(const double* x, double* y) {
        constexpr int B = 256;
        const int64_t rows_per_block = B / TPR;
        const int64_t g = ceil_div(n, rows_per_block);
        k_csr_apply<TPR, B><<<(unsigned)g, B, 0, ctx->stream>>>(n, indptr.p, indices.p, data.p, x, y);
        ctx->launches++;
    }
    template <int TPR>
    void step_t(const StepArgs& a) {
        constexpr int B = 256;
        const int64_t rows_per_block = B / TPR;
        const int64_t g = ceil_div(n, rows_per_block);
        k_csr_cdm<TPR, B><<<(unsigned)g, B, 0, ctx->stream>>>(n, indptr.p, indices.p, data.p, a);
        ctx->launches++;
    }
    void apply(const double* x, double* y) override {
        if (!n) return;
        if (sell) {
            StepArgs a;
            k_sell<false><<<(unsigned)ceil_div(n, 256), 256, 0, ctx->stream>>>(n, s_ptr.p, s_wid.p, s_idx.p,
                                                                               s_val.p, x, y, a);
            ctx->launches++;
            WCB_CHECK_LAUNCH();
            return;
        }
        switch (tpr) {
            case 1: apply_t<1>(x, y); break;
            case 2: apply_t<2>(x, y); break;
            case 4: apply_t<4>(x, y); break;
            case 8: apply_t<8>(x, y); break;
            case 16: apply_t<16>(x, y); break;
            default: apply_t<32>(x, y); break;
        }
        WCB_CHECK_LAUNCH();
    }
    void cdm_step(const StepArgs& a) override {
        if (!n) return;
        if (sell) {
            k_sell<true><<<(unsigned)ceil_div(n, 256), 256, 0, ctx->stream>>>(n, s_ptr.p, s_wid.p, s_idx.p,
                                                                              s_val.p, a.cur, nullptr, a);
            ctx->launches++;
            WCB_CHECK_LAUNCH();
            return;
        }
        switch (tpr) {
            case 1: step_t<1>(a); break;
            case 2: step_t<2>(a); break;
            case 4: step_t<4>(a); break;
            case 8: step_t<8>(a); break;
            case 16: step_t<16>(a); break;
            default: step_t<32>(a); break;
        }
        WCB_CHECK_LAUNCH();
    }
    // 12 B/nnz (fp64 value + int32 index) + 8 B indptr (int64 here)
    // + psi_k, psi_{k-1} read, psi_{k+1} write, 1/m read.
    double step_bytes() const override { return 12.0 * nnz + 8.0 * (n + 1) + 32.0 * n; }
};

Operator* make_csr_operator(Context* ctx, int64_t n, const int64_t* h_indptr,
                            const int32_t* h_indices, const double* h_data) {
    WCB_REQUIRE(h_indptr != nullptr, "indptr is NULL");
    WCB_REQUIRE(h_indptr[0] == 0, "indptr[0] must be 0");
    const int64_t nnz = h_indptr[n];
    WCB_REQUIRE(nnz >= 0, "negative nnz");
    WCB_REQUIRE(nnz == 0 || (h_indices && h_data), "indices/data NULL");
    for (int64_t i = 0; i < n; ++i)
        WCB_REQUIRE(h_indptr[i + 1] >= h_indptr[i], "indptr not monotone");
    for (int64_t j = 0; j < nnz; ++j)
        WCB_REQUIRE(h_indices[j] >= 0 && h_indices[j] < n, "column index out of range");
    auto* op = new CsrOperator();
    op->ctx = ctx;
    op->n = n;
    op->n_state = n;
    op->nnz = nnz;
    cudaStream_t s = ctx->stream;
    op->indptr.alloc(n + 1);
    op->indptr.upload(h_indptr, n + 1, s);
    op->indices.alloc(std::max<int64_t>(nnz, 1));
    op->indices.upload(h_indices, nnz, s);
    op->data.alloc(std::max<int64_t>(nnz, 1));
    op->data.upload(h_data, nnz, s);
    op->sidx.resize(n);
    std::iota(op->sidx.begin(), op->sidx.end(), (int64_t)0);
    // ~6 entries per lane: several rows per warp keep independent load chains
    // in flight (one row per warp is latency-bound at ~50 nnz/row)
    const double mean = n ? (double)nnz / (double)n : 0.0;
    int t = 1;
    while (t < 32 && t * 6 < mean) t <<= 1;
    op->tpr = std::max(1, std::min(32, t));
    // SELL-32 copy when padding stays small (regular stencil rows, e.g. IGA)
    const int64_t n_sl = ceil_div(n, 32);
    std::vector<int64_t> sp(n_sl + 1, 0);
    std::vector<int32_t> sw(std::max<int64_t>(n_sl, 1), 0);
    for (int64_t sl = 0; sl < n_sl; ++sl) {
        int64_t w = 0;
        for (int64_t r = sl * 32; r < std::min(n, sl * 32 + 32); ++r)
            w = std::max(w, h_indptr[r + 1] - h_indptr[r]);
        sw[sl] = (int32_t)w;
        sp[sl + 1] = sp[sl] + 32 * w;
    }
    if (n >= 32 && sp[n_sl] <= nnz + nnz / 4 && nnz > 0) {
        std::vector<int32_t> si(sp[n_sl]);
        std::vector<double> sv(sp[n_sl], 0.0);
        for (int64_t sl = 0; sl < n_sl; ++sl)
            for (int64_t r = sl * 32; r < sl * 32 + 32; ++r)
                for (int64_t k = 0; k < sw[sl]; ++k) {
                    const int64_t dst = sp[sl] + 32 * k + (r - sl * 32);
                    const int64_t src = r < n ? h_indptr[r] + k : -1;
                    if (r < n && src < h_indptr[r + 1]) {
                        si[dst] = h_indices[src];
                        sv[dst] = h_data[src];
                    } else {
                        si[dst] = (int32_t)std::min<int64_t>(r, n - 1);
                        sv[dst] = 0.0;
                    }
                }
        op->s_ptr.alloc(sp.size()); op->s_ptr.upload(sp.data(), sp.size(), s);
        op->s_wid.alloc(sw.size()); op->s_wid.upload(sw.data(), sw.size(), s);
        op->s_idx.alloc(si.size()); op->s_idx.upload(si.data(), si.size(), s);
        op->s_val.alloc(sv.size()); op->s_val.upload(sv.data(), sv.size(), s);
        op->sell = true;
    }
    WCB_CUDA(cudaStreamSynchronize(s));
    return op;
}

}  // namespace wcb
