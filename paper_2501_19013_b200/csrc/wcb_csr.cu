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
        for (int64_t j = b + lane; j < e; j += TPR) s += __ldg(data + j) * __ldg(x + __ldg(indices + j));
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
    double Ku = row_dot<TPR>(indptr, indices, data, a.cur, row, lane, valid);
    unsigned long long amp = 0ULL;
    if (valid && lane == 0) {
        const double f = a.ft[a.k];
        const double u = a.cur[row];
        const double up = a.prev[row];
        const double mi = a.minv[row];
        const double v = leapfrog(u, up, Ku, mi, f * source_at(a.F, row), a.dt2);
        a.out[row] = v;
        amp = mi != 0.0 ? amp_bits(v) : 0ULL;
    }
    block_amp_max<BLOCK>(amp, a.amp);
}

struct CsrOperator final : Operator {
    DevBuf<int64_t> indptr;
    DevBuf<int32_t> indices;
    DevBuf<double> data;
    DevBuf<int64_t> ident;  // identity map (state == compact)
    std::vector<int64_t> sidx;
    int64_t nnz = 0;
    int tpr = 8;

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
    const double mean = n ? (double)nnz / (double)n : 0.0;
    int t = 1;
    while (t < 32 && t < mean) t <<= 1;
    // a few lanes idle is cheaper than a serial tail per lane
    op->tpr = std::max(1, std::min(32, t));
    WCB_CUDA(cudaStreamSynchronize(s));
    return op;
}

}  // namespace wcb
