// Eigenvalue stabilisation of cut-cell mass matrices:
// batched cyclic-Jacobi eigensolver and the EVS update on the device.
//
// Reference: jacobi_eig src/linalg.py:133-212 (row-cyclic sweeps, the
// (tau, t, c, s) rotation with hypot, columns then rows then V, stop when
// max |off-diagonal| <= tol * max |A|), evs_stabilize
// src/stabilization.py:73-102 (projector onto the eigenvectors whose
// eigenvalue is below f_lambda * lambda_max, scaled to max |M_f|, weight
// epsilon).  One CTA per matrix, matrix and eigenvectors in shared memory;
// the rotation sequence is the reference's, so the results agree to
// rounding.
#include "wcb_internal.cuh"

#include <cmath>
#include <cstring>

namespace wcb {

// A: n x L x L (overwritten by the rotated matrix), lam: n x L ascending,
// V: n x L x L (eigenvectors as columns, same order).  status[b] = sweeps
// used, or -1 when max_sweeps was not enough.
__global__ void k_jacobi_batch(int64_t n, int L, double* __restrict__ Ag, double* __restrict__ lam,
                               double* __restrict__ Vg, int max_sweeps, double tol, int* __restrict__ status) {
    extern __shared__ double sm[];
    double* A = sm;              // L x L
    double* V = sm + L * L;      // L x L
    __shared__ double cs[2][2];   // (c, s) by rotation parity: thread 0 writes the next
    __shared__ int flag[2];       // rotation's while slow threads read this one's
    __shared__ double red[32];
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int64_t b = blockIdx.x; b < n; b += gridDim.x) {
        const double* Ab = Ag + b * L * L;
        // symmetrise, V = I
        for (int e = tid; e < L * L; e += nt) {
            const int i = e / L, j = e % L;
            A[e] = 0.5 * (Ab[i * L + j] + Ab[j * L + i]);
            V[e] = i == j ? 1.0 : 0.0;
        }
        __syncthreads();
        auto block_max = [&](bool offdiag) {
            double m = 0.0;
            for (int e = tid; e < L * L; e += nt)
                if (!offdiag || (e / L) != (e % L)) m = fmax(m, fabs(A[e]));
            for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            if ((tid & 31) == 0) red[tid >> 5] = m;
            __syncthreads();
            if (tid == 0) {
                double r = 0.0;
                for (int w = 0; w < (nt + 31) / 32; ++w) r = fmax(r, red[w]);
                red[0] = r;
            }
            __syncthreads();
            const double r = red[0];
            __syncthreads();
            return r;
        };
        double scale = block_max(false);
        if (scale == 0.0) scale = 1.0;
        int sweeps = -1;
        for (int sw = 0; sw <= max_sweeps; ++sw) {
            if (block_max(true) <= tol * scale) { sweeps = sw; break; }
            if (sw == max_sweeps) break;
            int rot = 0;
            for (int p = 0; p < L - 1; ++p)
                for (int q = p + 1; q < L; ++q, ++rot) {
                    const int par = rot & 1;
                    if (tid == 0) {
                        const double apq = A[p * L + q];
                        flag[par] = fabs(apq) > 1e-300;
                        if (flag[par]) {
                            const double tau = (A[q * L + q] - A[p * L + p]) / (2.0 * apq);
                            const double sg = (tau + (tau == 0.0 ? 1.0 : 0.0)) >= 0.0 ? 1.0 : -1.0;
                            const double t = sg / (fabs(tau) + hypot(1.0, tau));
                            const double c = 1.0 / sqrt(1.0 + t * t);
                            cs[par][0] = c;
                            cs[par][1] = t * c;
                        }
                    }
                    __syncthreads();
                    if (!flag[par]) continue;   // uniform
                    const double c = cs[par][0], s = cs[par][1];
                    for (int i = tid; i < L; i += nt) {   // columns p, q
                        const double cp = A[i * L + p], cq = A[i * L + q];
                        A[i * L + p] = c * cp - s * cq;
                        A[i * L + q] = s * cp + c * cq;
                    }
                    __syncthreads();
                    for (int i = tid; i < L; i += nt) {   // rows p, q; eigenvectors
                        const double rp = A[p * L + i], rq = A[q * L + i];
                        A[p * L + i] = c * rp - s * rq;
                        A[q * L + i] = s * rp + c * rq;
                        const double vp = V[i * L + p], vq = V[i * L + q];
                        V[i * L + p] = c * vp - s * vq;
                        V[i * L + q] = s * vp + c * vq;
                    }
                    __syncthreads();
                    if (tid == 0) {
                        A[p * L + q] = 0.0;
                        A[q * L + p] = 0.0;
                    }
                    // the next rotation's thread 0 reads after its own write
                }
            __syncthreads();
        }
        // ascending eigenvalues (stable order of the diagonal), V columns alike
        if (tid == 0) status[b] = sweeps;
        for (int i = tid; i < L; i += nt) {
            const double li = A[i * L + i];
            int rank = 0;
            for (int j = 0; j < L; ++j) {
                const double lj = A[j * L + j];
                rank += (lj < li) || (lj == li && j < i);
            }
            lam[b * L + rank] = li;
            for (int r = 0; r < L; ++r) Vg[b * L * L + (int64_t)r * L + rank] = V[r * L + i];
        }
        __syncthreads();
    }
}

// out = M_o + eps * scale * Phi_s Phi_s^T (src/stabilization.py:90-101)
__global__ void k_evs_update(int64_t n, int L, const double* __restrict__ lam, const double* __restrict__ V,
                             const double* __restrict__ mf_absmax, double eps, double f_lambda,
                             double* __restrict__ M) {
    extern __shared__ double sm[];
    double* Ms = sm;   // L x L
    __shared__ double red[32];
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int64_t b = blockIdx.x; b < n; b += gridDim.x) {
        const double* lb = lam + b * L;
        const double lmax = lb[L - 1];
        const double* Vb = V + b * L * L;
        double m = 0.0;
        for (int e = tid; e < L * L; e += nt) {
            const int i = e / L, j = e % L;
            double s = 0.0;
            for (int k = 0; k < L; ++k) s += Vb[i * L + k] * (lb[k] < f_lambda * lmax ? 1.0 : 0.0) * Vb[j * L + k];
            Ms[e] = s;
            m = fmax(m, fabs(s));
        }
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((tid & 31) == 0) red[tid >> 5] = m;
        __syncthreads();
        double denom = 0.0;
        for (int w = 0; w < (nt + 31) / 32; ++w) denom = fmax(denom, red[w]);
        const double scale = denom > 0.0 ? mf_absmax[b] / denom : 0.0;
        for (int e = tid; e < L * L; e += nt) M[b * L * L + e] = M[b * L * L + e] + eps * scale * Ms[e];
        __syncthreads();
    }
}

}  // namespace wcb

using namespace wcb;

namespace {
int jacobi_device(Context* ctx, int64_t n, int L, const double* A, double* lam, double* V, int max_sweeps,
                  double tol, DevBuf<double>& dA, DevBuf<double>& dlam, DevBuf<double>& dV) {
    WCB_REQUIRE(n >= 0 && L >= 1 && L <= 100, "matrix size must be 1..100");
    cudaStream_t s = ctx->stream;
    const size_t LL = (size_t)L * L;
    dA.alloc(std::max<size_t>(1, n * LL), s);
    dlam.alloc(std::max<size_t>(1, n * L), s);
    dV.alloc(std::max<size_t>(1, n * LL), s);
    DevBuf<int> st(std::max<int64_t>(n, 1));
    if (n) dA.upload(A, n * LL, s);
    const size_t smem = 2 * LL * sizeof(double);
    ensure_smem_attr((const void*)k_jacobi_batch, ctx->device, smem);
    const int threads = std::min(256, (L + 31) / 32 * 32);
    const int64_t blocks = std::min<int64_t>(std::max<int64_t>(n, 1), (int64_t)ctx->sm_count * 8);
    if (n) {
        k_jacobi_batch<<<(unsigned)blocks, threads, smem, s>>>(n, L, dA.p, dlam.p, dV.p, max_sweeps, tol, st.p);
        ctx->launches++;
        WCB_CHECK_LAUNCH();
    }
    std::vector<int> hs(std::max<int64_t>(n, 1));
    if (n) WCB_CUDA(cudaMemcpyAsync(hs.data(), st.p, n * sizeof(int), cudaMemcpyDeviceToHost, s));
    if (lam && n) WCB_CUDA(cudaMemcpyAsync(lam, dlam.p, n * L * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (V && n) WCB_CUDA(cudaMemcpyAsync(V, dV.p, n * LL * sizeof(double), cudaMemcpyDeviceToHost, s));
    WCB_CUDA(cudaStreamSynchronize(s));
    for (int64_t b = 0; b < n; ++b)
        if (hs[b] < 0) {
            char buf[128];
            std::snprintf(buf, sizeof(buf), "Jacobi iteration did not converge in %d sweeps", max_sweeps);
            throw Error{WCB_E_NOCONV, buf};
        }
    return WCB_OK;
}
}  // namespace

extern "C" {

int wcb_jacobi_eig(wcb_context* ctx, int64_t n, int L, const double* A, int max_sweeps, double tol,
                   double* lam, double* V) {
    try {
        WCB_REQUIRE(ctx && (n == 0 || (A && lam && V)), "NULL argument");
        Context* c = &ctx->c;
        WCB_CUDA(cudaSetDevice(c->device));
        DevBuf<double> dA, dl, dV;
        return jacobi_device(c, n, L, A, lam, V, max_sweeps, tol, dA, dl, dV);
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    }
}

int wcb_evs_stabilize(wcb_context* ctx, int64_t n, int L, double* M_o, const double* mf_absmax, double epsilon,
                      double f_lambda) {
    try {
        WCB_REQUIRE(ctx && (n == 0 || (M_o && mf_absmax)), "NULL argument");
        if (epsilon == 0.0 || n == 0) return WCB_OK;
        Context* c = &ctx->c;
        WCB_CUDA(cudaSetDevice(c->device));
        cudaStream_t s = c->stream;
        DevBuf<double> dA, dl, dV, dM(n * L * L), dmf(n);
        jacobi_device(c, n, L, M_o, nullptr, nullptr, 100, 1e-12, dA, dl, dV);
        dM.upload(M_o, n * L * L, s);
        dmf.upload(mf_absmax, n, s);
        const int threads = std::min(256, (L + 31) / 32 * 32);
        const size_t smem = (size_t)L * L * sizeof(double);
        ensure_smem_attr((const void*)k_evs_update, c->device, smem);
        k_evs_update<<<(unsigned)std::min<int64_t>(n, (int64_t)c->sm_count * 8), threads, smem, s>>>(
            n, L, dl.p, dV.p, dmf.p, epsilon, f_lambda, dM.p);
        c->launches++;
        WCB_CHECK_LAUNCH();
        copy_d2h(M_o, dM.p, n * L * L * sizeof(double), s);
        WCB_CUDA(cudaStreamSynchronize(s));
        return WCB_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    }
}

}  // extern "C"
