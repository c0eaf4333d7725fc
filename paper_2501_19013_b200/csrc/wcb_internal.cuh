// Internal declarations shared by the wavecell_b200 CUDA translation units.
// Everything here is C++ behind the extern "C" boundary of include/wavecell_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <algorithm>
#include <cstdlib>
#include <vector>
#include <thread>
#include <functional>

#include "../../include/wavecell_b200.h"

namespace wcb {

// ---------------------------------------------------------------- errors ----
void set_error(const std::string& msg);
struct Error {
    int code;
    std::string msg;
};

#define WCB_CUDA(call)                                                          \
    do {                                                                        \
        cudaError_t _e = (call);                                                \
        if (_e != cudaSuccess)                                                  \
            throw ::wcb::Error{WCB_E_CUDA, std::string(#call) + ": " +          \
                                               cudaGetErrorString(_e)};        \
    } while (0)

// Host<->device copies of (pageable) host arrays; large ones are staged through
// pinned chunks (wcb_core.cu).  copy_h2d returns once h may be reused,
// copy_d2h once h holds the data.
void copy_h2d(void* d, const void* h, size_t bytes, cudaStream_t s);
void copy_d2h(void* h, const void* d, size_t bytes, cudaStream_t s);
// Writes zeros over a large host output buffer on background threads (its
// pages are faulted in while the device works); join() before copy_d2h.
struct Prefault {
    std::vector<std::thread> th;
    Prefault(void* p, size_t bytes);
    ~Prefault();
    void join();
};

#define WCB_CHECK_LAUNCH() WCB_CUDA(cudaGetLastError())

#define WCB_REQUIRE(cond, msg)                                                  \
    do {                                                                        \
        if (!(cond)) throw ::wcb::Error{WCB_E_ARG, (msg)};                      \
    } while (0)

// ------------------------------------------------------------ device buf ----
// WAVECELL_B200_NO_POOL=1 turns the stream-ordered pool off (plain cudaMalloc)
inline bool use_pool() {
    static const bool on = [] {
        const char* e = getenv("WAVECELL_B200_NO_POOL");
        return !(e && e[0] == '1');
    }();
    return on;
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), st(o.st) { o.p = nullptr; o.n = 0; o.st = nullptr; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p; n = o.n; st = o.st;
            o.p = nullptr; o.n = 0; o.st = nullptr;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    cudaStream_t st = nullptr;   // stream-ordered allocation (pool) when set
    void alloc(size_t count) {
        release();
        n = count;
        if (count) WCB_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    // Stream-ordered allocation from the device's memory pool: per-run
    // buffers are recycled without the device-wide sync of cudaFree.
    void alloc(size_t count, cudaStream_t s) {
        if (!use_pool()) { alloc(count); return; }
        release();
        n = count;
        st = s;
        if (count) WCB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
    }
    void release() {
        if (p) {
            if (!st || cudaFreeAsync(p, st) != cudaSuccess) {
                cudaGetLastError();
                cudaFree(p);
            }
        }
        p = nullptr;
        st = nullptr;
        n = 0;
    }
    void upload(const T* h, size_t count, cudaStream_t s) { copy_h2d(p, h, count * sizeof(T), s); }
    void zero(cudaStream_t s) {
        if (n) WCB_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
};

// ---------------------------------------------------------------- context ----
struct Nccl;
struct Context {
    // lifetime: operators and plans retain their context; wcb_context_destroy
    // only marks it closing while they live (the last release tears it down)
    int refs = 0;
    bool closing = false;
    Nccl* nccl = nullptr;   // slab decomposition communicator (wcb_dist_init)
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    int64_t launches = 0;
    // scratch for deterministic reductions
    DevBuf<double> partials;   // per-block partial sums
    DevBuf<double> scalars;    // small scalar slots
    double* h_scalars = nullptr;  // pinned mirror
};

// ----------------------------------------------------------- step inputs ----
// Spatial load F_s in the operator's state layout, stored as a dense window
// over the state-index range [lo, hi] of its nonzeros (a point source spans
// a few rows; a distributed load spans the state), so a lookup is one load.
struct Source {
    const double* win = nullptr;     // win[i - lo] = F_s at state index i
    int64_t lo = 1, hi = 0;          // window range (empty when lo > hi)
};

__device__ __forceinline__ double source_at(const Source& s, int64_t i) {
    return (i < s.lo || i > s.hi) ? 0.0 : s.win[i - s.lo];
}

// Host: build the window from (state index, value) pairs.
inline Source make_source(std::vector<std::pair<int64_t, double>> nz, DevBuf<double>& buf,
                          cudaStream_t s) {
    Source src;
    if (nz.empty()) return src;
    std::sort(nz.begin(), nz.end());
    src.lo = nz.front().first;
    src.hi = nz.back().first;
    std::vector<double> w((size_t)(src.hi - src.lo + 1), 0.0);
    for (auto& q : nz) w[(size_t)(q.first - src.lo)] = q.second;
    buf.alloc(w.size(), s);
    buf.upload(w.data(), w.size(), s);
    WCB_CUDA(cudaStreamSynchronize(s));
    src.win = buf.p;
    return src;
}

// One explicit CDM step, src/timeint.py:179-190, fused:
//   out = 2 cur - prev + dt^2 * minv * (f F - K cur);  amp[0] = max |out|
// out may alias prev (each entry is read before it is written by one thread).
struct StepArgs {
    const double* cur = nullptr;
    const double* prev = nullptr;
    double* out = nullptr;
    const double* minv = nullptr;    // 1/m, 0 at non-DOF state slots
    Source F;
    const double* ft = nullptr;      // force table on device
    int64_t k = 0;                   // f = ft[k]
    double dt2 = 0.0;
    unsigned long long* amp = nullptr;
    // observer recording of psi_k (= cur) into obs_out[:, k], fused into the
    // step kernel (one block does it; src/timeint.py:97-106)
    int64_t n_obs = 0;
    const int64_t* obs_ptr = nullptr;
    const int64_t* obs_idx = nullptr;   // state indices
    const double* obs_val = nullptr;
    double* obs_out = nullptr;
    int64_t obs_stride = 0;
    int64_t obs_col = -1;               // column written (default: k)
};

// obs[:, k] = obs_mat @ psi_k in CSR order (scipy csr_matvec); call from
// every thread of exactly one block.
__device__ __forceinline__ void record_observers(const StepArgs& a) {
    if (!a.obs_out) return;
    for (int64_t r = threadIdx.x; r < a.n_obs; r += blockDim.x) {
        double s = 0.0;
        for (int64_t j = a.obs_ptr[r]; j < a.obs_ptr[r + 1]; ++j) s += a.obs_val[j] * a.cur[a.obs_idx[j]];
        a.obs_out[r * a.obs_stride + (a.obs_col >= 0 ? a.obs_col : a.k)] = s;
    }
}

// Programmatic dependent launch (time-step chains): a step kernel lets the
// next one launch as soon as all its CTAs are resident, and waits for the
// previous grid's completion (and memory) before touching any state.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("WAVECELL_B200_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Reference operation order of src/timeint.py:185:
//   psi_new = 2.0*psi - psi_prev + (dt*dt) * (rhs / m),  rhs = f*F - K psi
// Every operation is rounded on its own (__d*_rn: no FMA contraction, as in
// NumPy).  Two deviations remain and are bounded by the parity tests (fields
// rel. L2 <= 1e-10): 1/m is precomputed (rhs * (1/m) is within 1 ulp of
// rhs / m), and K psi is summed in another order than SciPy's csr_matvec.
__device__ __forceinline__ double leapfrog(double u, double up, double Ku, double minv,
                                           double fF, double dt2) {
    const double rhs = __dsub_rn(fF, Ku);
    return __dadd_rn(__dsub_rn(__dmul_rn(2.0, u), up), __dmul_rn(dt2, __dmul_rn(rhs, minv)));
}

__device__ __forceinline__ unsigned long long amp_bits(double v) {
    // |v| as ordered uint64: NaN (any payload) > +inf > finite.
    unsigned long long b = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffULL;
    return b;
}

// Warp-wide max of per-thread amp bits, one atomic per warp (no block
// barrier: warps that finish early leave at once).
__device__ __forceinline__ void warp_amp_max(unsigned long long v, unsigned long long* slot) {
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    if ((threadIdx.x & 31) == 0 && v) atomicMax(slot, v);
}

// Block-wide max of per-thread amp bits, one atomic per block.
template <int BLOCK>
__device__ __forceinline__ void block_amp_max(unsigned long long v, unsigned long long* slot) {
    __shared__ unsigned long long red[BLOCK / 32];
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < BLOCK / 32 ? red[lane] : 0ULL;
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
            v = w > v ? w : v;
        }
        if (lane == 0 && v) atomicMax(slot, v);
    }
}

// Deterministic block sum (fixed shuffle tree + fixed warp order).
template <int BLOCK>
__device__ __forceinline__ double block_sum(double v) {
    __shared__ double red[BLOCK / 32];
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        for (int w = 0; w < BLOCK / 32; ++w) s += red[w];
    }
    return s;  // valid in thread 0
}

// ---------------------------------------------------------------- operator ----
struct Operator {
    Context* ctx = nullptr;
    int64_t n = 0;          // compact DOFs
    int64_t n_state = 0;    // length of a state vector on the device
    virtual ~Operator() = default;
    virtual const char* name() const = 0;
    // the kernel(s) one fused time step launches (bench / profile labels)
    virtual std::string step_kernel() const { return name(); }
    // state index of each compact DOF (host copy, for observers / sources)
    virtual const std::vector<int64_t>& state_index() const = 0;
    // compact <-> state (state slots without a DOF are zero)
    virtual void scatter(const double* d_compact, double* d_state) = 0;
    virtual void gather(const double* d_state, double* d_compact) = 0;
    // y = K x in state layout
    virtual void apply(const double* d_x, double* d_y) = 0;
    // fused explicit step
    virtual void cdm_step(const StepArgs& a) = 0;
    // y = K x at (at least) the rows of a DOF subset fixed beforehand by
    // set_apply_subset (other rows of y are unspecified); default: full apply
    virtual bool set_apply_subset(const int64_t* /*compact_ids*/, int64_t /*n*/) { return false; }
    virtual void apply_subset(const double* x, double* y) { apply(x, y); }
    // (K x) at a fixed set of DOF rows, in the order given (IMEX c rows): the
    // operator may restrict the work to the cells touching those rows.
    // apply_rows returns false when not supported (caller: apply_subset + gather)
    virtual bool set_row_subset(const int64_t* /*compact_ids*/, int64_t /*n*/) { return false; }
    virtual bool apply_rows(const double* /*x_state*/, double* /*out_rows*/) { return false; }
    // split of the fused step into tiles whose input footprint holds none of
    // the given DOFs (part 0, "far") and the rest (part 1, "near"), so the far
    // part of step k+1 can overlap the implicit solve of step k; false when
    // the operator cannot split (then only cdm_step is used)
    virtual bool set_step_split(const int64_t* /*ids*/, int64_t /*n*/) { return false; }
    // slab steps overlapped with the halo exchange: part 0 computes the node
    // rows the neighbours need (and everything else that must precede the
    // exchange), part 1 the interior.  false: not split (cdm_step does all).
    virtual bool halo_split_ready() { return false; }
    virtual void cdm_step_halo_part(const StepArgs& a, int part) { if (part == 0) cdm_step(a); }
    virtual void cdm_step_part(const StepArgs& a, int part) { if (part == 1) cdm_step(a); }
    // the plan's 1/m state vector (fixed for the plan's lifetime): operators
    // may precompute which cells read it (default: every node loads 1/m)
    // zero_is_dead: slots with 1/m == 0 are not DOFs of any kind (plain CDM plan
    // with a diagonal mass), so the step may leave them untouched; false when
    // they are the implicit rows of an IMEX / consistent-mass plan
    virtual void bind_minv(const double* /*d_minv*/, bool /*zero_is_dead*/ = false) {}
    double minv_skipped = 0.0;   // DOFs whose 1/m the bound step takes from a table (no 8 B load)
    int halo_nplanes = 1;        // component planes of the state (slab halo exchange)
    int64_t halo_pstride = 0;    // doubles between component planes
    // algorithmic bytes of one fused step (for the roofline)
    virtual double step_bytes() const = 0;
    // slab halo layout (state rows of out[0] doubles), see wcb_operator_halo;
    // false when the operator is not a slab of a larger grid
    virtual bool halo(int64_t* out8) const {
        for (int i = 0; i < 8; ++i) out8[i] = 0;
        return false;
    }
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `fn` on `device`,
// raised only when `bytes` exceeds what was set there before (the attribute
// is per device; the record is mutex-protected, so several devices and host
// threads can launch the same kernel)
void ensure_smem_attr(const void* fn, int device, size_t bytes);

// consistent-mass hooks of the power iteration (mass blockdiag(diag(m), M_cc))
struct MassHooks {
    std::function<void(const double* t_state, double* y_state)> solve_c;   // y_c = M_cc^-1 t_c
    std::function<void(const double* x_state, double* mx_state)> apply_c;  // (M x)_c = M_cc x_c
};
struct Operator;
// power iteration of src/linalg.py:89-122 on op (throws Error)
void max_gen_eig_core(Operator* op, const double* m_diag, const double* x0, double tol, int64_t max_iter,
                      double* lam, int64_t* n_iter, const MassHooks* hooks);

void ctx_retain(Context* ctx);
void ctx_release(Context* ctx);

// NCCL (loaded with dlopen on first use; the library does not link it)
struct Nccl;
Nccl* nccl_for(Context* ctx);   // null unless wcb_dist_init was called on ctx
// +-1 neighbours; nplanes component planes `pstride` doubles apart
void nccl_exchange_halo(Context* ctx, double* state, const int64_t* h, int nplanes = 1, int64_t pstride = 0);
// the same exchange between consecutive slab states of one process (device copies)
struct Operator;
void copy_exchange_halo(const std::vector<Operator*>& ops, const std::vector<double*>& states, cudaStream_t s);
void nccl_allreduce_max_u64(Context* ctx, unsigned long long* d, int64_t n);
void nccl_allreduce_sum_f64(Context* ctx, double* d, int64_t n);
// true only for a slab operator (op->halo()) whose context holds a communicator
// of more than one rank: the loops run their collectives only then, so a plain
// (non-slab) run on a context that once joined a slab group stays rank-local
bool dist_slab(const Operator* op);

Operator* make_csr_operator(Context* ctx, int64_t n, const int64_t* indptr,
                            const int32_t* indices, const double* data);
Operator* make_scm_operator(Context* ctx, const wcb_scm_desc* d);
Operator* make_elastic_operator(Context* ctx, const wcb_elastic_desc* d);

// one-block observer recording (wcb_core.cu)
void launch_record_observers(Context* ctx, const StepArgs& a);

// generic elementwise kernels (wcb_core.cu)
void launch_scatter(Context* ctx, int64_t n, const int64_t* d_map, const double* src,
                    double* dst_state);
void launch_gather(Context* ctx, int64_t n, const int64_t* d_map, const double* src_state,
                   double* dst);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace wcb

struct wcb_context {
    wcb::Context c;
};
struct wcb_operator {
    wcb::Operator* op;
};
