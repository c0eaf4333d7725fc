// Context, error plumbing, generic vector kernels, the CDM time loop driver
// (src/timeint.py:159-193) and the power iteration (src/linalg.py:89-130).
#include "wcb_internal.cuh"

#include <atomic>
#include <thread>

#include <mutex>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>

namespace wcb {

// Host loop split over up to 16 threads in chunks of >= 256k iterations.
template <class F>
static void host_par_for(int64_t n, F&& f) {
    const int64_t min_chunk = 1 << 18;
    int nt = (int)std::min<int64_t>(std::max<int64_t>(1, n / min_chunk),
                                    std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
    if (nt <= 1) { f(0, n); return; }
    std::vector<std::thread> th;
    const int64_t chunk = (n + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) {
        const int64_t a = t * chunk, b = std::min<int64_t>(n, a + chunk);
        if (a < b) th.emplace_back([&f, a, b] { f(a, b); });
    }
    for (auto& x : th) x.join();
}

void ensure_smem_attr(const void* fn, int device, size_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void*, int>, size_t>> done;
    std::lock_guard<std::mutex> lock(mu);
    for (auto& e : done)
        if (e.first.first == fn && e.first.second == device) {
            if (e.second >= bytes) return;
            WCB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
            e.second = bytes;
            return;
        }
    WCB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    done.push_back({{fn, device}, bytes});
}

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

template <class F>
static int guarded(F&& f) {
    try {
        return f();
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return WCB_E_ARG;
    } catch (const std::exception& e) {
        set_error(e.what());
        return WCB_E_ARG;
    }
}

static int grid_for(const Context* ctx, int64_t n, int block = 256) {
    int64_t g = ceil_div(std::max<int64_t>(n, 1), block);
    int64_t cap = (int64_t)ctx->sm_count * 8;
    return (int)std::min(g, cap);
}

// ------------------------------------------------------------ kernels -----
__global__ void k_scatter(int64_t n, const int64_t* __restrict__ map,
                          const double* __restrict__ src, double* __restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[map[i]] = src[i];
}
__global__ void k_gather(int64_t n, const int64_t* __restrict__ map,
                         const double* __restrict__ src, double* __restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[map[i]];
}

void launch_scatter(Context* ctx, int64_t n, const int64_t* d_map, const double* src,
                    double* dst_state) {
    if (n == 0) return;
    k_scatter<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, d_map, src, dst_state);
    ctx->launches++;
    WCB_CHECK_LAUNCH();
}
void launch_gather(Context* ctx, int64_t n, const int64_t* d_map, const double* src_state,
                   double* dst) {
    if (n == 0) return;
    k_gather<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(n, d_map, src_state, dst);
    ctx->launches++;
    WCB_CHECK_LAUNCH();
}

// m_state = m at DOF slots, 1 elsewhere; minv = 1/m at DOF slots, 0 elsewhere.
__global__ void k_mass_state(int64_t n, const int64_t* __restrict__ map,
                             const double* __restrict__ m, double* __restrict__ m_state,
                             double* __restrict__ minv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t s = map[i];
        m_state[s] = m[i];
        minv[s] = 1.0 / m[i];
    }
}
// in: minv holds m at DOF slots and 0 elsewhere; out: m_state = m (1 at
// non-DOF slots), minv = 1/m (0 at non-DOF slots)
__global__ void k_mass_from_state(int64_t ns, double* __restrict__ minv, double* __restrict__ m_state) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double m = minv[i];
        m_state[i] = m != 0.0 ? m : 1.0;
        minv[i] = m != 0.0 ? 1.0 / m : 0.0;
    }
}
__global__ void k_fill(int64_t n, double v, double* __restrict__ x) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = v;
}

// CDM bootstrap, src/timeint.py:175-176:
//   a = (f0 F - K psi) / m;  psi_prev = psi - dt v + (0.5 dt dt) a
__global__ void k_cdm_bootstrap(int64_t ns, const double* __restrict__ psi,
                                const double* __restrict__ v, const double* __restrict__ Kpsi,
                                const double* __restrict__ m_state, Source F,
                                const double* __restrict__ ft, double dt,
                                double* __restrict__ prev) {
    const double f0 = ft[0];
    const double c = 0.5 * dt * dt;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns;
         i += (int64_t)gridDim.x * blockDim.x) {
        // src/timeint.py:175-176, each operation rounded on its own (no FMA)
        const double a = __ddiv_rn(__dsub_rn(__dmul_rn(f0, source_at(F, i)), Kpsi[i]), m_state[i]);
        prev[i] = __dadd_rn(__dsub_rn(psi[i], __dmul_rn(dt, v[i])), __dmul_rn(c, a));
    }
}

// obs[:, k] = obs_mat @ psi, CSR order (scipy csr_matvec), src/timeint.py:105-106.
__global__ void k_obs_record(int64_t n_obs, const int64_t* __restrict__ indptr,
                             const int64_t* __restrict__ sidx, const double* __restrict__ val,
                             const double* __restrict__ psi, double* __restrict__ out,
                             int64_t stride, int64_t k) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n_obs) return;
    double s = 0.0;
    for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j) s += val[j] * psi[sidx[j]];
    out[r * stride + k] = s;
}

__global__ void k_record_observers(StepArgs a) { record_observers(a); }

void launch_record_observers(Context* ctx, const StepArgs& a) {
    k_record_observers<<<1, 64, 0, ctx->stream>>>(a);
    ctx->launches++;
}

// ---- power iteration pieces (src/linalg.py:108-119) ----
constexpr int RB = 256;

// y = t / m ; partial[b] = sum y^2
__global__ void k_pow_y(int64_t ns, const double* __restrict__ t, const double* __restrict__ m,
                        double* __restrict__ y, double* __restrict__ part,
                        const double* __restrict__ sc) {
    if (sc[3] != 0.0) return;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < ns; i += (int64_t)gridDim.x * RB) {
        double yi = t[i] / m[i];
        y[i] = yi;
        acc += yi * yi;
    }
    double s = block_sum<RB>(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}
// sc[0] = ||y||; zero norm -> done (lam = 0)
__global__ void k_pow_norm(int nparts, const double* __restrict__ part, double* __restrict__ sc,
                           int64_t it) {
    if (sc[3] != 0.0) return;
    double acc = 0.0;
    for (int i = threadIdx.x; i < nparts; i += RB) acc += part[i];
    double s = block_sum<RB>(acc);
    if (threadIdx.x == 0) {
        double ny = sqrt(s);
        sc[0] = ny;
        if (ny == 0.0) { sc[1] = 0.0; sc[3] = 2.0; sc[4] = (double)it; }
    }
}
__global__ void k_pow_x(int64_t ns, const double* __restrict__ y, double* __restrict__ x,
                        const double* __restrict__ sc) {
    if (sc[3] != 0.0) return;
    const double ny = sc[0];
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < ns; i += (int64_t)gridDim.x * RB)
        x[i] = y[i] / ny;
}
// partials of x.Kx and x.(m x) (m = 1 at non-DOF slots where x = 0)
__global__ void k_pow_dots(int64_t ns, const double* __restrict__ x, const double* __restrict__ Kx,
                           const double* __restrict__ m, double* __restrict__ part,
                           const double* __restrict__ sc) {
    if (sc[3] != 0.0) return;
    double a = 0.0, b = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < ns; i += (int64_t)gridDim.x * RB) {
        double xi = x[i];
        a += xi * Kx[i];
        b += xi == 0.0 ? 0.0 : xi * (m[i] * xi);   // frozen DOFs carry m = inf
    }
    double sa = block_sum<RB>(a);
    double sb = block_sum<RB>(b);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = sa;
        part[2 * blockIdx.x + 1] = sb;
    }
}
// lam = xKx / xMx ; stop when |lam - lam_old| <= tol |lam| (src/linalg.py:116-117)
__global__ void k_pow_lambda(int nparts, const double* __restrict__ part, double* __restrict__ sc,
                             double tol, int64_t it) {
    if (sc[3] != 0.0) return;
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < nparts; i += RB) {
        a += part[2 * i];
        b += part[2 * i + 1];
    }
    double sa = block_sum<RB>(a);
    double sb = block_sum<RB>(b);
    if (threadIdx.x == 0) {
        double lam = sa / sb;
        double lam_old = sc[2];
        sc[1] = lam;
        if (fabs(lam - lam_old) <= tol * fabs(lam)) {
            sc[3] = 1.0;
            sc[4] = (double)it;
        }
        sc[2] = lam;
    }
}

// ------------------------------------------------- staged host copies ----
// Pageable host arrays (NumPy) move through a per-device ring of pinned
// chunks: the host side of each chunk is a memcpy split over threads (which
// also faults in fresh destination pages in parallel), overlapped with the
// DMA of the neighbouring chunk.  The driver's own pageable path stages
// through one thread.
namespace {
size_t env_size(const char* name, size_t dflt, size_t lo, size_t hi) {
    const char* e = getenv(name);
    const long long v = e ? atoll(e) : 0;
    return v > 0 ? std::min(hi, std::max(lo, (size_t)v)) : dflt;
}
// chunk MiB / host threads: WAVECELL_B200_STAGE_MB, WAVECELL_B200_STAGE_THREADS
const size_t STAGE_CHUNK = env_size("WAVECELL_B200_STAGE_MB", 32, 1, 256) << 20;
constexpr int STAGE_NBUF = 3;
constexpr size_t STAGE_MIN = size_t(2) << 20;   // smaller copies use cudaMemcpyAsync
bool stage_off() {   // WAVECELL_B200_NO_STAGE=1: plain cudaMemcpyAsync (A/B runs)
    static const bool off = [] {
        const char* e = getenv("WAVECELL_B200_NO_STAGE");
        return e && e[0] == '1';
    }();
    return off;
}
struct StageRing {
    unsigned char* buf[STAGE_NBUF] = {};
    cudaEvent_t ev[STAGE_NBUF] = {};
    std::mutex mu;
};
StageRing* stage_ring(int dev) {
    static std::mutex mu;
    static std::vector<std::unique_ptr<StageRing>> rings;
    std::lock_guard<std::mutex> g(mu);
    if ((int)rings.size() <= dev) rings.resize(dev + 1);
    if (!rings[dev]) {
        auto r = std::make_unique<StageRing>();
        for (int b = 0; b < STAGE_NBUF; ++b) {
            WCB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&r->buf[b]), STAGE_CHUNK,
                                   cudaHostAllocPortable));
            WCB_CUDA(cudaEventCreateWithFlags(&r->ev[b], cudaEventDisableTiming));
        }
        rings[dev] = std::move(r);
    }
    return rings[dev].get();
}
void par_memcpy(void* dst, const void* src, size_t bytes) {
    static const int nthr = (int)env_size("WAVECELL_B200_STAGE_THREADS",
                                          std::max(1u, std::min(16u, std::thread::hardware_concurrency())), 1, 64);
    const size_t piece = ((bytes + nthr - 1) / nthr + 4095) & ~size_t(4095);
    std::vector<std::thread> th;
    for (int t = 1; t < nthr && t * piece < bytes; ++t)
        th.emplace_back([=] {
            std::memcpy(static_cast<char*>(dst) + t * piece, static_cast<const char*>(src) + t * piece,
                        std::min(piece, bytes - t * piece));
        });
    std::memcpy(dst, src, std::min(piece, bytes));
    for (auto& x : th) x.join();
}
struct DevGuard {   // events are recorded on the stream's device
    int prev = -1;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) WCB_CUDA(cudaSetDevice(dev));
    }
    ~DevGuard() {
        int cur;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};
int stream_device(cudaStream_t s) {
    int dev;
    if (s) WCB_CUDA(cudaStreamGetDevice(s, &dev));
    else WCB_CUDA(cudaGetDevice(&dev));
    return dev;
}
}  // namespace

void copy_h2d(void* d, const void* h, size_t bytes, cudaStream_t s) {
    if (bytes < STAGE_MIN || stage_off()) {
        if (bytes) WCB_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    const int dev = stream_device(s);
    DevGuard g(dev);
    StageRing* r = stage_ring(dev);
    std::lock_guard<std::mutex> lk(r->mu);
    for (size_t off = 0, i = 0; off < bytes; off += STAGE_CHUNK, ++i) {
        const int b = (int)(i % STAGE_NBUF);
        const size_t len = std::min(STAGE_CHUNK, bytes - off);
        WCB_CUDA(cudaEventSynchronize(r->ev[b]));   // this chunk's last DMA is done
        par_memcpy(r->buf[b], static_cast<const char*>(h) + off, len);
        WCB_CUDA(cudaMemcpyAsync(static_cast<char*>(d) + off, r->buf[b], len,
                                 cudaMemcpyHostToDevice, s));
        WCB_CUDA(cudaEventRecord(r->ev[b], s));
    }
}

Prefault::Prefault(void* p, size_t bytes) {
    if (!p || bytes < STAGE_MIN || stage_off()) return;
    const int nt = std::max(1, std::min(8, (int)std::thread::hardware_concurrency() / 2));
    const size_t piece = ((bytes + nt - 1) / nt + 4095) & ~size_t(4095);
    for (int t = 0; t < nt && t * piece < bytes; ++t)
        th.emplace_back([=] {
            std::memset(static_cast<char*>(p) + t * piece, 0, std::min(piece, bytes - t * piece));
        });
}
Prefault::~Prefault() { join(); }
void Prefault::join() {
    for (auto& x : th) x.join();
    th.clear();
}

void copy_d2h(void* h, const void* d, size_t bytes, cudaStream_t s) {
    if (bytes < STAGE_MIN || stage_off()) {
        if (bytes) {
            WCB_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
            WCB_CUDA(cudaStreamSynchronize(s));
        }
        return;
    }
    const int dev = stream_device(s);
    DevGuard g(dev);
    StageRing* r = stage_ring(dev);
    std::lock_guard<std::mutex> lk(r->mu);
    const size_t n = (bytes + STAGE_CHUNK - 1) / STAGE_CHUNK;
    auto issue = [&](size_t i) {
        const int b = (int)(i % STAGE_NBUF);
        const size_t off = i * STAGE_CHUNK;
        WCB_CUDA(cudaStreamWaitEvent(s, r->ev[b], 0));   // an H2D on another stream may read it
        WCB_CUDA(cudaMemcpyAsync(r->buf[b], static_cast<const char*>(d) + off,
                                 std::min(STAGE_CHUNK, bytes - off), cudaMemcpyDeviceToHost, s));
        WCB_CUDA(cudaEventRecord(r->ev[b], s));
    };
    for (size_t i = 0; i < std::min<size_t>(n, STAGE_NBUF - 1); ++i) issue(i);
    for (size_t i = 0; i < n; ++i) {
        // buffer (i + NBUF - 1) % NBUF was drained by chunk i - 1's host copy
        if (i + STAGE_NBUF - 1 < n) issue(i + STAGE_NBUF - 1);
        const int b = (int)(i % STAGE_NBUF);
        const size_t off = i * STAGE_CHUNK;
        WCB_CUDA(cudaEventSynchronize(r->ev[b]));
        par_memcpy(static_cast<char*>(h) + off, r->buf[b], std::min(STAGE_CHUNK, bytes - off));
    }
}

}  // namespace wcb

using namespace wcb;

// ====================================================================== ABI ==
extern "C" {

int wcb_abi_version(void) { return WCB_ABI_VERSION; }
const char* wcb_last_error(void) { return g_last_error.c_str(); }

int wcb_device_count(int* out) {
    return guarded([&] {
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) n = 0;
        *out = n;
        return WCB_OK;
    });
}

int wcb_context_create(int device, wcb_context** out) {
    return guarded([&] {
        WCB_REQUIRE(out != nullptr, "out is NULL");
        std::unique_ptr<wcb_context> c(new wcb_context());
        Context& x = c->c;
        x.device = device;
        WCB_CUDA(cudaSetDevice(device));
        int major = 0;
        WCB_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        if (major != 10)
            throw Error{WCB_E_UNSUPPORTED,
                        "wavecell_b200 is built for sm_100a (B200); device has compute "
                        "capability major " + std::to_string(major)};
        WCB_CUDA(cudaDeviceGetAttribute(&x.sm_count, cudaDevAttrMultiProcessorCount, device));
        // highest priority: helper streams (IMEX far tiles) yield to it
        int lo_prio = 0, hi_prio = 0;
        WCB_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
        WCB_CUDA(cudaStreamCreateWithPriority(&x.stream, cudaStreamNonBlocking, hi_prio));
        {   // keep freed run buffers in the device pool (no release to the OS)
            cudaMemPool_t pool;
            WCB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
            uint64_t keep = ~0ULL;
            WCB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        }
        WCB_CUDA(cudaEventCreate(&x.ev0));
        WCB_CUDA(cudaEventCreate(&x.ev1));
        WCB_CUDA(cudaEventCreate(&x.ev2));
        x.partials.alloc(2 * (size_t)x.sm_count * 8 + 64);
        x.scalars.alloc(16);
        WCB_CUDA(cudaMallocHost(&x.h_scalars, 16 * sizeof(double)));
        *out = c.release();
        return WCB_OK;
    });
}

static std::mutex g_ctx_mutex;

static void ctx_teardown(wcb_context* ctx) {
    Context& x = ctx->c;
    cudaSetDevice(x.device);
    cudaStreamSynchronize(x.stream);
    x.partials.release();
    x.scalars.release();
    if (x.h_scalars) cudaFreeHost(x.h_scalars);
    cudaEventDestroy(x.ev0);
    cudaEventDestroy(x.ev1);
    cudaEventDestroy(x.ev2);
    cudaStreamDestroy(x.stream);
    delete ctx;
}

}  // extern "C"

namespace wcb {
void ctx_retain(Context* ctx) {
    std::lock_guard<std::mutex> g(g_ctx_mutex);
    ++ctx->refs;
}
void ctx_release(Context* ctx) {
    bool last = false;
    {
        std::lock_guard<std::mutex> g(g_ctx_mutex);
        last = --ctx->refs == 0 && ctx->closing;
    }
    // wcb_context's first member is the Context
    if (last) ctx_teardown(reinterpret_cast<wcb_context*>(ctx));
}
}  // namespace wcb

extern "C" {

int wcb_context_destroy(wcb_context* ctx) {
    if (!ctx) return WCB_OK;
    return guarded([&] {
        bool now = false;
        {
            std::lock_guard<std::mutex> g(g_ctx_mutex);
            ctx->c.closing = true;
            now = ctx->c.refs == 0;
        }
        if (now) ctx_teardown(ctx);
        return WCB_OK;
    });
}

void* wcb_context_stream(wcb_context* ctx) { return ctx ? (void*)ctx->c.stream : nullptr; }
int64_t wcb_context_launches(wcb_context* ctx) { return ctx ? ctx->c.launches : 0; }

int wcb_operator_csr_create(wcb_context* ctx, int64_t n, const int64_t* indptr,
                            const int32_t* indices, const double* data, wcb_operator** out) {
    return guarded([&] {
        WCB_REQUIRE(ctx && out, "NULL argument");
        WCB_REQUIRE(n >= 0, "negative n");
        WCB_CUDA(cudaSetDevice(ctx->c.device));
        std::unique_ptr<wcb_operator> o(new wcb_operator());
        o->op = make_csr_operator(&ctx->c, n, indptr, indices, data);
        ctx_retain(o->op->ctx);
        *out = o.release();
        return WCB_OK;
    });
}

int wcb_operator_scm_create(wcb_context* ctx, const wcb_scm_desc* desc, wcb_operator** out) {
    return guarded([&] {
        WCB_REQUIRE(ctx && desc && out, "NULL argument");
        WCB_CUDA(cudaSetDevice(ctx->c.device));
        std::unique_ptr<wcb_operator> o(new wcb_operator());
        o->op = make_scm_operator(&ctx->c, desc);
        ctx_retain(o->op->ctx);
        *out = o.release();
        return WCB_OK;
    });
}

int wcb_operator_elastic_create(wcb_context* ctx, const wcb_elastic_desc* desc, wcb_operator** out) {
    return guarded([&] {
        WCB_REQUIRE(ctx && desc && out, "NULL argument");
        WCB_CUDA(cudaSetDevice(ctx->c.device));
        std::unique_ptr<wcb_operator> o(new wcb_operator());
        o->op = make_elastic_operator(&ctx->c, desc);
        ctx_retain(o->op->ctx);
        *out = o.release();
        return WCB_OK;
    });
}

int wcb_operator_destroy(wcb_operator* op) {
    if (!op) return WCB_OK;
    return guarded([&] {
        Context* cx = op->op->ctx;
        cudaSetDevice(cx->device);
        cudaStreamSynchronize(cx->stream);
        delete op->op;
        delete op;
        ctx_release(cx);
        return WCB_OK;
    });
}

int64_t wcb_operator_n(const wcb_operator* op) { return op ? op->op->n : -1; }

int wcb_operator_apply(wcb_operator* o, const double* x, double* y) {
    return guarded([&] {
        WCB_REQUIRE(o && x && y, "NULL argument");
        Operator* op = o->op;
        Context* ctx = op->ctx;
        WCB_CUDA(cudaSetDevice(ctx->device));
        const int64_t n = op->n;
        if (n == 0) return WCB_OK;
        DevBuf<double> dx(n), dy(n), sx(op->n_state), sy(op->n_state);
        dx.upload(x, n, ctx->stream);
        sx.zero(ctx->stream);
        op->scatter(dx.p, sx.p);
        op->apply(sx.p, sy.p);
        op->gather(sy.p, dy.p);
        copy_d2h(y, dy.p, n * sizeof(double), ctx->stream);
        WCB_CUDA(cudaStreamSynchronize(ctx->stream));
        return WCB_OK;
    });
}

// ---------------------------------------------------------- max_gen_eig ----
// Power iteration of M^-1 K on the state (src/linalg.py:89-122); DOFs with
// m = +inf are frozen at zero (principal sub-problem, wcb_max_gen_eig_sub).
// With `hooks` the mass is blockdiag(diag(m), M_cc): m_diag holds 1 at the c
// rows, hooks->solve_c overwrites the c slots of y = M^-1 t and
// hooks->apply_c the c slots of M x (factorize()'s SuperLU path).
}  // extern "C"
namespace wcb {
__global__ void k_div_state(int64_t ns, const double* __restrict__ t, const double* __restrict__ m,
                            double* __restrict__ y, const double* __restrict__ sc) {
    if (sc[3] != 0.0) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = t[i] / m[i];
}
__global__ void k_sumsq(int64_t ns, const double* __restrict__ y, double* __restrict__ part,
                        const double* __restrict__ sc) {
    if (sc[3] != 0.0) return;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < ns; i += (int64_t)gridDim.x * RB)
        acc += y[i] * y[i];
    double s = block_sum<RB>(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void k_mul_state(int64_t ns, const double* __restrict__ m, const double* __restrict__ x,
                            double* __restrict__ mx, const double* __restrict__ sc) {
    if (sc[3] != 0.0) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x)
        mx[i] = m[i] * x[i];
}
// partials of x.Kx and x.Mx with M x given
__global__ void k_pow_dots_mx(int64_t ns, const double* __restrict__ x, const double* __restrict__ Kx,
                              const double* __restrict__ Mx, double* __restrict__ part,
                              const double* __restrict__ sc) {
    if (sc[3] != 0.0) return;
    double a = 0.0, b = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < ns; i += (int64_t)gridDim.x * RB) {
        const double xi = x[i];
        a += xi * Kx[i];
        b += xi * Mx[i];
    }
    double sa = block_sum<RB>(a);
    double sb = block_sum<RB>(b);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = sa;
        part[2 * blockIdx.x + 1] = sb;
    }
}

void max_gen_eig_core(Operator* op, const double* m_diag, const double* x0, double tol, int64_t max_iter,
                      double* lam, int64_t* n_iter, const MassHooks* hooks) {
    Context* ctx = op->ctx;
    WCB_CUDA(cudaSetDevice(ctx->device));
    const int64_t n = op->n, ns = op->n_state;
    WCB_REQUIRE(n > 0, "empty operator");
    cudaStream_t s = ctx->stream;
    DevBuf<double> dm(n), dx0(n), m_state(ns), minv(ns), x(ns), t(ns), y(ns), mx;
    DevBuf<int64_t> map;
    if (hooks) mx.alloc(ns, s);
    dm.upload(m_diag, n, s);
    dx0.upload(x0, n, s);
    // mass in state layout (1 at non-DOF slots so y = 0/1 = 0 there)
    k_fill<<<grid_for(ctx, ns), 256, 0, s>>>(ns, 1.0, m_state.p);
    ctx->launches++;
    {
        const std::vector<int64_t>& si = op->state_index();
        map.alloc(n);
        map.upload(si.data(), n, s);
        k_mass_state<<<grid_for(ctx, n), 256, 0, s>>>(n, map.p, dm.p, m_state.p, minv.p);
        ctx->launches++;
    }
    x.zero(s);
    op->scatter(dx0.p, x.p);
    t.zero(s);
    y.zero(s);
    WCB_CHECK_LAUNCH();
    const int gb = grid_for(ctx, ns, RB);
    double init[8] = {0.0, 0.0, INFINITY, 0.0, 0.0, 0.0, 0.0, 0.0};
    WCB_CUDA(cudaMemcpyAsync(ctx->scalars.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
    double* sc = ctx->scalars.p;
    double* part = ctx->partials.p;
    const int64_t batch = 16;
    int64_t it = 1;
    bool done = false;
    while (!done && it <= max_iter) {
        int64_t end = std::min<int64_t>(max_iter, it + batch - 1);
        for (; it <= end; ++it) {
            op->apply(x.p, t.p);
            if (hooks) {
                k_div_state<<<grid_for(ctx, ns), 256, 0, s>>>(ns, t.p, m_state.p, y.p, sc);
                hooks->solve_c(t.p, y.p);
                k_sumsq<<<gb, RB, 0, s>>>(ns, y.p, part, sc);
                ctx->launches += 2;
            } else {
                k_pow_y<<<gb, RB, 0, s>>>(ns, t.p, m_state.p, y.p, part, sc);
                ctx->launches++;
            }
            k_pow_norm<<<1, RB, 0, s>>>(gb, part, sc, it);
            k_pow_x<<<gb, RB, 0, s>>>(ns, y.p, x.p, sc);
            op->apply(x.p, t.p);
            if (hooks) {
                k_mul_state<<<grid_for(ctx, ns), 256, 0, s>>>(ns, m_state.p, x.p, mx.p, sc);
                hooks->apply_c(x.p, mx.p);
                k_pow_dots_mx<<<gb, RB, 0, s>>>(ns, x.p, t.p, mx.p, part, sc);
                ctx->launches += 2;
            } else {
                k_pow_dots<<<gb, RB, 0, s>>>(ns, x.p, t.p, m_state.p, part, sc);
                ctx->launches++;
            }
            k_pow_lambda<<<1, RB, 0, s>>>(gb, part, sc, tol, it);
            ctx->launches += 3;
        }
        WCB_CHECK_LAUNCH();
        WCB_CUDA(cudaMemcpyAsync(ctx->h_scalars, sc, 8 * sizeof(double),
                                 cudaMemcpyDeviceToHost, s));
        WCB_CUDA(cudaStreamSynchronize(s));
        done = ctx->h_scalars[3] != 0.0;
    }
    if (!done) {
        char buf[160];
        snprintf(buf, sizeof(buf),
                 "power iteration did not converge in %lld iterations (last estimate %.6e)",
                 (long long)max_iter, ctx->h_scalars[2]);
        throw Error{WCB_E_NOCONV, buf};
    }
    *lam = ctx->h_scalars[1];
    *n_iter = (int64_t)ctx->h_scalars[4];
}
}  // namespace wcb
extern "C" {

static int max_gen_eig_impl(wcb_operator* o, const double* m_diag, const double* x0, double tol,
                            int64_t max_iter, double* lam, int64_t* n_iter) {
    return guarded([&] {
        WCB_REQUIRE(o && m_diag && x0 && lam && n_iter, "NULL argument");
        max_gen_eig_core(o->op, m_diag, x0, tol, max_iter, lam, n_iter, nullptr);
        return WCB_OK;
    });
}

int wcb_max_gen_eig(wcb_operator* o, const double* m_diag, const double* x0, double tol,
                    int64_t max_iter, double* lam, int64_t* n_iter) {
    return max_gen_eig_impl(o, m_diag, x0, tol, max_iter, lam, n_iter);
}

int wcb_max_gen_eig_sub(wcb_operator* o, const double* m_diag, int64_t n_sub,
                        const int64_t* sub_idx, const double* x0_sub, double tol,
                        int64_t max_iter, double* lam, int64_t* n_iter) {
    int64_t n = 0;
    int code = guarded([&] {
        WCB_REQUIRE(o && m_diag && sub_idx && x0_sub, "NULL argument");
        n = o->op->n;
        WCB_REQUIRE(n_sub >= 1 && n_sub <= n, "sub-problem size must be in 1..n");
        return WCB_OK;
    });
    if (code != WCB_OK) return code;
    std::vector<double> m(n, INFINITY), x(n, 0.0);
    for (int64_t k = 0; k < n_sub; ++k) {
        const int64_t i = sub_idx[k];
        if (i < 0 || i >= n || (k && sub_idx[k - 1] >= i))
            return guarded([&] { throw Error{WCB_E_ARG, "sub_idx must be ascending DOF ids"}; return 0; });
        m[i] = m_diag[i];
        x[i] = x0_sub[k];
    }
    return max_gen_eig_impl(o, m.data(), x.data(), tol, max_iter, lam, n_iter);
}

}  // extern "C"

// ============================================================= CDM plan ====
struct wcb_cdm_plan {
    Operator* op = nullptr;
    Context* ctx = nullptr;   // retained
    DevBuf<double> m_state, minv;
    DevBuf<double> F_win;
    Source src;
    int64_t n_obs = 0;
    DevBuf<int64_t> obs_indptr, obs_idx;
    DevBuf<double> obs_val;
    DevBuf<double> AB, V, T, cin, cout;   // AB: psi_k / psi_{k-1} ping-pong, one allocation
    double* pA = nullptr;
    double* pB = nullptr;
    DevBuf<double> ft;
    DevBuf<unsigned long long> amp;
    std::vector<unsigned long long> h_amp;
};

namespace wcb {

// Halo exchange of state buffers cur[r] between consecutive slabs: device
// copies for an emulated group (one context), NCCL for one plan per process.
static void exchange_halos(std::vector<wcb_cdm_plan*>& Ps, std::vector<double*>& cur,
                           cudaStream_t on = nullptr) {
    const size_t n = Ps.size();
    Context* ctx = Ps[0]->op->ctx;
    cudaStream_t s = on ? on : ctx->stream;
    if (n == 1) {
        int64_t h[8];
        Operator* op = Ps[0]->op;
        if (dist_slab(op) && op->halo(h)) {
            cudaStream_t save = ctx->stream;
            ctx->stream = s;
            try {
                nccl_exchange_halo(ctx, cur[0], h, op->halo_nplanes, op->halo_pstride);
            } catch (...) {
                ctx->stream = save;
                throw;
            }
            ctx->stream = save;
        }
        return;
    }
    std::vector<Operator*> ops;
    for (auto* P : Ps) ops.push_back(P->op);
    copy_exchange_halo(ops, cur, s);
}

// RAII second stream + events for the halo exchange overlapped with the
// interior part of a slab step
struct HaloOverlap {
    cudaStream_t s2 = nullptr;
    cudaEvent_t e_b = nullptr, e_x = nullptr;
    explicit HaloOverlap(int device) {
        WCB_CUDA(cudaSetDevice(device));
        int lo = 0, hi = 0;
        WCB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        WCB_CUDA(cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, hi));   // the exchange first
        WCB_CUDA(cudaEventCreateWithFlags(&e_b, cudaEventDisableTiming));
        WCB_CUDA(cudaEventCreateWithFlags(&e_x, cudaEventDisableTiming));
    }
    ~HaloOverlap() {
        if (s2) { cudaStreamSynchronize(s2); cudaStreamDestroy(s2); }
        if (e_b) cudaEventDestroy(e_b);
        if (e_x) cudaEventDestroy(e_x);
    }
};

// The CDM loop of src/timeint.py:159-193 for one plan or a group of slab
// plans sharing one context (emulated ranks) or one plan per process with an
// NCCL communicator on its context.
static void run_cdm_group(std::vector<wcb_cdm_plan*>& Ps, const double* d_ft, double dt, int64_t n_t,
                          const std::vector<const double*>& d_psi0, const std::vector<const double*>& d_v0,
                          const std::vector<double*>& d_psi_out, const std::vector<double*>& d_obs_out,
                          wcb_divergence* div, wcb_timings* tm, int64_t rec = 1) {
    // rec > 1: observers recorded every rec steps only (column k / rec), the
    // exact step hits src/harness.py:101-131 samples when rec divides n_t
    const size_t G = Ps.size();
    Context* ctx = Ps[0]->op->ctx;
    for (auto* P : Ps) WCB_REQUIRE(P->op->ctx == ctx, "group plans must share one context");
    cudaStream_t s = ctx->stream;
    if (div) { div->step = -1; div->amplitude = 0.0; }
    if (tm) { tm->factorization = 0.0; tm->rhs = 0.0; tm->backward_insertion = 0.0; }
    WCB_REQUIRE(rec >= 1, "record_every must be >= 1");
    const int64_t stride = n_t / rec + 1;
    std::vector<double*> cur(G), prev(G);
    for (size_t r = 0; r < G; ++r) {
        wcb_cdm_plan* P = Ps[r];
        Operator* op = P->op;
        const int64_t ns = op->n_state;
        if (P->AB.n != (size_t)(2 * ns)) {
            P->AB.alloc(2 * ns, s); P->V.alloc(ns, s); P->T.alloc(ns, s);
            P->pA = P->AB.p;
            P->pB = P->AB.p + ns;
            P->AB.zero(s); P->T.zero(s);
        }
        if (P->amp.n < (size_t)(n_t + 1)) P->amp.alloc(n_t + 1, s);
        P->amp.zero(s);
        // initial state: zeros unless given (src/timeint.py:162-163)
        WCB_CUDA(cudaMemsetAsync(P->pA, 0, ns * sizeof(double), s));
        P->V.zero(s);
        if (d_psi0[r]) op->scatter(d_psi0[r], P->pA);
        if (d_v0[r]) op->scatter(d_v0[r], P->V.p);
        cur[r] = P->pA;
        prev[r] = P->pB;
    }
    exchange_halos(Ps, cur);   // psi_0 halos for the bootstrap apply
    std::vector<StepArgs> args(G);
    for (size_t r = 0; r < G; ++r) {
        wcb_cdm_plan* P = Ps[r];
        Operator* op = P->op;
        const int64_t ns = op->n_state;
        // bootstrap a0, psi_{-1} (src/timeint.py:175-176)
        op->apply(P->pA, P->T.p);
        k_cdm_bootstrap<<<grid_for(ctx, ns), 256, 0, s>>>(ns, P->pA, P->V.p, P->T.p, P->m_state.p, P->src,
                                                          d_ft, dt, P->pB);
        ctx->launches++;
        StepArgs& a = args[r];
        a.minv = P->minv.p;
        a.F = P->src;
        a.ft = d_ft;
        a.dt2 = dt * dt;
        if (P->n_obs && d_obs_out[r]) {
            a.n_obs = P->n_obs;
            a.obs_ptr = P->obs_indptr.p;
            a.obs_idx = P->obs_idx.p;
            a.obs_val = P->obs_val.p;
            a.obs_out = d_obs_out[r];
            a.obs_stride = stride;
        }
    }
    WCB_CHECK_LAUNCH();
    auto gate_obs = [&](size_t r, StepArgs& a, int64_t k) {
        if (rec == 1) return;
        a.obs_out = (k % rec == 0 && Ps[r]->n_obs) ? d_obs_out[r] : nullptr;
        a.obs_col = k / rec;
    };
    // Keep the psi_k / psi_{k-1} pair resident in L2 across time steps
    // (persisting access-policy window on the stream) when the pair fits the
    // access-policy window and at most twice the persisting set-aside (hit
    // ratio = set-aside / pair; config 2: 72 MB, -6 % per step).
    // WAVECELL_B200_L2_PERSIST=0 turns it off.
    bool persist = false;
    int maxp = 0, maxw = 0;
    if (G == 1 && !(getenv("WAVECELL_B200_L2_PERSIST") && getenv("WAVECELL_B200_L2_PERSIST")[0] == '0')) {
        WCB_CUDA(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, ctx->device));
        WCB_CUDA(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device));
        const size_t pair = 2 * (size_t)Ps[0]->op->n_state * sizeof(double);
        persist = maxp > 0 && pair <= (size_t)maxw && pair <= 2 * (size_t)maxp;
    }
    if (persist) {
        const size_t bytes = 2 * (size_t)Ps[0]->op->n_state * sizeof(double);
        WCB_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp));
        cudaStreamAttrValue v{};
        v.accessPolicyWindow.base_ptr = Ps[0]->AB.p;
        v.accessPolicyWindow.num_bytes = bytes;
        v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)maxp / (float)bytes);
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        WCB_CUDA(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v));
    }
    std::vector<unsigned long long> h_amp(G * (n_t + 1), 0ULL);
    const int64_t check_every = 256;
    int64_t checked = 0;   // amp[1..checked] inspected
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
            unsigned long long b = 0ULL;
            for (size_t r = 0; r < G; ++r) b = std::max(b, h_amp[r * (n_t + 1) + k]);
            double v;
            std::memcpy(&v, &b, sizeof(v));
            if (!std::isfinite(v) || v > 1.0e12) {
                if (div) { div->step = k; div->amplitude = v; }
                return true;
            }
        }
        checked = upto;
        return false;
    };
    // slab steps: the node rows the neighbours need first, their exchange on a
    // second stream while the interior rows are computed (north star (d));
    // WAVECELL_B200_HALO_OVERLAP=0 runs step and exchange back to back
    bool overlap = !(getenv("WAVECELL_B200_HALO_OVERLAP") && getenv("WAVECELL_B200_HALO_OVERLAP")[0] == '0');
    for (size_t r = 0; r < G && overlap; ++r) {
        int64_t h[8];
        overlap = (G > 1 || dist_slab(Ps[r]->op)) && Ps[r]->op->halo(h) && Ps[r]->op->halo_split_ready();
    }
    std::unique_ptr<HaloOverlap> hov;
    if (overlap) hov.reset(new HaloOverlap(ctx->device));
    WCB_CUDA(cudaEventRecord(ctx->ev0, s));
    bool diverged = false;
    for (int64_t k = 0; k < n_t; ++k) {
        if (overlap) {
            for (size_t r = 0; r < G; ++r) {
                StepArgs& a = args[r];
                a.cur = cur[r];
                a.prev = prev[r];
                a.out = prev[r];
                a.k = k;
                a.amp = Ps[r]->amp.p + (k + 1);
                gate_obs(r, a, k);
                Ps[r]->op->cdm_step_halo_part(a, 0);   // exchanged rows (+ observers of psi_k)
            }
            WCB_CUDA(cudaEventRecord(hov->e_b, s));
            WCB_CUDA(cudaStreamWaitEvent(hov->s2, hov->e_b, 0));
            exchange_halos(Ps, prev, hov->s2);        // psi_{k+1} halos, overlapped with ...
            WCB_CUDA(cudaEventRecord(hov->e_x, hov->s2));
            for (size_t r = 0; r < G; ++r) Ps[r]->op->cdm_step_halo_part(args[r], 1);   // ... the interior
            WCB_CUDA(cudaStreamWaitEvent(s, hov->e_x, 0));
            for (size_t r = 0; r < G; ++r) std::swap(cur[r], prev[r]);
            if ((k + 1) % check_every == 0) {
                WCB_CHECK_LAUNCH();
                if (inspect(k + 1)) { diverged = true; break; }
            }
            continue;
        }
        for (size_t r = 0; r < G; ++r) {
            StepArgs& a = args[r];
            a.cur = cur[r];
            a.prev = prev[r];
            a.out = prev[r];   // psi_{k+1} overwrites psi_{k-1} in place
            a.k = k;
            a.amp = Ps[r]->amp.p + (k + 1);
            gate_obs(r, a, k);
            Ps[r]->op->cdm_step(a);   // also records obs[:, k] from psi_k
            std::swap(cur[r], prev[r]);
        }
        exchange_halos(Ps, cur);
        if ((k + 1) % check_every == 0) {
            WCB_CHECK_LAUNCH();
            if (inspect(k + 1)) { diverged = true; break; }
        }
    }
    if (!diverged)
        for (size_t r = 0; r < G; ++r)
            if (Ps[r]->n_obs && d_obs_out[r]) {
                StepArgs a = args[r];
                a.cur = cur[r];
                a.k = n_t;
                a.obs_out = d_obs_out[r];
                a.obs_col = rec > 1 ? (n_t % rec == 0 ? n_t / rec : -2) : -1;
                if (a.obs_col != -2) launch_record_observers(ctx, a);
            }
    WCB_CUDA(cudaEventRecord(ctx->ev1, s));
    WCB_CHECK_LAUNCH();
    if (persist) {   // release the window and the persisting lines
        cudaStreamAttrValue v{};
        v.accessPolicyWindow.num_bytes = 0;
        WCB_CUDA(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v));
        WCB_CUDA(cudaCtxResetPersistingL2Cache());
    }
    if (!diverged) diverged = inspect(n_t);
    WCB_CUDA(cudaEventSynchronize(ctx->ev1));
    float ms = 0.f;
    WCB_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    // The K apply and the update are one fused kernel: the whole loop is
    // reported under "rhs" (src/timeint.py:181-188 splits them in two).
    if (tm) tm->rhs = ms * 1e-3;
    if (diverged) throw Error{WCB_E_DIVERGED, "solution diverged"};
    for (size_t r = 0; r < G; ++r) {
        if (Ps[r]->n_obs && d_obs_out[r] && G == 1 && dist_slab(Ps[r]->op)) nccl_allreduce_sum_f64(ctx, d_obs_out[r], Ps[r]->n_obs * stride);
        Ps[r]->op->gather(cur[r], d_psi_out[r]);
    }
    WCB_CUDA(cudaStreamSynchronize(s));
}

static void run_cdm_device(wcb_cdm_plan* P, const double* d_ft, double dt, int64_t n_t,
                           const double* d_psi0, const double* d_v0, double* d_psi_out,
                           double* d_obs_out, wcb_divergence* div, wcb_timings* tm) {
    std::vector<wcb_cdm_plan*> Ps{P};
    run_cdm_group(Ps, d_ft, dt, n_t, {d_psi0}, {d_v0}, {d_psi_out}, {d_obs_out}, div, tm);
}

}  // namespace wcb

extern "C" {

int wcb_csr_diagonal_check(int64_t n, const void* indptr, const void* indices, int index_bytes,
                           const double* data) {
    if (n < 0 || !indptr || !indices || !data || (index_bytes != 4 && index_bytes != 8)) return -1;
    std::atomic<int> pattern_ok{1}, values_ok{1};
    host_par_for(n, [&](int64_t a, int64_t b) {
        bool pat = true, val = true;
        if (index_bytes == 4) {
            const int32_t* ip = static_cast<const int32_t*>(indptr);
            const int32_t* ix = static_cast<const int32_t*>(indices);
            for (int64_t i = a; i < b && pat; ++i) pat = ip[i] == i && ix[i] == i;
            if (b == n) pat = pat && ip[n] == n;
        } else {
            const int64_t* ip = static_cast<const int64_t*>(indptr);
            const int64_t* ix = static_cast<const int64_t*>(indices);
            for (int64_t i = a; i < b && pat; ++i) pat = ip[i] == i && ix[i] == i;
            if (b == n) pat = pat && ip[n] == n;
        }
        for (int64_t i = a; i < b && val; ++i) val = data[i] > 0.0 && std::isfinite(data[i]);
        if (!pat) pattern_ok = 0;
        if (!val) values_ok = 0;
    });
    if (!pattern_ok) return -1;
    return values_ok ? 1 : 0;
}

int wcb_cdm_plan_create(wcb_operator* o, const double* m_diag, const double* F_s,
                        const wcb_observer* obs, wcb_cdm_plan** out) {
    return guarded([&] {
        WCB_REQUIRE(o && m_diag && F_s && out, "NULL argument");
        Operator* op = o->op;
        Context* ctx = op->ctx;
        WCB_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        const int64_t n = op->n, ns = op->n_state;
        std::atomic<int> m_ok{1};
        host_par_for(n, [&](int64_t a, int64_t b) {
            for (int64_t i = a; i < b; ++i)
                if (!(m_diag[i] > 0.0 && std::isfinite(m_diag[i]))) { m_ok = 0; return; }
        });
        WCB_REQUIRE(m_ok, "diagonal mass has non-positive entries");
        std::unique_ptr<wcb_cdm_plan> P(new wcb_cdm_plan());
        P->op = op;
        P->ctx = ctx;
        const std::vector<int64_t>& si = op->state_index();
        // m into the state layout through the operator's own device map
        // (scatter), then m_state = m / 1 and minv = 1/m / 0 at DOF / other slots
        DevBuf<double> dm;
        dm.alloc(n, s);
        dm.upload(m_diag, n, s);
        P->m_state.alloc(ns, s);
        P->minv.alloc(ns, s);
        P->minv.zero(s);
        if (n) op->scatter(dm.p, P->minv.p);
        k_mass_from_state<<<grid_for(ctx, ns), 256, 0, s>>>(ns, P->minv.p, P->m_state.p);
        ctx->launches += 2;
        WCB_CHECK_LAUNCH();
        op->bind_minv(P->minv.p, true);   // diagonal mass: 1/m == 0 only at non-DOF slots
        // source: dense window over its nonzeros' state-index range
        {
            std::mutex mu;
            std::vector<std::pair<int64_t, double>> nz;
            host_par_for(n, [&](int64_t a, int64_t b) {
                std::vector<std::pair<int64_t, double>> loc;
                for (int64_t i = a; i < b; ++i)
                    if (F_s[i] != 0.0) loc.emplace_back(si[i], F_s[i]);
                if (!loc.empty()) {
                    std::lock_guard<std::mutex> g(mu);
                    nz.insert(nz.end(), loc.begin(), loc.end());
                }
            });
            P->src = make_source(std::move(nz), P->F_win, s);   // sorts by state index
        }
        if (obs && obs->n_obs > 0) {
            P->n_obs = obs->n_obs;
            int64_t nnz = obs->indptr[obs->n_obs];
            std::vector<int64_t> sidx(nnz);
            for (int64_t j = 0; j < nnz; ++j) {
                int64_t c = obs->indices[j];
                WCB_REQUIRE(c >= 0 && c < n, "observer column out of range");
                sidx[j] = si[c];
            }
            P->obs_indptr.alloc(obs->n_obs + 1, s);
            P->obs_indptr.upload(obs->indptr, obs->n_obs + 1, s);
            P->obs_idx.alloc(std::max<int64_t>(nnz, 1), s);
            P->obs_idx.upload(sidx.data(), nnz, s);
            P->obs_val.alloc(std::max<int64_t>(nnz, 1), s);
            P->obs_val.upload(obs->data, nnz, s);
        }
        WCB_CUDA(cudaStreamSynchronize(s));
        ctx_retain(ctx);
        *out = P.release();
        return WCB_OK;
    });
}

int wcb_cdm_plan_destroy(wcb_cdm_plan* plan) {
    if (!plan) return WCB_OK;
    return guarded([&] {
        Context* cx = plan->ctx;
        cudaSetDevice(cx->device);
        cudaStreamSynchronize(cx->stream);
        delete plan;
        ctx_release(cx);
        return WCB_OK;
    });
}

int wcb_cdm_plan_run_device(wcb_cdm_plan* P, const double* d_ft, double dt, int64_t n_t,
                            const double* d_psi0, const double* d_v0, double* d_psi_out,
                            double* d_obs_out, wcb_divergence* div, wcb_timings* tm) {
    return guarded([&] {
        WCB_REQUIRE(P && d_psi_out, "NULL argument");
        WCB_REQUIRE(n_t >= 0, "negative n_t");
        WCB_REQUIRE(d_ft, "force table is NULL (it holds max(n_t,1) entries, ft[0] = f_t(0.0))");
        WCB_CUDA(cudaSetDevice(P->op->ctx->device));
        run_cdm_device(P, d_ft, dt, n_t, d_psi0, d_v0, d_psi_out, d_obs_out, div, tm);
        return WCB_OK;
    });
}

int wcb_cdm_plan_run(wcb_cdm_plan* P, const double* ft, double dt, int64_t n_t,
                     const double* psi0, const double* v0, double* psi_out, double* obs_out,
                     wcb_divergence* div, wcb_timings* tm) {
    return wcb_cdm_plan_run_sampled(P, ft, dt, n_t, 1, psi0, v0, psi_out, obs_out, div, tm);
}

int wcb_cdm_plan_run_sampled(wcb_cdm_plan* P, const double* ft, double dt, int64_t n_t, int64_t record_every,
                             const double* psi0, const double* v0, double* psi_out, double* obs_out,
                             wcb_divergence* div, wcb_timings* tm) {
    return guarded([&] {
        WCB_REQUIRE(record_every >= 1, "record_every must be >= 1");
        WCB_REQUIRE(P && psi_out, "NULL argument");
        WCB_REQUIRE(n_t >= 0, "negative n_t");
        Operator* op = P->op;
        Context* ctx = op->ctx;
        WCB_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        const int64_t n = op->n;
        DevBuf<double> dft, dpsi0, dv0, dout, dobs;
        dft.alloc(std::max<int64_t>(n_t, 1), s);
        dout.alloc(std::max<int64_t>(n, 1), s);
        WCB_REQUIRE(ft, "force table is NULL (it holds max(n_t,1) entries, ft[0] = f_t(0.0))");
        dft.upload(ft, std::max<int64_t>(n_t, 1), s);
        if (psi0) { dpsi0.alloc(n, s); dpsi0.upload(psi0, n, s); }
        if (v0) { dv0.alloc(n, s); dv0.upload(v0, n, s); }
        const int64_t ncol = n_t / record_every + 1;
        if (obs_out && P->n_obs) dobs.alloc(P->n_obs * ncol, s);
        Prefault pf(psi_out, n * sizeof(double));   // fault the output in while the loop runs
        {
            std::vector<wcb_cdm_plan*> Ps{P};
            run_cdm_group(Ps, dft.p, dt, n_t, {dpsi0.p}, {dv0.p}, {dout.p}, {dobs.p}, div, tm, record_every);
        }
        pf.join();
        copy_d2h(psi_out, dout.p, n * sizeof(double), s);
        if (obs_out && P->n_obs)
            WCB_CUDA(cudaMemcpyAsync(obs_out, dobs.p, P->n_obs * ncol * sizeof(double),
                                     cudaMemcpyDeviceToHost, s));
        WCB_CUDA(cudaStreamSynchronize(s));
        return WCB_OK;
    });
}

int wcb_cdm_group_run(int n_plans, wcb_cdm_plan** plans, const double* ft, double dt,
                      int64_t n_t, double** psi_out, double* obs_out, wcb_divergence* div,
                      wcb_timings* tm) {
    return guarded([&] {
        WCB_REQUIRE(n_plans >= 1 && plans && psi_out && ft, "NULL argument");
        std::vector<wcb_cdm_plan*> Ps(plans, plans + n_plans);
        Context* ctx = Ps[0]->op->ctx;
        WCB_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        DevBuf<double> dft(std::max<int64_t>(n_t, 1));
        dft.upload(ft, std::max<int64_t>(n_t, 1), s);
        std::vector<DevBuf<double>> outs(n_plans), obs(n_plans);
        std::vector<double*> pout(n_plans), pobs(n_plans, nullptr);
        const int64_t n_obs = Ps[0]->n_obs;
        for (int r = 0; r < n_plans; ++r) {
            WCB_REQUIRE(Ps[r]->n_obs == n_obs, "plans must share the observer count");
            outs[r].alloc(std::max<int64_t>(Ps[r]->op->n, 1));
            pout[r] = outs[r].p;
            if (obs_out && n_obs) {
                obs[r].alloc(n_obs * (n_t + 1));
                pobs[r] = obs[r].p;
            }
        }
        std::vector<const double*> none(n_plans, nullptr);
        std::vector<std::unique_ptr<Prefault>> pfs;
        for (int r = 0; r < n_plans; ++r)
            pfs.emplace_back(new Prefault(psi_out[r], Ps[r]->op->n * sizeof(double)));
        run_cdm_group(Ps, dft.p, dt, n_t, none, none, pout, pobs, div, tm);
        for (auto& pf : pfs) pf->join();
        for (int r = 0; r < n_plans; ++r)
            if (Ps[r]->op->n)
                copy_d2h(psi_out[r], pout[r], Ps[r]->op->n * sizeof(double), s);
        if (obs_out && n_obs) {
            // sum of the per-slab partial observers, in slab order
            std::vector<double> acc(n_obs * (n_t + 1), 0.0), part(n_obs * (n_t + 1));
            for (int r = 0; r < n_plans; ++r) {
                WCB_CUDA(cudaMemcpyAsync(part.data(), pobs[r], part.size() * sizeof(double),
                                         cudaMemcpyDeviceToHost, s));
                WCB_CUDA(cudaStreamSynchronize(s));
                for (size_t i = 0; i < acc.size(); ++i) acc[i] += part[i];
            }
            std::memcpy(obs_out, acc.data(), acc.size() * sizeof(double));
        }
        WCB_CUDA(cudaStreamSynchronize(s));
        return WCB_OK;
    });
}

int wcb_cdm_plan_step_bytes(const wcb_cdm_plan* plan, double* out) {
    return guarded([&] {
        WCB_REQUIRE(plan && out, "NULL argument");
        const Operator* op = plan->op;
        *out = op->step_bytes() - 8.0 * op->minv_skipped;
        return WCB_OK;
    });
}

int wcb_operator_halo(const wcb_operator* op, int64_t* out8) {
    if (!op || !out8) return WCB_E_ARG;
    return op->op->halo(out8) ? 1 : 0;
}

int wcb_operator_step_kernel(const wcb_operator* op, char* out, int64_t cap) {
    if (!op || !out || cap <= 0) return WCB_E_ARG;
    const std::string k = op->op->step_kernel();
    std::snprintf(out, (size_t)cap, "%s", k.c_str());
    return WCB_OK;
}

}  // extern "C"
