// Slab decomposition across GPUs: one process per GPU, x slabs,
// per step one halo exchange with the +-1 neighbours (p node rows travel
// "down" the slab order, one node row "up"), plus scalar all-reduces for the
// divergence amplitude and the observers.  NCCL is loaded with dlopen (the
// library does not link it); the communicator is created from a unique id the
// caller broadcasts (torch.distributed in paper_2501_19013_b200/dist.py).
#include "wcb_internal.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>

namespace wcb {

struct Nccl {
    void* lib = nullptr;
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    decltype(&ncclCommInitRank) init = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) gstart = nullptr;
    decltype(&ncclGroupEnd) gend = nullptr;
    decltype(&ncclAllReduce) allreduce = nullptr;
    decltype(&ncclGetErrorString) errstr = nullptr;
    decltype(&ncclGetUniqueId) uid = nullptr;
};

static void* nccl_dl() {
    static void* h = nullptr;
    if (!h) {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names)
            if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    }
    if (!h) throw Error{WCB_E_UNSUPPORTED, "libnccl.so.2 not found (needed for multi-GPU slabs)"};
    return h;
}

template <class F>
static F sym(void* h, const char* name) {
    void* p = dlsym(h, name);
    if (!p) throw Error{WCB_E_UNSUPPORTED, std::string("NCCL symbol missing: ") + name};
    return reinterpret_cast<F>(p);
}

#define NCCL_CHECK(N, call)                                                             \
    do {                                                                                \
        ncclResult_t _r = (call);                                                       \
        if (_r != ncclSuccess)                                                          \
            throw Error{WCB_E_CUDA, std::string("NCCL: ") + (N)->errstr(_r)};          \
    } while (0)

Nccl* nccl_for(Context* ctx) { return ctx->nccl; }

void nccl_exchange_halo(Context* ctx, double* state, const int64_t* h, int nplanes, int64_t pstride) {
    Nccl* N = ctx->nccl;
    if (!N || N->world == 1) return;
    const int64_t xs = h[0];
    const int up = N->rank + 1, down = N->rank - 1;
    NCCL_CHECK(N, N->gstart());
    for (int pl = 0; pl < nplanes; ++pl) {
        double* st = state + pl * pstride;
        if (h[2] > 0 && down >= 0) {
            // top halo (p rows) <- previous slab's last p rows; our first row -> its bottom halo
            NCCL_CHECK(N, N->recv(st + h[1] * xs, (size_t)(h[2] * xs), ncclDouble, down, N->comm, ctx->stream));
            NCCL_CHECK(N, N->send(st + h[7] * xs, (size_t)xs, ncclDouble, down, N->comm, ctx->stream));
        }
        if (h[4] > 0 && up < N->world) {
            // our last p rows -> next slab's top halo; its first row -> our bottom halo
            NCCL_CHECK(N, N->send(st + h[5] * xs, (size_t)(h[6] * xs), ncclDouble, up, N->comm, ctx->stream));
            NCCL_CHECK(N, N->recv(st + h[3] * xs, (size_t)(h[4] * xs), ncclDouble, up, N->comm, ctx->stream));
        }
    }
    NCCL_CHECK(N, N->gend());
}

void copy_exchange_halo(const std::vector<Operator*>& ops, const std::vector<double*>& st, cudaStream_t s) {
    for (size_t r = 0; r + 1 < ops.size(); ++r) {
        int64_t a[8], b[8];
        ops[r]->halo(a);
        ops[r + 1]->halo(b);
        WCB_REQUIRE(a[0] == b[0] && a[6] == b[2] && b[2] > 0 && a[4] == 1,
                    "plans are not consecutive slabs of one grid");
        const size_t xs = (size_t)a[0];
        for (int pl = 0; pl < ops[r]->halo_nplanes; ++pl) {
            double* A = st[r] + pl * ops[r]->halo_pstride;
            double* B = st[r + 1] + pl * ops[r + 1]->halo_pstride;
            WCB_CUDA(cudaMemcpyAsync(B + b[1] * xs, A + a[5] * xs, a[6] * xs * sizeof(double),
                                     cudaMemcpyDeviceToDevice, s));
            WCB_CUDA(cudaMemcpyAsync(A + a[3] * xs, B + b[7] * xs, xs * sizeof(double),
                                     cudaMemcpyDeviceToDevice, s));
        }
    }
}

bool dist_slab(const Operator* op) {
    const Nccl* N = op->ctx->nccl;
    int64_t h[8];
    return N && N->world > 1 && op->halo(h);
}

void nccl_allreduce_max_u64(Context* ctx, unsigned long long* d, int64_t n) {
    Nccl* N = ctx->nccl;
    if (!N || N->world == 1 || n <= 0) return;
    NCCL_CHECK(N, N->allreduce(d, d, (size_t)n, ncclUint64, ncclMax, N->comm, ctx->stream));
}

void nccl_allreduce_sum_f64(Context* ctx, double* d, int64_t n) {
    Nccl* N = ctx->nccl;
    if (!N || N->world == 1 || n <= 0) return;
    NCCL_CHECK(N, N->allreduce(d, d, (size_t)n, ncclDouble, ncclSum, N->comm, ctx->stream));
}

}  // namespace wcb

using namespace wcb;

extern "C" {

int wcb_dist_unique_id(char* out128) {
    try {
        void* h = nccl_dl();
        auto uid = sym<decltype(&ncclGetUniqueId)>(h, "ncclGetUniqueId");
        ncclUniqueId id;
        if (uid(&id) != ncclSuccess) throw Error{WCB_E_CUDA, "ncclGetUniqueId failed"};
        static_assert(sizeof(id.internal) == 128, "NCCL unique id size");
        std::memcpy(out128, id.internal, 128);
        return WCB_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    }
}

int wcb_dist_init(wcb_context* c, int rank, int world, const char* id128) {
    try {
        WCB_REQUIRE(c && id128, "NULL argument");
        WCB_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad rank/world");
        Context* ctx = &c->c;
        WCB_CUDA(cudaSetDevice(ctx->device));
        std::unique_ptr<Nccl> N(new Nccl());
        void* h = nccl_dl();
        N->init = sym<decltype(&ncclCommInitRank)>(h, "ncclCommInitRank");
        N->destroy = sym<decltype(&ncclCommDestroy)>(h, "ncclCommDestroy");
        N->send = sym<decltype(&ncclSend)>(h, "ncclSend");
        N->recv = sym<decltype(&ncclRecv)>(h, "ncclRecv");
        N->gstart = sym<decltype(&ncclGroupStart)>(h, "ncclGroupStart");
        N->gend = sym<decltype(&ncclGroupEnd)>(h, "ncclGroupEnd");
        N->allreduce = sym<decltype(&ncclAllReduce)>(h, "ncclAllReduce");
        N->errstr = sym<decltype(&ncclGetErrorString)>(h, "ncclGetErrorString");
        ncclUniqueId id;
        std::memcpy(id.internal, id128, 128);
        N->rank = rank;
        N->world = world;
        NCCL_CHECK(N.get(), N->init(&N->comm, world, id, rank));
        ctx->nccl = N.release();
        return WCB_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    }
}

int wcb_dist_finalize(wcb_context* c) {
    if (!c || !c->c.nccl) return WCB_OK;
    Nccl* N = c->c.nccl;
    cudaStreamSynchronize(c->c.stream);
    if (N->comm && N->destroy) N->destroy(N->comm);
    delete N;
    c->c.nccl = nullptr;
    return WCB_OK;
}

}  // extern "C"
