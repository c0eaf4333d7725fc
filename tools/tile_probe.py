"""Data-path probe for the 2D step kernel (not product code): moves the step's
bytes (psi_k with halo, psi_{k-1}, 1/m in; psi_{k+1} out) over a config-2
sized padded state with different tile/load schemes, no stencil arithmetic.
    python tools/tile_probe.py"""
import torch
from torch.utils.cpp_extension import load_inline

src = r"""
#include <torch/extension.h>
#include <ATen/cuda/CUDAContext.h>
#include <cuda.h>
#include <cudaTypedefs.h>

constexpr int TJ = 128, TI = 16, UW = 136, UH = 21, PAD = 32;

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k_elem(long n, const double* __restrict__ u, const double* __restrict__ p,
                       const double* __restrict__ m, double* __restrict__ o, double c) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    o[i] = 2.0 * u[i] - p[i] + c * m[i] * u[i];
}

// one CTA per 16x128 tile, 4 warps x 4 rows, lane owns 4 consecutive columns
__global__ void k_tile_ldg(int n_rt, long pitch, const double* __restrict__ u, const double* __restrict__ p,
                           const double* __restrict__ m, double* __restrict__ o, double c) {
  const int strip = blockIdx.x / n_rt, rt = blockIdx.x % n_rt;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  #pragma unroll
  for (int r = 0; r < 4; ++r) {
    const long base = (long)(rt * TI + w * 4 + r + 4) * pitch + strip * TJ + PAD + lane * 4;
    const double4 a = *reinterpret_cast<const double4*>(u + base);
    const double4 b = *reinterpret_cast<const double4*>(p + base);
    const double4 d = *reinterpret_cast<const double4*>(m + base);
    double4 v;
    v.x = 2.0 * a.x - b.x + c * d.x * a.x; v.y = 2.0 * a.y - b.y + c * d.y * a.y;
    v.z = 2.0 * a.z - b.z + c * d.z * a.z; v.w = 2.0 * a.w - b.w + c * d.w * a.w;
    *reinterpret_cast<double4*>(o + base) = v;
  }
}

__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               :: "r"(su(dst)), "l"((unsigned long long)map), "r"(x), "r"(y), "r"(su(bar)) : "memory");
}

// one CTA per tile: TMA u (with halo box), p, m into smem; MODE 0: lane reads
// its 4 columns (32 B stride), MODE 1: conflict-free double2 at lane + 32 h
template <int MODE>
__global__ void __launch_bounds__(160, 3) k_tile_tma(int n_rt, long pitch, const __grid_constant__ CUtensorMap tu,
    const __grid_constant__ CUtensorMap tp, const __grid_constant__ CUtensorMap tm, double* __restrict__ o, double c) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* us = (double*)sm;
  double* ps = (double*)(sm + 22912);
  double* ms = (double*)(sm + 22912 + 16384);
  uint64_t* bar = (uint64_t*)(sm + 22912 + 32768);
  const int strip = blockIdx.x / n_rt, rt = blockIdx.x % n_rt;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int J0 = strip * TJ, I0 = rt * TI;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(bar)), "r"(22848 + 32768) : "memory");
    tma2(us, &tu, J0 + PAD - 4, I0, bar);
    tma2(ps, &tp, J0 + PAD, I0 + 4, bar);
    tma2(ms, &tm, J0 + PAD, I0 + 4, bar);
  }
  __syncthreads();
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0; selp.u32 %0, 1, 0, q; }"
                 : "=r"(done) : "r"(su(bar)) : "memory");
  if (w == 4) return;
  #pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int tr = w * 4 + r;
    const long grow = (long)(I0 + tr + 4) * pitch + J0 + PAD;
    if (MODE == 0) {
      const double* ur = us + (tr + 4) * UW + 4 + lane * 4;
      const double* pr = ps + tr * TJ + lane * 4;
      const double* mr = ms + tr * TJ + lane * 4;
      double v[4];
      #pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = 2.0 * ur[j] - pr[j] + c * mr[j] * ur[j];
      *reinterpret_cast<double4*>(o + grow + lane * 4) = make_double4(v[0], v[1], v[2], v[3]);
    } else {
      #pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = 2 * (lane + 32 * h);
        const double2 a = *reinterpret_cast<const double2*>(us + (tr + 4) * UW + 4 + col);
        const double2 b = *reinterpret_cast<const double2*>(ps + tr * TJ + col);
        const double2 d = *reinterpret_cast<const double2*>(ms + tr * TJ + col);
        *reinterpret_cast<double2*>(o + grow + col) =
            make_double2(2.0 * a.x - b.x + c * d.x * a.x, 2.0 * a.y - b.y + c * d.y * a.y);
      }
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  static PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
  if (!f) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&f, cudaEnableDefault, &q);
  }
  return f;
}
#include <map>
static CUtensorMap mk(const double* base, long pitch, long rows, int bw, int bh) {
  static std::map<std::pair<const double*, int>, CUtensorMap> cache;
  auto key = std::make_pair(base, bw);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  CUtensorMap mp;
  cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)pitch * 8};
  cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh}, es[2] = {1, 1};
  enc()(&mp, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cache[key] = mp;
  return mp;
}

void run(torch::Tensor u, torch::Tensor p, torch::Tensor m, long pitch, long rows, int n_strips, int n_rt,
         int kind) {
  auto s = at::cuda::getCurrentCUDAStream();
  const long n = u.numel();
  const double *U = u.data_ptr<double>(), *Pp = p.data_ptr<double>(), *M = m.data_ptr<double>();
  double* O = p.data_ptr<double>();
  if (kind == 0) k_elem<<<148 * 8, 256, 0, s>>>(n, U, Pp, M, O, 1e-9);
  else if (kind == 1) k_tile_ldg<<<n_strips * n_rt, 128, 0, s>>>(n_rt, pitch, U, Pp, M, O, 1e-9);
  else {
    CUtensorMap a = mk(U, pitch, rows, UW, UH), b = mk(Pp, pitch, rows, TJ, TI), c = mk(M, pitch, rows, TJ, TI);
    const int smem = 22912 + 32768 + 64;
    if (kind == 2) {
      cudaFuncSetAttribute(k_tile_tma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k_tile_tma<0><<<n_strips * n_rt, 160, smem, s>>>(n_rt, pitch, a, b, c, O, 1e-9);
    } else {
      cudaFuncSetAttribute(k_tile_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k_tile_tma<1><<<n_strips * n_rt, 160, smem, s>>>(n_rt, pitch, a, b, c, O, 1e-9);
    }
  }
}
"""
mod = load_inline("tile_probe", cpp_sources="void run(torch::Tensor u, torch::Tensor p, torch::Tensor m, long pitch, long rows, int n_strips, int n_rt, int kind);",
                  cuda_sources=src, functions=["run"],
                  extra_cuda_cflags=["-gencode=arch=compute_100a,code=sm_100a", "-O3"], verbose=False)
n1, P = 2049, 4
n_strips, n_rt = 17, 129
pitch = 2208
rows = n_rt * 16 + 2 * P + 1
n = rows * pitch
dofs = n1 * n1
for name, kind in (("elementwise", 0), ("tile-ldg", 1), ("tile-tma lane-stride", 2), ("tile-tma conflict-free", 3)):
    u = torch.rand(n, dtype=torch.float64, device="cuda")
    p = torch.rand(n, dtype=torch.float64, device="cuda")
    m = torch.rand(n, dtype=torch.float64, device="cuda")
    for _ in range(20):
        mod.run(u, p, m, pitch, rows, n_strips, n_rt, kind); u, p = p, u
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 200
    e0.record()
    for _ in range(it):
        mod.run(u, p, m, pitch, rows, n_strips, n_rt, kind); u, p = p, u
    e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / it
    print(f"{name}: {us:.2f} us/step  {32 * dofs / us / 1e3:.0f} GB/s (32 B/DOF, {dofs} DOFs)", flush=True)
