"""Memory-roofline probe for the step loop's data volume: a fused elementwise
leapfrog (3 reads + 1 write per node, no stencil) over config-2-sized state
vectors, ping-ponging like the real loop.  Not product code."""
import torch
from torch.utils.cpp_extension import load_inline

src = r"""
#include <torch/extension.h>
__global__ void k(long n, const double* __restrict__ u, const double* __restrict__ p,
                  const double* __restrict__ m, double* __restrict__ o, double c) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    o[i] = 2.0 * u[i] - p[i] + c * m[i] * u[i];
}
__global__ void k2(long n, const double2* __restrict__ u, const double2* __restrict__ p,
                  const double2* __restrict__ m, double2* __restrict__ o, double c) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double2 a = u[i], b = p[i], d = m[i];
    o[i] = make_double2(2.0 * a.x - b.x + c * d.x * a.x, 2.0 * a.y - b.y + c * d.y * a.y);
  }
}
void run(torch::Tensor u, torch::Tensor p, torch::Tensor m, int blocks, int vec) {
  long n = u.numel();
  auto s = at::cuda::getCurrentCUDAStream();
  if (vec) k2<<<blocks, 256, 0, s>>>(n / 2, (const double2*)u.data_ptr<double>(), (const double2*)p.data_ptr<double>(),
                                     (const double2*)m.data_ptr<double>(), (double2*)p.data_ptr<double>(), 1e-9);
  else k<<<blocks, 256, 0, s>>>(n, u.data_ptr<double>(), p.data_ptr<double>(), m.data_ptr<double>(), p.data_ptr<double>(), 1e-9);
}
"""
mod = load_inline("probe", cpp_sources="void run(torch::Tensor u, torch::Tensor p, torch::Tensor m, int blocks, int vec);",
                  cuda_sources="#include <ATen/cuda/CUDAContext.h>\n" + src, functions=["run"],
                  extra_cuda_cflags=["-gencode=arch=compute_100a,code=sm_100a", "-O3"], verbose=False)
for n in (4_350_000, 16_000_000, 64_000_000):
    u = torch.rand(n, dtype=torch.float64, device="cuda")
    p = torch.rand(n, dtype=torch.float64, device="cuda")
    m = torch.rand(n, dtype=torch.float64, device="cuda")
    for vec in (0, 1):
        for blocks in (148 * 8, 148 * 32, (n + 255) // 256):
            for _ in range(20):
                mod.run(u, p, m, blocks, vec); u, p = p, u
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            it = 200
            e0.record()
            for _ in range(it):
                mod.run(u, p, m, blocks, vec); u, p = p, u
            e1.record(); e1.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / it
            print(f"n={n} vec={vec} blocks={blocks}: {us:.2f} us/step  {32 * n / us / 1e3:.0f} GB/s")
