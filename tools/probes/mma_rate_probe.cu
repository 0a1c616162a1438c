// MMA issue-rate probe: cycles per tcgen05.mma instruction (M = 128, cta_group::1)
// for kind::tf32 with A in smem or TMEM and kind::f16, N = 32..256, issued back to
// back by one thread into one accumulator, one CTA per SM (148 CTAs).  Decides
// whether the 3xTF32 k-loop at small P is bound by MMA instructions or by flops.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1509_09308_b200/csrc \
//        -o mma_rate_probe mma_rate_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100_ptx.cuh"
using namespace wino;

template <int KIND, int N, bool ATM>
__global__ void __launch_bounds__(128, 1) probe(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* s = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += 128) reinterpret_cast<float*>(s)[i] = 0.f;
  if (warp == 0) ptx::tmem_alloc(&slot, 512);
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  ptx::fence_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = ptx::umma_idesc(KIND ? 2u : 1u, 128, N);
    const uint64_t da = ptx::umma_desc_sw128(ptx::smem_u32(s));
    const uint64_t db = ptx::umma_desc_sw128(ptx::smem_u32(s + 16384));
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if constexpr (ATM)
          ptx::umma_tf32_tmem_a(tm, tm + 256 + 8 * k, db + 2 * k, idesc, 1u);
        else
          ptx::umma<KIND>(tm, da + 2 * k, db + 2 * k, idesc, 1u);
      }
    }
    ptx::umma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tm, 512);
}

template <int KIND, int N, bool ATM>
void run(const char* name, unsigned long long* d) {
  const int iters = 2000;
  auto k = probe<KIND, N, ATM>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<148, 128, 64 * 1024>>>(d, iters);
  k<<<148, 128, 64 * 1024>>>(d, iters);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double cyc = double(mx) / (iters * 4);
  const double flop = 2.0 * 128 * N * (KIND ? 8 : 16);
  printf("%-28s N=%3d: %6.1f cycles/MMA, %7.0f flop/clk/SM (%s)\n", name, N, cyc, flop / cyc,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  run<1, 32, false>("tf32 A smem", d);
  run<1, 64, false>("tf32 A smem", d);
  run<1, 128, false>("tf32 A smem", d);
  run<1, 256, false>("tf32 A smem", d);
  run<1, 32, true>("tf32 A tmem", d);
  run<1, 64, true>("tf32 A tmem", d);
  run<1, 128, true>("tf32 A tmem", d);
  run<1, 256, true>("tf32 A tmem", d);
  run<0, 64, false>("bf16 A smem", d);
  run<0, 128, false>("bf16 A smem", d);
  run<0, 256, false>("bf16 A smem", d);
  return 0;
}
