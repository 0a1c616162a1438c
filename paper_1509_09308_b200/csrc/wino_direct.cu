// Direct correlation with zero padding on CUDA cores: the reference's
// `direct` / `direct-fp32` algorithms and the fp64 accuracy oracle of
// cmd_accuracy (direct.py:82-114, commands.py:31-38, 64-92).  Not on the
// Winograd hot path; it lets `run_layer` / `cmd_accuracy` run on the GPU.
//
// One thread per output (n, k, x, y).  The accumulation order and rounding
// follow the reference exactly: for c, then v (column tap), then u (row tap),
// p = round(d * g) and acc = round(acc + p) in the accumulator type (the
// NumPy broadcast multiply, then the in-place add; no fused multiply-add), with
// out-of-image taps skipped rather than added as zero.  The result is
// therefore bitwise identical to the reference's direct_forward.
#include <cstdio>

#include "wino_internal.h"

namespace wino {

template <typename TI, typename TA>
__device__ __forceinline__ TA mul_rn(TI a, TI b);
template <>
__device__ __forceinline__ float mul_rn<float, float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_rn<float, double>(float a, float b) {
  return __dmul_rn(static_cast<double>(a), static_cast<double>(b));
}
template <>
__device__ __forceinline__ double mul_rn<double, double>(double a, double b) {
  return __dmul_rn(a, b);
}
template <>
__device__ __forceinline__ float mul_rn<double, float>(double a, double b) {
  return __fmul_rn(static_cast<float>(a), static_cast<float>(b));
}
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <typename TI, typename TA>
__global__ void __launch_bounds__(256) direct_conv_kernel(const TI* __restrict__ d,
                                                          const TI* __restrict__ g,
                                                          TA* __restrict__ y, int N, int C, int H,
                                                          int W, int K, int R, int S, int pad,
                                                          int oh, int ow) {
  // launched with PDL like every library kernel: wait for the predecessor's
  // writes (d may be the output of the previous launch on this stream)
  griddep_wait();
  griddep_launch();
  const long long o = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long total = static_cast<long long>(N) * K * oh * ow;
  if (o >= total) return;
  const int xy = static_cast<int>(o % (static_cast<long long>(oh) * ow));
  const long long nk = o / (static_cast<long long>(oh) * ow);
  const int k = static_cast<int>(nk % K), n = static_cast<int>(nk / K);
  const int x = xy / ow, yy = xy - (xy / ow) * ow;
  TA acc = TA(0);
  for (int c = 0; c < C; ++c) {
    const TI* dc = d + (static_cast<size_t>(n) * C + c) * H * W;
    const TI* gc = g + (static_cast<size_t>(k) * C + c) * R * S;
    for (int v = 0; v < S; ++v) {
      const int col = yy + v - pad;
      if (col < 0 || col >= W) continue;
      for (int u = 0; u < R; ++u) {
        const int row = x + u - pad;
        if (row < 0 || row >= H) continue;
        acc = add_rn(acc, mul_rn<TI, TA>(dc[static_cast<size_t>(row) * W + col], gc[u * S + v]));
      }
    }
  }
  y[o] = acc;
}

cudaError_t launch_direct(int in_prec, int acc_prec, const void* d, const void* g, void* y, int N,
                          int C, int H, int W, int K, int R, int S, int pad, int oh, int ow,
                          cudaStream_t s) {
  const long long total = static_cast<long long>(N) * K * oh * ow;
  if (total <= 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((total + 255) / 256));
  const bool in64 = in_prec == kFP64, acc64 = acc_prec == kFP64;
  if (in64 && acc64)
    launch_k(direct_conv_kernel<double, double>, grid, dim3(256), 0, s,
             static_cast<const double*>(d), static_cast<const double*>(g), static_cast<double*>(y),
             N, C, H, W, K, R, S, pad, oh, ow);
  else if (in64)
    launch_k(direct_conv_kernel<double, float>, grid, dim3(256), 0, s,
             static_cast<const double*>(d), static_cast<const double*>(g), static_cast<float*>(y),
             N, C, H, W, K, R, S, pad, oh, ow);
  else if (acc64)
    launch_k(direct_conv_kernel<float, double>, grid, dim3(256), 0, s,
             static_cast<const float*>(d), static_cast<const float*>(g), static_cast<double*>(y),
             N, C, H, W, K, R, S, pad, oh, ow);
  else
    launch_k(direct_conv_kernel<float, float>, grid, dim3(256), 0, s,
             static_cast<const float*>(d), static_cast<const float*>(g), static_cast<float*>(y), N,
             C, H, W, K, R, S, pad, oh, ow);
  return cudaGetLastError();
}

}  // namespace wino
