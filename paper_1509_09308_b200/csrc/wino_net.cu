// Glue for chaining layers into the VGG-E conv stack (network.py): ReLU, with
// an optional 2x2 / stride-2 max-pool, between two Winograd layers.  Not on the
// reference's path (winoconv has no activations or pooling); it lets layer i's
// output feed layer i+1 at the shapes VGG network E uses.
//
// HBM-bound elementwise pass: one thread per output element, its 2x2 window
// read as two float2 row loads (W even), so a warp's loads cover 64 contiguous
// input floats per row.
#include "wino_internal.h"

namespace wino {

__global__ void __launch_bounds__(256) relu_pool_kernel(const float* __restrict__ x,
                                                        float* __restrict__ y, long long planes,
                                                        int H, int W, int pool) {
  griddep_launch();
  griddep_wait();
  const int oh = pool ? H / 2 : H, ow = pool ? W / 2 : W;
  const long long total = planes * oh * ow;
  for (long long o = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long pl = o / (static_cast<long long>(oh) * ow);
    const int r = static_cast<int>(o - pl * oh * ow);
    const int oy = r / ow, ox = r - (r / ow) * ow;
    const float* src = x + pl * H * W;
    float v;
    if (pool) {
      const float2 a = *reinterpret_cast<const float2*>(src + (2 * oy) * W + 2 * ox);
      const float2 b = *reinterpret_cast<const float2*>(src + (2 * oy + 1) * W + 2 * ox);
      v = fmaxf(fmaxf(a.x, a.y), fmaxf(b.x, b.y));
    } else {
      v = src[oy * W + ox];
    }
    y[o] = fmaxf(v, 0.f);
  }
}

cudaError_t launch_relu_pool(const float* x, float* y, int N, int C, int H, int W, int pool,
                             cudaStream_t s) {
  const long long planes = static_cast<long long>(N) * C;
  const long long total = planes * (pool ? (H / 2) * (W / 2) : static_cast<long long>(H) * W);
  if (total <= 0) return cudaSuccess;
  long long blocks = (total + 255) / 256;
  const long long cap = static_cast<long long>(device_sms()) * 8;
  if (blocks > cap) blocks = cap;
  launch_k(relu_pool_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, s, x, y, planes,
           H, W, pool);
  return cudaGetLastError();
}

}  // namespace wino

extern "C" int wino_relu_pool(const float* x, float* y, int N, int C, int H, int W, int pool,
                              void* stream) {
  using namespace wino;
  if (!x || !y || N < 1 || C < 1 || H < 1 || W < 1) {
    set_error("relu_pool: bad arguments");
    return WINO_EINVAL;
  }
  if (pool && ((H | W) & 1)) {
    set_error("relu_pool: 2x2 pooling needs even H and W (got %dx%d)", H, W);
    return WINO_EINVAL;
  }
  if (pool && ((reinterpret_cast<uintptr_t>(x) & 7) != 0)) {
    set_error("relu_pool: input must be 8-byte aligned");
    return WINO_EINVAL;
  }
  cudaError_t e = launch_relu_pool(x, y, N, C, H, W, pool, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    set_error("relu_pool: %s", cudaGetErrorString(e));
    return WINO_ECUDA;
  }
  return WINO_OK;
}
