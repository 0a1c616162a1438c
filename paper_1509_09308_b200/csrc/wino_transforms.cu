// Winograd transform kernels: filter transform G g G^T, input-tile transform
// B^T d B, and the inverse transform A^T M A with clipped write-back.
// These are HBM-bandwidth-bound CUDA-core kernels; coalescing is arranged
// through shared-memory staging so every global access is a contiguous row.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "wino_internal.h"
#include "winograd_mats.cuh"

namespace wino {

// --------------------------------------------------------------- operand store
// Writes one transform-space value in the GEMM operand format at element index
// `idx` of split plane 0; split plane s lives `plane` elements further.
template <int PREC>
struct OpStore;

template <>
struct OpStore<kFP32> {  // 3xTF32: hi = rna_tf32(x), lo = x - hi (exact in fp32)
  using T = float;
  __device__ static void put(void* base, size_t idx, size_t plane, float x) {
    uint32_t hi_bits;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi_bits) : "f"(x));
    const float hi = __uint_as_float(hi_bits);
    float* p = static_cast<float*>(base);
    p[idx] = hi;
    p[idx + plane] = x - hi;
  }
};
template <>
struct OpStore<kTF32> {
  using T = float;
  __device__ static void put(void* base, size_t idx, size_t, float x) {
    uint32_t b;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(x));
    static_cast<float*>(base)[idx] = __uint_as_float(b);
  }
};
template <>
struct OpStore<kBF16> {
  using T = float;
  __device__ static void put(void* base, size_t idx, size_t, float x) {
    static_cast<__nv_bfloat16*>(base)[idx] = __float2bfloat16_rn(x);
  }
};
template <>
struct OpStore<kFP16> {
  using T = float;
  __device__ static void put(void* base, size_t idx, size_t, float x) {
    static_cast<__half*>(base)[idx] = __float2half_rn(x);
  }
};
template <>
struct OpStore<kFP64> {
  using T = double;
  __device__ static void put(void* base, size_t idx, size_t, double x) {
    static_cast<double*>(base)[idx] = x;
  }
};

// ============================================================ filter transform
// One thread per (k, c).  U[s][comp][k][c] with c fastest: consecutive threads
// write consecutive c (coalesced).  (engine.py:104-114)
template <int M, int PREC>
__global__ void __launch_bounds__(256) filter_transform_kernel(
    const typename OpStore<PREC>::T* __restrict__ g, void* __restrict__ U, int K, int C,
    int c_pad) {
  using T = typename OpStore<PREC>::T;
  using A = Alg<M>;
  constexpr int AL = A::alpha;
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long long>(K) * C) return;
  const int k = static_cast<int>(t / C);
  const int c = static_cast<int>(t - static_cast<long long>(k) * C);
  T in[3][3];
  const T* src = g + t * 9;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) in[i][j] = src[i * 3 + j];
  T out[AL][AL];
  sandwich<T, AL, 3>(in, out, [](int i, int j) { return A::G(i, j); });
  const size_t plane = static_cast<size_t>(AL) * AL * K * c_pad;
#pragma unroll
  for (int xi = 0; xi < AL; ++xi)
#pragma unroll
    for (int nu = 0; nu < AL; ++nu) {
      const size_t idx = (static_cast<size_t>(xi * AL + nu) * K + k) * c_pad + c;
      OpStore<PREC>::put(U, idx, plane, out[xi][nu]);
    }
}

// ============================================================= input transform
// Block = 32 channels x TPX consecutive tiles of one tile row (n, ty).
// Phase 1 stages the alpha input rows of every channel in shared memory with
// x-contiguous (coalesced) loads; out-of-image pixels are written as 0, so the
// zero padding is never materialised in HBM (engine.py:13-16, 170-191).
// Phase 2: lane = channel, warp = tile; each thread forms B^T d B for its
// patch and writes the alpha^2 values to V[s][comp][p][c] (c fastest -> a
// warp writes one contiguous 32-channel row per component).  (engine.py:232-237)
constexpr int kInCB = 32;
template <int M>
struct InCfg {
  static constexpr int alpha = M + 2;
  static constexpr int tpx = (M == 2) ? 32 : 16;      // tiles per block along x
  static constexpr int xw = tpx * M + 2;              // staged row width (halo r-1 = 2)
  static constexpr int plane = alpha * xw + 1;        // odd stride: conflict-free per-lane reads
};

template <int M, int PREC>
__global__ void __launch_bounds__(256) input_transform_kernel(
    const typename OpStore<PREC>::T* __restrict__ d, void* __restrict__ V, int N, int C, int H,
    int W, int pad, int th, int tw, int row0, long long Pc, int c_pad) {
  using T = typename OpStore<PREC>::T;
  using A = Alg<M>;
  using Cfg = InCfg<M>;
  constexpr int AL = A::alpha;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s = reinterpret_cast<T*>(smem_raw);

  const int row = row0 + blockIdx.y;  // global tile row = n*th + ty
  const int n = row / th;
  const int ty = row - n * th;
  const int tx0 = blockIdx.x * Cfg::tpx;
  const int c0 = blockIdx.z * kInCB;
  const int y0 = M * ty - pad;
  const int x0 = M * tx0 - pad;

  // ---- phase 1: stage [32 ch][alpha rows][xw] with zero fill
  const int total = kInCB * AL * Cfg::xw;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int x = e % Cfg::xw;
    const int rest = e / Cfg::xw;
    const int i = rest % AL;
    const int cl = rest / AL;
    const int c = c0 + cl;
    const int gy = y0 + i, gx = x0 + x;
    T v = T(0);
    if (c < C && gy >= 0 && gy < H && gx >= 0 && gx < W)
      v = __ldg(d + ((static_cast<size_t>(n) * C + c) * H + gy) * W + gx);
    s[cl * Cfg::plane + i * Cfg::xw + x] = v;
  }
  __syncthreads();

  // ---- phase 2: transform and scatter
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int c = c0 + lane;
  const int ntiles = min(Cfg::tpx, tw - tx0);
  const size_t plane = static_cast<size_t>(AL) * AL * Pc * c_pad;
  for (int t = warp; t < ntiles; t += blockDim.x >> 5) {
    if (c >= C) continue;
    T in[AL][AL];
    const T* src = s + lane * Cfg::plane + t * M;
#pragma unroll
    for (int i = 0; i < AL; ++i)
#pragma unroll
      for (int j = 0; j < AL; ++j) in[i][j] = src[i * Cfg::xw + j];
    T out[AL][AL];
    sandwich<T, AL, AL>(in, out, [](int i, int j) { return A::BT(i, j); });
    const long long p = static_cast<long long>(blockIdx.y) * tw + tx0 + t;  // chunk-local tile
#pragma unroll
    for (int xi = 0; xi < AL; ++xi)
#pragma unroll
      for (int nu = 0; nu < AL; ++nu) {
        const size_t idx = (static_cast<size_t>(xi * AL + nu) * Pc + p) * c_pad + c;
        OpStore<PREC>::put(V, idx, plane, out[xi][nu]);
      }
  }
}

// ============================================================ output transform
// One thread per (chunk tile p, filter k): reads the alpha^2 accumulators
// M[comp][k][p] (coalesced over p), forms A^T M A and writes the valid
// vr x vc corner of the m x m tile (edge tiles clipped, engine.py:241-254).
template <int M, typename TA>
__global__ void __launch_bounds__(128) output_transform_kernel(const TA* __restrict__ Mbuf,
                                                               TA* __restrict__ y, int N, int K,
                                                               int th, int tw, int oh, int ow,
                                                               int row0, long long Pc) {
  using A = Alg<M>;
  constexpr int AL = A::alpha;
  const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (p >= Pc) return;
  TA in[AL][AL];
#pragma unroll
  for (int xi = 0; xi < AL; ++xi)
#pragma unroll
    for (int nu = 0; nu < AL; ++nu)
      in[xi][nu] = Mbuf[(static_cast<size_t>(xi * AL + nu) * K + k) * Pc + p];
  TA out[M][M];
  sandwich<TA, M, AL>(in, out, [](int i, int j) { return A::AT(i, j); });
  const long long gp = static_cast<long long>(row0) * tw + p;
  const int n = static_cast<int>(gp / (static_cast<long long>(th) * tw));
  const int rest = static_cast<int>(gp - static_cast<long long>(n) * th * tw);
  const int ty = rest / tw, tx = rest - (rest / tw) * tw;
  const int vr = min(M, oh - M * ty), vc = min(M, ow - M * tx);
  TA* dst = y + ((static_cast<size_t>(n) * K + k) * oh + M * ty) * ow + M * tx;
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j < M; ++j)
      if (i < vr && j < vc) dst[static_cast<size_t>(i) * ow + j] = out[i][j];
}

// ================================================================ launchers
template <int M>
static cudaError_t filter_dispatch(int prec, const void* g, void* U, int K, int C, int c_pad,
                                   cudaStream_t s) {
  const long long n = static_cast<long long>(K) * C;
  const dim3 grid(static_cast<unsigned>((n + 255) / 256));
  switch (prec) {
    case kFP32:
      filter_transform_kernel<M, kFP32><<<grid, 256, 0, s>>>(static_cast<const float*>(g), U, K,
                                                             C, c_pad);
      break;
    case kTF32:
      filter_transform_kernel<M, kTF32><<<grid, 256, 0, s>>>(static_cast<const float*>(g), U, K,
                                                             C, c_pad);
      break;
    case kBF16:
      filter_transform_kernel<M, kBF16><<<grid, 256, 0, s>>>(static_cast<const float*>(g), U, K,
                                                             C, c_pad);
      break;
    case kFP16:
      filter_transform_kernel<M, kFP16><<<grid, 256, 0, s>>>(static_cast<const float*>(g), U, K,
                                                             C, c_pad);
      break;
    case kFP64:
      filter_transform_kernel<M, kFP64><<<grid, 256, 0, s>>>(static_cast<const double*>(g), U,
                                                             K, C, c_pad);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_filter_transform(int m, int prec, const void* g, void* U, int K, int C,
                                    int c_pad, cudaStream_t s) {
  if (K <= 0 || C <= 0) return cudaSuccess;
  return m == 2 ? filter_dispatch<2>(prec, g, U, K, C, c_pad, s)
                : filter_dispatch<4>(prec, g, U, K, C, c_pad, s);
}

template <int M, int PREC>
static cudaError_t input_one(const void* d, void* V, int N, int C, int H, int W, int pad, int th,
                             int tw, int row0, int rows, long long Pc, int c_pad,
                             cudaStream_t s) {
  using T = typename OpStore<PREC>::T;
  using Cfg = InCfg<M>;
  const size_t smem = sizeof(T) * kInCB * Cfg::plane;
  auto kern = input_transform_kernel<M, PREC>;
  static bool configured = false;  // benign race: idempotent attribute set
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    configured = true;
  }
  const dim3 grid((tw + Cfg::tpx - 1) / Cfg::tpx, rows, (C + kInCB - 1) / kInCB);
  kern<<<grid, 256, smem, s>>>(static_cast<const T*>(d), V, N, C, H, W, pad, th, tw, row0, Pc,
                               c_pad);
  return cudaGetLastError();
}

template <int M>
static cudaError_t input_dispatch(int prec, const void* d, void* V, int N, int C, int H, int W,
                                  int pad, int th, int tw, int row0, int rows, long long Pc,
                                  int c_pad, cudaStream_t s) {
  switch (prec) {
    case kFP32: return input_one<M, kFP32>(d, V, N, C, H, W, pad, th, tw, row0, rows, Pc, c_pad, s);
    case kTF32: return input_one<M, kTF32>(d, V, N, C, H, W, pad, th, tw, row0, rows, Pc, c_pad, s);
    case kBF16: return input_one<M, kBF16>(d, V, N, C, H, W, pad, th, tw, row0, rows, Pc, c_pad, s);
    case kFP16: return input_one<M, kFP16>(d, V, N, C, H, W, pad, th, tw, row0, rows, Pc, c_pad, s);
    case kFP64: return input_one<M, kFP64>(d, V, N, C, H, W, pad, th, tw, row0, rows, Pc, c_pad, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_input_transform(int m, int prec, const void* d, void* V, int N, int C, int H,
                                   int W, int pad, int th, int tw, int row0, int rows,
                                   long long Pc, int c_pad, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  return m == 2 ? input_dispatch<2>(prec, d, V, N, C, H, W, pad, th, tw, row0, rows, Pc, c_pad, s)
                : input_dispatch<4>(prec, d, V, N, C, H, W, pad, th, tw, row0, rows, Pc, c_pad, s);
}

cudaError_t launch_output_transform(int m, int prec, const void* Mbuf, void* y, int N, int K,
                                    int th, int tw, int oh, int ow, int row0, long long Pc,
                                    cudaStream_t s) {
  if (Pc <= 0 || K <= 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((Pc + 127) / 128), K);
  if (prec == kFP64) {
    if (m == 2)
      output_transform_kernel<2, double><<<grid, 128, 0, s>>>(
          static_cast<const double*>(Mbuf), static_cast<double*>(y), N, K, th, tw, oh, ow, row0, Pc);
    else
      output_transform_kernel<4, double><<<grid, 128, 0, s>>>(
          static_cast<const double*>(Mbuf), static_cast<double*>(y), N, K, th, tw, oh, ow, row0, Pc);
  } else {
    if (m == 2)
      output_transform_kernel<2, float><<<grid, 128, 0, s>>>(
          static_cast<const float*>(Mbuf), static_cast<float*>(y), N, K, th, tw, oh, ow, row0, Pc);
    else
      output_transform_kernel<4, float><<<grid, 128, 0, s>>>(
          static_cast<const float*>(Mbuf), static_cast<float*>(y), N, K, th, tw, oh, ow, row0, Pc);
  }
  return cudaGetLastError();
}

}  // namespace wino
