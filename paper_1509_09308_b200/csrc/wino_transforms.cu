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
// Block = 256 consecutive (k, c) pairs = 256 contiguous 3x3 filters: staged
// through shared memory with coalesced loads (the 36-byte records would
// otherwise give strided warp loads), then one thread per (k, c) writes
// U[s][comp][k][c] with c fastest (coalesced across the warp).
// (engine.py:104-114)
template <int M, int PREC>
__global__ void __launch_bounds__(256) filter_transform_kernel(
    const typename OpStore<PREC>::T* __restrict__ g, void* __restrict__ U, int K, int C,
    int c_pad) {
  using T = typename OpStore<PREC>::T;
  using A = Alg<M>;
  constexpr int AL = A::alpha;
  __shared__ T sg[256 * 9 + 1];
  const long long total = static_cast<long long>(K) * C;
  const long long t0 = static_cast<long long>(blockIdx.x) * 256;
  const int nloc = static_cast<int>(min(256LL, total - t0));
  const T* src = g + t0 * 9;
  for (int e = threadIdx.x; e < nloc * 9; e += 256) sg[e] = __ldg(src + e);
  __syncthreads();
  if (static_cast<int>(threadIdx.x) >= nloc) return;
  const long long t = t0 + threadIdx.x;
  const int k = static_cast<int>(t / C);
  const int c = static_cast<int>(t - static_cast<long long>(k) * C);
  T in[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) in[i][j] = sg[threadIdx.x * 9 + i * 3 + j];
  T out[AL][AL];
  sandwich<T, AL, 3>(in, out, [](int i, int j) { return A::G(i, j); });
  const size_t plane = static_cast<size_t>(AL) * AL * K * c_pad;
  const size_t cstride = static_cast<size_t>(K) * c_pad;
  size_t idx = static_cast<size_t>(k) * c_pad + c;
#pragma unroll
  for (int xi = 0; xi < AL; ++xi)
#pragma unroll
    for (int nu = 0; nu < AL; ++nu) {
      OpStore<PREC>::put(U, idx, plane, out[xi][nu]);
      idx += cstride;
    }
}

// ============================================================= input transform
// Block = CB channels x TPX consecutive tiles of one tile row (n, ty).
// Phase 1 stages the alpha input rows of every channel in shared memory with
// x-contiguous (coalesced) loads; out-of-image pixels are written as 0, so the
// zero padding is never materialised in HBM (engine.py:13-16, 170-191).
// Phase 2: lane = channel group (CPL consecutive channels), warp = tile; each
// thread forms B^T d B for its patch(es) and writes the alpha^2 values to
// V[s][comp][p][c] (c fastest): every warp store is one contiguous 128-byte
// row segment (32 lanes x CPL channels x operand bytes).  (engine.py:232-237)
template <int PREC>
struct InPack {  // channels per lane: 2 for 16-bit operands (packed 4-byte stores)
  static constexpr int cpl = (PREC == kBF16 || PREC == kFP16) ? 2 : 1;
};
template <int M, int PREC>
struct InCfg {
  static constexpr int alpha = M + 2;
  static constexpr int cpl = InPack<PREC>::cpl;
  static constexpr int cb = 32 * cpl;  // channels per block
  static constexpr bool wide = (cpl == 2) || (PREC == kFP64);
  static constexpr int tpx = (M == 2) ? (wide ? 16 : 32) : (wide ? 8 : 16);
  static constexpr int xw = tpx * M + 2;        // staged row width (halo r-1 = 2)
  static constexpr int plane = alpha * xw + 1;  // odd stride: conflict-free per-lane reads
};

template <int PREC>
__device__ __forceinline__ void put_ops(void* base, size_t idx, size_t plane, const float* v) {
  if constexpr (PREC == kBF16) {
    *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(base) + idx) =
        __floats2bfloat162_rn(v[0], v[1]);
  } else if constexpr (PREC == kFP16) {
    *reinterpret_cast<__half2*>(static_cast<__half*>(base) + idx) = __floats2half2_rn(v[0], v[1]);
  } else {
    OpStore<PREC>::put(base, idx, plane, v[0]);
  }
}
template <int PREC>
__device__ __forceinline__ void put_ops(void* base, size_t idx, size_t plane, const double* v) {
  OpStore<PREC>::put(base, idx, plane, v[0]);
}

template <int M, int PREC>
__global__ void __launch_bounds__(256) input_transform_kernel(
    const typename OpStore<PREC>::T* __restrict__ d, void* __restrict__ V, int N, int C, int H,
    int W, int pad, int th, int tw, int row0, long long Pc, int c_pad) {
  using T = typename OpStore<PREC>::T;
  using A = Alg<M>;
  using Cfg = InCfg<M, PREC>;
  constexpr int AL = A::alpha;
  constexpr int CPL = Cfg::cpl;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s = reinterpret_cast<T*>(smem_raw);

  const int row = row0 + blockIdx.y;  // global tile row = n*th + ty
  const int n = row / th;
  const int ty = row - n * th;
  const int tx0 = blockIdx.x * Cfg::tpx;
  const int c0 = blockIdx.z * Cfg::cb;
  const int y0 = M * ty - pad;
  const int x0 = M * tx0 - pad;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  constexpr int NW = 256 / 32;

  // ---- phase 1: stage [cb ch][alpha rows][xw] with zero fill.  Every element
  // is an independent cp.async (zero-filled when out of range), so all loads of
  // the block are in flight at once instead of one latency per row.
  // Warp w stages rows (channel, i) = w, w+8, ...; lane l covers x = l, l+32.
  // Row-level bounds/addresses are computed once per row, so each element is a
  // compare, a select and one cp.async.
  const size_t img = static_cast<size_t>(n) * C * H * W;
  constexpr int XH = (Cfg::xw + 31) / 32;
  int gx_l[XH];
  bool okx[XH];
#pragma unroll
  for (int h = 0; h < XH; ++h) {
    gx_l[h] = x0 + lane + 32 * h;
    okx[h] = (lane + 32 * h < Cfg::xw) && gx_l[h] >= 0 && gx_l[h] < W;
  }
  for (int cr = warp; cr < Cfg::cb * AL; cr += NW) {
    const int cl = cr / AL;
    const int i = cr - cl * AL;
    const int c = c0 + cl, gy = y0 + i;
    const bool rowok = (c < C) && (gy >= 0) && (gy < H);
    const T* row = d + img + (rowok ? (static_cast<size_t>(c) * H + gy) * W : 0);
    const uint32_t dst0 = static_cast<uint32_t>(
        __cvta_generic_to_shared(s + cl * Cfg::plane + i * Cfg::xw + lane));
#pragma unroll
    for (int h = 0; h < XH; ++h) {
      if (lane + 32 * h >= Cfg::xw) break;
      const bool ok = rowok && okx[h];
      const T* src = ok ? row + gx_l[h] : d;
      const uint32_t dst = dst0 + 32 * h * sizeof(T);
      if constexpr (sizeof(T) == 8) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
                     "r"(ok ? 8 : 0)
                     : "memory");
      } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src),
                     "r"(ok ? 4 : 0)
                     : "memory");
      }
    }
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
  __syncthreads();

  // ---- phase 2: transform and scatter
  const int cbase = c0 + lane * CPL;
  if (cbase >= C) return;
  const int ntiles = min(Cfg::tpx, tw - tx0);
  const size_t plane = static_cast<size_t>(AL) * AL * Pc * c_pad;
  const size_t comp_stride = static_cast<size_t>(Pc) * c_pad;
  for (int t = warp; t < ntiles; t += NW) {
    T out[CPL][AL][AL];
#pragma unroll
    for (int h = 0; h < CPL; ++h) {
      T in[AL][AL];
      const T* src = s + (lane * CPL + h) * Cfg::plane + t * M;
#pragma unroll
      for (int i = 0; i < AL; ++i)
#pragma unroll
        for (int j = 0; j < AL; ++j) in[i][j] = src[i * Cfg::xw + j];
      sandwich<T, AL, AL>(in, out[h], [](int i, int j) { return A::BT(i, j); });
    }
    const long long p = static_cast<long long>(blockIdx.y) * tw + tx0 + t;  // chunk-local tile
    size_t idx = static_cast<size_t>(p) * c_pad + cbase;
#pragma unroll
    for (int xi = 0; xi < AL; ++xi)
#pragma unroll
      for (int nu = 0; nu < AL; ++nu) {
        T v[CPL];
#pragma unroll
        for (int h = 0; h < CPL; ++h) v[h] = out[h][xi][nu];
        put_ops<PREC>(V, idx, plane, v);
        idx += comp_stride;
      }
  }
}

// ============================================================ output transform
// One thread per (chunk tile p, filter k): reads the alpha^2 accumulators
// M[s][comp][k][p] (coalesced over p; split-C slices summed in ascending s),
// forms A^T M A and writes the valid vr x vc corner of the m x m tile (edge
// tiles clipped, engine.py:241-254).
template <int M, typename TA>
__global__ void __launch_bounds__(128) output_transform_kernel(const TA* __restrict__ Mbuf,
                                                               TA* __restrict__ y, int N, int K,
                                                               int th, int tw, int oh, int ow,
                                                               int row0, long long Pc,
                                                               long long m_ld, int splits) {
  using A = Alg<M>;
  constexpr int AL = A::alpha;
  const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (p >= Pc) return;
  const size_t cstride = static_cast<size_t>(K) * m_ld;
  const size_t sstride = cstride * AL * AL;
  const TA* src = Mbuf + static_cast<size_t>(k) * m_ld + p;
  TA in[AL][AL];
#pragma unroll
  for (int xi = 0; xi < AL; ++xi)
#pragma unroll
    for (int nu = 0; nu < AL; ++nu) in[xi][nu] = __ldg(src + (xi * AL + nu) * cstride);
  for (int sp = 1; sp < splits; ++sp) {
    src += sstride;
#pragma unroll
    for (int xi = 0; xi < AL; ++xi)
#pragma unroll
      for (int nu = 0; nu < AL; ++nu) in[xi][nu] += __ldg(src + (xi * AL + nu) * cstride);
  }
  TA out[M][M];
  sandwich<TA, M, AL>(in, out, [](int i, int j) { return A::AT(i, j); });
  const long long gp = static_cast<long long>(row0) * tw + p;
  const long long per_img = static_cast<long long>(th) * tw;
  const int n = static_cast<int>(gp / per_img);
  const int rest = static_cast<int>(gp - n * per_img);
  const int ty = rest / tw, tx = rest - ty * tw;
  const int vr = min(M, oh - M * ty), vc = min(M, ow - M * tx);
  TA* dst = y + ((static_cast<size_t>(n) * K + k) * oh + M * ty) * ow + M * tx;
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int j = 0; j < M; ++j)
      if (i < vr && j < vc) dst[static_cast<size_t>(i) * ow + j] = out[i][j];
}

// ================================================================ launchers
// Every kernel of the pipeline runs with the same (maximum) shared-memory
// carveout as the GEMM, so consecutive launches never wait for an L1/smem
// reconfiguration of the SMs.
template <typename F>
static void max_carveout(F kern) {
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
}

template <int M, int PREC>
static void filter_launch(const void* g, void* U, int K, int C, int c_pad, cudaStream_t s) {
  using T = typename OpStore<PREC>::T;
  const long long n = static_cast<long long>(K) * C;
  auto kern = filter_transform_kernel<M, PREC>;
  static bool configured = false;
  if (!configured) {
    max_carveout(kern);
    configured = true;
  }
  kern<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(static_cast<const T*>(g), U, K, C,
                                                              c_pad);
}

template <int M>
static cudaError_t filter_dispatch(int prec, const void* g, void* U, int K, int C, int c_pad,
                                   cudaStream_t s) {
  switch (prec) {
    case kFP32: filter_launch<M, kFP32>(g, U, K, C, c_pad, s); break;
    case kTF32: filter_launch<M, kTF32>(g, U, K, C, c_pad, s); break;
    case kBF16: filter_launch<M, kBF16>(g, U, K, C, c_pad, s); break;
    case kFP16: filter_launch<M, kFP16>(g, U, K, C, c_pad, s); break;
    case kFP64: filter_launch<M, kFP64>(g, U, K, C, c_pad, s); break;
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
  using Cfg = InCfg<M, PREC>;
  const size_t smem = sizeof(T) * Cfg::cb * Cfg::plane;
  auto kern = input_transform_kernel<M, PREC>;
  static bool configured = false;  // benign race: idempotent attribute set
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    max_carveout(kern);
    configured = true;
  }
  const dim3 grid((tw + Cfg::tpx - 1) / Cfg::tpx, rows, (C + Cfg::cb - 1) / Cfg::cb);
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
                                    long long m_ld, int splits, cudaStream_t s) {
  if (Pc <= 0 || K <= 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((Pc + 127) / 128), K);
  static bool configured = false;
  if (!configured) {
    max_carveout(output_transform_kernel<2, double>);
    max_carveout(output_transform_kernel<4, double>);
    max_carveout(output_transform_kernel<2, float>);
    max_carveout(output_transform_kernel<4, float>);
    configured = true;
  }
  if (prec == kFP64) {
    if (m == 2)
      output_transform_kernel<2, double><<<grid, 128, 0, s>>>(
          static_cast<const double*>(Mbuf), static_cast<double*>(y), N, K, th, tw, oh, ow, row0, Pc,
          m_ld, splits);
    else
      output_transform_kernel<4, double><<<grid, 128, 0, s>>>(
          static_cast<const double*>(Mbuf), static_cast<double*>(y), N, K, th, tw, oh, ow, row0, Pc,
          m_ld, splits);
  } else {
    if (m == 2)
      output_transform_kernel<2, float><<<grid, 128, 0, s>>>(
          static_cast<const float*>(Mbuf), static_cast<float*>(y), N, K, th, tw, oh, ow, row0, Pc,
          m_ld, splits);
    else
      output_transform_kernel<4, float><<<grid, 128, 0, s>>>(
          static_cast<const float*>(Mbuf), static_cast<float*>(y), N, K, th, tw, oh, ow, row0, Pc,
          m_ld, splits);
  }
  return cudaGetLastError();
}

}  // namespace wino
