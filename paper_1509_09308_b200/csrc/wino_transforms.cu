// Winograd transform kernels: filter transform G g G^T, input-tile transform
// B^T d B, and the inverse transform A^T M A with clipped write-back.
// These are HBM-bandwidth-bound CUDA-core kernels; coalescing is arranged
// through shared-memory staging so every global access is a contiguous row.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdlib>

#include "sm100_ptx.cuh"
#include <type_traits>

#include "wino_internal.h"
#include "winograd_mats.cuh"

namespace wino {

// --------------------------------------------------------------- operand store
// Writes one transform-space value in the GEMM operand format at element index
// `idx` of split plane 0; split plane s lives `plane` elements further.
template <int PREC>
struct OpStore;

template <>
struct OpStore<kFP32> {  // 3xTF32: plain fp32 in memory; the GEMM splits hi/lo on chip
  using T = float;
  __device__ static void put(void* base, size_t idx, size_t, float x) {
    static_cast<float*>(base)[idx] = x;
  }
};
template <>
struct OpStore<kFP32S> {  // 3xTF32 pre-split: hi = rna_tf32(x) at idx, lo = x - hi one plane on
  using T = float;
  __device__ static void put(void* base, size_t idx, size_t plane, float x) {
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    static_cast<float*>(base)[idx] = __uint_as_float(h);
    static_cast<float*>(base)[idx + plane] = x - __uint_as_float(h);
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

template <int M, typename TA>
__device__ __forceinline__ void store_tile(TA* dst, int ow, int vr, int vc, const TA (&out)[M][M]);

// Write one output tile of (n, k) at tile (ty, tx) with the forward's epilogue
// activation (wino_forward_act; the chained network's ReLU and 2x2 max-pool,
// fused here instead of a separate pass over y): kActNone stores the tile,
// kActRelu stores max(x, 0), kActReluPool stores the 2x2 / stride-2 max of
// max(x, 0) into y (N, K, oh/2, ow/2).  Tile origins are multiples of m (even)
// and oh, ow are even, so a tile holds whole pooling windows and its valid rows
// / columns are even.
template <int M, typename TA>
__device__ __forceinline__ void emit_tile(TA* __restrict__ y, int act, int n, int K, int k,
                                          int oh, int ow, int ty, int tx, int vr, int vc,
                                          TA (&out)[M][M]) {
  if (act == kActReluPool) {
    constexpr int P = M / 2;
    TA pooled[P][P];
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
      for (int j = 0; j < P; ++j) {
        // fmax semantics, as the separate wino_relu_pool pass (wino_net.cu)
        const TA a = fmax(out[2 * i][2 * j], out[2 * i][2 * j + 1]);
        const TA b = fmax(out[2 * i + 1][2 * j], out[2 * i + 1][2 * j + 1]);
        pooled[i][j] = fmax(fmax(a, b), TA(0));
      }
    const int ph = oh >> 1, pw = ow >> 1;
    TA* dst = y + ((static_cast<size_t>(n) * K + k) * ph + P * ty) * pw + P * tx;
    store_tile<P>(dst, pw, vr >> 1, vc >> 1, pooled);
    return;
  }
  if (act == kActRelu) {
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
      for (int j = 0; j < M; ++j) out[i][j] = fmax(out[i][j], TA(0));
  }
  TA* dst = y + ((static_cast<size_t>(n) * K + k) * oh + M * ty) * ow + M * tx;
  store_tile<M>(dst, ow, vr, vc, out);
}

// ============================================================ filter transform
// Block = 256 x FPT consecutive (k, c) pairs = contiguous 3x3 filters, staged through shared memory with coalesced 16-byte loads (all
// of a thread's loads in flight at once; the 36-byte records would otherwise
// give strided warp loads), then thread t forms G g G^T for pairs t, t+256, ... and writes
// U[s][comp][k][c] with c fastest (coalesced across the warp).
// (engine.py:104-114)
// One block's work (block index `blk`, staging buffer `sg` of 256*FPT*9 T).
template <int M, int PREC, int FPT, bool SPLIT2>
__device__ __forceinline__ void filter_block(const typename OpStore<PREC>::T* __restrict__ g,
                                             void* __restrict__ U, int K, int C, int c_pad,
                                             int blk, typename OpStore<PREC>::T* sg) {
  using T = typename OpStore<PREC>::T;
  using A = Alg<M>;
  constexpr int AL = A::alpha;
  constexpr int NP = 256 * FPT;  // pairs per block
  const long long total = static_cast<long long>(K) * C;
  const long long t0 = static_cast<long long>(blk) * NP;
  const int nloc = static_cast<int>(min(static_cast<long long>(NP), total - t0));
  const T* src = g + t0 * 9;
  constexpr int VE = 16 / sizeof(T);  // elements per 16-byte load
  if (nloc == NP && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    constexpr int NVT = NP * 9 / VE;           // 16-byte chunks in the block (NP % 4 == 0)
    constexpr int NV = (NVT + 255) / 256;      // per thread, all in flight
    // cp.async straight into shared memory: every chunk's load is in flight at
    // once (register staging let the compiler interleave loads and stores,
    // i.e. several dependent round trips)
    const uint32_t s0 = static_cast<uint32_t>(__cvta_generic_to_shared(sg));
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int i = threadIdx.x + 256 * q;
      if (NVT % 256 == 0 || i < NVT)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s0 + 16 * i),
                     "l"(reinterpret_cast<const uint4*>(src) + i)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
  } else {
    for (int e = threadIdx.x; e < nloc * 9; e += 256) sg[e] = __ldg(src + e);
  }
  __syncthreads();
  const size_t plane = static_cast<size_t>(AL) * AL * K * c_pad;
  const size_t cstride = static_cast<size_t>(K) * c_pad;
#pragma unroll
  for (int q = 0; q < FPT; ++q) {
    const int j = threadIdx.x + 256 * q;
    if (j >= nloc) break;
    const long long t = t0 + j;
    const int k = static_cast<int>(t / C);
    const int c = static_cast<int>(t - static_cast<long long>(k) * C);
    T in[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int jj = 0; jj < 3; ++jj) in[i][jj] = sg[j * 9 + i * 3 + jj];
    T out[AL][AL];
    sandwich<T, AL, 3>(in, out, [](int i, int jj) { return A::G(i, jj); });
    size_t idx = static_cast<size_t>(k) * c_pad + c;
#pragma unroll
    for (int xi = 0; xi < AL; ++xi)
#pragma unroll
      for (int nu = 0; nu < AL; ++nu) {
        if constexpr (SPLIT2) {  // 3xTF32 hi / lo planes
          uint32_t h;
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(out[xi][nu]));
          static_cast<float*>(U)[idx] = __uint_as_float(h);
          static_cast<float*>(U)[idx + plane] = out[xi][nu] - __uint_as_float(h);
        } else {
          OpStore<PREC>::put(U, idx, plane, out[xi][nu]);
        }
        idx += cstride;
      }
  }
}

template <int M, int PREC, int FPT, bool SPLIT2 = false>
__global__ void __launch_bounds__(256) filter_transform_kernel(
    const typename OpStore<PREC>::T* __restrict__ g, void* __restrict__ U, int K, int C,
    int c_pad) {
  using T = typename OpStore<PREC>::T;
  __shared__ __align__(16) T sg[256 * FPT * 9];
  griddep_launch();
  griddep_wait();
  filter_block<M, PREC, FPT, SPLIT2>(g, U, K, C, c_pad, blockIdx.x, sg);
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

template <int PREC, int CPL = InPack<PREC>::cpl>
__device__ __forceinline__ void put_ops(void* base, size_t idx, size_t plane, const float* v) {
  if constexpr (CPL == 1) {
    OpStore<PREC>::put(base, idx, plane, v[0]);
  } else if constexpr (PREC == kBF16) {
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
  extern __shared__ __align__(128) unsigned char smem_raw[];
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
  griddep_launch();
  griddep_wait();

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
      if constexpr (M == 4)
        bt6_2d(in, out[h]);
      else
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

// ----------------------------------------- whole-plane input transform (small)
// Small images whose rows are not 16-byte aligned (VGG conv5: 14 x 14, W*4 = 56
// bytes, so no TMA box): the CB channel planes of one image are one contiguous,
// 16-byte-aligned run of HBM (HW % 4 == 0), read with coalesced 16-byte loads
// into [channel][PS] shared planes (PS odd: per-lane patch reads hit distinct
// banks).  Warp w then transforms tiles w, w+8, ... of the image's tile rows
// that fall inside the chunk; the patch bounds are warp-uniform, so padding is
// a uniform select, not a memory access.  Same V layout as the kernels above.
template <int M, int PREC, int CPL>
__global__ void __launch_bounds__(256) input_transform_plane_kernel(
    const float* __restrict__ d, void* __restrict__ V, int C, int H, int W, int pad, int th,
    int tw, int row0, int rows, long long Pc, int c_pad, int ps) {
  using A = Alg<M>;
  constexpr int AL = A::alpha;
  constexpr int CB = 32 * CPL;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* s = reinterpret_cast<float*>(smem_raw);
  const int n = row0 / th + blockIdx.x;
  const int c0 = blockIdx.y * CB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hw = H * W;
  griddep_launch();
  griddep_wait();

  // ---- stage CB planes (channels >= C left unread: their lanes exit below)
  const int nch = min(CB, C - c0);
  const float4* src = reinterpret_cast<const float4*>(d + (static_cast<size_t>(n) * C + c0) * hw);
  const int q_per_plane = hw >> 2;
  const int nq = nch * q_per_plane;
  constexpr int B = 4;  // loads in flight per thread
  for (int base = threadIdx.x; base < nq; base += 256 * B) {
    float4 v[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int q = base + b * 256;
      if (q < nq) v[b] = __ldg(src + q);
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int q = base + b * 256;
      if (q < nq) {
        const int ch = q / q_per_plane, off = (q - ch * q_per_plane) * 4;
        float* dst = s + ch * ps + off;
        dst[0] = v[b].x; dst[1] = v[b].y; dst[2] = v[b].z; dst[3] = v[b].w;
      }
    }
  }
  __syncthreads();

  const int cbase = c0 + lane * CPL;
  if (cbase >= C) return;
  const int r_lo = max(row0, n * th), r_hi = min(row0 + rows, (n + 1) * th);
  const int ntile = (r_hi - r_lo) * tw;
  const size_t plane_v = static_cast<size_t>(AL) * AL * Pc * c_pad;
  const size_t comp_stride = static_cast<size_t>(Pc) * c_pad;
  for (int t = warp; t < ntile; t += 8) {
    const int ty = r_lo - n * th + t / tw, tx = t - (t / tw) * tw;
    const int y0 = M * ty - pad, x0 = M * tx - pad;
    float out[CPL][AL][AL];
#pragma unroll
    for (int h = 0; h < CPL; ++h) {
      const float* sc = s + (lane * CPL + h) * ps;
      float in[AL][AL];
#pragma unroll
      for (int i = 0; i < AL; ++i) {
        const int gy = y0 + i;
        const bool rok = gy >= 0 && gy < H;
#pragma unroll
        for (int j = 0; j < AL; ++j) {
          const int gx = x0 + j;
          in[i][j] = (rok && gx >= 0 && gx < W) ? sc[gy * W + gx] : 0.f;
        }
      }
      if constexpr (M == 4)
        bt6_2d(in, out[h]);
      else
        sandwich<float, AL, AL>(in, out[h], [](int i, int j) { return A::BT(i, j); });
    }
    const long long p = static_cast<long long>(r_lo - row0) * tw + t;  // chunk-local tile
    size_t idx = static_cast<size_t>(p) * c_pad + cbase;
#pragma unroll
    for (int xi = 0; xi < AL; ++xi)
#pragma unroll
      for (int nu = 0; nu < AL; ++nu) {
        float v[CPL];
#pragma unroll
        for (int h = 0; h < CPL; ++h) v[h] = out[h][xi][nu];
        put_ops<PREC, CPL>(V, idx, plane_v, v);
        idx += comp_stride;
      }
  }
}

// z = A^T x for one alpha-vector (F(4,3): 10 flops with shared subexpressions;
// F(2,3): coefficient-folded).
template <int M, typename T>
__device__ __forceinline__ void at_vec(const T (&x)[M + 2], T (&z)[M]) {
  if constexpr (M == 4) {
    const T s1 = x[1] + x[2], d1 = x[1] - x[2], s2 = x[3] + x[4], d2 = x[3] - x[4];
    z[0] = x[0] + s1 + s2;
    z[1] = fma(T(2), d2, d1);
    z[2] = fma(T(4), s2, s1);
    z[3] = fma(T(8), d2, d1) + x[5];
  } else {
    z[0] = x[0] + x[1] + x[2];
    z[1] = x[1] - x[2] - x[3];
  }
}

// out = A^T in A with at_vec over the columns, then over the rows.
template <int M, typename T>
__device__ __forceinline__ void at_2d(const T (&in)[M + 2][M + 2], T (&out)[M][M]) {
  constexpr int AL = M + 2;
  T tmp[M][AL];
#pragma unroll
  for (int v = 0; v < AL; ++v) {
    T col[AL], z[M];
#pragma unroll
    for (int u = 0; u < AL; ++u) col[u] = in[u][v];
    at_vec<M, T>(col, z);
#pragma unroll
    for (int i = 0; i < M; ++i) tmp[i][v] = z[i];
  }
#pragma unroll
  for (int i = 0; i < M; ++i) at_vec<M, T>(tmp[i], out[i]);
}

// ============================================================ output transform
// One thread per (chunk tile p, filter k): reads the alpha^2 accumulators
// M[s][comp][k][p] (coalesced over p; split-C slices summed in ascending s),
// forms A^T M A and writes the valid vr x vc corner of the m x m tile (edge
// tiles clipped, engine.py:241-254).
// 128 threads x >= 8 blocks/SM: a latency-bound stream needs the occupancy
// (unbounded, ptxas spends 168 registers on 36 live addresses).
template <int M, typename TA>
__global__ void __launch_bounds__(128, 8) output_transform_kernel(const TA* __restrict__ Mbuf,
                                                               TA* __restrict__ y, int N, int K,
                                                               int th, int tw, int oh, int ow,
                                                               int row0, long long Pc,
                                                               long long m_ld, int splits,
                                                               int act) {
  using A = Alg<M>;
  constexpr int AL = A::alpha;
  const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  griddep_launch();
  griddep_wait();
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
  at_2d<M, TA>(in, out);
  const long long gp = static_cast<long long>(row0) * tw + p;
  const long long per_img = static_cast<long long>(th) * tw;
  const int n = static_cast<int>(gp / per_img);
  const int rest = static_cast<int>(gp - n * per_img);
  const int ty = rest / tw, tx = rest - ty * tw;
  const int vr = min(M, oh - M * ty), vc = min(M, ow - M * tx);
  emit_tile<M>(y, act, n, K, k, oh, ow, ty, tx, vr, vc, out);
}

// TMA-staged variant (fp32, no split-C): one 3D TMA box brings a block's
// M[comp][k0..k0+OF)[p0..p0+128) (alpha^2 x OF x 128 fp32) into shared memory
// -- all of the block's loads in flight at once without any register cost --
// then thread = tile forms A^T M A for each of the OF filters from smem
// (lane-contiguous, conflict-free) and stores the clipped tiles.
constexpr int kOutTP = 128;  // tiles per block
// MT = the staged M element: float, or bf16 for the bf16 GEMM (wino_api.cu).
template <int M, typename MT = float>
struct OutTma {
  static constexpr int alpha = M + 2;
  static constexpr int OF = (M == 4) ? (sizeof(MT) == 2 ? 2 : 1) : 4;  // filters per block
  static constexpr int bytes = alpha * alpha * OF * kOutTP * static_cast<int>(sizeof(MT));
};

template <int M, typename MT>
__global__ void __launch_bounds__(kOutTP) output_transform_tma_kernel(
    const __grid_constant__ CUtensorMap tmM, float* __restrict__ y, int K, int th, int tw, int oh,
    int ow, int row0, long long Pc, const char* __restrict__ mbase, long long m_ld, int discard,
    const char* __restrict__ dead, long long dead_lines, int act) {
  using A = Alg<M>;
  using Cfg = OutTma<M, MT>;
  constexpr int AL = A::alpha;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  MT* s = reinterpret_cast<MT*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                ~static_cast<uintptr_t>(127));
  __shared__ uint64_t bar;
  const int p0 = blockIdx.x * kOutTP;
  const int k0 = blockIdx.y * Cfg::OF;
  griddep_launch();
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bar, Cfg::bytes);
    ptx::tma_load_3d(s, &tmM, &bar, p0, k0, 0);
  }
  if (dead_lines > 0) {
    // the chunk's V is dead (the GEMM has completed): this block's share of
    // its 128-byte lines leaves L2 without a write-back, under the box load
    const long long nb = static_cast<long long>(gridDim.x) * gridDim.y;
    const long long per = (dead_lines + nb - 1) / nb;
    const long long l0 = (static_cast<long long>(blockIdx.y) * gridDim.x + blockIdx.x) * per;
    const long long l1 = min(dead_lines, l0 + per);
    for (long long l = l0 + threadIdx.x; l < l1; l += kOutTP)
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(dead + 128 * l) : "memory");
  }
  ptx::mbar_wait(&bar, 0);
  if (discard) {
    // M is dead once this box is in smem: drop its (dirty) L2 lines so they are
    // never written back to HBM.  Rows start 128-byte aligned (m_ld % 64 == 0);
    // lines past the row's m_ld belong to the next row and are left alone.
    constexpr int EPL = 128 / static_cast<int>(sizeof(MT));  // elements per line
    constexpr int LPR = kOutTP / EPL;                         // lines per box row
    constexpr int NL = Cfg::alpha * Cfg::alpha * Cfg::OF * LPR;
    for (int i = threadIdx.x; i < NL; i += kOutTP) {
      const int row = i / LPR, l = i - (i / LPR) * LPR;
      const int comp = row / Cfg::OF, k = k0 + (row - comp * Cfg::OF);
      const long long e0 = static_cast<long long>(p0) + l * EPL;
      if (k < K && e0 < m_ld) {
        const char* a = mbase + ((static_cast<long long>(comp) * K + k) * m_ld + e0) *
                                    static_cast<long long>(sizeof(MT));
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
      }
    }
  }
  const int t = threadIdx.x;
  const long long p = static_cast<long long>(p0) + t;
  if (p >= Pc) return;
  const long long gp = static_cast<long long>(row0) * tw + p;
  const long long per_img = static_cast<long long>(th) * tw;
  const int n = static_cast<int>(gp / per_img);
  const int rest = static_cast<int>(gp - n * per_img);
  const int ty = rest / tw, tx = rest - ty * tw;
  const int vr = min(M, oh - M * ty), vc = min(M, ow - M * tx);
#pragma unroll
  for (int f = 0; f < Cfg::OF; ++f) {
    const int k = k0 + f;
    if (k >= K) break;
    float in[AL][AL];
#pragma unroll
    for (int xi = 0; xi < AL; ++xi)
#pragma unroll
      for (int nu = 0; nu < AL; ++nu) {
        if constexpr (std::is_same<MT, __half>::value)
          in[xi][nu] = __half2float(s[((xi * AL + nu) * Cfg::OF + f) * kOutTP + t]) *
                       static_cast<float>(1 << kM16Shift);
        else if constexpr (sizeof(MT) == 2)
          in[xi][nu] = __bfloat162float(s[((xi * AL + nu) * Cfg::OF + f) * kOutTP + t]);
        else
          in[xi][nu] = s[((xi * AL + nu) * Cfg::OF + f) * kOutTP + t];
      }
    float out[M][M];
    at_2d<M, float>(in, out);
    emit_tile<M>(y, act, n, K, k, oh, ow, ty, tx, vr, vc, out);
  }
}

// Write an m x m output tile: one vector store per row for full tiles whose
// rows are vector-aligned (a warp then writes 32 adjacent tiles = whole lines),
// clipped scalar stores for edge tiles (engine.py:246-253).
template <int M, typename TA>
__device__ __forceinline__ void store_tile(TA* dst, int ow, int vr, int vc, const TA (&out)[M][M]) {
  constexpr int VB = M * sizeof(TA);  // bytes per tile row
  const bool vec = (vr == M) && (vc == M) && (VB == 8 || VB == 16 || VB == 32) &&
                   ((reinterpret_cast<uintptr_t>(dst) | (static_cast<size_t>(ow) * sizeof(TA))) %
                        (VB > 16 ? 16 : VB) ==
                    0);
  if (vec) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
      TA* row = dst + static_cast<size_t>(i) * ow;
      if constexpr (VB == 8) {
        if constexpr (sizeof(TA) == 4)
          *reinterpret_cast<float2*>(row) = make_float2(out[i][0], out[i][1]);
        else
          *reinterpret_cast<double*>(row) = out[i][0];
      } else {
#pragma unroll
        for (int h = 0; h < VB / 16; ++h) {
          if constexpr (sizeof(TA) == 4)
            reinterpret_cast<float4*>(row)[h] =
                make_float4(out[i][4 * h], out[i][4 * h + 1], out[i][4 * h + 2], out[i][4 * h + 3]);
          else
            reinterpret_cast<double2*>(row)[h] = make_double2(out[i][2 * h], out[i][2 * h + 1]);
        }
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
      for (int j = 0; j < M; ++j)
        if (i < vr && j < vc) dst[static_cast<size_t>(i) * ow + j] = out[i][j];
  }
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
static void filter_launch(const void* g, void* U, int K, int C, int c_pad, cudaStream_t s,
                          bool split2) {
  using T = typename OpStore<PREC>::T;
  const long long n = static_cast<long long>(K) * C;
  static const int fpt_env = getenv("WINO_FILTER_FPT") ? atoi(getenv("WINO_FILTER_FPT")) : 0;
  // (k,c) pairs per thread.  Alone on the GPU one per thread is twice as fast
  // (512 x 512 F2 fp32: 4.1 vs 8.3 us).  For the 3xTF32 plans four stay faster
  // in the pass, where the transform runs beside the input transform or just
  // ahead of the GEMM, whose CTAs launch early (PDL) and co-reside only while
  // the transform leaves SMs free: VGG-E F2 fp32 N=1 0.380 ms at four per
  // thread vs 0.397 at one.  For the single-pass GEMMs (tf32 / bf16 / fp16) one
  // per thread measured faster: F4 tf32 N=8 0.859 -> 0.819 ms, N=1 0.336 ->
  // 0.325; F4 bf16 N=8 0.589 -> 0.577; F4 fp16 N=8 0.593 -> 0.580.  fp64: two.
  const int fpt = fpt_env == 1 || fpt_env == 2 || fpt_env == 4
                      ? fpt_env
                      : (PREC == kFP32 ? 4 : PREC == kFP64 ? 2 : 1);
  auto go = [&](auto kern, int FPT) {
    max_carveout(kern);
    launch_k(kern, dim3(static_cast<unsigned>((n + 256 * FPT - 1) / (256 * FPT))), dim3(256), 0, s,
             static_cast<const T*>(g), U, K, C, c_pad);
  };
  if constexpr (PREC == kFP32) {
    if (split2) {
      go(filter_transform_kernel<M, PREC, 4, true>, 4);
      return;
    }
  }
  if (fpt == 1) go(filter_transform_kernel<M, PREC, 1>, 1);
  else if (fpt == 2) go(filter_transform_kernel<M, PREC, 2>, 2);
  else if constexpr (sizeof(T) == 4) go(filter_transform_kernel<M, PREC, 4>, 4);
  else go(filter_transform_kernel<M, PREC, 2>, 2);
}

template <int M>
static cudaError_t filter_dispatch(int prec, const void* g, void* U, int K, int C, int c_pad,
                                   cudaStream_t s, bool split2) {
  switch (prec) {
    case kFP32: filter_launch<M, kFP32>(g, U, K, C, c_pad, s, split2); break;
    case kTF32: filter_launch<M, kTF32>(g, U, K, C, c_pad, s, false); break;
    case kBF16: filter_launch<M, kBF16>(g, U, K, C, c_pad, s, false); break;
    case kFP16: filter_launch<M, kFP16>(g, U, K, C, c_pad, s, false); break;
    case kFP64: filter_launch<M, kFP64>(g, U, K, C, c_pad, s, false); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_filter_transform(int m, int prec, const void* g, void* U, int K, int C,
                                    int c_pad, cudaStream_t s, bool split2) {
  if (K <= 0 || C <= 0) return cudaSuccess;
  return m == 2 ? filter_dispatch<2>(prec, g, U, K, C, c_pad, s, split2)
                : filter_dispatch<4>(prec, g, U, K, C, c_pad, s, split2);
}

// ------------------------------------------------ TMA-staged input transform
// Fast path for fp32 data with 16-byte-aligned rows (W % 4 == 0): one 4D TMA
// box (x, y, channel) per block stages the window, zero-filling the padding
// and channels >= C in hardware (negative start coordinates are legal).
// The box's innermost start coordinate must be 16-byte aligned (otherwise the
// load faults -- tools/probes/tma_grid_probe.cu), so the box starts SH = (-pad)
// mod 4 columns left of the window.  It carries alpha+1 rows and XWB = 4*odd
// columns so each channel plane is an odd number of 16-byte units: lane =
// channel then reads its patch rows with conflict-free LDS.128.
// Block = 32 channels x TPX tiles (16 for F(2x2), 8 for F(4x4): a 32-56 KB
// box, so 4-5 blocks share an SM); warp w transforms tiles w (and w+8).
template <int M, int SH>
struct InTma {
  static constexpr int alpha = M + 2;
  static constexpr int tpx = (M == 2) ? 16 : 8;
  static constexpr int rows = alpha + 1;
  static constexpr int xwb = 44;  // >= SH + tpx*M + 2 (and the last float4 patch read), 4*odd
  static constexpr int plane = rows * xwb;
  static constexpr int bytes = 32 * plane * 4;
  static constexpr int nv = (M == 2) ? 2 : 3;     // float4 reads per patch row
  static_assert((plane / 4) % 2 == 1, "plane must be an odd number of 16-byte units");
  static_assert(SH + tpx * M + 2 <= xwb, "box too narrow");
};

template <int M, int AL, int NV, int OFF>
__device__ __forceinline__ void load_patch(const float* sc, int xwb, int base, float (&in)[AL][AL]) {
#pragma unroll
  for (int i = 0; i < AL; ++i) {
    float r[4 * NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const float4 q = *reinterpret_cast<const float4*>(sc + i * xwb + base + 4 * v);
      r[4 * v] = q.x;
      r[4 * v + 1] = q.y;
      r[4 * v + 2] = q.z;
      r[4 * v + 3] = q.w;
    }
#pragma unroll
    for (int j = 0; j < AL; ++j) in[i][j] = r[OFF + j];
  }
}

// One block's work: box (bx, by, bz) of the chunk, staged at `s` with `bar`.
template <int M, int PREC, int SH>
__device__ __forceinline__ void input_tma_block(const CUtensorMap* tmD, void* __restrict__ V,
                                                int C, int pad, int th, int tw, int row0,
                                                long long Pc, int c_pad, int bx, int by, int bz,
                                                float* s, uint64_t& bar) {
  using A = Alg<M>;
  using Cfg = InTma<M, SH>;
  constexpr int AL = A::alpha;
  const int row = row0 + by;
  const int n = row / th;
  const int ty = row - n * th;
  const int tx0 = bx * Cfg::tpx;
  const int c0 = bz * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bar, Cfg::bytes);
    ptx::tma_load_4d(s, tmD, &bar, M * tx0 - pad - SH, M * ty - pad, c0, n);
  }
  ptx::mbar_wait(&bar, 0);

  const int c = c0 + lane;
  if (c >= C) return;
  const size_t plane_v = static_cast<size_t>(AL) * AL * Pc * c_pad;
  const size_t comp_stride = static_cast<size_t>(Pc) * c_pad;
  const float* sc = s + lane * Cfg::plane;
#pragma unroll
  for (int h = 0; h < Cfg::tpx / 8; ++h) {
    const int t = warp + 8 * h;
    if (tx0 + t >= tw) break;
    float in[AL][AL];
    const int x = SH + t * M;  // window column of the patch
    if constexpr (M == 4) {
      load_patch<M, AL, Cfg::nv, SH>(sc, Cfg::xwb, x - SH, in);
    } else {  // F(2x2): the in-float4 offset depends on the (warp-uniform) tile parity
      constexpr int O0 = SH & 3, O1 = (SH + 2) & 3;
      if (t & 1)
        load_patch<M, AL, Cfg::nv, O1>(sc, Cfg::xwb, x - O1, in);
      else
        load_patch<M, AL, Cfg::nv, O0>(sc, Cfg::xwb, x - O0, in);
    }
    float out[AL][AL];
    if constexpr (M == 4)
      bt6_2d(in, out);
    else
      sandwich<float, AL, AL>(in, out, [](int i, int j) { return A::BT(i, j); });
    const long long p = static_cast<long long>(by) * tw + tx0 + t;
    size_t idx = static_cast<size_t>(p) * c_pad + c;
#pragma unroll
    for (int xi = 0; xi < AL; ++xi)
#pragma unroll
      for (int nu = 0; nu < AL; ++nu) {
        OpStore<PREC>::put(V, idx, plane_v, out[xi][nu]);
        idx += comp_stride;
      }
  }
}

template <int M, int PREC, int SH>
__global__ void __launch_bounds__(256) input_transform_tma_kernel(
    const __grid_constant__ CUtensorMap tmD, void* __restrict__ V, int C, int pad, int th,
    int tw, int row0, long long Pc, int c_pad) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* s = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~static_cast<uintptr_t>(1023));
  __shared__ uint64_t bar;
  griddep_launch();
  input_tma_block<M, PREC, SH>(&tmD, V, C, pad, th, tw, row0, Pc, c_pad, blockIdx.x, blockIdx.y,
                               blockIdx.z, s, bar);
}

// Filter transform and (single-chunk) TMA input transform in ONE launch:
// blocks [0, n_in) take input boxes, the rest take 1024 (k, c) filter pairs.
// Saves the side-stream fork/join and a launch per layer; the GEMM follows
// in-stream behind one predecessor (PDL).
template <int M, int PREC, int SH, bool SPLIT2>
__global__ void __launch_bounds__(256) transforms_kernel(
    const __grid_constant__ CUtensorMap tmD, void* __restrict__ V, int C, int pad, int th,
    int tw, int rows, long long Pc, int c_pad, int nx, int ncb,
    const typename OpStore<PREC>::T* __restrict__ g, void* __restrict__ U, int K) {
  using T = typename OpStore<PREC>::T;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bar;
  griddep_launch();
  const int n_in = nx * rows * ncb;
  const int b = blockIdx.x;
  if (b < n_in) {
    float* s = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                        ~static_cast<uintptr_t>(1023));
    const int bx = b % nx, r = b / nx;
    input_tma_block<M, PREC, SH>(&tmD, V, C, pad, th, tw, 0, Pc, c_pad, bx, r % rows, r / rows,
                                 s, bar);
  } else {
    griddep_wait();
    T* sg = reinterpret_cast<T*>((reinterpret_cast<uintptr_t>(smem_raw) + 15) &
                                 ~static_cast<uintptr_t>(15));
    // (kFP32S splits V only: U stays one fp32 plane, the A operand split on chip)
    filter_block<M, PREC == kFP32S ? kFP32 : PREC, 4, SPLIT2>(g, U, K, C, c_pad, b - n_in, sg);
  }
}

template <int M, int PREC, int SH>
static cudaError_t input_tma_launch(const void* d, void* V, int N, int C, int H, int W, int pad,
                                    int th, int tw, int row0, int rows, long long Pc, int c_pad,
                                    cudaStream_t s) {
  using Cfg = InTma<M, SH>;
  alignas(64) CUtensorMap tmD;
  if (!encode_tmap_nchw_f32(&tmD, d, N, C, H, W, Cfg::xwb, Cfg::rows, 32))
    return cudaErrorInvalidValue;
  auto kern = input_transform_tma_kernel<M, PREC, SH>;
  static DeviceOnce configured;
  if (configured.first()) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::bytes + 1024);
    max_carveout(kern);
    configured.done();
  }
  const dim3 grid((tw + Cfg::tpx - 1) / Cfg::tpx, rows, (C + 31) / 32);
  launch_k(kern, grid, dim3(256), static_cast<size_t>(Cfg::bytes + 1024), s, tmD, V, C, pad, th,
           tw, row0, Pc, c_pad);
  return cudaGetLastError();
}

template <int M, int PREC, int SH, bool SPLIT2>
static cudaError_t transforms_launch(const void* d, void* V, int N, int C, int H, int W, int pad,
                                     int th, int tw, int rows, long long Pc, int c_pad,
                                     const void* g, void* U, int K, cudaStream_t s) {
  using Cfg = InTma<M, SH>;
  using T = typename OpStore<PREC>::T;
  alignas(64) CUtensorMap tmD;
  if (!encode_tmap_nchw_f32(&tmD, d, N, C, H, W, Cfg::xwb, Cfg::rows, 32))
    return cudaErrorInvalidValue;
  auto kern = transforms_kernel<M, PREC, SH, SPLIT2>;
  constexpr size_t in_smem = Cfg::bytes + 1024;
  constexpr size_t f_smem = 256 * 4 * 9 * sizeof(T) + 16;
  constexpr size_t smem = in_smem > f_smem ? in_smem : f_smem;
  static DeviceOnce configured;
  if (configured.first()) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    max_carveout(kern);
    configured.done();
  }
  const int nx = (tw + Cfg::tpx - 1) / Cfg::tpx, ncb = (C + 31) / 32;
  const long long nf = (static_cast<long long>(K) * C + 1023) / 1024;
  const long long blocks = static_cast<long long>(nx) * rows * ncb + nf;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  launch_k(kern, dim3(static_cast<unsigned>(blocks)), dim3(256), smem, s, tmD, V, C, pad, th, tw,
           rows, Pc, c_pad, nx, ncb, static_cast<const T*>(g), U, K);
  return cudaGetLastError();
}

template <int M, int PREC>
static cudaError_t transforms_sh(const void* d, void* V, int N, int C, int H, int W, int pad,
                                 int th, int tw, int rows, long long Pc, int c_pad, const void* g,
                                 void* U, int K, bool split2, cudaStream_t s) {
  const int sh = (4 - pad % 4) % 4;
#define WINO_TR(SHV, SP) \
  return transforms_launch<M, PREC, SHV, SP>(d, V, N, C, H, W, pad, th, tw, rows, Pc, c_pad, g, U, K, s)
  if (split2) {
    if constexpr (PREC == kFP32) {
      switch (sh) {
        case 0: WINO_TR(0, true);
        case 1: WINO_TR(1, true);
        case 2: WINO_TR(2, true);
        default: WINO_TR(3, true);
      }
    }
    return cudaErrorInvalidValue;
  }
  switch (sh) {
    case 0: WINO_TR(0, false);
    case 1: WINO_TR(1, false);
    case 2: WINO_TR(2, false);
    default: WINO_TR(3, false);
  }
#undef WINO_TR
}

bool transforms_combinable(int prec, int W, int pad) {
  return prec != kFP64 && W % 4 == 0 && pad <= 3 && getenv("WINO_NO_TMA_INPUT") == nullptr &&
         getenv("WINO_NO_COMBINED") == nullptr;
}

cudaError_t launch_transforms(int m, int prec, const void* d, void* V, int N, int C, int H, int W,
                              int pad, int th, int tw, int rows, long long Pc, int c_pad,
                              const void* g, void* U, int K, bool split2, cudaStream_t s) {
  if (!transforms_combinable(prec, W, pad)) return cudaErrorInvalidValue;
#define WINO_TP(MM, P) \
  return transforms_sh<MM, P>(d, V, N, C, H, W, pad, th, tw, rows, Pc, c_pad, g, U, K, split2, s)
  if (m == 2) {
    switch (prec) {
      case kFP32: WINO_TP(2, kFP32);
      case kFP32S: WINO_TP(2, kFP32S);
      case kTF32: WINO_TP(2, kTF32);
      case kBF16: WINO_TP(2, kBF16);
      case kFP16: WINO_TP(2, kFP16);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (prec) {
    case kFP32: WINO_TP(4, kFP32);
    case kFP32S: WINO_TP(4, kFP32S);
    case kTF32: WINO_TP(4, kTF32);
    case kBF16: WINO_TP(4, kBF16);
    case kFP16: WINO_TP(4, kFP16);
    default: return cudaErrorInvalidValue;
  }
#undef WINO_TP
}

// The whole-plane input transform needs enough blocks (images x channel
// groups) to spread; below 32 the tile-row kernel is faster (conv5 at N = 1:
// 16 blocks).  At N = 8 (64 blocks) the plane kernel wins: VGG-E F4 fp16 N=8
// 0.611 -> 0.598 ms, F2 fp32 N=8 1.529 -> 1.513 ms (the bound was 148).
static long long plane_min_blocks() {
  static const long long v =
      getenv("WINO_PLANE_MIN_BLOCKS") ? atoll(getenv("WINO_PLANE_MIN_BLOCKS")) : 32;
  return v;
}

template <int M, int PREC>
static cudaError_t input_one(const void* d, void* V, int N, int C, int H, int W, int pad, int th,
                             int tw, int row0, int rows, long long Pc, int c_pad,
                             cudaStream_t s) {
  using T = typename OpStore<PREC>::T;
  if constexpr (PREC != kFP64) {
    if (W % 4 == 0 && pad <= 3 && getenv("WINO_NO_TMA_INPUT") == nullptr) {
      switch ((4 - pad % 4) % 4) {  // box shift that makes the start column 16-byte aligned
        case 0: return input_tma_launch<M, PREC, 0>(d, V, N, C, H, W, pad, th, tw, row0, rows, Pc, c_pad, s);
        case 1: return input_tma_launch<M, PREC, 1>(d, V, N, C, H, W, pad, th, tw, row0, rows, Pc, c_pad, s);
        case 2: return input_tma_launch<M, PREC, 2>(d, V, N, C, H, W, pad, th, tw, row0, rows, Pc, c_pad, s);
        default: return input_tma_launch<M, PREC, 3>(d, V, N, C, H, W, pad, th, tw, row0, rows, Pc, c_pad, s);
      }
    }
  }
  if constexpr (PREC != kFP64) {
    // small image planes, 16-byte-aligned runs: whole-plane staging (2 channels
    // per lane for 16-bit operands: packed stores; measured faster than 1)
    constexpr int CPL = InPack<PREC>::cpl;
    constexpr int CB = 32 * CPL;
    const int hw = H * W;
    const int ps = hw | 1;
    const size_t psmem = sizeof(float) * CB * ps;
    const long long blocks = static_cast<long long>((row0 + rows - 1) / th - row0 / th + 1) *
                             ((C + CB - 1) / CB);
    // enough blocks to cover the SMs (else the tile-row kernel spreads wider)
    if (hw % 4 == 0 && psmem <= 100 * 1024 && (reinterpret_cast<uintptr_t>(d) & 15) == 0 &&
        (blocks >= plane_min_blocks() || getenv("WINO_FORCE_PLANE_INPUT") != nullptr) &&
        getenv("WINO_NO_PLANE_INPUT") == nullptr) {
      auto kp = input_transform_plane_kernel<M, PREC, CPL>;
      static DeviceOnce pconf;
      if (pconf.first()) {
        cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        max_carveout(kp);
        pconf.done();
      }
      const int n0 = row0 / th, n1 = (row0 + rows - 1) / th;
      const dim3 grid(n1 - n0 + 1, (C + CB - 1) / CB);
      launch_k(kp, grid, dim3(256), psmem, s, static_cast<const float*>(d), V, C, H, W, pad, th,
               tw, row0, rows, Pc, c_pad, ps);
      return cudaGetLastError();
    }
  }
  using Cfg = InCfg<M, PREC>;
  const size_t smem = sizeof(T) * Cfg::cb * Cfg::plane;
  auto kern = input_transform_kernel<M, PREC>;
  static DeviceOnce configured;
  if (configured.first()) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    max_carveout(kern);
    configured.done();
  }
  const dim3 grid((tw + Cfg::tpx - 1) / Cfg::tpx, rows, (C + Cfg::cb - 1) / Cfg::cb);
  launch_k(kern, grid, dim3(256), smem, s, static_cast<const T*>(d), V, N, C, H, W, pad, th, tw,
           row0, Pc, c_pad);
  return cudaGetLastError();
}

template <int M>
static cudaError_t input_dispatch(int prec, const void* d, void* V, int N, int C, int H, int W,
                                  int pad, int th, int tw, int row0, int rows, long long Pc,
                                  int c_pad, cudaStream_t s) {
  switch (prec) {
    case kFP32: return input_one<M, kFP32>(d, V, N, C, H, W, pad, th, tw, row0, rows, Pc, c_pad, s);
    case kFP32S: return input_one<M, kFP32S>(d, V, N, C, H, W, pad, th, tw, row0, rows, Pc, c_pad, s);
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

template <int M, typename MT>
static cudaError_t output_tma_launch(const void* Mbuf, void* y, int K, int th, int tw, int oh,
                                     int ow, int row0, long long Pc, long long m_ld,
                                     cudaStream_t s, const void* dead, size_t dead_bytes,
                                     int act) {
  using Cfg = OutTma<M, MT>;
  alignas(64) CUtensorMap tmM;
  // M [a2][K][m_ld] (fp32 or bf16), box (128 tiles, OF filters, a2 components), no swizzle
  constexpr uint64_t es = sizeof(MT);
  if (!encode_tmap_3d_box(&tmM, Mbuf, static_cast<uint64_t>(Pc), static_cast<uint64_t>(K),
                          static_cast<uint64_t>(Cfg::alpha * Cfg::alpha), m_ld * es,
                          static_cast<uint64_t>(K) * m_ld * es, kOutTP, Cfg::OF,
                          Cfg::alpha * Cfg::alpha, es == 2))
    return cudaErrorInvalidValue;
  auto kern = output_transform_tma_kernel<M, MT>;
  static DeviceOnce configured;
  if (configured.first()) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::bytes + 128);
    max_carveout(kern);
    configured.done();
  }
  const dim3 grid(static_cast<unsigned>((Pc + kOutTP - 1) / kOutTP), (K + Cfg::OF - 1) / Cfg::OF);
  static const bool no_discard = getenv("WINO_NO_DISCARD") != nullptr;
  const int discard = !no_discard && m_ld % 64 == 0 && (reinterpret_cast<uintptr_t>(Mbuf) & 127) == 0;
  // V discard is opt-in (WINO_VDISCARD=1): it takes conv3.2 F4 bf16 N=64 from 432 to
  // 288 MB of DRAM writes per forward (1.40x the compulsory y) but the pass gets
  // 1-2% slower (profiles/r2/vdiscard.txt)
  static const bool vdiscard = !no_discard && getenv("WINO_VDISCARD") != nullptr;
  const long long dead_lines =
      (vdiscard && dead && (reinterpret_cast<uintptr_t>(dead) & 127) == 0)
          ? static_cast<long long>(dead_bytes / 128) : 0;
  launch_k(kern, grid, dim3(kOutTP), static_cast<size_t>(Cfg::bytes + 128), s, tmM,
           static_cast<float*>(y), K, th, tw, oh, ow, row0, Pc,
           static_cast<const char*>(Mbuf), m_ld, discard, static_cast<const char*>(dead),
           dead_lines, act);
  return cudaGetLastError();
}

long long output_tma_min_tiles(int prec) {
  static const char* e = getenv("WINO_OUT_TMA_MIN");
  if (e) return atoll(e);
  return (prec == kBF16 || prec == kFP16) ? 0 : 256;
}

cudaError_t launch_output_transform(int m, int prec, const void* Mbuf, void* y, int N, int K,
                                    int th, int tw, int oh, int ow, int row0, long long Pc,
                                    long long m_ld, int splits, cudaStream_t s, int m_bf16,
                                    const void* dead, size_t dead_bytes, int act) {
  if (Pc <= 0 || K <= 0) return cudaSuccess;
  if (m_bf16 == 2) {  // fp16-staged M (x 2^-kM16Shift; fp16 GEMM, no split-C): TMA path only
    if (splits != 1) return cudaErrorInvalidValue;
    return m == 2 ? output_tma_launch<2, __half>(Mbuf, y, K, th, tw, oh, ow, row0, Pc, m_ld, s,
                                                 dead, dead_bytes, act)
                  : output_tma_launch<4, __half>(Mbuf, y, K, th, tw, oh, ow, row0, Pc, m_ld, s,
                                                 dead, dead_bytes, act);
  }
  if (m_bf16) {  // bf16-staged M (bf16 GEMM, no split-C): TMA path only
    if (splits != 1) return cudaErrorInvalidValue;
    return m == 2 ? output_tma_launch<2, __nv_bfloat16>(Mbuf, y, K, th, tw, oh, ow, row0, Pc, m_ld, s,
                                                        dead, dead_bytes, act)
                  : output_tma_launch<4, __nv_bfloat16>(Mbuf, y, K, th, tw, oh, ow, row0, Pc, m_ld, s,
                                                        dead, dead_bytes, act);
  }
  // F(4x4) chunks of <= output_tma_min_tiles(prec) tiles take the per-thread
  // kernel: 256 for fp32 / tf32 (F4 tf32 N=1 0.300 -> 0.289 ms), 0 for the
  // 16-bit GEMMs, whose small chunks then stage 16-bit M too (F4 N=1 fp16
  // 0.267 -> 0.264, bf16 0.266 -> 0.263 ms).  WINO_OUT_TMA_MIN overrides.  For
  // F(2x2) the TMA box is always taken.
  const long long tma_min = output_tma_min_tiles(prec);
  if (prec != kFP64 && splits == 1 && (m == 2 || Pc > tma_min) &&
      getenv("WINO_NO_TMA_OUTPUT") == nullptr)
    return m == 2 ? output_tma_launch<2, float>(Mbuf, y, K, th, tw, oh, ow, row0, Pc, m_ld, s,
                                                dead, dead_bytes, act)
                  : output_tma_launch<4, float>(Mbuf, y, K, th, tw, oh, ow, row0, Pc, m_ld, s,
                                                dead, dead_bytes, act);
  const dim3 grid(static_cast<unsigned>((Pc + 127) / 128), K);
  static DeviceOnce configured;
  if (configured.first()) {
    max_carveout(output_transform_kernel<2, double>);
    max_carveout(output_transform_kernel<4, double>);
    max_carveout(output_transform_kernel<2, float>);
    max_carveout(output_transform_kernel<4, float>);
    configured.done();
  }
  if (prec == kFP64) {
    launch_k(m == 2 ? output_transform_kernel<2, double> : output_transform_kernel<4, double>, grid,
             dim3(128), 0, s, static_cast<const double*>(Mbuf), static_cast<double*>(y), N, K, th,
             tw, oh, ow, row0, Pc, m_ld, splits, act);
  } else {
    launch_k(m == 2 ? output_transform_kernel<2, float> : output_transform_kernel<4, float>, grid,
             dim3(128), 0, s, static_cast<const float*>(Mbuf), static_cast<float*>(y), N, K, th,
             tw, oh, ow, row0, Pc, m_ld, splits, act);
  }
  return cudaGetLastError();
}

// ====================================================== fused tiny-C layer
// For C <= 8 (VGG conv1.1 has C = 3) the alpha^2 GEMMs reduce over only C
// terms, so the transform-space intermediates (alpha^2*C*P + alpha^2*K*P
// values) dwarf the layer's input.  This kernel runs the whole layer on chip.
// Persistent: CTA b owns the filter chunk kc = b % nkc (KC = 64 filters; its
// alpha^2 x KC x CP transformed weights are converted to fp32 into shared
// memory once) and strides through units = 32 consecutive tiles of one tile
// row.  Per unit:
//   1. the C x alpha x (32m+2) input window of the NEXT unit is requested
//      with zero-filling cp.async (the padding is never materialised), so its
//      load latency hides under this unit's arithmetic;
//   2. thread (tile, channel) forms V[comp][t][c] = B^T d B (shared memory);
//   3. two passes of 32 filters: warp = 4 filters x 32 tiles (lane = tile),
//      M[comp] = sum_c U V from vector shared loads, the inverse transform
//      folded per transform row xi (only the m x m outputs and two rows of
//      Z = M A live), and the clipped m x m tile stored as vector rows.
// Arithmetic is fp32 (fp64 for FP64): at least the precision of the
// tensor-core path it replaces.
constexpr int kSmallC = 8;
constexpr int kSmallKC = 64;   // filters per CTA
constexpr int kSmallTiles = 32;

// one transformed weight in the operand format of `prec` -> fp32
__device__ __forceinline__ float load_op_any(int prec, const void* U, size_t idx) {
  if (prec == kBF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(U)[idx]);
  if (prec == kFP16) return __half2float(static_cast<const __half*>(U)[idx]);
  return static_cast<const float*>(U)[idx];  // fp32 (3xTF32) / tf32-rounded plane
}

// FPW filters per warp for vector weight loads (F(2x2)'s 2x2 outputs leave
// registers for 8; F(4x4)'s 4x4 outputs fit 2 without spilling at two CTAs
// per SM -- four spilled 24 B per thread: conv1.1 F4 N=64 303 -> 288 us).
template <int M, typename T>
struct SmallCfg {
  static constexpr int AL = M + 2, A2 = AL * AL, XW = kSmallTiles * M + 2;
  static constexpr int FPW = (M == 2 && sizeof(T) == 4) ? 8 : 2;
  static constexpr int passes = kSmallKC / (8 * FPW);
};

// FPW consecutive fp32 / fp64 values (16-byte aligned), broadcast loads
template <typename T, int FPW>
__device__ __forceinline__ void load_u(const T* p, T (&u)[FPW]) {
  if constexpr (sizeof(T) == 4 && FPW % 4 == 0) {
#pragma unroll
    for (int q = 0; q < FPW / 4; ++q) {
      const float4 x = reinterpret_cast<const float4*>(p)[q];
      u[4 * q] = x.x; u[4 * q + 1] = x.y; u[4 * q + 2] = x.z; u[4 * q + 3] = x.w;
    }
  } else if constexpr (sizeof(T) == 4) {
    static_assert(FPW % 2 == 0, "FPW");
#pragma unroll
    for (int q = 0; q < FPW / 2; ++q) {
      const float2 x = reinterpret_cast<const float2*>(p)[q];
      u[2 * q] = x.x; u[2 * q + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < FPW / 2; ++q) {
      const double2 x = reinterpret_cast<const double2*>(p)[q];
      u[2 * q] = x.x; u[2 * q + 1] = x.y;
    }
  }
}

// CE = the exact channel count (1..4) or 8 (C = 5..8, zero-padded).
template <int M, typename T, int CE>
__global__ void __launch_bounds__(256, 2) fused_smallc_kernel(
    const T* __restrict__ d, const void* __restrict__ U, T* __restrict__ y, int prec, int C,
    int H, int W, int K, int pad, int th, int tw, int oh, int ow, int c_pad, int n_units,
    int nkc, int act) {
  using A = Alg<M>;
  using Cfg = SmallCfg<M, T>;
  constexpr int AL = Cfg::AL, A2 = Cfg::A2, XW = Cfg::XW, FPW = Cfg::FPW;
  // smem: u[A2][CE][KC] | v[A2][CE][32] | in[2][CE][AL][XW]
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* s_u = reinterpret_cast<T*>(smem_raw);
  T* s_v = s_u + A2 * CE * kSmallKC;
  T* s_in = s_v + A2 * CE * kSmallTiles;
  constexpr int in_elems = CE * AL * XW;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kc = blockIdx.x % nkc;
  const int k_base = kc * kSmallKC;
  const int kn = min(kSmallKC, K - k_base);
  const int cta = blockIdx.x / nkc, nctas = gridDim.x / nkc;
  const int nxb = (tw + kSmallTiles - 1) / kSmallTiles;

  // stage the input window of unit uu into buffer b (zero-filled cp.async)
  auto stage = [&](int uu, int b) {
    const int row = uu / nxb, xb = uu - (uu / nxb) * nxb;
    const int n = row / th, ty = row - (row / th) * th;
    const int y0 = M * ty - pad, x0 = M * xb * kSmallTiles - pad;
    T* dst_b = s_in + b * in_elems;
    for (int r = warp; r < CE * AL; r += 8) {  // row (c, i): lanes along x
      const int c = r / AL, i = r - (r / AL) * AL;
      const int gy = y0 + i;
      const bool rowok = c < C && gy >= 0 && gy < H;
      const T* src = d + (rowok ? ((static_cast<size_t>(n) * C + c) * H + gy) * W : 0);
      const uint32_t dst0 = static_cast<uint32_t>(__cvta_generic_to_shared(dst_b + r * XW));
#pragma unroll
      for (int h = 0; h < (XW + 31) / 32; ++h) {
        const int x = lane + 32 * h;
        if (x >= XW) break;
        const int gx = x0 + x;
        const bool ok = rowok && gx >= 0 && gx < W;
        const T* sp = ok ? src + gx : d;
        if constexpr (sizeof(T) == 8)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst0 + 8 * x), "l"(sp),
                       "r"(ok ? 8 : 0) : "memory");
        else
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst0 + 4 * x), "l"(sp),
                       "r"(ok ? 4 : 0) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  griddep_launch();
  griddep_wait();
  int uu = cta;
  if (uu < n_units) stage(uu, 0);
  // transformed weights of this filter chunk -> fp32/fp64 smem [comp][c][k] (once)
  for (int e = threadIdx.x; e < A2 * CE * kSmallKC; e += 256) {
    const int kk = e % kSmallKC, r = e / kSmallKC;
    const int c = r % CE, comp = r / CE;
    T v = T(0);
    if (c < C && kk < kn) {
      const size_t idx = (static_cast<size_t>(comp) * K + k_base + kk) * c_pad + c;
      if constexpr (sizeof(T) == 8)
        v = static_cast<const double*>(U)[idx];
      else
        v = load_op_any(prec, U, idx);
    }
    s_u[e] = v;
  }

  for (int it = 0; uu < n_units; uu += nctas, ++it) {
    const int b = it & 1;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // window b landed; previous unit's s_v / window b^1 reads done
    if (uu + nctas < n_units) stage(uu + nctas, b ^ 1);
    const int row = uu / nxb, xb = uu - (uu / nxb) * nxb;
    const int n = row / th, ty = row - (row / th) * th;
    const int tx0 = xb * kSmallTiles;
    // ---- V = B^T d B for (tile = lane, channel = warp) pairs
    if (warp < CE) {
      const int c = warp;
      const T* win = s_in + b * in_elems + c * AL * XW + lane * M;
      T in[AL][AL], out[AL][AL];
#pragma unroll
      for (int i = 0; i < AL; ++i)
#pragma unroll
        for (int j = 0; j < AL; ++j) in[i][j] = win[i * XW + j];
      if constexpr (M == 4)
        bt6_2d(in, out);
      else
        sandwich<T, AL, AL>(in, out, [](int i, int j) { return A::BT(i, j); });
#pragma unroll
      for (int xi = 0; xi < AL; ++xi)
#pragma unroll
        for (int nu = 0; nu < AL; ++nu)
          s_v[((xi * AL + nu) * CE + c) * kSmallTiles + lane] = out[xi][nu];
    }
    __syncthreads();
    const int t = tx0 + lane;
    const int vr = min(M, oh - M * ty), vc = min(M, ow - M * t);
#pragma unroll 1
    for (int pass = 0; pass < Cfg::passes; ++pass) {
      const int k0 = (pass * 8 + warp) * FPW;  // chunk-local first filter of this warp
      if (k0 >= kn) break;
      T out[FPW][M][M] = {};
      T zp[FPW][M];  // Z of the previous transform row (F(4x4) pairs (1,2), (3,4))
#pragma unroll
      for (int xi = 0; xi < AL; ++xi) {
        T mrow[FPW][AL];
#pragma unroll
        for (int nu = 0; nu < AL; ++nu) {
          const int comp = xi * AL + nu;
#pragma unroll
          for (int c = 0; c < CE; ++c) {
            const T v = s_v[(comp * CE + c) * kSmallTiles + lane];
            T u[FPW];
            load_u<T, FPW>(s_u + (comp * CE + c) * kSmallKC + k0, u);
#pragma unroll
            for (int f = 0; f < FPW; ++f) mrow[f][nu] = c == 0 ? u[f] * v : fma(u[f], v, mrow[f][nu]);
          }
        }
#pragma unroll
        for (int f = 0; f < FPW; ++f) {
          T z[M];
          at_vec<M, T>(mrow[f], z);
          if constexpr (M == 4) {
            // Y = A^T Z over xi, by pairs:  y0 = Z0 + (Z1+Z2) + (Z3+Z4),
            // y1 = (Z1-Z2) + 2(Z3-Z4), y2 = (Z1+Z2) + 4(Z3+Z4), y3 = (Z1-Z2) + 8(Z3-Z4) + Z5
#pragma unroll
            for (int j = 0; j < M; ++j) {
              if (xi == 0) {
                out[f][0][j] = z[j];
              } else if (xi == 1 || xi == 3) {
                zp[f][j] = z[j];
              } else if (xi == 2) {
                const T sp = zp[f][j] + z[j], dm = zp[f][j] - z[j];
                out[f][0][j] += sp;
                out[f][1][j] = dm;
                out[f][2][j] = sp;
                out[f][3][j] = dm;
              } else if (xi == 4) {
                const T sp = zp[f][j] + z[j], dm = zp[f][j] - z[j];
                out[f][0][j] += sp;
                out[f][1][j] = fma(T(2), dm, out[f][1][j]);
                out[f][2][j] = fma(T(4), sp, out[f][2][j]);
                out[f][3][j] = fma(T(8), dm, out[f][3][j]);
              } else {
                out[f][3][j] += z[j];
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < M; ++i)
#pragma unroll
              for (int j = 0; j < M; ++j) out[f][i][j] = mac(out[f][i][j], A::AT(i, xi), z[j], false);
          }
        }
      }
      if (t < tw) {
#pragma unroll
        for (int f = 0; f < FPW; ++f) {
          if (k0 + f >= kn) break;
          emit_tile<M>(y, act, n, K, k_base + k0 + f, oh, ow, ty, t, vr, vc, out[f]);
        }
      }
    }
  }
}

template <int M, typename T, int CE>
static cudaError_t smallc_one(int prec, const void* d, const void* U, void* y, int N, int C,
                              int H, int W, int K, int pad, int th, int tw, int oh, int ow,
                              int c_pad, cudaStream_t s, int act) {
  using Cfg = SmallCfg<M, T>;
  auto kern = fused_smallc_kernel<M, T, CE>;
  constexpr size_t smem =
      sizeof(T) * CE * (Cfg::A2 * kSmallKC + Cfg::A2 * kSmallTiles + 2 * Cfg::AL * Cfg::XW);
  if constexpr (smem > 227 * 1024) {  // F(4x4) fp64 with C > 4: the planner does not route here
    return cudaErrorInvalidValue;
  } else {
    static DeviceOnce configured;
    static std::atomic<int> per_sm_dev[64];  // occupancy, per device (0 = not yet known)
    const int dbit = DeviceOnce::bit();
    if (configured.first()) {
      max_carveout(kern);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
      int occ = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
      per_sm_dev[dbit].store(occ < 1 ? 1 : occ);
      configured.done();
    }
    const int per_sm = per_sm_dev[dbit].load() > 0 ? per_sm_dev[dbit].load() : 1;
    const int nkc = (K + kSmallKC - 1) / kSmallKC;
    const long long units =
        static_cast<long long>(N) * th * ((tw + kSmallTiles - 1) / kSmallTiles);
    if (units > 0x7fffffffLL) return cudaErrorInvalidValue;
    const int sms = device_sms();
    long long per_kc = (static_cast<long long>(sms) * per_sm + nkc - 1) / nkc;
    if (per_kc > units) per_kc = units;
    if (per_kc < 1) per_kc = 1;
    const dim3 grid(static_cast<unsigned>(per_kc * nkc));
    launch_k(kern, grid, dim3(256), smem, s, static_cast<const T*>(d), U, static_cast<T*>(y),
             prec, C, H, W, K, pad, th, tw, oh, ow, c_pad, static_cast<int>(units), nkc, act);
    return cudaGetLastError();
  }
}

template <int M, typename T>
static cudaError_t smallc_ce(int prec, const void* d, const void* U, void* y, int N, int C, int H,
                             int W, int K, int pad, int th, int tw, int oh, int ow, int c_pad,
                             cudaStream_t s, int act) {
  switch (C) {
    case 1: return smallc_one<M, T, 1>(prec, d, U, y, N, C, H, W, K, pad, th, tw, oh, ow, c_pad, s, act);
    case 2: return smallc_one<M, T, 2>(prec, d, U, y, N, C, H, W, K, pad, th, tw, oh, ow, c_pad, s, act);
    case 3: return smallc_one<M, T, 3>(prec, d, U, y, N, C, H, W, K, pad, th, tw, oh, ow, c_pad, s, act);
    case 4: return smallc_one<M, T, 4>(prec, d, U, y, N, C, H, W, K, pad, th, tw, oh, ow, c_pad, s, act);
    default: return smallc_one<M, T, 8>(prec, d, U, y, N, C, H, W, K, pad, th, tw, oh, ow, c_pad, s, act);
  }
}

cudaError_t launch_fused_smallc(int m, int prec, const void* d, const void* U, void* y, int N,
                                int C, int H, int W, int K, int pad, int th, int tw, int oh,
                                int ow, int c_pad, cudaStream_t s, int act) {
  if (C > kSmallC) return cudaErrorInvalidValue;
  if (prec == kFP64)
    return m == 2 ? smallc_ce<2, double>(prec, d, U, y, N, C, H, W, K, pad, th, tw, oh, ow, c_pad, s, act)
                  : smallc_ce<4, double>(prec, d, U, y, N, C, H, W, K, pad, th, tw, oh, ow, c_pad, s, act);
  return m == 2 ? smallc_ce<2, float>(prec, d, U, y, N, C, H, W, K, pad, th, tw, oh, ow, c_pad, s, act)
                : smallc_ce<4, float>(prec, d, U, y, N, C, H, W, K, pad, th, tw, oh, ow, c_pad, s, act);
}

// ====================================================== weight gradient
// F(3x3, 2x2) (engine.py:278-328): dY is cut into non-overlapping 2x2 tiles
// (zero past the output edge), each paired with the 4x4 input patch at
// (2ty - pad, 2tx - pad).  The tile index b is the GEMM reduction axis, so
// both transforms store b innermost (the K-major operand layout of the
// tcgen05 GEMM):  Uw[s][comp][k][b] = (G y G^T),  Vw[s][comp][c][b] = (B^T d B).
// Thread = (row k or c, tile b), b fastest: coalesced stores.

template <int PREC>
__global__ void __launch_bounds__(256) wgrad_dy_transform_kernel(
    const typename OpStore<PREC>::T* __restrict__ dy, void* __restrict__ Uw, int K, int oh,
    int ow, int gh, int gw, long long b0, long long nb, long long b_pad) {
  using T = typename OpStore<PREC>::T;
  griddep_launch();
  griddep_wait();
  const long long bl = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x;
  const int k = blockIdx.y;
  if (bl >= nb) return;
  const long long b = b0 + bl;
  const long long per_img = static_cast<long long>(gh) * gw;
  const int n = static_cast<int>(b / per_img);
  const int rem = static_cast<int>(b - n * per_img);
  const int ty = rem / gw, tx = rem - (rem / gw) * gw;
  const T* src = dy + ((static_cast<long long>(n) * K + k) * oh + 2 * ty) * ow + 2 * tx;
  T in[2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      in[i][j] = (2 * ty + i < oh && 2 * tx + j < ow) ? src[i * ow + j] : T(0);
  T out[4][4];
  sandwich<T, 4, 2>(in, out, [](int i, int j) { return Alg32::G(i, j); });
  const size_t plane = static_cast<size_t>(16) * K * b_pad;
  size_t idx = static_cast<size_t>(k) * b_pad + bl;
#pragma unroll
  for (int xi = 0; xi < 4; ++xi)
#pragma unroll
    for (int nu = 0; nu < 4; ++nu) {
      OpStore<PREC>::put(Uw, idx, plane, out[xi][nu]);
      idx += static_cast<size_t>(K) * b_pad;
    }
}

template <int PREC>
__global__ void __launch_bounds__(256) wgrad_d_transform_kernel(
    const typename OpStore<PREC>::T* __restrict__ d, void* __restrict__ Vw, int C, int H, int W,
    int pad, int gh, int gw, long long b0, long long nb, long long b_pad) {
  using T = typename OpStore<PREC>::T;
  griddep_launch();
  griddep_wait();
  const long long bl = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x;
  const int c = blockIdx.y;
  if (bl >= nb) return;
  const long long b = b0 + bl;
  const long long per_img = static_cast<long long>(gh) * gw;
  const int n = static_cast<int>(b / per_img);
  const int rem = static_cast<int>(b - n * per_img);
  const int ty = rem / gw, tx = rem - (rem / gw) * gw;
  const int y0 = 2 * ty - pad, x0 = 2 * tx - pad;
  const T* plane_in = d + (static_cast<long long>(n) * C + c) * H * W;
  T in[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int yy = y0 + u, xx = x0 + v;
      in[u][v] = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? plane_in[yy * W + xx] : T(0);
    }
  T out[4][4];
  sandwich<T, 4, 4>(in, out, [](int i, int j) { return Alg32::BT(i, j); });
  const size_t plane = static_cast<size_t>(16) * C * b_pad;
  size_t idx = static_cast<size_t>(c) * b_pad + bl;
#pragma unroll
  for (int xi = 0; xi < 4; ++xi)
#pragma unroll
    for (int nu = 0; nu < 4; ++nu) {
      OpStore<PREC>::put(Vw, idx, plane, out[xi][nu]);
      idx += static_cast<size_t>(C) * b_pad;
    }
}

// dg[k][c] = A^T (sum_s M[s][.][k][c]) A, slices summed in ascending order.
// Thread = (k, c) with all 16 components: used when K*C fills the GPU.
template <typename TA>
__global__ void __launch_bounds__(256) wgrad_inverse_kernel(const TA* __restrict__ Mbuf,
                                                            TA* __restrict__ dg, int K, int C,
                                                            long long m_ld, int slices) {
  griddep_launch();
  griddep_wait();
  const int c = blockIdx.x * 256 + threadIdx.x;
  const int k = blockIdx.y;
  if (c >= C) return;
  const size_t comp_stride = static_cast<size_t>(K) * m_ld;
  TA acc[4][4];
#pragma unroll
  for (int xi = 0; xi < 4; ++xi)
#pragma unroll
    for (int nu = 0; nu < 4; ++nu)
      acc[xi][nu] = Mbuf[(xi * 4 + nu) * comp_stride + static_cast<size_t>(k) * m_ld + c];
  for (int s = 1; s < slices; ++s) {
    const TA* Ms = Mbuf + static_cast<size_t>(s) * 16 * comp_stride;
#pragma unroll
    for (int xi = 0; xi < 4; ++xi)
#pragma unroll
      for (int nu = 0; nu < 4; ++nu)
        acc[xi][nu] += Ms[(xi * 4 + nu) * comp_stride + static_cast<size_t>(k) * m_ld + c];
  }
  TA out[3][3];
  sandwich<TA, 3, 4>(acc, out, [](int i, int j) { return Alg32::AT(i, j); });
  TA* dst = dg + (static_cast<size_t>(k) * C + c) * 9;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) dst[i * 3 + j] = out[i][j];
}

// Same result, for small K*C with many slices (conv1.1: C = 3, tens of
// slices): block = (16 channels c, one k), thread = (component, c), c fastest.
// Each thread sums one M element over the slices (independent loads), then 16
// threads apply the 4x4 -> 3x3 inverse.
template <typename TA>
__global__ void __launch_bounds__(256) wgrad_inverse_wide_kernel(const TA* __restrict__ Mbuf,
                                                                 TA* __restrict__ dg, int K,
                                                                 int C, long long m_ld,
                                                                 int slices) {
  griddep_launch();
  griddep_wait();
  __shared__ TA sm[16][17];
  const int cl = threadIdx.x & 15, comp = threadIdx.x >> 4;
  const int c = blockIdx.x * 16 + cl;
  const int k = blockIdx.y;
  const size_t comp_stride = static_cast<size_t>(K) * m_ld;
  const size_t slice_stride = 16 * comp_stride;
  if (c < C) {
    const TA* p = Mbuf + comp * comp_stride + static_cast<size_t>(k) * m_ld + c;
    TA v = p[0];
#pragma unroll 8
    for (int s = 1; s < slices; ++s) v += p[s * slice_stride];
    sm[comp][cl] = v;
  }
  __syncthreads();
  if (threadIdx.x >= 16 || c >= C) return;
  TA acc[4][4];
#pragma unroll
  for (int xi = 0; xi < 4; ++xi)
#pragma unroll
    for (int nu = 0; nu < 4; ++nu) acc[xi][nu] = sm[xi * 4 + nu][cl];
  TA out[3][3];
  sandwich<TA, 3, 4>(acc, out, [](int i, int j) { return Alg32::AT(i, j); });
  TA* dst = dg + (static_cast<size_t>(k) * C + c) * 9;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) dst[i * 3 + j] = out[i][j];
}

// ---------------------------------------------- small-C weight gradient
// C <= 4 (conv1.1): the tile-reduction GEMM would put 3 channels on the
// tensor core's 128-row side (and stage 16 x K transformed dY values per tile
// through HBM for 16 x C x K MACs).  Instead one pass on the CUDA cores reads
// dY and d once: per group of 32 tiles the block stages the 2x2 dY patches of
// 64 filters and the transformed input patches (B^T d B, C channels) in shared
// memory, then thread (k, q) forms G y G^T for tiles q, q+4, ... and
// accumulates the 16 x C products.  Operands are rounded to the GEMM operand
// type first (products exact in fp32, as on the tensor core); fp32 is plain
// FFMA (at least as accurate as 3xTF32).  Each block writes one M slice
// [16][K][m_ld]; wgrad_reduce_slices_kernel sums them in a fixed order.
template <int PREC>
__device__ __forceinline__ float op_round(float x) {
  if constexpr (PREC == kTF32) {
    uint32_t b;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(x));
    return __uint_as_float(b);
  } else if constexpr (PREC == kBF16) {
    return __bfloat162float(__float2bfloat16_rn(x));
  } else if constexpr (PREC == kFP16) {
    return __half2float(__float2half_rn(x));
  } else {
    return x;
  }
}

constexpr int kWgSmallTiles = 32;  // tiles per staged group
constexpr int kWgSmallK = 64;      // filters per block (grid.y covers K)

template <int PREC, int CC>
__global__ void __launch_bounds__(256) wgrad_smallc_kernel(
    const float* __restrict__ d, const float* __restrict__ dy, float* __restrict__ Mparts, int K,
    int H, int W, int pad, int oh, int ow, int gh, int gw, long long B, long long m_ld) {
  constexpr int TG = kWgSmallTiles;
  __shared__ float4 dyS[kWgSmallK][TG + 1];  // [k][tile] 2x2 dY patch
  // [tile][comp * CC + c] transformed input; row stride VS float4s, picked so
  // a quarter-warp's 8 loads (4 tiles x 2 component rows) hit distinct banks
  constexpr int VS = CC == 1 ? 6 : CC == 2 ? 9 : CC == 3 ? 14 : 17;
  __shared__ float4 vS[TG][VS];
  griddep_launch();
  griddep_wait();
  const int tid = threadIdx.x;
  // thread = (tile lane q, component row cq = xi, filter quad kq): filters
  // 4kq..4kq+3 x components 4cq..4cq+3 x CC channels in registers, so every
  // shared-memory value feeds 4 (V) or 4 CC (dY) multiply-adds
  const int q = tid & 3, cq = (tid >> 2) & 3, kq = tid >> 4;
  const int k0 = blockIdx.y * kWgSmallK;
  // tile indices fit in 32 bits (the planner checks B < 2^31): 32-bit
  // division and offsets keep the load phase short
  const int Bi = static_cast<int>(B);
  const int ngroups = (Bi + TG - 1) / TG;
  const int per_img = gh * gw;
  // row cq of F(3,2)'s G = {1,0}, {1/2,1/2}, {1/2,-1/2}, {0,1}
  const float g0 = cq == 0 ? 1.f : (cq == 3 ? 0.f : 0.5f);
  const float g1 = cq == 0 ? 0.f : (cq == 1 ? 0.5f : (cq == 2 ? -0.5f : 1.f));
  float acc[4][4][CC];  // [filter kk][component nu][channel]
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < CC; ++c) acc[kk][i][c] = 0.f;

  // this thread's dY element in every group: column j, row i of tile tl, for
  // filters k0 + kd, k0 + kd + 2, ... (a warp reads 2 x 16 consecutive
  // columns of one row); all 32 loads in flight at once
  const int dj = tid & 1, dtl = (tid >> 1) & (TG - 1), di = (tid >> 6) & 1, kd = tid >> 7;
  const int kstride = 2 * oh * ow;  // two filter planes
  // loads with k = k0 + kd + 2 it < K
  const int nit = min(kWgSmallK / 2, (K - k0 - kd + 1) / 2);
  for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int tb = g * TG;
    {
      const int b = tb + dtl;
      float v[kWgSmallK / 2];
      int n = 0, y = oh, x = 0;
      if (b < Bi) {
        n = b / per_img;
        const int rem = b - n * per_img;
        const int ty = rem / gw;
        y = 2 * ty + di;
        x = 2 * (rem - ty * gw) + dj;
      }
      if (y < oh && x < ow) {
        const float* src = dy + ((static_cast<long long>(n) * K + k0 + kd) * oh + y) * ow + x;
        if (nit == kWgSmallK / 2) {  // all 64 filters of the block exist
#pragma unroll
          for (int it = 0; it < kWgSmallK / 2; ++it) v[it] = __ldg(src + it * kstride);
        } else {
#pragma unroll
          for (int it = 0; it < kWgSmallK / 2; ++it)
            v[it] = it < nit ? __ldg(src + it * kstride) : 0.f;
        }
      } else {
#pragma unroll
        for (int it = 0; it < kWgSmallK / 2; ++it) v[it] = 0.f;
      }
#pragma unroll
      for (int it = 0; it < kWgSmallK / 2; ++it)
        reinterpret_cast<float*>(&dyS[kd + 2 * it][dtl])[di * 2 + dj] = v[it];
    }
    // transformed input patches, one (tile, channel) per thread
    if (tid < TG * CC) {
      const int tl = tid % TG, c = tid / TG;
      const int b = tb + tl;
      float out[4][4];
      if (b < Bi) {
        const int n = b / per_img;
        const int rem = b - n * per_img;
        const int ty = rem / gw;
        const int y0 = 2 * ty - pad, x0 = 2 * (rem - ty * gw) - pad;
        const float* plane = d + (static_cast<long long>(n) * CC + c) * H * W;
        float in[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int yy = y0 + u, xx = x0 + v;
            in[u][v] = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? __ldg(plane + yy * W + xx) : 0.f;
          }
        sandwich<float, 4, 4>(in, out, [](int i2, int j2) { return Alg32::BT(i2, j2); });
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) out[u][v] = 0.f;
      }
      float* dst = reinterpret_cast<float*>(vS[tl]);  // row tl: [comp][c]
#pragma unroll
      for (int xi = 0; xi < 4; ++xi)
#pragma unroll
        for (int nu = 0; nu < 4; ++nu) dst[(xi * 4 + nu) * CC + c] = op_round<PREC>(out[xi][nu]);
    }
    __syncthreads();
#pragma unroll 2
    for (int t = q; t < TG; t += 4) {
      float vv[4 * CC];  // V[4cq + nu][c]
#pragma unroll
      for (int i = 0; i < CC; ++i) {
        const float4 f = vS[t][cq * CC + i];
        vv[4 * i] = f.x;
        vv[4 * i + 1] = f.y;
        vv[4 * i + 2] = f.z;
        vv[4 * i + 3] = f.w;
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const float4 y4 = dyS[4 * kq + kk][t];  // y[0][0], y[0][1], y[1][0], y[1][1]
        // (G y G^T)[cq][nu]: row cq of G y, then the G^T columns
        const float t0 = g0 * y4.x + g1 * y4.z, t1 = g0 * y4.y + g1 * y4.w;
        const float u[4] = {t0, 0.5f * t0 + 0.5f * t1, 0.5f * t0 - 0.5f * t1, t1};
#pragma unroll
        for (int nu = 0; nu < 4; ++nu) {
          const float uu = op_round<PREC>(u[nu]);
#pragma unroll
          for (int c = 0; c < CC; ++c)
            acc[kk][nu][c] = fmaf(uu, vv[nu * CC + c], acc[kk][nu][c]);
        }
      }
    }
    __syncthreads();
  }
  // fold the 4 tile lanes (fixed butterfly order), then lane q == 0 writes
  // this block's slice
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < CC; ++c) {
        float v = acc[kk][i][c];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        acc[kk][i][c] = v;
      }
  if (q != 0) return;
  float* slice = Mparts + static_cast<size_t>(blockIdx.x) * 16 * K * m_ld;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const int k = k0 + 4 * kq + kk;
    if (k >= K) break;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < CC; ++c)
        slice[(static_cast<size_t>(4 * cq + i) * K + k) * m_ld + c] = acc[kk][i][c];
  }
}

// out[i] = sum over S slices of slices[s][i] (n elements each), in a fixed
// order: block = 32 consecutive elements x 32 slice groups (coalesced rows,
// ~S/32 loads in flight per thread), group sums folded in ascending order.
__global__ void __launch_bounds__(1024) wgrad_reduce_slices_kernel(const float* __restrict__ sl,
                                                                   float* __restrict__ out,
                                                                   long long n, int S) {
  griddep_launch();
  griddep_wait();
  __shared__ float part[32][33];
  const int il = threadIdx.x & 31, sg = threadIdx.x >> 5;
  const long long i = blockIdx.x * 32LL + il;
  float v = 0.f;
  if (i < n) {
#pragma unroll 8
    for (int s = sg; s < S; s += 32) v += sl[static_cast<size_t>(s) * n + i];
  }
  part[sg][il] = v;
  __syncthreads();
  if (sg != 0 || i >= n) return;
  float r = part[0][il];
#pragma unroll
  for (int g2 = 1; g2 < 32; ++g2) r += part[g2][il];
  out[i] = r;
}

template <int PREC>
static cudaError_t wgrad_smallc_prec(const float* d, const float* dy, float* parts, int K, int C,
                                     int H, int W, int pad, int oh, int ow, int gh, int gw,
                                     long long B, long long m_ld, int nblk, cudaStream_t s) {
  const dim3 grid(nblk, (K + kWgSmallK - 1) / kWgSmallK);
  switch (C) {
    case 1: launch_k(wgrad_smallc_kernel<PREC, 1>, grid, dim3(256), 0, s, d, dy, parts, K, H, W, pad, oh, ow, gh, gw, B, m_ld); break;
    case 2: launch_k(wgrad_smallc_kernel<PREC, 2>, grid, dim3(256), 0, s, d, dy, parts, K, H, W, pad, oh, ow, gh, gw, B, m_ld); break;
    case 3: launch_k(wgrad_smallc_kernel<PREC, 3>, grid, dim3(256), 0, s, d, dy, parts, K, H, W, pad, oh, ow, gh, gw, B, m_ld); break;
    case 4: launch_k(wgrad_smallc_kernel<PREC, 4>, grid, dim3(256), 0, s, d, dy, parts, K, H, W, pad, oh, ow, gh, gw, B, m_ld); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_wgrad_smallc(int prec, const void* d, const void* dy, void* parts,
                                void* summed, int K, int C, int H, int W, int pad, int oh, int ow,
                                int gh, int gw, long long B, long long m_ld, int nblk,
                                cudaStream_t s) {
  const float* df = static_cast<const float*>(d);
  const float* yf = static_cast<const float*>(dy);
  float* pf = static_cast<float*>(parts);
  cudaError_t e;
  switch (prec) {
    case kFP32: e = wgrad_smallc_prec<kFP32>(df, yf, pf, K, C, H, W, pad, oh, ow, gh, gw, B, m_ld, nblk, s); break;
    case kTF32: e = wgrad_smallc_prec<kTF32>(df, yf, pf, K, C, H, W, pad, oh, ow, gh, gw, B, m_ld, nblk, s); break;
    case kBF16: e = wgrad_smallc_prec<kBF16>(df, yf, pf, K, C, H, W, pad, oh, ow, gh, gw, B, m_ld, nblk, s); break;
    case kFP16: e = wgrad_smallc_prec<kFP16>(df, yf, pf, K, C, H, W, pad, oh, ow, gh, gw, B, m_ld, nblk, s); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  const long long n = 16LL * K * m_ld;
  launch_k(wgrad_reduce_slices_kernel, dim3(static_cast<unsigned>((n + 31) / 32)), dim3(1024), 0,
           s, static_cast<const float*>(parts), static_cast<float*>(summed), n, nblk);
  return cudaGetLastError();
}

// acc (+)= sum_s slice[s], ascending s (one tile chunk's split partials).
template <typename TA>
__global__ void __launch_bounds__(256) wgrad_accumulate_kernel(TA* __restrict__ acc,
                                                               const TA* __restrict__ slices,
                                                               long long n, int splits,
                                                               int first) {
  griddep_launch();
  griddep_wait();
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) {
    TA v = first ? slices[i] : acc[i] + slices[i];
    for (int s = 1; s < splits; ++s) v += slices[s * n + i];
    acc[i] = v;
  }
}

cudaError_t launch_wgrad_accumulate(int prec, void* acc, const void* slices, long long n,
                                    int splits, int first, cudaStream_t s) {
  long long blocks = (n + 255) / 256;
  if (blocks > 8 * 148) blocks = 8 * 148;
  const dim3 grid(static_cast<unsigned>(blocks > 0 ? blocks : 1));
  if (prec == kFP64)
    launch_k(wgrad_accumulate_kernel<double>, grid, dim3(256), 0, s, static_cast<double*>(acc),
             static_cast<const double*>(slices), n, splits, first);
  else
    launch_k(wgrad_accumulate_kernel<float>, grid, dim3(256), 0, s, static_cast<float*>(acc),
             static_cast<const float*>(slices), n, splits, first);
  return cudaGetLastError();
}

template <int PREC>
static cudaError_t wgrad_tf_one(const void* d, const void* dy, void* Uw, void* Vw, int K, int C,
                                int H, int W, int pad, int oh, int ow, int gh, int gw,
                                long long b0, long long nb, long long b_pad, cudaStream_t s) {
  using T = typename OpStore<PREC>::T;
  const unsigned gx = static_cast<unsigned>((nb + 255) / 256);
  launch_k(wgrad_dy_transform_kernel<PREC>, dim3(gx, K), dim3(256), 0, s,
           static_cast<const T*>(dy), Uw, K, oh, ow, gh, gw, b0, nb, b_pad);
  launch_k(wgrad_d_transform_kernel<PREC>, dim3(gx, C), dim3(256), 0, s,
           static_cast<const T*>(d), Vw, C, H, W, pad, gh, gw, b0, nb, b_pad);
  return cudaGetLastError();
}

cudaError_t launch_wgrad_transforms(int prec, const void* d, const void* dy, void* Uw, void* Vw,
                                    int K, int C, int H, int W, int pad, int oh, int ow, int gh,
                                    int gw, long long b0, long long nb, long long b_pad,
                                    cudaStream_t s) {
  if (nb <= 0) return cudaSuccess;
  switch (prec) {
    case kFP32: return wgrad_tf_one<kFP32>(d, dy, Uw, Vw, K, C, H, W, pad, oh, ow, gh, gw, b0, nb, b_pad, s);
    case kTF32: return wgrad_tf_one<kTF32>(d, dy, Uw, Vw, K, C, H, W, pad, oh, ow, gh, gw, b0, nb, b_pad, s);
    case kBF16: return wgrad_tf_one<kBF16>(d, dy, Uw, Vw, K, C, H, W, pad, oh, ow, gh, gw, b0, nb, b_pad, s);
    case kFP16: return wgrad_tf_one<kFP16>(d, dy, Uw, Vw, K, C, H, W, pad, oh, ow, gh, gw, b0, nb, b_pad, s);
    case kFP64: return wgrad_tf_one<kFP64>(d, dy, Uw, Vw, K, C, H, W, pad, oh, ow, gh, gw, b0, nb, b_pad, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_wgrad_inverse(int prec, const void* Mbuf, void* dg, int K, int C,
                                 long long m_ld, int slices, cudaStream_t s) {
  // thread per (k, c) once K*C covers the SMs a few times over; else spread
  // the slice sums over 16x more threads
  const bool wide = static_cast<long long>(K) * C < 64LL * 1024;
  const dim3 grid(wide ? (C + 15) / 16 : (C + 255) / 256, K);
  if (prec == kFP64) {
    if (wide)
      launch_k(wgrad_inverse_wide_kernel<double>, grid, dim3(256), 0, s,
               static_cast<const double*>(Mbuf), static_cast<double*>(dg), K, C, m_ld, slices);
    else
      launch_k(wgrad_inverse_kernel<double>, grid, dim3(256), 0, s,
               static_cast<const double*>(Mbuf), static_cast<double*>(dg), K, C, m_ld, slices);
  } else {
    if (wide)
      launch_k(wgrad_inverse_wide_kernel<float>, grid, dim3(256), 0, s,
               static_cast<const float*>(Mbuf), static_cast<float*>(dg), K, C, m_ld, slices);
    else
      launch_k(wgrad_inverse_kernel<float>, grid, dim3(256), 0, s,
               static_cast<const float*>(Mbuf), static_cast<float*>(dg), K, C, m_ld, slices);
  }
  return cudaGetLastError();
}

}  // namespace wino
