// Fused Winograd-GEMM for F(2x2,3x3) and F(4x4,3x3) on sm_100a: the input-tile
// transform runs in the GEMM's producer warps, the alpha^2 transform-space
// products run on tcgen05 with TMEM accumulators, and the inverse transform
// runs in the epilogue, so V and M never leave the chip.
// (Reference stages fused here: engine.py:226-254 -- data transform
// engine.py:235-237, batched_matmul kernels.py:50-65, inverse transform and
// clip engine.py:241-254.)
//
// The alpha^2 accumulators of one (filter block x tile block) do not fit one
// SM's TMEM (F(4x4): 36 x 128 x 64 fp32 = 1.2 MB vs 256 KB), so a thread-block
// CLUSTER of alpha CTAs shares the unit: CTA s owns the alpha components of
// transform row xi = s,
//   M[s][nu][k][p] = sum_c U[s*alpha+nu][k][c] * V[s*alpha+nu][p][c],
// as alpha accumulators of 128 filters (TMEM lanes) x Pb tiles (columns).
//   producer : warp 0 TMAs U[s*alpha+nu] boxes (128 filters x one swizzle row
//              of channels) for every nu into a 3-stage ring;
//   transform: warps 2-9 read the raw NCHW input (read-only path, zero padding
//              by predication -- never materialised), form row s of B^T d B
//              for every nu (r = B^T[s,:] d, then V[s][nu] = r B[:,nu]) and
//              write it, rounded to the operand format, straight into the
//              swizzled K-major smem layout tcgen05 reads;
//   MMA      : warp 1, one thread, alpha tcgen05.mma per K step (3 per nu for
//              3xTF32: lo*hi + hi*lo + hi*hi);
//   epilogue : warps 2-9 fold their row with A^T along nu,
//              Z_s[j] = sum_nu A^T[j][nu] M[s][nu]   (m values per filter/tile),
//              push Z_s through distributed shared memory to the CTA that owns
//              the filter (filters are partitioned alpha ways), and after a
//              cluster barrier the owner forms Y[i][j] = sum_s A^T[i][s] Z_s[j]
//              in fixed s order (deterministic) and writes the clipped m x m
//              tile to NCHW y (engine.py:246-254).
// Split-C (small tile counts): each split writes its partial y slice and a
// small kernel sums the slices in ascending order.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>

#include "sm100_ptx.cuh"
#include "wino_internal.h"
#include "winograd_mats.cuh"

namespace wino {

template <int M, int PREC>
struct FCfg {
  static constexpr int alpha = M + 2;
  static constexpr int a2 = alpha * alpha;
  static constexpr int Kb = 128;                  // filters per unit (UMMA M, TMEM lanes)
  static constexpr int Pb = (M == 4) ? 64 : 128;  // tiles per unit (UMMA N); alpha*Pb <= 512
  static constexpr int kind = (PREC == kFP32 || PREC == kTF32) ? 1 : 0;
  static constexpr int esize = kind ? 4 : 2;
  static constexpr int nsplit = (PREC == kFP32) ? 2 : 1;
  static constexpr int swz = (PREC == kFP32) ? 32 : 64;  // operand row bytes per stage
  static constexpr int bkc = swz / esize;                // channels per stage
  static constexpr int uk = 32 / esize;                  // channels per tcgen05.mma
  static constexpr int chunks = swz / 16;                // 16-byte chunks per operand row
  static constexpr int cpc = 16 / esize;                 // channels per chunk
  static constexpr int u_slot = Kb * swz;
  static constexpr int v_slot = Pb * swz;
  static constexpr int u_bytes = nsplit * alpha * u_slot;
  static constexpr int v_bytes = nsplit * alpha * v_slot;
  static constexpr int stage_bytes = u_bytes + v_bytes;
  static constexpr int stages = 3;
  static constexpr int NT = 256;                   // transform / epilogue threads
  static constexpr int threads = NT + 64;          // + producer warp + MMA warp
  static constexpr int fo = (Kb + alpha - 1) / alpha;  // filters owned per CTA in the epilogue
  static constexpr int fls = Pb * M + 4;           // floats per (src, filter) row, +16 B: no bank conflicts
  static constexpr int xbytes = alpha * fo * fls * 4;  // Z receive buffer (aliases the ring)
  static constexpr int ring = stages * stage_bytes;
  static constexpr int bar_off = ring > xbytes ? ring : xbytes;
  static constexpr int smem = bar_off + 512 + 1024;
  static constexpr int tmem_cols = 512;
  static constexpr int TT = 8;                     // tiles per TMEM load in the epilogue
  static_assert(alpha * Pb <= tmem_cols, "accumulators exceed TMEM");
  static_assert(smem <= 227 * 1024, "shared memory budget");
  static_assert(NT % Pb == 0, "thread/tile mapping");
};

struct FusedParams {
  const float* d;
  float* y;       // output (splits == 1) or partial slices [split][N][K][oh][ow]
  long long P;
  int N, C, H, W, K, pad, th, tw, oh, ow;
  int num_kb, kb_per_split;
  int vec;                   // 1: pad == 1 and W % m == 0 (vector row loads)
  long long p0;              // global index of local tile 0 (row chunk offset; V-TMA mode)
  long long y_split_stride;  // elements between split slices (0 when splits == 1)
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pack_f16x2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t b;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(x));
  return b;
}

// One 16-byte operand chunk (cpc channels of one tile, one component) in the
// operand format; 3xTF32 also writes the lo plane.
template <int PREC, int CPC>
__device__ __forceinline__ void store_chunk(unsigned char* hi, unsigned char* lo,
                                            const float (&v)[CPC]) {
  uint4 q;
  if constexpr (PREC == kBF16) {
    q = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                   pack_bf16x2(v[6], v[7]));
  } else if constexpr (PREC == kFP16) {
    q = make_uint4(pack_f16x2(v[0], v[1]), pack_f16x2(v[2], v[3]), pack_f16x2(v[4], v[5]),
                   pack_f16x2(v[6], v[7]));
  } else if constexpr (PREC == kTF32) {
    q = make_uint4(tf32_rna(v[0]), tf32_rna(v[1]), tf32_rna(v[2]), tf32_rna(v[3]));
  } else {  // 3xTF32: hi = rna_tf32(x), lo = x - hi (exact in fp32)
    uint32_t h[4];
    float l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      h[i] = tf32_rna(v[i]);
      l[i] = v[i] - __uint_as_float(h[i]);
    }
    q = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(lo) = make_uint4(__float_as_uint(l[0]), __float_as_uint(l[1]),
                                               __float_as_uint(l[2]), __float_as_uint(l[3]));
  }
  *reinterpret_cast<uint4*>(hi) = q;
}

// Per-tile input geometry, fixed for the whole channel loop.
struct TileGeo {
  long long base;   // offset of the patch origin (y0, x0) in channel 0 of image n
  uint32_t rmask;   // bit u: input row y0+u inside the image
  uint32_t cmask;   // bit x: input column x0+x inside the image
};

// One input-patch row d[u][0..alpha) of one channel.  VEC (pad == 1 and
// W % m == 0): the middle m values start at column m*tx, m-float aligned and
// always inside the image, so a row is one scalar + one vector (float4 for
// F(4x4), float2 for F(2x2)) + one scalar load.  Out-of-image elements are
// predicated to 0 (the zero padding is never materialised); there is no
// edge/interior branch, so warps never diverge on tile position.
template <int M, bool VEC>
__device__ __forceinline__ void load_row(const float* __restrict__ row, int u, const TileGeo& g,
                                         float (&x)[M + 2]) {
  constexpr int AL = M + 2;
  const bool rok = (g.rmask >> u) & 1u;
  if constexpr (VEC) {
    float a = 0.f, b = 0.f;
    if (rok && (g.cmask & 1u)) a = __ldg(row);
    if (rok && ((g.cmask >> (AL - 1)) & 1u)) b = __ldg(row + AL - 1);
    x[0] = a;
    x[AL - 1] = b;
    if constexpr (M == 4) {
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
      if (rok) q = __ldg(reinterpret_cast<const float4*>(row + 1));
      x[1] = q.x; x[2] = q.y; x[3] = q.z; x[4] = q.w;
    } else {
      float2 q = make_float2(0.f, 0.f);
      if (rok) q = __ldg(reinterpret_cast<const float2*>(row + 1));
      x[1] = q.x; x[2] = q.y;
    }
  } else {
#pragma unroll
    for (int v = 0; v < AL; ++v) {
      float e = 0.f;
      if (rok && ((g.cmask >> v) & 1u)) e = __ldg(row + v);
      x[v] = e;
    }
  }
}

// Row S of B^T d B for one channel: r[x] = sum_u BT[S][u] d[u][x], then
// V[nu] = sum_x BT[nu][x] r[x] (for F(4,3) with the shared-subexpression bt6).
// Rows with BT[S][u] == 0 are never loaded.
template <int M, int S, bool VEC>
__device__ __forceinline__ void v_row(const float* __restrict__ src, int W, const TileGeo& g,
                                      float (&v)[M + 2]) {
  using A = Alg<M>;
  constexpr int AL = M + 2;
  float dr[AL][AL];
#pragma unroll
  for (int u = 0; u < AL; ++u) {
    if (A::BT(S, u) != 0.0) load_row<M, VEC>(src + u * W, u, g, dr[u]);
  }
  float r[AL];
#pragma unroll
  for (int x = 0; x < AL; ++x) {
    float acc = 0.f;
    bool first = true;
#pragma unroll
    for (int u = 0; u < AL; ++u) {
      const double c = A::BT(S, u);
      if (c != 0.0) {
        acc = mac(acc, c, dr[u][x], first);
        first = false;
      }
    }
    r[x] = acc;
  }
  if constexpr (M == 4) {
    bt6(r, v);  // shared-subexpression F(4,3) column transform (winograd_mats.cuh)
  } else {
#pragma unroll
    for (int nu = 0; nu < AL; ++nu) {
      float acc = 0.f;
      bool first = true;
#pragma unroll
      for (int x = 0; x < AL; ++x) {
        const double c = A::BT(nu, x);
        acc = mac(acc, c, r[x], first);
        if (c != 0.0) first = false;
      }
      v[nu] = acc;
    }
  }
}

// Transform warps' main loop for cluster rank S.  Thread = (tile t, 16-byte
// channel chunk j): it forms V[S][nu] for cpc channels and stores one 16-byte
// chunk per nu.  The loads and arithmetic of a stage run before the wait for
// the ring slot, so they overlap the MMAs still reading it.
// 3xTF32 keeps one fp32 plane of U (and of a staged V) in HBM: once the TMA
// bytes of the stage have landed (tmaf), the transform warps split them into
// hi = rna_tf32(x) in place and lo = x - hi before releasing the stage.
template <int PREC>
__device__ __forceinline__ void split_stage(unsigned char* base, int bytes_hi, int tid,
                                            int nthreads) {
  if constexpr (PREC == kFP32) {
    float4* hi = reinterpret_cast<float4*>(base);
    float4* lo = reinterpret_cast<float4*>(base + bytes_hi);
    for (int i = tid; i < bytes_hi / 16; i += nthreads) ptx::split_tf32_chunk(hi + i, lo + i);
  }
}

template <int M, int PREC, int S, bool VEC>
__device__ __forceinline__ void transform_loop_v(const FusedParams& a, unsigned char* smem,
                                                 uint64_t* full, uint64_t* empty, uint64_t* tmaf,
                                                 int tid, int pb, int kb0, int kb1) {
  using Cf = FCfg<M, PREC>;
  constexpr int AL = Cf::alpha, Pb = Cf::Pb, CPC = Cf::cpc, NG = Cf::NT / Pb;
  const int t = tid % Pb, jg = tid / Pb;
  const long long p = static_cast<long long>(pb) * Pb + t;
  const bool valid = p < a.P;
  int n = 0, ty = 0, tx = 0;
  if (valid) {
    const long long per_img = static_cast<long long>(a.th) * a.tw;
    n = static_cast<int>(p / per_img);
    const int rem = static_cast<int>(p - n * per_img);
    ty = rem / a.tw;
    tx = rem - ty * a.tw;
  }
  const int y0 = M * ty - a.pad, x0 = M * tx - a.pad;
  TileGeo g;
  g.rmask = 0;
  g.cmask = 0;
#pragma unroll
  for (int u = 0; u < AL; ++u) {
    if (valid && y0 + u >= 0 && y0 + u < a.H) g.rmask |= 1u << u;
    if (x0 + u >= 0 && x0 + u < a.W) g.cmask |= 1u << u;
  }
  g.base = (static_cast<long long>(n) * a.C * a.H + y0) * a.W + x0;
  const long long plane = static_cast<long long>(a.H) * a.W;
  const int lane = tid & 31;
  int it = 0;
  for (int kb = kb0; kb < kb1; ++kb, ++it) {
    const int st = it % Cf::stages;
    unsigned char* vst = smem + st * Cf::stage_bytes + Cf::u_bytes;
    bool waited = false;
    for (int j = jg; j < Cf::chunks; j += NG) {
      const int c0 = kb * Cf::bkc + j * CPC;
      float v[AL][CPC];
#pragma unroll
      for (int cc = 0; cc < CPC; ++cc) {
        const int c = c0 + cc;
        TileGeo gc = g;
        if (c >= a.C) gc.rmask = 0;  // channel padding: zeros, no loads
        const float* src = a.d + g.base + static_cast<long long>(c < a.C ? c : 0) * plane;
        float vv[AL];
        v_row<M, S, VEC>(src, a.W, gc, vv);
#pragma unroll
        for (int nu = 0; nu < AL; ++nu) v[nu][cc] = vv[nu];
      }
      if (!waited) {
        ptx::mbar_wait(&empty[st], ((it / Cf::stages) & 1) ^ 1);
        waited = true;
      }
      const uint32_t off = t * Cf::swz + ptx::swz_chunk<Cf::swz>(t, j) * 16;
#pragma unroll
      for (int nu = 0; nu < AL; ++nu)
        store_chunk<PREC, CPC>(vst + nu * Cf::v_slot + off, vst + (AL + nu) * Cf::v_slot + off,
                               v[nu]);
    }
    // idle threads must also see the slot free before their warp re-arms it
    if (!waited) ptx::mbar_wait(&empty[st], ((it / Cf::stages) & 1) ^ 1);
    if constexpr (PREC == kFP32) {
      ptx::mbar_wait(&tmaf[st], (it / Cf::stages) & 1);
      split_stage<PREC>(smem + st * Cf::stage_bytes, Cf::alpha * Cf::u_slot, tid, Cf::NT);
    }
    ptx::fence_async_smem();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&full[st]);
  }
}

template <int M, int PREC, int S>
__device__ __forceinline__ void transform_loop(const FusedParams& a, unsigned char* smem,
                                               uint64_t* full, uint64_t* empty, uint64_t* tmaf,
                                               int tid, int pb, int kb0, int kb1) {
  if (a.vec)
    transform_loop_v<M, PREC, S, true>(a, smem, full, empty, tmaf, tid, pb, kb0, kb1);
  else
    transform_loop_v<M, PREC, S, false>(a, smem, full, empty, tmaf, tid, pb, kb0, kb1);
}

template <int M, int PREC>
__device__ __forceinline__ void transform_dispatch(int s, const FusedParams& a, unsigned char* smem,
                                                   uint64_t* full, uint64_t* empty, uint64_t* tmaf,
                                                   int tid, int pb, int kb0, int kb1) {
  switch (s) {
    case 0: transform_loop<M, PREC, 0>(a, smem, full, empty, tmaf, tid, pb, kb0, kb1); break;
    case 1: transform_loop<M, PREC, 1>(a, smem, full, empty, tmaf, tid, pb, kb0, kb1); break;
    case 2: transform_loop<M, PREC, 2>(a, smem, full, empty, tmaf, tid, pb, kb0, kb1); break;
    case 3: transform_loop<M, PREC, 3>(a, smem, full, empty, tmaf, tid, pb, kb0, kb1); break;
    default:
      if constexpr (M == 4) {
        if (s == 4) transform_loop<M, PREC, 4>(a, smem, full, empty, tmaf, tid, pb, kb0, kb1);
        else transform_loop<M, PREC, 5>(a, smem, full, empty, tmaf, tid, pb, kb0, kb1);
      }
      break;
  }
}

// ------------------------------------------------------------------ kernel
// VT = false: V is formed in-kernel from d by the transform warps (fully fused).
// VT = true : V (written by the staged input transform into an L2-resident row
//             chunk) is TMA-loaded like U; the transform warps only run the
//             epilogue.  Either way M never leaves the chip.
template <int M, int PREC, bool VT>
__global__ void __launch_bounds__(FCfg<M, PREC>::threads, 1)
    wfused_kernel(const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmV,
                  const FusedParams a) {
  using Cf = FCfg<M, PREC>;
  using A = Alg<M>;
  constexpr int AL = Cf::alpha, Pb = Cf::Pb, STAGES = Cf::stages;

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cf::bar_off);
  uint64_t* empty = full + STAGES;
  uint64_t* accf = empty + STAGES;
  uint64_t* tmaf = accf + 1;  // [STAGES] 3xTF32: TMA bytes landed (split pending)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmaf + STAGES);
  constexpr bool SPLIT = (PREC == kFP32);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int s = static_cast<int>(ptx::cluster_ctarank());  // transform row xi owned here
  const int pb = blockIdx.x / AL;
  const int kblk = blockIdx.y;
  const int kb0 = blockIdx.z * a.kb_per_split;
  const int kb1 = min(a.num_kb, kb0 + a.kb_per_split);

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmU);
    if constexpr (VT) ptx::prefetch_tmap(&tmV);
    for (int i = 0; i < STAGES; ++i) {
      // TMA expect_tx (+ one arrive per transform warp when V is formed in-kernel)
      // 3xTF32: one arrive per transform warp once the hi/lo split is done
      ptx::mbar_init(&full[i], SPLIT ? Cf::NT / 32 : (VT ? 1 : 1 + Cf::NT / 32));
      ptx::mbar_init(&empty[i], 1);
      ptx::mbar_init(&tmaf[i], 1);
    }
    ptx::mbar_init(accf, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, Cf::tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch();
  griddep_wait();

  if (warp == 0) {
    // ---------------------------------------------------------- U producer
    if (lane == 0) {
      int it = 0;
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int st = it % STAGES;
        ptx::mbar_wait(&empty[st], ((it / STAGES) & 1) ^ 1);
        unsigned char* ust = smem + st * Cf::stage_bytes;
        // HBM holds one operand plane (3xTF32 lo planes are made on chip)
        uint64_t* tb = SPLIT ? &tmaf[st] : &full[st];
        ptx::mbar_arrive_expect_tx(tb, AL * (Cf::u_slot + (VT ? Cf::v_slot : 0)));
#pragma unroll
        for (int nu = 0; nu < AL; ++nu)
          ptx::tma_load_3d(ust + nu * Cf::u_slot, &tmU, tb, kb * Cf::bkc, kblk * Cf::Kb,
                           s * AL + nu);
        if constexpr (VT) {
#pragma unroll
          for (int nu = 0; nu < AL; ++nu)
            ptx::tma_load_3d(ust + Cf::u_bytes + nu * Cf::v_slot, &tmV, tb, kb * Cf::bkc, pb * Pb,
                             s * AL + nu);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc =
          ptx::umma_idesc(PREC == kBF16 ? 1u : (PREC == kFP16 ? 0u : 2u), Cf::Kb, Pb);
      int it = 0;
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int st = it % STAGES;
        ptx::mbar_wait(&full[st], (it / STAGES) & 1);
        ptx::tc_fence_after();
        const uint32_t ub = ptx::smem_u32(smem + st * Cf::stage_bytes);
        const uint32_t vb = ub + Cf::u_bytes;
#pragma unroll
        for (int nu = 0; nu < AL; ++nu) {
          const uint32_t dt = tmem_base + nu * Pb;
#pragma unroll
          for (int k = 0; k < Cf::bkc / Cf::uk; ++k) {
            const uint32_t off = k * 32;
            const uint32_t acc = (kb != kb0 || k != 0) ? 1u : 0u;
            const uint32_t a_hi = ub + nu * Cf::u_slot + off;
            const uint32_t b_hi = vb + nu * Cf::v_slot + off;
            if constexpr (Cf::nsplit == 2) {
              const uint32_t a_lo = a_hi + AL * Cf::u_slot;
              const uint32_t b_lo = b_hi + AL * Cf::v_slot;
              ptx::umma<1>(dt, ptx::umma_desc_sw<Cf::swz>(a_lo), ptx::umma_desc_sw<Cf::swz>(b_hi),
                           idesc, acc);
              ptx::umma<1>(dt, ptx::umma_desc_sw<Cf::swz>(a_hi), ptx::umma_desc_sw<Cf::swz>(b_lo),
                           idesc, 1u);
              ptx::umma<1>(dt, ptx::umma_desc_sw<Cf::swz>(a_hi), ptx::umma_desc_sw<Cf::swz>(b_hi),
                           idesc, 1u);
            } else {
              ptx::umma<Cf::kind>(dt, ptx::umma_desc_sw<Cf::swz>(a_hi),
                                  ptx::umma_desc_sw<Cf::swz>(b_hi), idesc, acc);
            }
          }
        }
        ptx::umma_commit(&empty[st]);
      }
      ptx::umma_commit(accf);
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------- transform
    if constexpr (!VT) {
      transform_dispatch<M, PREC>(s, a, smem, full, empty, tmaf, threadIdx.x - 64, pb, kb0, kb1);
    } else if constexpr (SPLIT) {  // staged V and U: only the on-chip hi/lo split
      const int tid = threadIdx.x - 64;
      int it = 0;
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int st = it % STAGES;
        ptx::mbar_wait(&tmaf[st], (it / STAGES) & 1);
        unsigned char* base = smem + st * Cf::stage_bytes;
        split_stage<PREC>(base, AL * Cf::u_slot, tid, Cf::NT);
        split_stage<PREC>(base + Cf::u_bytes, AL * Cf::v_slot, tid, Cf::NT);
        ptx::fence_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&full[st]);
      }
    }
  }

  // ============================================================ epilogue
  const bool epi = warp >= 2;
  if (epi) {
    ptx::mbar_wait(accf, 0);
    ptx::tc_fence_after();
  }
  // every CTA of the cluster has retired its MMAs (smem ring no longer read):
  // the ring can now receive Z rows from the other CTAs
  ptx::cluster_sync();
  float* xbuf = reinterpret_cast<float*>(smem);
  if (epi) {
    const int q = warp & 3;                // TMEM lane quarter this warp may read
    const int half = (warp - 2) >> 2;      // which half of the tile block
    const int f = q * 32 + lane;           // filter within the block (TMEM lane)
    const int o = f / Cf::fo;              // owner CTA of this filter
    const int fl = f - o * Cf::fo;
    const uint32_t rbase =
        ptx::mapa(ptx::smem_u32(xbuf + (s * Cf::fo + fl) * Cf::fls), static_cast<uint32_t>(o));
    constexpr int TH = Pb / 2;
#pragma unroll 1
    for (int t0 = half * TH; t0 < (half + 1) * TH; t0 += Cf::TT) {
      uint32_t r[AL][Cf::TT];
#pragma unroll
      for (int nu = 0; nu < AL; ++nu)
        ptx::tmem_ld_32x32b_x8(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + nu * Pb + t0,
                               r[nu]);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int tt = 0; tt < Cf::TT; ++tt) {
        float z[M];
#pragma unroll
        for (int j = 0; j < M; ++j) {
          float acc = 0.f;
          bool first = true;
#pragma unroll
          for (int nu = 0; nu < AL; ++nu) {
            const double c = A::AT(j, nu);
            acc = mac(acc, c, __uint_as_float(r[nu][tt]), first);
            if (c != 0.0) first = false;
          }
          z[j] = acc;
        }
        const uint32_t ra = rbase + (t0 + tt) * M * 4;
        if constexpr (M == 4)
          ptx::st_cluster_v4(ra, z[0], z[1], z[2], z[3]);
        else
          ptx::st_cluster_v2(ra, z[0], z[1]);
      }
    }
  }
  ptx::cluster_sync();
  if (epi) {
    // owner reduce: Y[i][j] = sum_src AT[i][src] Z_src[j], clipped store
    const int tid = threadIdx.x - 64;
    const int f_lo = s * Cf::fo;
    const int nf = min(Cf::fo, Cf::Kb - f_lo);
    const long long per_img = static_cast<long long>(a.th) * a.tw;
    float* yout = a.y + static_cast<long long>(blockIdx.z) * a.y_split_stride;
    for (int item = tid; item < nf * Pb; item += Cf::NT) {
      const int fl = item / Pb, t = item - (item / Pb) * Pb;
      const int k = kblk * Cf::Kb + f_lo + fl;
      const long long pl = static_cast<long long>(pb) * Pb + t;  // tile within the chunk
      if (k >= a.K || pl >= a.P) continue;
      const long long p = a.p0 + pl;
      float z[AL][M];
#pragma unroll
      for (int src = 0; src < AL; ++src) {
        const float* zp = xbuf + (src * Cf::fo + fl) * Cf::fls + t * M;
        if constexpr (M == 4) {
          const float4 q4 = *reinterpret_cast<const float4*>(zp);
          z[src][0] = q4.x; z[src][1] = q4.y; z[src][2] = q4.z; z[src][3] = q4.w;
        } else {
          const float2 q2 = *reinterpret_cast<const float2*>(zp);
          z[src][0] = q2.x; z[src][1] = q2.y;
        }
      }
      float yv[M][M];
#pragma unroll
      for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < M; ++j) {
          float acc = 0.f;
          bool first = true;
#pragma unroll
          for (int src = 0; src < AL; ++src) {
            const double c = A::AT(i, src);
            acc = mac(acc, c, z[src][j], first);
            if (c != 0.0) first = false;
          }
          yv[i][j] = acc;
        }
      const int n = static_cast<int>(p / per_img);
      const int rem = static_cast<int>(p - n * per_img);
      const int ty = rem / a.tw, tx = rem - (rem / a.tw) * a.tw;
      const int oy = M * ty, ox = M * tx;
      const int vr = min(M, a.oh - oy), vc = min(M, a.ow - ox);
      float* dst = yout + ((static_cast<long long>(n) * a.K + k) * a.oh + oy) * a.ow + ox;
      if (vc == M && (a.ow % M) == 0) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
          if (i < vr) {
            if constexpr (M == 4)
              *reinterpret_cast<float4*>(dst + i * a.ow) =
                  make_float4(yv[i][0], yv[i][1], yv[i][2], yv[i][3]);
            else
              *reinterpret_cast<float2*>(dst + i * a.ow) = make_float2(yv[i][0], yv[i][1]);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
          for (int j = 0; j < M; ++j)
            if (i < vr && j < vc) dst[i * a.ow + j] = yv[i][j];
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    ptx::tmem_dealloc(tmem_base, Cf::tmem_cols);
  }
}

// Sum of split-C partial outputs in ascending split order (deterministic).
// Slices are `stride` floats apart (a multiple of 4, so float4 loads stay aligned).
static __global__ void __launch_bounds__(256) split_sum_kernel(const float* __restrict__ part,
                                                        float* __restrict__ y, long long n,
                                                        long long stride, int splits) {
  griddep_launch();
  griddep_wait();
  const long long n4 = n / 4, s4 = stride / 4;
  const float4* p4 = reinterpret_cast<const float4*>(part);
  float4* y4 = reinterpret_cast<float4*>(y);
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += 256LL * gridDim.x) {
    float4 acc = __ldg(p4 + i);
    for (int s = 1; s < splits; ++s) {
      const float4 v = __ldg(p4 + s * s4 + i);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    y4[i] = acc;
  }
  for (long long i = n4 * 4 + blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) {
    float acc = part[i];
    for (int s = 1; s < splits; ++s) acc += part[s * stride + i];
    y[i] = acc;
  }
}

// ------------------------------------------------------------------ launch
template <int M, int PREC, bool VT>
static cudaError_t launch_fused_t(const FusedArgs& f, cudaStream_t s) {
  using Cf = FCfg<M, PREC>;
  alignas(64) CUtensorMap tmU, tmV;
  const uint64_t es = Cf::esize;
  const uint64_t planes = static_cast<uint64_t>(op_splits(PREC)) * Cf::a2;  // planes in HBM
  if (!encode_tmap_3d_sw(&tmU, PREC, f.U, f.C, f.K, planes, f.c_pad * es,
                         static_cast<uint64_t>(f.K) * f.c_pad * es, Cf::bkc, Cf::Kb, Cf::swz))
    return cudaErrorInvalidValue;
  if (VT) {  // V chunk [nsplit][a2][P][c_pad]: rows = tiles (B operand, K-major)
    if (!encode_tmap_3d_sw(&tmV, PREC, f.V, f.C, static_cast<uint64_t>(f.P), planes, f.c_pad * es,
                           static_cast<uint64_t>(f.P) * f.c_pad * es, Cf::bkc, Cf::Pb, Cf::swz))
      return cudaErrorInvalidValue;
  } else {
    tmV = tmU;  // unused
  }
  auto kern = wfused_kernel<M, PREC, VT>;
  static DeviceOnce configured;
  if (configured.first()) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::smem);
    if (e != cudaSuccess) return e;
    configured.done();
  }
  const int splits = f.splits < 1 ? 1 : f.splits;
  const int num_kb = (f.C + Cf::bkc - 1) / Cf::bkc;
  const int kbps = (num_kb + splits - 1) / splits;
  const long long n_pblk = (f.P + Cf::Pb - 1) / Cf::Pb;
  const int n_kblk = (f.K + Cf::Kb - 1) / Cf::Kb;
  if (n_pblk * Cf::alpha > 0x7fffffffLL || n_kblk > 65535 || splits > 65535)
    return cudaErrorInvalidValue;
  FusedParams a;
  a.d = static_cast<const float*>(f.d);
  a.P = f.P;
  a.N = f.N; a.C = f.C; a.H = f.H; a.W = f.W; a.K = f.K; a.pad = f.pad;
  a.th = f.th; a.tw = f.tw; a.oh = f.oh; a.ow = f.ow;
  a.num_kb = num_kb;
  a.kb_per_split = kbps;
  a.vec = (f.pad == 1 && f.W % M == 0) ? 1 : 0;
  a.p0 = f.p0;
  const long long ysz = static_cast<long long>(f.N) * f.K * f.oh * f.ow;
  a.y = static_cast<float*>(splits > 1 ? f.ypart : f.y);
  const long long ystride = (ysz + 3) / 4 * 4;
  a.y_split_stride = splits > 1 ? ystride : 0;

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(n_pblk * Cf::alpha), n_kblk, splits);
  cfg.blockDim = dim3(Cf::threads);
  cfg.dynamicSmemBytes = Cf::smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = Cf::alpha;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  static DeviceOnce reported;
  if (reported.first()) {
    reported.done();
    const char* dbg = getenv("WINO_DEBUG");
    if (dbg && dbg[0] == '1') {
      int ncl = -1;
      cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
      fprintf(stderr, "[wino] fused F(%d) prec %d vtma %d: cluster %d x %d threads, smem %d B, "
              "max active clusters %d\n", M, PREC, VT ? 1 : 0, Cf::alpha, Cf::threads, Cf::smem,
              ncl);
    }
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmU, tmV, a);
  if (e != cudaSuccess) return e;
  if (splits > 1) {
    const long long blocks = (ysz / 4 + 255) / 256;
    const int grid = static_cast<int>(blocks < 4 * 148 ? (blocks > 0 ? blocks : 1) : 4 * 148);
    e = launch_k(split_sum_kernel, dim3(grid), dim3(256), 0, s,
                 static_cast<const float*>(f.ypart), static_cast<float*>(f.y), ysz, ystride,
                 splits);
  }
  return e;
}

// Per-F(m) precision dispatch (instantiated in wino_fused_f2.cu / wino_fused_f4.cu).
template <int M, bool VT>
cudaError_t launch_fused_mv(int prec, const FusedArgs& f, cudaStream_t s) {
  switch (prec) {
    case kFP32: return launch_fused_t<M, kFP32, VT>(f, s);
    case kTF32: return launch_fused_t<M, kTF32, VT>(f, s);
    case kBF16: return launch_fused_t<M, kBF16, VT>(f, s);
    case kFP16: return launch_fused_t<M, kFP16, VT>(f, s);
    default: return cudaErrorInvalidValue;
  }
}
template <int M>
cudaError_t launch_fused_m(int prec, const FusedArgs& f, cudaStream_t s) {
  return f.V ? launch_fused_mv<M, true>(prec, f, s) : launch_fused_mv<M, false>(prec, f, s);
}

}  // namespace wino
