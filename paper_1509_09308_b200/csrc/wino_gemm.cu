// The alpha^2 independent transform-space GEMMs
//   M[comp][k][p] = sum_c U[comp][k][c] * V[comp][p][c]
// (reference: batched_matmul -> _bgemm, kernels.py:31-65; engine.py:239).
//
// sm_100a tensor-core kernel, persistent: each CTA strides through work units
// (one 128-tile x BN-filter block of one component, optionally one split of
// the channel reduction).  Warp-specialised:
//   warp 0   : TMA producer (one elected lane), STAGES-deep mbarrier ring
//   warp 1   : TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5: epilogue, tcgen05.ld TMEM -> registers -> coalesced fp32 stores
// TMEM holds two BN-column accumulators so the epilogue of one unit overlaps
// the MMAs of the next.
// Operands are K-major (channels contiguous) in the 128-byte-swizzle canonical
// layout the TMA box writes; the accumulator (128 lanes x BN fp32 columns)
// lives in TMEM.  The MMA M dimension runs over tiles P (so a warp's epilogue
// store covers 32 consecutive tiles = one 128 B line), N over filters K.
//
// Precisions: kind::f16 (bf16 / fp16 operands), kind::tf32 (single pass), and
// 3xTF32 (hi*hi + hi*lo + lo*hi into the same TMEM accumulator) which keeps the
// fp32 accuracy the reference's test tolerances assume (test_engine.py:97-112).
//
// FP64 (the reference's fp64 precision, test_engine.py:114-119) runs on a
// small CUDA-core tiled kernel: there is no fp64 tensor-core path worth using.
#include <cstdio>
#include <cstdlib>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "sm100_ptx.cuh"
#include "wino_internal.h"

namespace wino {

// Diagnostic timeline (WINO_GEMM_DBG bit 64; tools/gemm_trace.py): per CTA,
// globaltimer stamps 0 entry, 1 after griddepcontrol.wait, 2 first stage at the
// MMA warp, 3 last commit issued, 4 first accumulator at the epilogue, 5
// epilogue done, 6 exit, 7 first stage landed (3xTF32 split warp); slots 8-11
// accumulate the ns the producer waited on `empty`, the MMA warp on `full` /
// `sfull`, the MMA warp on `tempty`, and the first epilogue warp on `tfull`.
// Compiled in only with -DWINO_GEMM_TRACE (WINO_BUILD_TRACE=1 python -m
// paper_1509_09308_b200.build): even untaken trace branches in the MMA-issue
// loop measurably slow it (VGG-E N=1 0.381 -> 0.389 ms).
__device__ unsigned long long g_gemm_trace[1024][16];
#ifdef WINO_GEMM_TRACE
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_stamp(int dbg, int slot) {
  if ((dbg & 64) && blockIdx.x < 1024) g_gemm_trace[blockIdx.x][slot] = gtimer();
}
__device__ __forceinline__ void trace_add(int dbg, int slot, unsigned long long t0) {
  if ((dbg & 64) && blockIdx.x < 1024) g_gemm_trace[blockIdx.x][slot] += gtimer() - t0;
}
#define TRACE_T0 ((dbg & 64) ? gtimer() : 0ull)
#else
__device__ __forceinline__ void trace_stamp(int, int) {}
__device__ __forceinline__ void trace_add(int, int, unsigned long long) {}
#define TRACE_T0 0ull
#endif

// warp 0 producer, warp 1 MMA, then the epilogue warps (4 for 3xTF32, whose
// 8 split warps follow them; 8 otherwise: two per TMEM lane quarter, each
// draining every other 32-column chunk -- the 16-bit GEMMs at large P were
// epilogue-bound with 4: the MMA warp spent its time waiting on tempty)
constexpr int kSplitWarps = 8;
template <int PREC>
__host__ __device__ constexpr int gemm_epi_warps() { return PREC == kFP32 ? 4 : 8; }
template <int PREC>
constexpr int gemm_threads() {
  return PREC == kFP32 ? 64 + 32 * (4 + kSplitWarps) : 64 + 32 * gemm_epi_warps<PREC>();
}
constexpr int kTileP = 128;        // UMMA M (tiles per CTA)

template <int PREC>
struct GemmTraits {
  static constexpr int kind = (PREC == kFP32 || PREC == kTF32) ? 1 : 0;  // 1 = tf32
  static constexpr int esize = kind ? 4 : 2;
  static constexpr int bk = 128 / esize;     // channels per stage (one 128 B swizzle row)
  static constexpr int uk = 32 / esize;      // channels per tcgen05.mma
  static constexpr int nsplit = (PREC == kFP32) ? 2 : 1;  // smem planes (HBM holds one)
  static constexpr uint32_t fmt = (PREC == kBF16) ? 1u : (PREC == kFP16 ? 0u : 2u);
};

constexpr int kEpiWarps = 4;
constexpr int kEpiBuf = 32 * 32 * 4;  // one 32-tile x 32-filter fp32 block

// TA: 3xTF32 with the A operand (V, 128 tiles) split straight into tensor
// memory -- smem holds one A plane and the B hi/lo planes, and the MMAs read A
// from TMEM, which takes the A traffic off the shared-memory port the split and
// the MMAs otherwise saturate.
template <int PREC, int BN, bool TA = false>
struct GemmSmem {
  using Tr = GemmTraits<PREC>;
  static constexpr int a_bytes = kTileP * 128;  // 128 rows x 128 B
  static constexpr int b_bytes = BN * 128;
  static constexpr int stage_bytes = TA ? a_bytes + 2 * b_bytes : Tr::nsplit * (a_bytes + b_bytes);
  static constexpr int epi_bytes = kEpiWarps * 2 * kEpiBuf;  // double-buffered per warp
  static constexpr int avail = 227 * 1024 - 1024 - 512 - epi_bytes;
  static constexpr int stages = avail / stage_bytes >= 6 ? 6 : avail / stage_bytes;
  static constexpr int epi_offset = stages * stage_bytes;
  static constexpr int bar_offset = epi_offset + epi_bytes;
  static constexpr int total = bar_offset + 512 + 1024;  // barriers + alignment slack
  // TMEM: two BN-column accumulators (+ hi/lo A columns per stage for TA)
  static constexpr int tmem_cols = TA ? 512 : 2 * BN;
  static constexpr int a_tmem_col = 2 * BN;             // stage s: hi at +64 s, lo at +64 s + 32
  static_assert(!TA || 2 * BN + 64 * stages <= 512, "TMEM budget");
};

// 3xTF32 split of `n` 16-byte chunks at shared address `hi` (lo plane `lo_off`
// bytes further) by the kSplitWarps split warps: batches of four loads in
// flight per thread, single chunks for the tail.
template <int NTS = 32 * kSplitWarps>
__device__ __forceinline__ void split_region_n(uint32_t hi, int n, int lo_off, int tid) {
  int base = 0;
  for (; base + 4 * NTS <= n; base += 4 * NTS) {
    const int i = base + tid;
    const uint32_t h[4] = {hi + 16 * i, hi + 16 * (i + NTS), hi + 16 * (i + 2 * NTS),
                           hi + 16 * (i + 3 * NTS)};
    const uint32_t l[4] = {h[0] + lo_off, h[1] + lo_off, h[2] + lo_off, h[3] + lo_off};
    ptx::split_tf32_chunk4_s(h, l);
  }
  for (int i = base + tid; i < n; i += NTS) ptx::split_tf32_chunk_s(hi + 16 * i, hi + 16 * i + lo_off);
}
__device__ __forceinline__ void split_region(uint32_t hi, int n, int lo_off, int tid) {
  split_region_n<>(hi, n, lo_off, tid);
}

// Persistent, warp-specialised tcgen05 GEMM.  Work unit = (split, comp,
// filter block, tile block); CTAs stride through units.  The accumulator is
// double-buffered in TMEM (2 x BN columns) so the epilogue of unit j overlaps
// the MMAs of unit j+1.  Split-C units (small-P layers) write partial sums to
// separate M slices that the output transform adds in a fixed order.
// MB: store M in 16 bits (bf16 for the bf16 GEMM, fp16 x 2^-kM16Shift for the
// fp16 GEMM: the staged M of the 16-bit plans, wino_api.cu planner).
// BS (with TA): U arrives as hi / lo planes (filter transform split2), so the
// B operand needs no on-chip split; TMA loads both planes into the stage.
// TRN (3xTF32, K > P layers): roles swapped -- A (M side, split into TMEM) is
// the filter block U[comp][128 filters][c], B (N side) a BN-tile block of V, so
// a 49-tile layer runs 128 x 64 MMAs instead of 128 x 128 with 79 empty rows;
// the epilogue writes the transposed TMEM tile into the same M[z][k][p] layout
// through a 128B-swizzled staging box.
template <int PREC, int BN, bool TA, bool MB, bool BS = false, bool TRN = false>
__global__ void __launch_bounds__(gemm_threads<PREC>(), 1)
    wgemm_tc_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmU,
                    const __grid_constant__ CUtensorMap tmM, int a2, int num_kb,
                    int kb_per_split, int n_pblk, int n_kblk, int n_units, int dbg) {
  using Tr = GemmTraits<PREC>;
  using Sm = GemmSmem<PREC, BN, TA>;
  static_assert(!TA || PREC == kFP32, "TMEM A operand is the 3xTF32 variant");
  constexpr int STAGES = Sm::stages;
  static_assert(STAGES >= 2, "pipeline needs at least two stages");
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Sm::bar_offset);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;       // [2] accumulator drained
  uint64_t* sfull = tempty + 2;       // [STAGES] 3xTF32: hi/lo split of the stage done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfull + STAGES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    trace_stamp(dbg, 0);
#ifdef WINO_GEMM_TRACE
    if ((dbg & 64) && blockIdx.x < 1024)
      for (int i = 8; i < 16; ++i) g_gemm_trace[blockIdx.x][i] = 0;
#endif
    ptx::prefetch_tmap(&tmV);
    ptx::prefetch_tmap(&tmU);
    ptx::prefetch_tmap(&tmM);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 32 * gemm_epi_warps<PREC>());
    }
    for (int s = 0; s < STAGES; ++s) ptx::mbar_init(&sfull[s], kSplitWarps);  // one per split warp
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, Sm::tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue above overlaps the predecessor (PDL); operands are read below
  griddep_launch();
  griddep_wait();
  if (warp == 0 && lane == 0) trace_stamp(dbg, 1);

  auto decode = [&](int u, int& pb, int& kbk, int& comp, int& split) {
    pb = u % n_pblk;
    int r = u / n_pblk;
    kbk = r % n_kblk;
    r /= n_kblk;
    comp = r % a2;
    split = r / a2;
  };
  // The CTA's units are u = blockIdx.x + i * gridDim.x; step the mixed-radix
  // (pb, kbk, comp, split) coordinates by the decoded stride instead of three
  // integer divisions per unit (the single MMA-issuing thread and the
  // producer are latency-bound on them at one k-block per unit, C <= 64).
  int st_pb, st_kb, st_c, st_s;
  decode(static_cast<int>(gridDim.x), st_pb, st_kb, st_c, st_s);
  auto advance = [&](int& pb, int& kbk, int& comp, int& split) {
    pb += st_pb;
    int c = pb >= n_pblk;
    pb -= c ? n_pblk : 0;
    kbk += st_kb + c;
    c = kbk >= n_kblk;
    kbk -= c ? n_kblk : 0;
    comp += st_c + c;
    c = comp >= a2;
    comp -= c ? a2 : 0;
    split += st_s + c;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int it = 0;
      int pb, kbk, comp, split;
      decode(blockIdx.x, pb, kbk, comp, split);
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, advance(pb, kbk, comp, split)) {
        const int kb0 = split * kb_per_split;
        const int kb1 = min(num_kb, kb0 + kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          const unsigned long long te0 = TRACE_T0;
          ptx::mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          trace_add(dbg, 8, te0);
          unsigned char* st = smem + s * Sm::stage_bytes;
          // HBM holds one plane; 3xTF32's lo planes are produced on chip
          if (dbg & 2) { ptx::mbar_arrive(&full[s]); continue; }
          ptx::mbar_arrive_expect_tx(&full[s], Sm::a_bytes + (BS ? 2 : 1) * Sm::b_bytes);
          ptx::tma_load_3d(st, &tmV, &full[s], kb * Tr::bk, pb * kTileP, comp);
          ptx::tma_load_3d(st + (TA ? 1 : Tr::nsplit) * Sm::a_bytes, &tmU, &full[s], kb * Tr::bk, kbk * BN,
                           comp);
          if constexpr (BS)  // lo plane of U right after the hi tile
            ptx::tma_load_3d(st + Sm::a_bytes + Sm::b_bytes, &tmU, &full[s], kb * Tr::bk,
                             kbk * BN, a2 + comp);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::umma_idesc(Tr::fmt, kTileP, BN);
      // descriptor of smem byte offset x = dbase + (x >> 4): the 14-bit start
      // field cannot carry (shared window < 256 KB), so per-MMA descriptors are
      // one 64-bit add instead of a shift / mask / or chain each
      const uint64_t dbase = ptx::umma_desc_sw128(ptx::smem_u32(smem));
      int it = 0, j = 0;
      int pb, kbk, comp, split;
      decode(blockIdx.x, pb, kbk, comp, split);
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++j, advance(pb, kbk, comp, split)) {
        const int kb0 = split * kb_per_split;
        const int kb1 = min(num_kb, kb0 + kb_per_split);
        const int acc = j & 1;
        const unsigned long long tt0 = TRACE_T0;
        ptx::mbar_wait(&tempty[acc], ((j >> 1) & 1) ^ 1);
        trace_add(dbg, 10, tt0);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          const unsigned long long tf0 = TRACE_T0;
          if constexpr (Tr::nsplit == 2)
            ptx::mbar_wait(&sfull[s], (it / STAGES) & 1);
          else
            ptx::mbar_wait(&full[s], (it / STAGES) & 1);
          trace_add(dbg, 9, tf0);
          if (it == 0) trace_stamp(dbg, 2);
          ptx::tc_fence_after();
          // stage descriptors: base + compile-time offsets (>> 4 of 16-B multiples)
          const uint64_t dst = dbase + static_cast<uint32_t>((s * Sm::stage_bytes) >> 4);
          constexpr uint32_t kAlo = Sm::a_bytes >> 4;
          constexpr uint32_t kBhi = ((TA ? 1 : Tr::nsplit) * Sm::a_bytes) >> 4;
          constexpr uint32_t kBlo = kBhi + (Sm::b_bytes >> 4);
          const uint32_t ta_hi = tmem_base + Sm::a_tmem_col + 64 * s, ta_lo = ta_hi + 32;
#pragma unroll
          for (int k = 0; k < Tr::bk / Tr::uk; ++k) {
            if (dbg & 8) break;
            const uint32_t off = k * 2;  // 32 bytes of K per MMA inside the swizzle atom (>> 4)
            const uint32_t accum = (kb != kb0 || k != 0) ? 1u : 0u;
            if constexpr (TA) {  // A (8 tf32 columns per MMA) from tensor memory
              ptx::umma_tf32_tmem_a(d_tmem, ta_lo + 8 * k, dst + (kBhi + off), idesc, accum);
              ptx::umma_tf32_tmem_a(d_tmem, ta_hi + 8 * k, dst + (kBlo + off), idesc, 1u);
              ptx::umma_tf32_tmem_a(d_tmem, ta_hi + 8 * k, dst + (kBhi + off), idesc, 1u);
            } else if constexpr (Tr::nsplit == 2) {
              ptx::umma<1>(d_tmem, dst + (kAlo + off), dst + (kBhi + off), idesc, accum);
              ptx::umma<1>(d_tmem, dst + off, dst + (kBlo + off), idesc, 1u);
              ptx::umma<1>(d_tmem, dst + off, dst + (kBhi + off), idesc, 1u);
            } else {
              ptx::umma<Tr::kind>(d_tmem, dst + off, dst + (kBhi + off), idesc, accum);
            }
          }
          ptx::umma_commit(&empty[s]);  // frees the smem slot when these MMAs retire
        }
        ptx::umma_commit(&tfull[acc]);  // accumulator complete
      }
      trace_stamp(dbg, 3);
    }
  } else if (PREC == kFP32 && warp >= 6) {
    // ------------------------------------------------------------ 3xTF32 split
    // (warps 6.. exist only for PREC == kFP32) hi = rna_tf32(x) in place,
    // lo = x - hi into the stage's lo planes, then release the stage to MMA.
    if constexpr (Tr::nsplit == 2) {
      const int tid = threadIdx.x - 192;
      int it = 0;
      int pb, kbk, comp, split;
      decode(blockIdx.x, pb, kbk, comp, split);
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, advance(pb, kbk, comp, split)) {
        const int kb0 = split * kb_per_split;
        const int kb1 = min(num_kb, kb0 + kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          ptx::mbar_wait(&full[s], (it / STAGES) & 1);
          if (it == 0 && warp == 6 && lane == 0) trace_stamp(dbg, 7);
          const uint32_t st = ptx::smem_u32(smem + s * Sm::stage_bytes);
          if constexpr (TA) {
            if (warp < 6 + 4 && !(dbg & 32)) {
              // A: thread = tile row r of its warp's TMEM lane quarter; the
              // 128-byte row (32 channels, 128B-swizzled) -> hi / lo columns
              const int q = warp & 3, r = 32 * q + lane;
              const uint32_t row = st + 128 * r;
              uint32_t hi[32], lo[32];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                float x0, x1, x2, x3;
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(x0), "=f"(x1), "=f"(x2), "=f"(x3)
                             : "r"(row + 16 * (j ^ (r & 7))));
                const float xs[4] = {x0, x1, x2, x3};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  uint32_t h;
                  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(xs[e]));
                  hi[4 * j + e] = h;
                  lo[4 * j + e] = __float_as_uint(xs[e] - __uint_as_float(h));
                }
              }
              const uint32_t t0 = tmem_base + (static_cast<uint32_t>(32 * q) << 16) +
                                  Sm::a_tmem_col + 64 * s;
              ptx::tmem_st_32x32b_x32(t0, hi);
              ptx::tmem_st_32x32b_x32(t0 + 32, lo);
              ptx::tmem_st_wait();
              ptx::tc_fence_before();
            } else if (!BS && warp >= 6 + 4 && !(dbg & 4)) {  // B: hi in place, lo plane, by the other 4 warps
              split_region_n<128>(st + Sm::a_bytes, Sm::b_bytes / 16, Sm::b_bytes, tid - 128);
            }
          } else if (!(dbg & 4)) {
            split_region(st, Sm::a_bytes / 16, Sm::a_bytes, tid);
            split_region(st + 2 * Sm::a_bytes, Sm::b_bytes / 16, Sm::b_bytes, tid);
          }
          ptx::fence_async_smem();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&sfull[s]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // TMEM -> registers -> smem [32 filters][32 tiles] -> TMA bulk store into
    // M[split*a2 + comp][k][p]; the tensor map clips tiles >= Pc / filters >= K.
    // The next 32-column TMEM load is in flight while the current one is
    // written to shared memory (two register sets, fully unrolled), and the
    // accumulator is released as soon as its last column is in registers.
    constexpr int NE = gemm_epi_warps<PREC>();
    constexpr int NH = NE / 4;   // epilogue warps per TMEM lane quarter
    constexpr int NB = 2 / NH;   // smem staging buffers per warp (32 KB in all)
    const int ew = warp - 2;     // epilogue warps are 2 .. 2+NE-1
    const int q = warp & 3;      // TMEM lane quarter this warp may access
    const int half = ew >> 2;    // this warp drains chunks ci = half, half+NH, ...
    float* buf0 = reinterpret_cast<float*>(smem + Sm::epi_offset + ew * NB * kEpiBuf);
    const uint32_t sbuf0 = ptx::smem_u32(buf0) + 4 * lane;
    int j = 0, nbuf = 0;
    int pb, kbk, comp, split;
    decode(blockIdx.x, pb, kbk, comp, split);
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++j, advance(pb, kbk, comp, split)) {
      const int acc = j & 1;
      const unsigned long long tw0 = TRACE_T0;
      ptx::mbar_wait(&tfull[acc], (j >> 1) & 1);
      if (ew == 0 && lane == 0) {
        trace_add(dbg, 11, tw0);
        if (j == 0) trace_stamp(dbg, 4);
      }
      ptx::tc_fence_after();
      const int p0 = pb * kTileP + q * 32;
      const int z = split * a2 + comp;
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      constexpr int NC = BN / 32;
      uint32_t r[2][32];
      if (half < NC) ptx::tmem_ld_32x32b_x32(taddr + 32 * half, r[0]);
#pragma unroll
      for (int c = 0; c < (NC + NH - 1) / NH; ++c) {
        const int ci = half + NH * c;
        if (ci >= NC) break;
        ptx::tmem_ld_wait();  // chunk ci in registers
        if (ci + NH < NC) {
          ptx::tmem_ld_32x32b_x32(taddr + 32 * (ci + NH), r[(c + 1) & 1]);
        } else {
          ptx::tc_fence_before();
          ptx::mbar_arrive(&tempty[acc]);  // this warp's columns drained to registers
        }
        if (dbg & 1) continue;
        const int b = NB == 2 ? (nbuf++ & 1) : 0;
        if (lane == 0) ptx::bulk_wait_read<NB - 1>();  // the store that last used buffer b has read it
        __syncwarp();
        const uint32_t sb = sbuf0 + b * kEpiBuf;
        if constexpr (TRN) {  // thread = filter row, r[jj] = tile jj: swizzled 128-B rows
          const uint32_t rowb = sb - 4 * lane + 128 * lane;  // sbuf0 carries 4*lane
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowb + ((c4 ^ (lane & 7)) << 4)),
                         "r"(r[c & 1][4 * c4]), "r"(r[c & 1][4 * c4 + 1]), "r"(r[c & 1][4 * c4 + 2]),
                         "r"(r[c & 1][4 * c4 + 3])
                         : "memory");
        } else if constexpr (MB) {  // [32 filters][32 tiles] bf16, or fp16 x 2^-kM16Shift
          const uint32_t sh = sb - 2 * lane;  // sbuf0 carries 4*lane
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            unsigned short h;
            if constexpr (PREC == kFP16)
              h = __half_as_ushort(__float2half_rn(__uint_as_float(r[c & 1][jj]) *
                                                   (1.0f / (1 << kM16Shift))));
            else
              h = __bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(r[c & 1][jj])));
            asm volatile("st.shared.b16 [%0], %1;" ::"r"(sh + jj * 64), "h"(h) : "memory");
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj)
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(sb + jj * 128), "r"(r[c & 1][jj]) : "memory");
        }
        ptx::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          if constexpr (TRN)  // (tile, filter) = (column block, TMEM lane block)
            ptx::tma_store_3d(&tmM, buf0 + b * (kEpiBuf / 4), kbk * BN + 32 * ci, p0, z);
          else
            ptx::tma_store_3d(&tmM, buf0 + b * (kEpiBuf / 4), p0, kbk * BN + 32 * ci, z);
          ptx::bulk_commit();
        }
      }
      if (half >= NC) {  // BN = 32 with two warps per quarter: nothing to drain
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
      }
    }
    if (lane == 0) ptx::bulk_wait_read<0>();  // smem read; the writes drain before grid completion
    if (ew == 0 && lane == 0) trace_stamp(dbg, 5);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    ptx::tmem_dealloc(tmem_base, Sm::tmem_cols);
    if (lane == 0) trace_stamp(dbg, 6);
  }
}

// ------------------------------------------------------------ CTA-pair 3xTF32
// cta_group::2 variant of the TMEM-A 3xTF32 GEMM: a cluster of two CTAs on one
// TPC computes a 256-tile x BN-filter block per unit.  Each CTA stages its own
// 128 tile rows (A, split into its own TMEM) and HALF of the filter block (B),
// so each SM's shared memory carries half the B bytes, half the B split and
// half the MMA's B reads of the single-CTA kernel.  The leader CTA issues
// tcgen05.mma.cta_group::2 (M = 256); D rows 0-127 land in the leader's TMEM,
// 128-255 in the peer's.  Synchronisation: each CTA waits on its own full
// barrier; both CTAs' split warps arrive on the leader's sfull; the leader's
// commits multicast to both CTAs' empty / tfull; both epilogues arrive on the
// leader's tempty.
template <int BN, bool BS>
__global__ void __launch_bounds__(gemm_threads<kFP32>(), 1)
    wgemm_tc2_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmU,
                     const __grid_constant__ CUtensorMap tmM, int a2, int num_kb,
                     int kb_per_split, int n_ppblk, int n_kblk, int n_units) {
  using Tr = GemmTraits<kFP32>;
  constexpr int HB = BN / 2;                 // filters staged per CTA
  constexpr int a_bytes = kTileP * 128;
  constexpr int b_bytes = HB * 128;
  constexpr int stage_bytes = a_bytes + 2 * b_bytes;
  constexpr int epi_bytes = kEpiWarps * 2 * kEpiBuf;
  constexpr int avail = 227 * 1024 - 1024 - 512 - epi_bytes;
  constexpr int STAGES = avail / stage_bytes >= 4 ? 4 : avail / stage_bytes;
  static_assert(2 * BN + 64 * STAGES <= 512, "TMEM budget");
  constexpr int epi_offset = STAGES * stage_bytes;
  constexpr int bar_offset = epi_offset + epi_bytes;
  constexpr int a_tmem_col = 2 * BN;

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + bar_offset);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfull + STAGES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmV);
    ptx::prefetch_tmap(&tmU);
    ptx::prefetch_tmap(&tmM);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
      ptx::mbar_init(&sfull[s], 2 * kSplitWarps);  // both CTAs' split warps (leader's copy used)
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 256);  // both CTAs' epilogue threads (leader's copy used)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     ptx::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch();
  griddep_wait();

  auto decode = [&](int u, int& pp, int& kbk, int& comp, int& split) {
    pp = u % n_ppblk;
    int r = u / n_ppblk;
    kbk = r % n_kblk;
    r /= n_kblk;
    comp = r % a2;
    split = r / a2;
  };
  const uint32_t mask2 = 3u;

  if (warp == 0) {
    if (lane == 0) {  // ---- producer: own A rows, own half of B
      int it = 0;
      for (int u = cid; u < n_units; u += ncl) {
        int pp, kbk, comp, split;
        decode(u, pp, kbk, comp, split);
        const int kb0 = split * kb_per_split;
        const int kb1 = min(num_kb, kb0 + kb_per_split);
        const int prow = (2 * pp + static_cast<int>(rank)) * kTileP;
        const int frow = kbk * BN + static_cast<int>(rank) * HB;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          ptx::mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          unsigned char* st = smem + s * stage_bytes;
          ptx::mbar_arrive_expect_tx(&full[s], a_bytes + (BS ? 2 : 1) * b_bytes);
          ptx::tma_load_3d(st, &tmV, &full[s], kb * Tr::bk, prow, comp);
          ptx::tma_load_3d(st + a_bytes, &tmU, &full[s], kb * Tr::bk, frow, comp);
          if constexpr (BS)
            ptx::tma_load_3d(st + a_bytes + b_bytes, &tmU, &full[s], kb * Tr::bk, frow, a2 + comp);
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ---- MMA issuer (leader only), M = 256
      constexpr uint32_t idesc = ptx::umma_idesc(Tr::fmt, 2 * kTileP, BN);
      int it = 0, j = 0;
      for (int u = cid; u < n_units; u += ncl, ++j) {
        int pp, kbk, comp, split;
        decode(u, pp, kbk, comp, split);
        const int kb0 = split * kb_per_split;
        const int kb1 = min(num_kb, kb0 + kb_per_split);
        const int acc = j & 1;
        ptx::mbar_wait(&tempty[acc], ((j >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          ptx::mbar_wait(&sfull[s], (it / STAGES) & 1);
          ptx::tc_fence_after();
          const uint32_t st = ptx::smem_u32(smem + s * stage_bytes);
          const uint32_t b_hi = st + a_bytes, b_lo = b_hi + b_bytes;
          const uint32_t ta_hi = tmem_base + a_tmem_col + 64 * s, ta_lo = ta_hi + 32;
#pragma unroll
          for (int k = 0; k < Tr::bk / Tr::uk; ++k) {
            const uint32_t off = k * 32;
            const uint32_t accum = (kb != kb0 || k != 0) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
                "r"(ta_lo + 8 * k), "l"(ptx::umma_desc_sw128(b_hi + off)), "r"(idesc), "r"(accum));
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
                "r"(ta_hi + 8 * k), "l"(ptx::umma_desc_sw128(b_lo + off)), "r"(idesc), "r"(1u));
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
                "r"(ta_hi + 8 * k), "l"(ptx::umma_desc_sw128(b_hi + off)), "r"(idesc), "r"(1u));
          }
          asm volatile(  // frees stage s in both CTAs
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  ptx::smem_u32(&empty[s])),
              "h"(static_cast<unsigned short>(mask2))
              : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                ptx::smem_u32(&tfull[acc])),
            "h"(static_cast<unsigned short>(mask2))
            : "memory");
      }
    }
  } else if (warp >= 6) {  // ---- split warps: A rows -> own TMEM, own B half in smem
    const int tid = threadIdx.x - 192;
    const uint32_t sfull_leader = ptx::mapa(ptx::smem_u32(sfull), 0);
    int it = 0;
    for (int u = cid; u < n_units; u += ncl) {
      int pp, kbk, comp, split;
      decode(u, pp, kbk, comp, split);
      const int kb0 = split * kb_per_split;
      const int kb1 = min(num_kb, kb0 + kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % STAGES;
        ptx::mbar_wait(&full[s], (it / STAGES) & 1);
        const uint32_t st = ptx::smem_u32(smem + s * stage_bytes);
        if (warp < 6 + 4) {
          const int q = warp & 3, r = 32 * q + lane;
          const uint32_t row = st + 128 * r;
          uint32_t hi[32], lo[32];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            float x0, x1, x2, x3;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(x0), "=f"(x1), "=f"(x2), "=f"(x3)
                         : "r"(row + 16 * (jj ^ (r & 7))));
            const float xs[4] = {x0, x1, x2, x3};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              uint32_t h;
              asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(xs[e]));
              hi[4 * jj + e] = h;
              lo[4 * jj + e] = __float_as_uint(xs[e] - __uint_as_float(h));
            }
          }
          const uint32_t t0 =
              tmem_base + (static_cast<uint32_t>(32 * q) << 16) + a_tmem_col + 64 * s;
          ptx::tmem_st_32x32b_x32(t0, hi);
          ptx::tmem_st_32x32b_x32(t0 + 32, lo);
          ptx::tmem_st_wait();
          ptx::tc_fence_before();
        } else if (!BS) {
          split_region_n<128>(st + a_bytes, b_bytes / 16, b_bytes, tid - 128);
        }
        ptx::fence_async_smem();
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                           sfull_leader + 8 * s)
                       : "memory");
      }
    }
  } else {  // ---- epilogue: own TMEM rows = own 128 tiles
    const int q = warp & 3;
    float* buf0 = reinterpret_cast<float*>(smem + epi_offset + (warp - 2) * 2 * kEpiBuf);
    const uint32_t sbuf0 = ptx::smem_u32(buf0) + 4 * lane;
    const uint32_t tempty_leader = ptx::mapa(ptx::smem_u32(tempty), 0);
    int j = 0, nbuf = 0;
    for (int u = cid; u < n_units; u += ncl, ++j) {
      int pp, kbk, comp, split;
      decode(u, pp, kbk, comp, split);
      const int acc = j & 1;
      ptx::mbar_wait(&tfull[acc], (j >> 1) & 1);
      ptx::tc_fence_after();
      const int p0 = (2 * pp + static_cast<int>(rank)) * kTileP + q * 32;
      const int z = split * a2 + comp;
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      constexpr int NC = BN / 32;
      uint32_t r[2][32];
      ptx::tmem_ld_32x32b_x32(taddr, r[0]);
#pragma unroll
      for (int ci = 0; ci < NC; ++ci) {
        ptx::tmem_ld_wait();
        if (ci + 1 < NC) {
          ptx::tmem_ld_32x32b_x32(taddr + 32 * (ci + 1), r[(ci + 1) & 1]);
        } else {
          ptx::tc_fence_before();
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                           tempty_leader + 8 * acc)
                       : "memory");
        }
        const int b = nbuf++ & 1;
        if (lane == 0) ptx::bulk_wait_read<1>();
        __syncwarp();
        const uint32_t sb = sbuf0 + b * kEpiBuf;
#pragma unroll
        for (int jj = 0; jj < 32; ++jj)
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(sb + jj * 128), "r"(r[ci & 1][jj]) : "memory");
        ptx::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          ptx::tma_store_3d(&tmM, buf0 + b * (kEpiBuf / 4), p0, kbk * BN + 32 * ci, z);
          ptx::bulk_commit();
        }
      }
    }
    if (lane == 0) ptx::bulk_wait_all();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

static int num_sms();

template <int BN, bool BS>
static cudaError_t launch_tc2(const GemmArgs& a, cudaStream_t s) {
  using Tr = GemmTraits<kFP32>;
  constexpr int HB = BN / 2;
  constexpr int stage_bytes = kTileP * 128 + 2 * HB * 128;
  constexpr int epi_bytes = kEpiWarps * 2 * kEpiBuf;
  constexpr int avail = 227 * 1024 - 1024 - 512 - epi_bytes;
  constexpr int STAGES = avail / stage_bytes >= 4 ? 4 : avail / stage_bytes;
  constexpr int total = STAGES * stage_bytes + epi_bytes + 512 + 1024;
  alignas(64) CUtensorMap tmV, tmU, tmM;
  const uint64_t es = 4;
  const uint64_t planes = static_cast<uint64_t>(a.a2);
  if (!encode_tmap_3d(&tmV, kFP32, a.V, a.C, a.Pc, planes, a.c_pad * es, a.Pc * a.c_pad * es,
                      Tr::bk, kTileP))
    return cudaErrorInvalidValue;
  if (!encode_tmap_3d(&tmU, kFP32, a.U, a.C, a.K, BS ? 2 * planes : planes, a.c_pad * es,
                      static_cast<uint64_t>(a.K) * a.c_pad * es, Tr::bk, HB))
    return cudaErrorInvalidValue;
  const int splits = a.splits < 1 ? 1 : a.splits;
  if (!encode_tmap_3d(&tmM, -1, a.M, a.Pc, a.K, static_cast<uint64_t>(splits) * a.a2, a.m_ld * 4ull,
                      static_cast<uint64_t>(a.K) * a.m_ld * 4ull, 32, 32))
    return cudaErrorInvalidValue;
  auto kern = wgemm_tc2_kernel<BN, BS>;
  static DeviceOnce configured;
  if (configured.first()) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, total);
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    configured.done();
  }
  const int num_kb = (a.C + Tr::bk - 1) / Tr::bk;
  const int kbps = (num_kb + splits - 1) / splits;
  const int n_ppblk = static_cast<int>((a.Pc + 2 * kTileP - 1) / (2 * kTileP));
  const int n_kblk = (a.K + BN - 1) / BN;
  const long long units = static_cast<long long>(n_ppblk) * n_kblk * a.a2 * splits;
  if (units > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int clusters = static_cast<int>(units < num_sms() / 2 ? units : num_sms() / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(gemm_threads<kFP32>());
  cfg.dynamicSmemBytes = total;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmV, tmU, tmM, a.a2, num_kb, kbps, n_ppblk,
                                     n_kblk, static_cast<int>(units));
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// ------------------------------------------------------------ fp64 CUDA-core
// 64 x 64 output block, 16-channel smem slices, c-ascending accumulation
// (deterministic, same reduction order as kernels.py:43-47).
__global__ void __launch_bounds__(256) wgemm_f64_kernel(const double* __restrict__ V,
                                                        const double* __restrict__ U,
                                                        double* __restrict__ Mout, int K,
                                                        long long Pc, int C, int c_pad,
                                                        long long m_ld) {
  __shared__ double sv[16][65];
  __shared__ double su[16][65];
  const int comp = blockIdx.z;
  const long long p0 = static_cast<long long>(blockIdx.x) * 64;
  const int k0 = blockIdx.y * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 each
  const double* Vc = V + static_cast<size_t>(comp) * Pc * c_pad;
  const double* Uc = U + static_cast<size_t>(comp) * K * c_pad;
  double acc[4][4] = {};
  griddep_launch();
  griddep_wait();
  for (int cb = 0; cb < C; cb += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int r = e / 16, cc = e % 16;
      const int c = cb + cc;
      const long long p = p0 + r;
      const int k = k0 + r;
      sv[cc][r] = (c < C && p < Pc) ? Vc[static_cast<size_t>(p) * c_pad + c] : 0.0;
      su[cc][r] = (c < C && k < K) ? Uc[static_cast<size_t>(k) * c_pad + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = su[cc][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sv[cc][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* Mc = Mout + static_cast<size_t>(comp) * K * m_ld;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + ty * 4 + i;
    if (k >= K) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long p = p0 + tx * 4 + j;
      if (p < Pc) Mc[static_cast<size_t>(k) * m_ld + p] = acc[i][j];
    }
  }
}

// ------------------------------------------------------------ launch
static int num_sms() { return device_sms(); }

int device_sms() {
  static std::atomic<int> cache[64];  // per device; benign race (idempotent)
  const int b = DeviceOnce::bit();
  int n = cache[b].load(std::memory_order_relaxed);
  if (n == 0) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n = v > 0 ? v : 148;
    cache[b].store(n, std::memory_order_relaxed);
  }
  return n;
}

static int gemm_dbg() {  // diagnostic: 1 = skip M stores, 2 = skip operand loads,
                         // 4 = skip the 3xTF32 (B) split, 8 = skip the MMAs,
                         // 32 = skip the TMEM-A split
  static int v = -1;
  if (v < 0) v = getenv("WINO_GEMM_DBG") ? atoi(getenv("WINO_GEMM_DBG")) : 0;
  return v;
}

template <int PREC, int BN, bool TA, bool MB = false, bool BS = false, bool TRN = false>
static cudaError_t launch_tc(const GemmArgs& a, cudaStream_t s) {
  using Tr = GemmTraits<PREC>;
  using Sm = GemmSmem<PREC, BN, TA>;
  static_assert(!TRN || !MB, "TRN: fp32 M");
  alignas(64) CUtensorMap tmV, tmU;  // the A (128-row) and B (BN-row) operand maps
  const uint64_t es = Tr::esize;
  const uint64_t planes = static_cast<uint64_t>(op_splits(PREC)) * a.a2;  // planes in HBM
  const uint64_t u_planes = BS ? 2 * planes : planes;
  const void* A = TRN ? a.U : a.V;
  const void* B = TRN ? a.V : a.U;
  const uint64_t a_rows = TRN ? static_cast<uint64_t>(a.K) : static_cast<uint64_t>(a.Pc);
  const uint64_t b_rows = TRN ? static_cast<uint64_t>(a.Pc) : static_cast<uint64_t>(a.K);
  if (!encode_tmap_3d(&tmV, PREC, A, a.C, a_rows, planes, a.c_pad * es, a_rows * a.c_pad * es,
                      Tr::bk, kTileP))
    return cudaErrorInvalidValue;
  if (!encode_tmap_3d(&tmU, PREC, B, a.C, b_rows, u_planes, a.c_pad * es,
                      b_rows * a.c_pad * es, Tr::bk, BN))
    return cudaErrorInvalidValue;
  const int splits = a.splits < 1 ? 1 : a.splits;
  alignas(64) CUtensorMap tmM;
  constexpr uint64_t mes = MB ? 2 : 4;  // M element bytes
  // TRN stages 128B-swizzled [32 filters][32 tiles] boxes (conflict-free row stores)
  if (!encode_tmap_3d(&tmM, TRN ? kFP32 : (MB ? -2 : -1), a.M, a.Pc, a.K,
                      static_cast<uint64_t>(splits) * a.a2, a.m_ld * mes,
                      static_cast<uint64_t>(a.K) * a.m_ld * mes, 32, 32))
    return cudaErrorInvalidValue;
  auto kern = wgemm_tc_kernel<PREC, BN, TA, MB, BS, TRN>;
  static DeviceOnce configured;
  if (configured.first()) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Sm::total);
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    configured.done();
  }
  const int num_kb = (a.C + Tr::bk - 1) / Tr::bk;
  const int kbps = (num_kb + splits - 1) / splits;
  // A-side (128-row) and B-side (BN-row) block counts
  const int n_pblk = static_cast<int>((a_rows + kTileP - 1) / kTileP);
  const int n_kblk = static_cast<int>((b_rows + BN - 1) / BN);
  const long long units = static_cast<long long>(n_pblk) * n_kblk * a.a2 * splits;
  if (units > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int grid = static_cast<int>(units < num_sms() ? units : num_sms());
  launch_k(kern, dim3(grid), dim3(gemm_threads<PREC>()), Sm::total, s, tmV, tmU, tmM, a.a2, num_kb, kbps,
           n_pblk, n_kblk, static_cast<int>(units), gemm_dbg());
  return cudaGetLastError();
}

int gemm_num_kblocks(int prec, int C) {
  const int bk = (prec == kBF16 || prec == kFP16) ? 64 : 32;
  return (C + bk - 1) / bk;
}

int gemm_device_sms() { return num_sms(); }

bool gemm_tmem_a_enabled() { return getenv("WINO_NO_TMEM_A") == nullptr; }

template <int PREC>
static cudaError_t launch_prec(const GemmArgs& a, cudaStream_t s) {
  if constexpr (PREC != kFP32) {  // single-pass GEMMs with the filters on the M side
    if (a.tr) {
      switch (a.bn) {
        case 32: return launch_tc<PREC, 32, false, false, false, true>(a, s);
        case 64: return launch_tc<PREC, 64, false, false, false, true>(a, s);
        case 128: return launch_tc<PREC, 128, false, false, false, true>(a, s);
        default: return cudaErrorInvalidValue;
      }
    }
  }
  if constexpr (PREC == kFP32) {  // 3xTF32: A operand through tensor memory (BN <= 128)
    static const bool tmem_a = getenv("WINO_NO_TMEM_A") == nullptr;
    static const bool pair = getenv("WINO_GEMM_2SM") != nullptr;
    if (tmem_a && pair && !a.tr && (a.bn == 64 || a.bn == 128)) {
      if (a.b_split)
        return a.bn == 64 ? launch_tc2<64, true>(a, s) : launch_tc2<128, true>(a, s);
      return a.bn == 64 ? launch_tc2<64, false>(a, s) : launch_tc2<128, false>(a, s);
    }
    if (tmem_a && a.tr) {  // b_split: V arrives as hi / lo planes (input transform)
      switch (a.bn * 2 + (a.b_split ? 1 : 0)) {
        case 64: return launch_tc<PREC, 32, true, false, false, true>(a, s);
        case 65: return launch_tc<PREC, 32, true, false, true, true>(a, s);
        case 128: return launch_tc<PREC, 64, true, false, false, true>(a, s);
        case 129: return launch_tc<PREC, 64, true, false, true, true>(a, s);
        case 256: return launch_tc<PREC, 128, true, false, false, true>(a, s);
        case 257: return launch_tc<PREC, 128, true, false, true, true>(a, s);
        default: return cudaErrorInvalidValue;
      }
    }
    if (tmem_a && a.b_split) {
      switch (a.bn) {
        case 32: return launch_tc<PREC, 32, true, false, true>(a, s);
        case 64: return launch_tc<PREC, 64, true, false, true>(a, s);
        case 128: return launch_tc<PREC, 128, true, false, true>(a, s);
        default: return cudaErrorInvalidValue;
      }
    }
    if (a.b_split) return cudaErrorInvalidValue;  // split planes need the TMEM-A kernel
    if (tmem_a) {
      switch (a.bn) {
        case 32: return launch_tc<PREC, 32, true>(a, s);
        case 64: return launch_tc<PREC, 64, true>(a, s);
        case 128: return launch_tc<PREC, 128, true>(a, s);
        default: break;
      }
    }
  }
  if constexpr (PREC == kBF16 || PREC == kFP16) {
    if (a.m_bf16) {
      switch (a.bn) {
        case 32: return launch_tc<PREC, 32, false, true>(a, s);
        case 64: return launch_tc<PREC, 64, false, true>(a, s);
        case 128: return launch_tc<PREC, 128, false, true>(a, s);
        case 256: return launch_tc<PREC, 256, false, true>(a, s);
        default: return cudaErrorInvalidValue;
      }
    }
  }
  switch (a.bn) {
    case 32: return launch_tc<PREC, 32, false>(a, s);
    case 64: return launch_tc<PREC, 64, false>(a, s);
    case 128: return launch_tc<PREC, 128, false>(a, s);
    case 256: return launch_tc<PREC, 256, false>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_batched_gemm(int prec, const GemmArgs& a, cudaStream_t s) {
  if (a.Pc <= 0 || a.K <= 0) return cudaSuccess;
  switch (prec) {
    case kFP32: return launch_prec<kFP32>(a, s);
    case kTF32: return launch_prec<kTF32>(a, s);
    case kBF16: return launch_prec<kBF16>(a, s);
    case kFP16: return launch_prec<kFP16>(a, s);
    case kFP64: {
      const dim3 grid(static_cast<unsigned>((a.Pc + 63) / 64), (a.K + 63) / 64, a.a2);
      launch_k(wgemm_f64_kernel, grid, dim3(256), 0, s, static_cast<const double*>(a.V),
               static_cast<const double*>(a.U), static_cast<double*>(a.M), a.K, a.Pc, a.C,
               a.c_pad, a.m_ld);
      return cudaGetLastError();
    }
    default: return cudaErrorInvalidValue;
  }
}

int gemm_kernels_per_launch(int) { return 1; }

}  // namespace wino

// Diagnostic only (not part of include/wino.h): copy the GEMM timeline of the
// last launch (WINO_GEMM_DBG=64), 16 values per CTA.
extern "C" int wino_debug_gemm_trace(unsigned long long* out, int ctas) {
  if (ctas > 1024) ctas = 1024;
  return cudaMemcpyFromSymbol(out, wino::g_gemm_trace, sizeof(unsigned long long) * 16 * ctas) ==
                 cudaSuccess ? 0 : -1;
}
