// Internal declarations shared by the kernel translation units and the C-ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include <atomic>
#include <utility>

#include "../../include/wino.h"

namespace wino {

// Operand precision of the alpha^2 batched GEMM (the transform-space data).
enum Prec : int {
  kFP32 = WINO_PREC_FP32,  // 3xTF32 split operands (hi + lo), fp32-accurate
  kTF32 = WINO_PREC_TF32,  // single-pass TF32
  kBF16 = WINO_PREC_BF16,
  kFP16 = WINO_PREC_FP16,
  kFP64 = WINO_PREC_FP64,  // fp64 data end to end (CUDA-core GEMM)
  // internal, input transform only: fp32 V written as tf32 hi / lo planes (the
  // 3xTF32 GEMM's B operand pre-split, WINO_PREC_FP32 plans with filters on M)
  kFP32S = 16,
};

inline int op_bytes(int prec) {
  switch (prec) {
    case kBF16:
    case kFP16: return 2;
    case kFP64: return 8;
    default: return 4;
  }
}
// Operand planes in HBM.  3xTF32 keeps ONE fp32 plane in memory; the GEMM
// kernels split each landed shared-memory stage into hi = rna_tf32(x) and
// lo = x - hi on chip, so U and V cost 4 bytes per element, not 8.
inline int op_splits(int) { return 1; }


// Kernel attributes (dynamic shared-memory opt-in, carveout) belong to a device
// context, so "already configured" is tracked per (kernel call site, device):
// a process that drives several GPUs opts every kernel in on each of them.
// Thread-safe; concurrent first calls just set the same attributes twice.
struct DeviceOnce {
  std::atomic<unsigned long long> mask{0};
  static int bit() {
    int d = 0;
    cudaGetDevice(&d);
    return d & 63;
  }
  bool first() const { return !((mask.load(std::memory_order_acquire) >> bit()) & 1ull); }
  void done() { mask.fetch_or(1ull << bit(), std::memory_order_release); }
};
// SM count of the current device (cached per device).
int device_sms();

// ---- launchers (defined in wino_transforms.cu / wino_gemm.cu) -------------
// All return cudaError_t of the launch.

// g (K,C,3,3) [float or double] -> U [nsplit][alpha^2][K][c_pad]
// split2 (FP32 only): write hi = rna_tf32(u) and lo = u - hi as two planes
// (the staged 3xTF32 GEMM then needs no on-chip split of U).
cudaError_t launch_filter_transform(int m, int prec, const void* g, void* U, int K, int C,
                                    int c_pad, cudaStream_t s, bool split2 = false);

// Filter transform + single-chunk TMA input transform in one launch (non-FX,
// W % 4 == 0, pad <= 3, not fp64): V for tile rows [0, rows), U as above.
bool transforms_combinable(int prec, int W, int pad);
cudaError_t launch_transforms(int m, int prec, const void* d, void* V, int N, int C, int H, int W,
                              int pad, int th, int tw, int rows, long long Pc, int c_pad,
                              const void* g, void* U, int K, bool split2, cudaStream_t s);

// d (N,C,H,W) -> V [nsplit][alpha^2][Pc][c_pad] for tile rows [row0, row0+rows)
cudaError_t launch_input_transform(int m, int prec, const void* d, void* V, int N, int C, int H,
                                   int W, int pad, int th, int tw, int row0, int rows,
                                   long long Pc, int c_pad, cudaStream_t s);

// M [splits][alpha^2][K][m_ld] (float, or double for FP64) -> y (N,K,oh,ow), clipped;
// split slices are summed in ascending order (deterministic).
// F(4x4) chunks of at most this many tiles take the per-thread output transform
// (fp32 M) instead of the TMA box (WINO_OUT_TMA_MIN, default 256).
long long output_tma_min_tiles(int prec);
// `dead`/`dead_bytes`: a 128-byte-aligned region (the chunk's V) that is dead once
// the GEMM has run; the TMA variant drops its L2 lines (no HBM write-back).
// `act`: epilogue activation of the written tiles (kActNone / kActRelu /
// kActReluPool: y is then (N, K, oh/2, ow/2)); see emit_tile.
enum : int { kActNone = 0, kActRelu = 1, kActReluPool = 2 };
cudaError_t launch_output_transform(int m, int prec, const void* Mbuf, void* y, int N, int K,
                                    int th, int tw, int oh, int ow, int row0, long long Pc,
                                    long long m_ld, int splits, cudaStream_t s, int m_bf16 = 0,
                                    const void* dead = nullptr, size_t dead_bytes = 0,
                                    int act = kActNone);

// Whole layer on chip for C <= 8 (input transform + C-term reduction + output
// transform in one kernel); U in the plan's operand format.
constexpr int kSmallCMax = 8;
// fp16-staged M holds M * 2^-kM16Shift (exact power of two): |M| up to 2^20 stays
// finite and |M| >= 2^-10 keeps full fp16 precision (the fp16 operands U, V
// already bound the data to fp16 range).
constexpr int kM16Shift = 4;
cudaError_t launch_fused_smallc(int m, int prec, const void* d, const void* U, void* y, int N,
                                int C, int H, int W, int K, int pad, int th, int tw, int oh,
                                int ow, int c_pad, cudaStream_t s, int act = kActNone);

// Weight gradient F(3x3,2x2) (engine.py:278-328): transforms of tiles
// [b0, b0+nb) into Uw [nsplit][16][K][b_pad] and Vw [nsplit][16][C][b_pad]
// (tile index innermost), and the inverse transform of the summed M slices
// [slices][16][K][m_ld] into dg (K,C,3,3).
cudaError_t launch_wgrad_transforms(int prec, const void* d, const void* dy, void* Uw, void* Vw,
                                    int K, int C, int H, int W, int pad, int oh, int ow, int gh,
                                    int gw, long long b0, long long nb, long long b_pad,
                                    cudaStream_t s);
cudaError_t launch_wgrad_accumulate(int prec, void* acc, const void* slices, long long n,
                                    int splits, int first, cudaStream_t s);
// Small-C (C <= 4, fp32 inputs, prec != FP64) weight gradient on the CUDA cores:
// nblk blocks each write one M slice [16][K][m_ld] of `parts`; the slices are
// summed into `summed` ([16][K][m_ld]).
cudaError_t launch_wgrad_smallc(int prec, const void* d, const void* dy, void* parts,
                                void* summed, int K, int C, int H, int W, int pad, int oh, int ow,
                                int gh, int gw, long long B, long long m_ld, int nblk,
                                cudaStream_t s);
cudaError_t launch_wgrad_inverse(int prec, const void* Mbuf, void* dg, int K, int C,
                                 long long m_ld, int slices, cudaStream_t s);

struct GemmArgs {
  const void* V;   // [nsplit][a2][Pc][c_pad]
  const void* U;   // [nsplit][a2][K][c_pad]
  void* M;         // [splits][a2][K][Pc]
  int a2, K, C, c_pad;
  long long Pc;
  int bn;          // filters per CTA (tcgen05 N)
  int splits;      // split-C factor: partial sums go to M slices [splits][a2][K][m_ld]
  long long m_ld;  // M row stride (>= Pc, multiple of 4 -- 8 for bf16 M -- for the TMA store)
  int m_bf16 = 0;  // 16-bit GEMMs: M staged in 16 bits (1 = bf16, 2 = fp16 x 2^-kM16Shift; planner)
  int b_split = 0; // 3xTF32 only: U holds [hi planes][lo planes] (no on-chip B split)
  int tr = 0;      // 3xTF32 TMEM-A only: filters on the MMA M side, bn = tiles per unit
};
int gemm_num_kblocks(int prec, int C);
int gemm_device_sms();
bool gemm_tmem_a_enabled();  // 3xTF32 A operand through TMEM (WINO_NO_TMEM_A=1 disables)
// Tensor-core (tcgen05) GEMM for FP32/TF32/BF16/FP16, CUDA-core fp64 for FP64.
cudaError_t launch_batched_gemm(int prec, const GemmArgs& a, cudaStream_t s);

// Direct correlation (reference order and rounding), input fp32/fp64 ->
// accumulator/output fp32/fp64 (wino_direct.cu).
cudaError_t launch_direct(int in_prec, int acc_prec, const void* d, const void* g, void* y, int N,
                          int C, int H, int W, int K, int R, int S, int pad, int oh, int ow,
                          cudaStream_t s);
int gemm_kernels_per_launch(int prec);

// Fused Winograd-GEMM (wino_fused.cu): input transform in the producer warps,
// tcgen05 GEMM, output transform in the epilogue; one cluster of alpha CTAs per
// (tile block, filter block).  splits > 1 writes partial y slices to ypart
// ([splits][N][K][oh][ow] fp32) and sums them in a second kernel.
struct FusedArgs {
  const void* d;  // (N,C,H,W) fp32
  const void* U;  // [nsplit][a2][K][c_pad] operand format
  const void* V;  // NULL: form V in-kernel from d; else staged V chunk [nsplit][a2][P][c_pad]
  void* y;        // (N,K,oh,ow) fp32
  void* ypart;    // split partials (splits > 1)
  long long P;    // tiles in this launch (the chunk)
  long long p0;   // global index of its first tile
  int N, C, H, W, K, pad, th, tw, oh, ow, c_pad;
  int splits;
};
int fused_num_kblocks(int prec, int C);
int fused_tiles_per_unit(int m);
cudaError_t launch_fused(int m, int prec, const FusedArgs& f, cudaStream_t s);

// ---- launch helper: every pipeline kernel is launched with Programmatic
// Dependent Launch allowed (disable with WINO_NO_PDL=1), so its launch and
// prologue overlap the previous kernel's tail; kernels call griddep_wait()
// before touching predecessor outputs and griddep_launch() at entry.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#ifdef __CUDACC__
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#endif

// Host helpers.
const char* set_error(const char* fmt, ...);
// 4D fp32 map over an NCHW tensor (dims W,H,C,N), no swizzle, zero OOB fill.
bool encode_tmap_nchw_f32(void* map_out, const void* base, int N, int C, int H, int W,
                          uint32_t box_w, uint32_t box_h, uint32_t box_c);
bool encode_tmap_3d_sw(void* map_out, int prec, const void* base, uint64_t d0, uint64_t d1,
                       uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0,
                       uint32_t box1, int swizzle_bytes);
bool encode_tmap_3d_box(void* map_out, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                        uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0,
                        uint32_t box1, uint32_t box2, bool bf16 = false);
bool encode_tmap_3d(void* map_out, int prec, const void* base, uint64_t d0, uint64_t d1,
                    uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0,
                    uint32_t box1);

}  // namespace wino
