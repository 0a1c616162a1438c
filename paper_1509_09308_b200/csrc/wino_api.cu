// C ABI (include/wino.h): plan creation with the tile/workspace planner,
// filter transform, and the chunked forward pipeline
//   input transform -> tcgen05 batched GEMM -> output transform
// per chunk of whole tile rows, sized so the chunk's transform-space staging
// (V and M) stays resident in the 126 MB L2 instead of round-tripping HBM.
#include <cudaTypedefs.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "wino_internal.h"

struct wino_plan_s {
  wino_layer_t L;
  int m, r, alpha, a2, prec;
  int oh, ow, th, tw;
  long long P;
  int c_pad, esize, nsplit, acc_bytes;
  int bn, splits;
  bool smallc;  // whole layer in the fused tiny-C kernel (no V/M staging)
  int path;     // kPathStaged / kPathFused / kPathHybrid (see plan_create)
  bool overlap; // staged, several chunks: nbuf chunks in flight on nbuf streams
  int nbuf;     // V/M buffer sets (1, or the streams in flight: 2 default, 3 by env)
  int fsplits;  // split-C factor of the fused kernel
  size_t ypart_bytes;
  int rows_total, rows_per_chunk, num_chunks;
  long long chunk_tiles;
  long long m_ld;                    // M row stride (tiles, multiple of 64: 128-byte rows)
  int m_bf16;                        // M staged as bf16 (bf16 GEMM, staged, no split-C)
  int m_es;                          // M element bytes
  size_t u_bytes, v_bytes, m_bytes;  // v/m per full chunk
  int u_split2;                      // non-FX 3xTF32 staged: U as hi/lo planes in the workspace
  int gemm_tr;                       // 3xTF32 small P: filters on the MMA M side (bn = tiles)
  int v_split2;                      // with gemm_tr: V written as tf32 hi / lo planes
  size_t u_ws;                       // workspace bytes of a forward-computed U
  size_t staging_bytes;              // V + M of the chunks in flight (+ fused partials)
  size_t ws_limit;                   // workspace_limit passed at creation (shard sub-plans)
};

namespace wino {

enum : int { kPathStaged = 0, kPathFused = 1, kPathHybrid = 2 };

static thread_local std::string g_err;

const char* set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return g_err.c_str();
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static bool load_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

bool encode_tmap_3d(void* map_out, int prec, const void* base, uint64_t d0, uint64_t d1,
                    uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0,
                    uint32_t box1) {
  if (!load_encode()) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return false;
  }
  CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  if (prec == kBF16 || prec == -2) dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if (prec == kFP16) dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  // operand maps use the 128B swizzle UMMA expects; the accumulator store maps
  // (prec -1 fp32, -2 bf16) are plain row-major boxes
  CUresult r = g_encode(reinterpret_cast<CUtensorMap*>(map_out), dt, 3, const_cast<void*>(base),
                        dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        prec < 0 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): dims %llu,%llu,%llu strides %llu,%llu", (int)r,
              (unsigned long long)d0, (unsigned long long)d1, (unsigned long long)d2,
              (unsigned long long)stride1_bytes, (unsigned long long)stride2_bytes);
    return false;
  }
  return true;
}

// Operand map with an explicit swizzle span (32 / 64 / 128 bytes per box row).
bool encode_tmap_3d_sw(void* map_out, int prec, const void* base, uint64_t d0, uint64_t d1,
                       uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0,
                       uint32_t box1, int swizzle_bytes) {
  if (!load_encode()) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return false;
  }
  CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  if (prec == kBF16) dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if (prec == kFP16) dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                      : CU_TENSOR_MAP_SWIZZLE_32B;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(reinterpret_cast<CUtensorMap*>(map_out), dt, 3, const_cast<void*>(base),
                        dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (swizzle %d) failed (%d)", swizzle_bytes, (int)r);
    return false;
  }
  return true;
}

// fp32 3D map with a 3D box (no swizzle, zero OOB fill): the output transform's
// M[comp][k][p] staging box.
bool encode_tmap_3d_box(void* map_out, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                        uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0,
                        uint32_t box1, uint32_t box2, bool bf16) {
  if (!load_encode()) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return false;
  }
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {box0, box1, box2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(reinterpret_cast<CUtensorMap*>(map_out),
                        bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        3, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (3d box) failed (%d)", (int)r);
    return false;
  }
  return true;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("WINO_NO_PDL");
    return !(v && v[0] == '1');
  }();
  return on;
}

bool encode_tmap_nchw_f32(void* map_out, const void* base, int N, int C, int H, int W,
                          uint32_t box_w, uint32_t box_h, uint32_t box_c) {
  if (!load_encode()) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return false;
  }
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(N)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(W) * 4, static_cast<cuuint64_t>(H) * W * 4,
                           static_cast<cuuint64_t>(C) * H * W * 4};
  cuuint32_t box[4] = {box_w, box_h, box_c, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = g_encode(reinterpret_cast<CUtensorMap*>(map_out), CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        4, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (NCHW) failed (%d)", (int)r);
    return false;
  }
  return true;
}

static int cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) {
    set_error("%s: out of device memory", what);
    return WINO_ENOMEM;
  }
  set_error("%s: %s", what, cudaGetErrorString(e));
  return WINO_ECUDA;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Default chunk budget: transform-space staging that stays L2-resident.
constexpr size_t kDefaultWorkspace = 128ull << 20;
// The staged input-transform kernels put a chunk's tile rows on grid.y.
constexpr long long kMaxChunkRows = 65535;

}  // namespace wino

using namespace wino;

extern "C" {

const char* wino_last_error(void) { return g_err.c_str(); }

#ifndef WINO_SRC_HASH
#define WINO_SRC_HASH "unknown000000000"
#endif
// The source hash lets build() detect a stale library (build.py).
const char* wino_version(void) { return "wino-b200 0.2.0 (sm_100a) src " WINO_SRC_HASH; }

int wino_plan_create(const wino_layer_t* layer, int m, int prec, size_t workspace_limit,
                     wino_plan_t* out) {
  g_err.clear();
  if (!layer || !out) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  *out = nullptr;
  const wino_layer_t& L = *layer;
  // LayerConfig validation (direct.py:48-55)
  if (L.N < 1 || L.C < 1 || L.H < 1 || L.W < 1 || L.K < 1 || L.R < 1 || L.S < 1) {
    set_error("N, C, H, W, K, R, S must be >= 1");
    return WINO_EINVAL;
  }
  if (L.pad < 0) {
    set_error("pad must be >= 0");
    return WINO_EINVAL;
  }
  const int oh = L.H + 2 * L.pad - L.R + 1, ow = L.W + 2 * L.pad - L.S + 1;
  if (oh < 1 || ow < 1) {
    set_error("output dimensions must be >= 1");
    return WINO_EINVAL;
  }
  if (m != 2 && m != 4) {  // builtin() lookup (winograd.py:225-232)
    set_error("no builtin algorithm for F(%d,3); available F(2,3), F(4,3)", m);
    return WINO_EUNSUPPORTED;
  }
  if (L.R != 3 || L.S != 3) {  // engine.py:217-218
    set_error("layer filter %dx%d but algorithm is F(%d,3)", L.R, L.S, m);
    return WINO_EUNSUPPORTED;
  }
  if (prec < WINO_PREC_FP32 || prec > WINO_PREC_FP64) {
    set_error("unknown precision %d", prec);
    return WINO_EINVAL;
  }
  wino_plan_s* p = new (std::nothrow) wino_plan_s();
  if (!p) {
    set_error("host allocation failed");
    return WINO_ENOMEM;
  }
  p->L = L;
  p->ws_limit = workspace_limit;
  p->m = m;
  p->r = 3;
  p->alpha = m + 2;
  p->a2 = p->alpha * p->alpha;
  p->prec = prec;
  p->oh = oh;
  p->ow = ow;
  p->th = (oh + m - 1) / m;
  p->tw = (ow + m - 1) / m;
  p->P = static_cast<long long>(L.N) * p->th * p->tw;
  p->esize = op_bytes(prec);
  p->nsplit = op_splits(prec);
  p->acc_bytes = prec == kFP64 ? 8 : 4;
  // channel stride padded so TMA row strides are 16-byte multiples
  p->c_pad = static_cast<int>(align_up(L.C, 16 / p->esize));
  p->u_bytes = align_up(static_cast<size_t>(p->nsplit) * p->a2 * L.K * p->c_pad * p->esize, 1024);

  // ---- GEMM tile: BN filters per CTA (tcgen05 N).  Prefer wide tiles, shrink
  // while the grid would leave SMs idle.
  int bn = 256;
  if (prec == kFP32) bn = 128;  // 3 split stages of 64 KB fit; 256 would leave 2
  while (bn > 32 && bn / 2 >= L.K) bn /= 2;
  const long long ptiles = (p->P + 127) / 128;
  // 3xTF32 streams twice the operand bytes: keep 128-wide tiles (less V
  // re-reading) and let split-C fill the SMs (measured: VGG-E N=1 -4%).
  const int bn_floor = prec == kFP32 ? 128 : 64;
  while (bn > bn_floor && ptiles * ((L.K + bn - 1) / bn) * p->a2 < 148) bn /= 2;
  if (const char* e = getenv("WINO_GEMM_BN")) {  // tuning override (32/64/128/256)
    const int v = atoi(e);
    if (v == 32 || v == 64 || v == 128 || v == 256) bn = v;
    if (prec == kFP32 && bn > 128) bn = 128;  // the 3xTF32 kernels stop at 128
  }
  p->bn = bn;

  // (F(4x4) fp64 with C > 4 would exceed the small-C kernel's shared memory)
  p->smallc = L.C <= ((prec == kFP64 && m == 4) ? 4 : kSmallCMax);

  // 3xTF32 with more filters than tiles (K > P: the deep layers at N = 1):
  // filters on the MMA's 128-row side (A, split into TMEM) and the tiles on N
  // (bn = 32 / 64 / 128 tiles), with V pre-split into tf32 hi / lo planes by
  // the input transform (off the critical path there: the filter transform is
  // longer), so no operand is split in shared memory.  WINO_NO_GEMM_TR=1
  // disables; WINO_GEMM_TR_MAXP bounds P (default 256).
  p->gemm_tr = 0;
  static const long long tr_maxp =
      getenv("WINO_GEMM_TR_MAXP") ? atoll(getenv("WINO_GEMM_TR_MAXP")) : 256;
  // The single-pass GEMMs (tf32 / bf16 / fp16) take the same orientation for
  // K > P <= 64 (their 128-row tile blocks would otherwise carry 16-49 real
  // tiles: conv4-5 at N = 1): VGG-E F4 N=1 tf32 0.324 -> 0.289 ms, fp16 0.278
  // -> 0.268, bf16 0.277 -> 0.268; at P = 128 (conv5, N = 8) it measured 1%
  // slower.  WINO_NO_GEMM_TR16=1 disables, WINO_GEMM_TR16_MAXP moves the bound.
  const bool tr16 = getenv("WINO_NO_GEMM_TR16") == nullptr;  // (read per plan: tests toggle it)
  static const long long tr16_maxp =
      getenv("WINO_GEMM_TR16_MAXP") ? atoll(getenv("WINO_GEMM_TR16_MAXP")) : 64;
  const bool single_pass = prec == kTF32 || prec == kBF16 || prec == kFP16;
  const bool tr_prec = (prec == kFP32 && gemm_tmem_a_enabled()) ||
                       (tr16 && single_pass && p->P <= tr16_maxp);
  if (tr_prec && !p->smallc && p->P <= tr_maxp &&
      static_cast<long long>(L.K) > p->P && L.K >= 128 && getenv("WINO_NO_GEMM_TR") == nullptr) {
    p->gemm_tr = 1;
    p->bn = p->P <= 32 ? 32 : p->P <= 64 ? 64 : 128;
  }

  // ---- chunk planner: whole tile rows, V + M staging within the budget
  const size_t budget = workspace_limit ? workspace_limit : kDefaultWorkspace;
  // bf16 GEMM: M is staged in bf16.  The accumulation stays fp32 (TMEM); the one
  // extra rounding of M is of the size of the bf16 operand roundings of U and V
  // that already dominate the variant's error (measured +22% rms),
  // and it halves the largest staged tensor.  WINO_M_FP32=1 keeps fp32 M.
  // fp16 GEMM: M staged as fp16 (scaled by 2^-kM16Shift) -- fp16's 11-bit
  // significand keeps the variant ~5x tighter than bf16 operands (emulated F4:
  // 0.77% -> 1.2% of max|y|, bf16 6-7%) at the bf16 plan's staging bytes;
  // WINO_FP16_M32=1 (or WINO_M_FP32=1) keeps fp32 M.
  const bool m16 = getenv("WINO_M_FP32") == nullptr &&
                   (prec == kBF16 || (prec == kFP16 && getenv("WINO_FP16_M32") == nullptr));
  p->m_es = m16 ? 2 : p->acc_bytes;
  const size_t per_tile = static_cast<size_t>(p->nsplit) * p->a2 * p->c_pad * p->esize +
                          static_cast<size_t>(p->a2) * L.K * p->m_es;
  const size_t per_row = per_tile * p->tw;
  p->rows_total = L.N * p->th;
  long long rows = static_cast<long long>(budget / (per_row ? per_row : 1));
  if (rows < 1) rows = 1;
  if (rows > p->rows_total) rows = p->rows_total;
  if (rows > kMaxChunkRows) rows = kMaxChunkRows;
  p->rows_per_chunk = static_cast<int>(rows);
  p->num_chunks = (p->rows_total + p->rows_per_chunk - 1) / p->rows_per_chunk;
  p->chunk_tiles = static_cast<long long>(p->rows_per_chunk) * p->tw;

  // ---- split-C for small-P layers (single chunk): enough GEMM work units to
  // cover the SMs; partial sums land in separate M slices.
  p->splits = 1;
  if (prec != kFP64 && p->num_chunks == 1) {
    const int sms = gemm_device_sms();
    const int num_kb = gemm_num_kblocks(prec, L.C);
    const long long units =
        p->gemm_tr ? ((L.K + 127) / 128) * ((p->chunk_tiles + p->bn - 1) / p->bn) * p->a2
                   : ((p->chunk_tiles + 127) / 128) * ((L.K + p->bn - 1) / p->bn) * p->a2;
    if (units < sms && num_kb > 1) {
      // waves x k-steps per unit (+2 for the unit's fill and epilogue) + half a
      // k-step per M slice the output transform sums; ties -> fewer splits
      double best = 1e30;
      for (int sp = 1; sp <= num_kb && sp <= 8; ++sp) {
        const int kbps = (num_kb + sp - 1) / sp;
        const int sp_eff = (num_kb + kbps - 1) / kbps;
        const long long waves = (units * sp_eff + sms - 1) / sms;
        const double cost = static_cast<double>(waves) * (kbps + 2) + 0.5 * sp_eff;
        if (cost < best - 1e-9) {
          best = cost;
          p->splits = sp_eff;
        }
      }
      if (const char* e = getenv("WINO_SPLITS")) {  // tuning override
        const int v = atoi(e);
        if (v >= 1 && v <= num_kb) {
          const int kbps = (num_kb + v - 1) / v;
          p->splits = (num_kb + kbps - 1) / kbps;
        }
      }
    }
  }
  // gemm_tr plans take V from the input transform as tf32 hi / lo planes, so
  // the GEMM's B operand needs no on-chip split (WINO_NO_VSPLIT=1 disables)
  p->v_split2 = (p->gemm_tr && prec == kFP32 && getenv("WINO_NO_VSPLIT") == nullptr) ? 1 : 0;
  p->v_bytes = p->smallc ? 0
                        : align_up(static_cast<size_t>(p->nsplit) * (p->v_split2 ? 2 : 1) *
                                       p->a2 * p->chunk_tiles * p->c_pad * p->esize,
                                   1024);
  if (p->smallc) {  // no transform-space staging at all
    p->num_chunks = 1;
    p->rows_per_chunk = p->rows_total;
    p->chunk_tiles = p->P;
    p->splits = 1;
  }
  p->m_ld = static_cast<long long>(align_up(static_cast<size_t>(p->chunk_tiles), 64));
  // ---- path (WINO_PATH=staged|fused|hybrid overrides the choice; read at
  // plan creation):
  //   staged : input transform -> GEMM -> output transform, V and M staged;
  //   fused  : one kernel, V formed in the GEMM producer, inverse transform in
  //            the epilogue (no V, no M);
  //   hybrid : staged input transform into an L2-sized V chunk, then the fused
  //            GEMM + inverse-transform kernel TMA-loads it (no M).
  // Default: staged -- on B200 it measured fastest on every VGG-E layer at
  // N = 1 and 64 (the alpha-way component split of the fused
  // kernels cuts TMEM tile reuse alpha-fold and adds an L2/DSMEM exchange).
  p->path = kPathStaged;
  if (!p->smallc && prec != kFP64) {
    const char* env = getenv("WINO_PATH");
    if (env && (strcmp(env, "staged") == 0 || strcmp(env, "unfused") == 0)) p->path = kPathStaged;
    if (env && strcmp(env, "fused") == 0) p->path = kPathFused;
    if (env && strcmp(env, "hybrid") == 0) p->path = kPathHybrid;
  }
  p->fsplits = 1;
  p->ypart_bytes = 0;
  if (p->path != kPathStaged) p->gemm_tr = p->v_split2 = 0;
  if (p->path != kPathStaged) {
    if (p->path == kPathFused) {
      p->num_chunks = 1;
      p->rows_per_chunk = p->rows_total;
      p->chunk_tiles = p->P;
      p->v_bytes = 0;
    } else {  // hybrid: the whole budget goes to the V chunk (no M)
      const size_t per_row_v =
          static_cast<size_t>(p->nsplit) * p->a2 * p->c_pad * p->esize * p->tw;
      long long r2 = static_cast<long long>(budget / (per_row_v ? per_row_v : 1));
      if (r2 < 1) r2 = 1;
      if (r2 > p->rows_total) r2 = p->rows_total;
      if (r2 > kMaxChunkRows) r2 = kMaxChunkRows;
      p->rows_per_chunk = static_cast<int>(r2);
      p->num_chunks = (p->rows_total + p->rows_per_chunk - 1) / p->rows_per_chunk;
      p->chunk_tiles = static_cast<long long>(p->rows_per_chunk) * p->tw;
      p->v_bytes = align_up(static_cast<size_t>(p->nsplit) * p->a2 * p->chunk_tiles * p->c_pad *
                                p->esize,
                            1024);
    }
    p->splits = 1;
    if (p->num_chunks == 1) {
      const int sms = gemm_device_sms();
      const int num_kb = fused_num_kblocks(prec, L.C);
      const int pbt = fused_tiles_per_unit(m);
      const long long ctas = ((p->P + pbt - 1) / pbt) * ((L.K + 127) / 128) * p->alpha;
      if (ctas < sms && num_kb > 1) {
        int sp = static_cast<int>((sms + ctas - 1) / ctas);
        if (sp > num_kb) sp = num_kb;
        const int kbps = (num_kb + sp - 1) / sp;
        p->fsplits = (num_kb + kbps - 1) / kbps;
      }
    }
    if (p->fsplits > 1)
      p->ypart_bytes = align_up(static_cast<size_t>(p->fsplits) *
                                    align_up(static_cast<size_t>(L.N) * L.K * oh * ow, 4) * 4,
                                1024);
  }
  // ---- staged path with several chunks: two chunks in flight (chunk i+1's
  // input transform runs under chunk i's GEMM and output transform, on a second
  // stream), each with half the budget so both stay L2-resident.
  p->overlap = false;
  p->nbuf = 1;
  if (p->path == kPathStaged && !p->smallc && p->num_chunks > 1) {
    int ns = 2;
    if (const char* e = getenv("WINO_CHUNK_STREAMS")) ns = atoi(e) == 3 ? 3 : 2;
    p->nbuf = ns;
    long long r2 = static_cast<long long>((budget / ns) / (per_row ? per_row : 1));
    if (r2 < 1) r2 = 1;
    if (r2 > kMaxChunkRows) r2 = kMaxChunkRows;
    p->rows_per_chunk = static_cast<int>(r2);
    p->num_chunks = (p->rows_total + p->rows_per_chunk - 1) / p->rows_per_chunk;
    p->chunk_tiles = static_cast<long long>(p->rows_per_chunk) * p->tw;
    p->v_bytes = align_up(static_cast<size_t>(p->nsplit) * (p->v_split2 ? 2 : 1) * p->a2 *
                              p->chunk_tiles * p->c_pad * p->esize,
                          1024);
    p->m_ld = static_cast<long long>(align_up(static_cast<size_t>(p->chunk_tiles), 64));
    p->overlap = p->num_chunks > 1;
    if (!p->overlap) p->nbuf = 1;
  }
  // (F(4x4) single chunks of <= output_tma_min_tiles(prec) tiles keep fp32 M for
  // the per-thread output transform; for the 16-bit GEMMs the threshold is 0 by
  // default (WINO_OUT_TMA_MIN raises it).  WINO_M16_SMALL=1 stages them in 16
  // bits regardless.)
  const bool small_f4 = m == 4 && p->num_chunks == 1 && p->chunk_tiles <= output_tma_min_tiles(prec) &&
                        getenv("WINO_M16_SMALL") == nullptr;
  p->m_bf16 = (p->m_es == 2 && p->splits == 1 && !p->smallc && p->path == kPathStaged && !small_f4 &&
               !p->gemm_tr)  // (the transposed epilogue stores fp32 M)
                  ? (prec == kFP16 ? 2 : 1) : 0;
  if (!p->m_bf16) p->m_es = p->acc_bytes;
  // Non-FX 3xTF32 staged plans: the filter transform writes U as hi / lo planes
  // in the workspace, so the GEMM's split warps only split V (into TMEM).
  // Worth it when U is re-read by several tile blocks; with few (the small-P deep
  // layers at N = 1) the doubled U write sits on the critical path instead.
  // Threshold (WINO_USPLIT_MIN_PBLK) measured on VGG-E F2 fp32 N=1: 16 -> 0.3755,
  // 4 -> 0.3705, 1 -> 0.385 ms; N=64: 11.6 -> 11.2 ms with it.
  static const int usplit_min = getenv("WINO_USPLIT_MIN_PBLK") ? atoi(getenv("WINO_USPLIT_MIN_PBLK")) : 4;
  p->u_split2 = (prec == kFP32 && p->path == kPathStaged && !p->smallc && !p->gemm_tr &&
                 gemm_tmem_a_enabled() && (p->P + 127) / 128 >= usplit_min &&
                 getenv("WINO_NO_USPLIT") == nullptr) ? 1 : 0;
  p->u_ws = p->u_split2 ? 2 * p->u_bytes : p->u_bytes;
  auto set_m_bytes = [&] {
    p->m_bytes = (p->smallc || p->path != kPathStaged) ? 0
                          : align_up(static_cast<size_t>(p->splits) * p->a2 * L.K * p->m_ld *
                                         p->m_es,
                                     1024);
  };
  set_m_bytes();
  // An explicit workspace_limit is a hard cap on the transform-space staging
  // (V + M of every chunk in flight, + fused split-C partials; U excluded -- it
  // is the FX filter workspace, or the caller passes it).  The chunk planner
  // sized V + M for one split; split-C multiplies M, so it is reduced here until
  // the staging fits (the paper's <= 16 MB mode).
  if (workspace_limit) {
    const int num_kb = gemm_num_kblocks(prec, L.C);
    while (p->splits > 1 && p->nbuf * (p->v_bytes + p->m_bytes) + p->ypart_bytes > workspace_limit) {
      const int kbps = (num_kb + p->splits - 2) / (p->splits - 1);
      p->splits = (num_kb + kbps - 1) / kbps;
      if (p->splits == 1 && m16 && !p->smallc && !small_f4 && !p->gemm_tr &&
          p->path == kPathStaged) {
        p->m_es = 2;
        p->m_bf16 = prec == kFP16 ? 2 : 1;
      }
      set_m_bytes();
    }
  }
  p->staging_bytes = p->nbuf * (p->v_bytes + p->m_bytes) + p->ypart_bytes;
  *out = p;
  return WINO_OK;
}

// Non-FX forwards of this plan launch the filter and input transforms as one
// kernel (staged, single chunk, 16-bit operands, TMA-eligible input).
// Only small layers (P <= 64 tiles: conv4-5 at N = 1) combine the transforms:
// on larger ones the separate kernels on two streams finish first (VGG-E F4
// fp16 N=1 0.2834 -> 0.2779 ms, N=8 0.611 -> 0.605 ms against combining every
// single-chunk 16-bit plan).  WINO_COMBINED_MAXP overrides the tile bound.
static bool plan_combines_transforms(const wino_plan_s* p) {
  static const bool fp32 = getenv("WINO_FP32_COMBINED") != nullptr;
  static const long long maxp =
      getenv("WINO_COMBINED_MAXP") ? atoll(getenv("WINO_COMBINED_MAXP")) : 64;
  return p->path == kPathStaged && !p->smallc &&
         (p->prec == kBF16 || p->prec == kFP16 || (fp32 && p->prec == kFP32)) &&
         p->num_chunks == 1 && p->P <= maxp && transforms_combinable(p->prec, p->L.W, p->L.pad);
}

int wino_plan_destroy(wino_plan_t plan) {
  delete plan;
  return WINO_OK;
}

int wino_plan_get_info(wino_plan_t p, wino_plan_info_t* info) {
  if (!p || !info) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  memset(info, 0, sizeof *info);
  info->m = p->m;
  info->r = p->r;
  info->alpha = p->alpha;
  info->out_h = p->oh;
  info->out_w = p->ow;
  info->tiles_h = p->th;
  info->tiles_w = p->tw;
  info->P = p->P;
  info->prec = p->prec;
  info->c_pad = p->c_pad;
  info->op_bytes = p->esize;
  info->op_splits = p->nsplit;
  info->gemm_bn = p->bn;
  info->gemm_splits = p->splits;
  info->rows_per_chunk = p->rows_per_chunk;
  info->num_chunks = p->num_chunks;
  info->chunk_tiles = p->chunk_tiles;
  info->u_bytes = p->u_bytes;
  info->workspace_bytes =
      p->u_ws + p->nbuf * (p->v_bytes + p->m_bytes) + p->ypart_bytes;
  info->launches_per_forward =
      p->smallc ? 1
                : p->path == kPathFused  ? 1 + (p->fsplits > 1)
                : p->path == kPathHybrid ? p->num_chunks * 2 + (p->fsplits > 1)
                                         : p->num_chunks * 3;
  info->fused = p->path;
  info->fused_splits = p->fsplits;
  info->m_bytes_per_elem = p->m_es;
  info->combined_transforms = plan_combines_transforms(p) ? 1 : 0;
  info->staging_bytes = p->staging_bytes;
  info->fused_small_c = p->smallc ? 1 : 0;
  info->multiplies = p->P * p->L.C * static_cast<long long>(p->L.K) * p->a2;
  return WINO_OK;
}

int wino_filter_transform(wino_plan_t p, const void* g, void* U, void* stream) {
  g_err.clear();
  if (!p || !g || !U) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  cudaError_t e = launch_filter_transform(p->m, p->prec, g, U, p->L.K, p->L.C, p->c_pad,
                                          static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? WINO_OK : cuda_fail(e, "filter transform");
}

// Stage timer: events recorded on the launch stream after every launch, read
// back later (no host synchronisation inside the forward, so host launch
// latency is not counted when the host runs ahead of the GPU).
struct wino_timer_s {
  static constexpr int kMax = 4096;
  cudaEvent_t ev[kMax];
  int stage[kMax];
  int n = 0;
  bool open = false;
};

namespace {
struct StageTimer {
  wino_timer_s* t;
  cudaStream_t s;
  StageTimer(cudaStream_t s_, wino_timer_s* t_) : t(t_), s(s_) {
    if (t && !t->open && t->n < wino_timer_s::kMax) {  // opening event of a sequence
      cudaEventRecord(t->ev[t->n], s);
      t->stage[t->n++] = -1;
      t->open = true;
    }
  }
  void mark(int st) {
    if (!t || t->n >= wino_timer_s::kMax) return;
    cudaEventRecord(t->ev[t->n], s);
    t->stage[t->n++] = st;
  }
};
}  // namespace

// Side stream on which the filter transform runs concurrently with the input
// transform (independent stages; the GEMM joins both).  One per host thread
// and device, created on first use; under stream capture the record/wait pair
// becomes a graph fork/join.
namespace {
struct SideStream {
  cudaStream_t st = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaStream_t st2 = nullptr;      // third chunk stream (created on first use)
  cudaEvent_t join2 = nullptr;
};
// One side stream per (host thread, device, caller stream): callers that
// pipeline independent forwards on several streams must not be coupled
// through a shared side stream.
SideStream* side_stream(cudaStream_t user) {
  struct Key {
    int dev;
    cudaStream_t user;
  };
  constexpr int kMax = 64;
  thread_local Key keys[kMax];
  thread_local SideStream ss[kMax];
  thread_local int n = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  for (int i = 0; i < n; ++i)
    if (keys[i].dev == dev && keys[i].user == user) return &ss[i];
  if (n == kMax) return nullptr;
  SideStream& x = ss[n];
  if (cudaStreamCreateWithFlags(&x.st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess) {
    x = SideStream();
    return nullptr;
  }
  keys[n] = Key{dev, user};
  return &ss[n++];
}
}  // namespace

static int forward_impl(wino_plan_t p, const void* d, const void* U, const void* g, void* y,
                        void* workspace, size_t workspace_bytes, void* stream,
                        wino_timer_s* timer, int act = kActNone) {
  g_err.clear();
  if (!p || !d || !y || (!U && !g) || !workspace) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  if (act != kActNone && act != kActRelu && act != kActReluPool) {
    set_error("unknown activation %d", act);
    return WINO_EINVAL;
  }
  if (act == kActReluPool && (p->oh % 2 != 0 || p->ow % 2 != 0)) {
    set_error("2x2 max-pool needs an even output size, got %dx%d", p->oh, p->ow);
    return WINO_EINVAL;
  }
  if (act != kActNone && !p->smallc && p->path != kPathStaged) {
    set_error("the activation epilogue runs on the staged path (WINO_PATH=staged)");
    return WINO_EUNSUPPORTED;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  StageTimer tm(s, timer);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  size_t need =
      p->nbuf * (p->v_bytes + p->m_bytes) + p->ypart_bytes + (U ? 0 : p->u_ws);
  if (workspace_bytes < need) {
    set_error("workspace too small: %zu < %zu bytes", workspace_bytes, need);
    return WINO_EINVAL;
  }
  // non-FX: G g G^T into the workspace.  Unless stage-timed, it runs on the
  // side stream alongside the input transform and is joined before the GEMM.
  // The side stream also carries every odd row chunk of a staged plan with
  // `overlap` (double-buffered V/M), joined back at the end.
  SideStream* side = nullptr;
  bool filt_side = false;
  const bool may_overlap = !timer && !p->smallc && p->path != kPathFused &&
                           getenv("WINO_NO_OVERLAP") == nullptr;
  const bool chunk_overlap = may_overlap && p->overlap && p->path == kPathStaged;
  // Non-FX single-chunk staged plans with 16-bit operands: filter and input
  // transforms in one launch (no side stream, one predecessor for the GEMM).
  // Measured: F4 bf16 N=1 VGG-E 0.328 -> 0.314 ms; for the fp32 (3xTF32) plans
  // the side-stream arrangement stays faster (0.385 vs 0.389 ms), so they keep it.
  const bool combined = !U && !timer && plan_combines_transforms(p);
  if (may_overlap && !combined && (!U || chunk_overlap)) {
    side = side_stream(s);
    if (side && (cudaEventRecord(side->fork, s) != cudaSuccess ||
                 cudaStreamWaitEvent(side->st, side->fork, 0) != cudaSuccess))
      side = nullptr;
  }
  // WINO_SIDE_SWAP=1: single-chunk staged plans with K > P swap the two, the
  // input transform on the side stream and the filter transform in-stream.
  // That was faster while the filter transform was the longer of the two; since
  // those plans' input transform writes V as tf32 hi / lo planes it is the
  // longer one, and keeping it in-stream (the GEMM launches behind it by PDL)
  // measured 0.3731 -> 0.3690 ms on VGG-E F2 fp32 N=1.
  bool input_enqueued = false;  // chunk 0's input transform already launched
  const bool u_split = !U && p->u_split2;  // U computed here as hi / lo planes
  if (combined) {
    const wino_layer_t& Lc = p->L;
    cudaError_t e = launch_transforms(p->m, p->v_split2 ? kFP32S : p->prec, d, ws + p->u_ws, Lc.N, Lc.C, Lc.H, Lc.W,
                                      Lc.pad, p->th, p->tw, p->rows_total, p->P, p->c_pad, g, ws,
                                      Lc.K, u_split, s);
    if (e != cudaSuccess) return cuda_fail(e, "filter + input transforms");
    input_enqueued = true;
    U = ws;
    ws += p->u_ws;
  } else if (!U) {
    static const bool swap = getenv("WINO_SIDE_SWAP") != nullptr;
    const bool in_side = side && p->path == kPathStaged && p->num_chunks == 1 &&
                         !chunk_overlap && static_cast<long long>(p->L.K) > p->P && swap;
    if (in_side) {
      input_enqueued = true;
      cudaError_t e = launch_input_transform(p->m, p->v_split2 ? kFP32S : p->prec, d, ws + p->u_ws, p->L.N, p->L.C,
                                             p->L.H, p->L.W, p->L.pad, p->th, p->tw, 0,
                                             p->rows_total, p->P, p->c_pad, side->st);
      if (e != cudaSuccess) return cuda_fail(e, "input transform");
      e = cudaEventRecord(side->join, side->st);
      if (e != cudaSuccess) return cuda_fail(e, "input transform join");
    }
    cudaError_t e = launch_filter_transform(p->m, p->prec, g, ws, p->L.K, p->L.C, p->c_pad,
                                            (side && !in_side) ? side->st : s, u_split);
    if (e != cudaSuccess) return cuda_fail(e, "filter transform");
    if (side && !in_side) {
      e = cudaEventRecord(side->join, side->st);
      if (e != cudaSuccess) return cuda_fail(e, "filter transform join");
      filt_side = true;
    }
    if (in_side) filt_side = true;  // the GEMM joins the side stream (now the input transform)
    tm.mark(0);
    U = ws;
    ws += p->u_ws;
  }
  int nstreams = (chunk_overlap && side) ? p->nbuf : 1;
  if (nstreams == 3) {  // third chunk stream: after the caller's prior work and U
    cudaError_t e = cudaSuccess;
    if (!side->st2) {
      e = cudaStreamCreateWithFlags(&side->st2, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&side->join2, cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side->st2, side->fork, 0);
    if (e == cudaSuccess && filt_side) e = cudaStreamWaitEvent(side->st2, side->join, 0);
    if (e != cudaSuccess) return cuda_fail(e, "third chunk stream");
  }
  auto join_filters = [&]() -> cudaError_t {
    if (!filt_side) return cudaSuccess;
    filt_side = false;
    return cudaStreamWaitEvent(s, side->join, 0);
  };
  const wino_layer_t& L = p->L;
  if (p->smallc) {
    cudaError_t e = launch_fused_smallc(p->m, p->prec, d, U, y, L.N, L.C, L.H, L.W, L.K, L.pad,
                                        p->th, p->tw, p->oh, p->ow, p->c_pad, s, act);
    if (e != cudaSuccess) return cuda_fail(e, "fused small-C layer");
    tm.mark(1);
    return WINO_OK;
  }
  if (p->path == kPathFused) {
    FusedArgs fa{d, U, nullptr, y, ws, p->P, 0, L.N, L.C, L.H, L.W, L.K, L.pad, p->th, p->tw,
                 p->oh, p->ow, p->c_pad, p->fsplits};
    cudaError_t e = launch_fused(p->m, p->prec, fa, s);
    if (e != cudaSuccess) {
      if (g_err.empty()) return cuda_fail(e, "fused winograd gemm");
      return WINO_ECUDA;
    }
    tm.mark(2);
    return WINO_OK;
  }
  if (p->path == kPathHybrid) {
    void* V = ws;
    void* yp = ws + p->v_bytes;
    for (int ch = 0; ch < p->num_chunks; ++ch) {
      const int row0 = ch * p->rows_per_chunk;
      const int rows = (row0 + p->rows_per_chunk <= p->rows_total) ? p->rows_per_chunk
                                                                    : p->rows_total - row0;
      const long long Pc = static_cast<long long>(rows) * p->tw;
      cudaError_t e = launch_input_transform(p->m, p->prec, d, V, L.N, L.C, L.H, L.W, L.pad,
                                             p->th, p->tw, row0, rows, Pc, p->c_pad, s);
      if (e != cudaSuccess) return cuda_fail(e, "input transform");
      tm.mark(1);
      FusedArgs fa{d, U, V, y, yp, Pc, static_cast<long long>(row0) * p->tw, L.N, L.C, L.H, L.W,
                   L.K, L.pad, p->th, p->tw, p->oh, p->ow, p->c_pad, p->fsplits};
      e = join_filters();
      if (e != cudaSuccess) return cuda_fail(e, "filter transform join");
      e = launch_fused(p->m, p->prec, fa, s);
      if (e != cudaSuccess) {
        if (g_err.empty()) return cuda_fail(e, "fused winograd gemm");
        return WINO_ECUDA;
      }
      tm.mark(2);
    }
    return WINO_OK;
  }
  const size_t vm = p->v_bytes + p->m_bytes;
  for (int ch = 0; ch < p->num_chunks; ++ch) {
    const int row0 = ch * p->rows_per_chunk;
    const int rows = (row0 + p->rows_per_chunk <= p->rows_total) ? p->rows_per_chunk
                                                                  : p->rows_total - row0;
    const long long Pc = static_cast<long long>(rows) * p->tw;
    // chunk ch on stream ch % nbuf with V/M buffer ch % nbuf (stream order
    // serialises chunks that share a buffer; U precedes on `side`, and the
    // third stream waited for it at the fork)
    const int bi = (chunk_overlap && side) ? ch % nstreams : 0;
    const bool side_chunk = bi != 0;  // U reached its stream at the fork / in order
    cudaStream_t cs = bi == 0 ? s : bi == 1 ? side->st : side->st2;
    unsigned char* V = ws + bi * vm;
    unsigned char* Mb = V + p->v_bytes;
    cudaError_t e = cudaSuccess;
    if (!(input_enqueued && ch == 0)) {
      e = launch_input_transform(p->m, p->v_split2 ? kFP32S : p->prec, d, V, L.N, L.C, L.H, L.W, L.pad, p->th, p->tw,
                                 row0, rows, Pc, p->c_pad, cs);
      if (e != cudaSuccess) return cuda_fail(e, "input transform");
    }
    tm.mark(1);
    GemmArgs ga{V, U, Mb, p->a2, L.K, L.C, p->c_pad, Pc, p->bn, p->splits, p->m_ld, p->m_bf16,
                (u_split || p->v_split2) ? 1 : 0, p->gemm_tr};
    if (!side_chunk) {
      e = join_filters();
      if (e != cudaSuccess) return cuda_fail(e, "filter transform join");
    }
    e = launch_batched_gemm(p->prec, ga, cs);
    if (e != cudaSuccess) {
      if (g_err.empty()) return cuda_fail(e, "batched gemm");
      return WINO_ECUDA;
    }
    tm.mark(2);
    e = launch_output_transform(p->m, p->prec, Mb, y, L.N, L.K, p->th, p->tw, p->oh, p->ow, row0,
                                Pc, p->m_ld, p->splits, cs, p->m_bf16, V, p->v_bytes, act);
    if (e != cudaSuccess) return cuda_fail(e, "output transform");
    tm.mark(3);
  }
  if (side && (chunk_overlap || filt_side)) {  // join the side stream(s) back into `s`
    cudaError_t e = cudaEventRecord(side->join, side->st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, side->join, 0);
    if (e == cudaSuccess && nstreams == 3) {
      e = cudaEventRecord(side->join2, side->st2);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s, side->join2, 0);
    }
    if (e != cudaSuccess) return cuda_fail(e, "side stream join");
  }
  return WINO_OK;
}

int wino_forward(wino_plan_t p, const void* d, const void* U, const void* g, void* y,
                 void* workspace, size_t workspace_bytes, void* stream) {
  return forward_impl(p, d, U, g, y, workspace, workspace_bytes, stream, nullptr);
}

int wino_forward_act(wino_plan_t p, const void* d, const void* U, const void* g, void* y,
                     void* workspace, size_t workspace_bytes, int act, void* stream) {
  return forward_impl(p, d, U, g, y, workspace, workspace_bytes, stream, nullptr, act);
}

int wino_timer_create(wino_timer_t* out) {
  if (!out) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  wino_timer_s* t = new (std::nothrow) wino_timer_s();
  if (!t) return WINO_ENOMEM;
  for (int i = 0; i < wino_timer_s::kMax; ++i) {
    cudaError_t e = cudaEventCreate(&t->ev[i]);
    if (e != cudaSuccess) {
      for (int j = 0; j < i; ++j) cudaEventDestroy(t->ev[j]);
      delete t;
      return cuda_fail(e, "timer events");
    }
  }
  *out = t;
  return WINO_OK;
}

int wino_timer_destroy(wino_timer_t t) {
  if (t) {
    for (int i = 0; i < wino_timer_s::kMax; ++i) cudaEventDestroy(t->ev[i]);
    delete t;
  }
  return WINO_OK;
}

int wino_timer_break(wino_timer_t t) {
  if (!t) return WINO_EINVAL;
  t->open = false;  // the next timed forward starts a new sequence
  return WINO_OK;
}

int wino_timer_read(wino_timer_t t, float* stage_ms, int* launches) {
  if (!t || !stage_ms || !launches) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  if (t->n > 0) {
    cudaError_t e = cudaEventSynchronize(t->ev[t->n - 1]);
    if (e != cudaSuccess) return cuda_fail(e, "timer sync");
  }
  for (int i = 1; i < t->n; ++i) {
    if (t->stage[i] < 0) continue;  // sequence opener
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t->ev[i - 1], t->ev[i]);
    stage_ms[t->stage[i]] += ms;
    launches[t->stage[i]] += 1;
  }
  t->n = 0;
  t->open = false;
  return WINO_OK;
}

int wino_forward_timed(wino_plan_t p, const void* d, const void* U, const void* g, void* y,
                       void* workspace, size_t workspace_bytes, void* stream, wino_timer_t timer) {
  if (!timer) {
    set_error("null timer");
    return WINO_EINVAL;
  }
  return forward_impl(p, d, U, g, y, workspace, workspace_bytes, stream, timer);
}

int wino_forward_host(wino_plan_t p, const void* d_host, const void* U, const void* g,
                      void* y_host, void* d_dev, void* y_dev, void* workspace,
                      size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (!p || !d_host || !y_host || !d_dev || !y_dev) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const wino_layer_t& L = p->L;
  const size_t db = static_cast<size_t>(L.N) * L.C * L.H * L.W * p->acc_bytes;
  const size_t yb = static_cast<size_t>(L.N) * L.K * p->oh * p->ow * p->acc_bytes;
  cudaError_t e = cudaMemcpyAsync(d_dev, d_host, db, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
  int rc = wino_forward(p, d_dev, U, g, y_dev, workspace, workspace_bytes, stream);
  if (rc != WINO_OK) return rc;
  e = cudaMemcpyAsync(y_host, y_dev, yb, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
  return WINO_OK;
}

// ---------------------------------------------------------------- batch shards
// Multi-GPU from one host thread (SURVEY.md §8(b) wino_forward_sharded, §8(e)):
// images are independent, so shard s runs the layer on its contiguous images
// with a sub-plan of batch `count` on devices[s]; no data crosses devices.  The
// U layout depends only on (m, prec, K, C), so the full plan's filter
// transform serves every sub-plan.  Sub-plans are built per call (host-only
// planning) and freed before returning; kernels already enqueued keep running.
int wino_shard_bounds(int N, int n_shards, int shard, int* start, int* count) {
  g_err.clear();
  if (!start || !count) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  if (n_shards < 1 || shard < 0 || shard >= n_shards) {
    set_error("bad shard %d of %d", shard, n_shards);
    return WINO_EINVAL;
  }
  if (N < 0) {
    set_error("N must be >= 0");
    return WINO_EINVAL;
  }
  const int base = N / n_shards, extra = N % n_shards;  // sharding.shard_bounds
  *start = shard * base + (shard < extra ? shard : extra);
  *count = base + (shard < extra ? 1 : 0);
  return WINO_OK;
}

static int shard_plan(wino_plan_t p, int n_shards, int shard, wino_plan_t* sub) {
  *sub = nullptr;
  int start = 0, count = 0;
  int rc = wino_shard_bounds(p->L.N, n_shards, shard, &start, &count);
  if (rc != WINO_OK || count == 0) return rc;
  wino_layer_t L = p->L;
  L.N = count;
  return wino_plan_create(&L, p->m, p->prec, p->ws_limit, sub);
}

int wino_shard_workspace(wino_plan_t p, int n_shards, int shard, int with_filters,
                         size_t* bytes) {
  g_err.clear();
  if (!p || !bytes) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  wino_plan_t sub = nullptr;
  const int rc = shard_plan(p, n_shards, shard, &sub);
  if (rc != WINO_OK) return rc;
  *bytes = 0;
  if (sub) {
    *bytes = with_filters ? sub->u_ws + sub->nbuf * (sub->v_bytes + sub->m_bytes) + sub->ypart_bytes
                          : sub->staging_bytes;
    wino_plan_destroy(sub);
  }
  return WINO_OK;
}

int wino_forward_sharded(wino_plan_t p, int n_shards, const int* devices,
                         const void* const* d, const void* const* U, const void* const* g,
                         void* const* y, void* const* workspace, const size_t* workspace_bytes,
                         void* const* streams) {
  g_err.clear();
  if (!p || n_shards < 1 || !devices || !d || !y || !workspace || !workspace_bytes ||
      (!U && !g)) {
    set_error("null argument or n_shards < 1");
    return WINO_EINVAL;
  }
  int dev0 = 0;
  cudaError_t e = cudaGetDevice(&dev0);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int rc = WINO_OK;
  for (int s = 0; s < n_shards && rc == WINO_OK; ++s) {
    e = cudaSetDevice(devices[s]);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "cudaSetDevice");
      break;
    }
    wino_plan_t sub = nullptr;
    rc = shard_plan(p, n_shards, s, &sub);
    if (rc != WINO_OK || !sub) continue;  // error, or a shard without images
    rc = forward_impl(sub, d[s], U ? U[s] : nullptr, g ? g[s] : nullptr, y[s], workspace[s],
                      workspace_bytes[s], streams ? streams[s] : nullptr, nullptr);
    wino_plan_destroy(sub);
    if (rc != WINO_OK) {
      const std::string msg = g_err;
      set_error("shard %d (device %d): %s", s, devices[s], msg.c_str());
    }
  }
  e = cudaSetDevice(dev0);
  if (rc == WINO_OK && e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  return rc;
}

// ---------------------------------------------------------------- weight gradient
// dL/dg via F(3x3, 2x2) (engine.py:278-328): transforms of dY tiles (Uw) and
// input patches (Vw) with the tile index innermost, the 16 tile-reduction
// GEMMs on the same tcgen05 kernel as the forward (reduction axis = tiles),
// and one inverse transform per (k, c).  Tiles are processed in chunks that
// fit the workspace budget; every chunk x split writes its own M slice and the
// inverse transform sums the slices in order (deterministic).
namespace {
struct WgPlan {
  int oh, ow, gh, gw;
  long long B, nb, b_pad;
  int nchunks, esize, nsplit, acc_bytes, bn, splits;
  int total_slices;  // M slices over all chunks (keep_all) -- each chunk's effective splits
  int keep_all;      // every chunk keeps its own slices; else a running sum is folded per chunk
  int smallc;        // C <= 4: one CUDA-core pass (wgrad_smallc_kernel), no staging
  int nblk;          // smallc: blocks = M slices
  long long m_ld;
  size_t u_bytes, v_bytes, m_bytes, slice_bytes;
};
// 1 GB: VGG-E layers at N = 8 run as one tile chunk (no per-chunk wave tails).
constexpr size_t kWgradDefaultWorkspace = 1ull << 30;

// Split count the GEMM actually runs for a chunk of nb tiles: the last split
// never ends up empty (the kernel's epilogue needs at least one k-block).
int wgrad_effective_splits(int prec, long long nb, int splits) {
  const int nkb = gemm_num_kblocks(prec, static_cast<int>(nb));
  if (splits <= 1 || nkb <= 1) return 1;
  const int kbps = (nkb + splits - 1) / splits;
  return (nkb + kbps - 1) / kbps;
}

int wgrad_plan(const wino_layer_t* layer, int prec, size_t limit, WgPlan* w) {
  if (!layer) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  const wino_layer_t& L = *layer;
  if (L.N < 1 || L.C < 1 || L.H < 1 || L.W < 1 || L.K < 1 || L.R < 1 || L.S < 1 || L.pad < 0) {
    set_error("N, C, H, W, K, R, S must be >= 1 and pad >= 0");
    return WINO_EINVAL;
  }
  if (L.R != 3 || L.S != 3) {  // engine.py:292-295
    set_error("default weight-gradient algorithm needs R=S=3, got %dx%d", L.R, L.S);
    return WINO_EUNSUPPORTED;
  }
  if (prec < WINO_PREC_FP32 || prec > WINO_PREC_FP64) {
    set_error("unknown precision %d", prec);
    return WINO_EINVAL;
  }
  w->oh = L.H + 2 * L.pad - 2;
  w->ow = L.W + 2 * L.pad - 2;
  if (w->oh < 1 || w->ow < 1) {
    set_error("output dimensions must be >= 1");
    return WINO_EINVAL;
  }
  w->gh = (w->oh + 1) / 2;
  w->gw = (w->ow + 1) / 2;
  w->B = static_cast<long long>(L.N) * w->gh * w->gw;
  w->esize = op_bytes(prec);
  w->nsplit = op_splits(prec);
  w->acc_bytes = prec == kFP64 ? 8 : 4;
  const size_t budget = limit ? limit : kWgradDefaultWorkspace;
  size_t stage = budget;  // Uw + Vw bytes per tile chunk
  if (const char* e = getenv("WINO_WGRAD_CHUNK_MB")) {  // tuning override
    const size_t v = static_cast<size_t>(atoll(e)) << 20;
    if (v > 0 && v < stage) stage = v;
  }
  const size_t per_tile = static_cast<size_t>(w->nsplit) * 16 * (L.K + L.C) * w->esize;
  long long nb = static_cast<long long>(stage / per_tile);
  if (nb < 64) nb = 64;
  if (nb >= w->B) nb = w->B;
  else nb = nb / 64 * 64;
  w->nb = nb;
  w->nchunks = static_cast<int>((w->B + nb - 1) / nb);
  w->b_pad = static_cast<long long>(align_up(static_cast<size_t>(nb), 16 / w->esize));
  int bn = prec == kFP32 ? 128 : 256;
  while (bn > 32 && bn / 2 >= L.K) bn /= 2;
  w->bn = bn;
  w->m_ld = static_cast<long long>(align_up(static_cast<size_t>(L.C), 4));
  w->slice_bytes = static_cast<size_t>(16) * L.K * w->m_ld * w->acc_bytes;
  // Split the tile reduction so the GEMM's work units fill whole waves: cost =
  // waves x (k-steps per unit + 2 for fill and epilogue) + each slice's HBM
  // write and re-read (~3 MB per k-step); ties -> fewer splits.
  w->splits = 1;
  if (prec != kFP64) {
    const int sms = gemm_device_sms();
    const int num_kb = gemm_num_kblocks(prec, static_cast<int>(nb));
    const long long units = ((L.C + 127) / 128) * ((L.K + bn - 1) / bn) * 16LL;
    const double slice_cost = 2.0 * static_cast<double>(w->slice_bytes) / 3e6;
    double best = 1e30;
    for (int sp = 1; sp <= num_kb && sp <= 512; ++sp) {
      const int kbps = (num_kb + sp - 1) / sp;
      const int sp_eff = (num_kb + kbps - 1) / kbps;
      if (sp_eff != sp) continue;
      const long long waves = (units * sp + sms - 1) / sms;
      const double cost = static_cast<double>(waves) * (kbps + 2) + sp * slice_cost;
      if (cost < best - 1e-9) {
        best = cost;
        w->splits = sp;
      }
    }
    if (const char* e = getenv("WINO_WGRAD_SPLITS")) {  // tuning override
      const int v = atoi(e);
      if (v >= 1 && v <= num_kb) w->splits = wgrad_effective_splits(prec, nb, v);
    }
  }
  // C <= 4: the tensor-core GEMM would waste 125 of 128 rows and stage 16 x K
  // values per tile through HBM; the small-C kernel reads d and dY once
  w->smallc = (L.C <= 4 && prec != kFP64 && w->B < (1LL << 31) - 64 &&
               static_cast<long long>(w->oh) * w->ow * 64 < (1LL << 31) &&  // 32-bit load offsets
               !getenv("WINO_NO_WGRAD_SMALLC")) ? 1 : 0;
  if (w->smallc) {
    const long long groups = (w->B + 31) / 32;
    const int per_y = (2 * gemm_device_sms()) / ((L.K + 63) / 64);
    w->nblk = static_cast<int>(groups < per_y ? groups : (per_y > 0 ? per_y : 1));
    w->nb = w->B;
    w->nchunks = 1;
    w->splits = 1;
    w->total_slices = w->nblk;
    w->keep_all = 1;
    w->u_bytes = w->v_bytes = 0;
    w->m_bytes = align_up(static_cast<size_t>(w->nblk + 1) * w->slice_bytes, 1024);
    return WINO_OK;
  }
  w->nblk = 0;
  w->total_slices = 0;
  for (int ch = 0; ch < w->nchunks; ++ch) {
    const long long b0 = static_cast<long long>(ch) * nb;
    w->total_slices += wgrad_effective_splits(prec, b0 + nb <= w->B ? nb : w->B - b0, w->splits);
  }
  w->keep_all = (w->nchunks == 1 ||
                 static_cast<size_t>(w->total_slices) * w->slice_bytes <= budget / 4) ? 1 : 0;
  w->u_bytes = align_up(static_cast<size_t>(w->nsplit) * 16 * L.K * w->b_pad * w->esize, 1024);
  w->v_bytes = align_up(static_cast<size_t>(w->nsplit) * 16 * L.C * w->b_pad * w->esize, 1024);
  // keep_all: every chunk's split slices, summed once by the inverse transform;
  // else one chunk's slices plus a running sum folded after every chunk
  // (bounded memory).  Either way the slices are summed in one fixed order.
  w->m_bytes = align_up((w->keep_all ? static_cast<size_t>(w->total_slices)
                                     : static_cast<size_t>(w->splits + 1)) * w->slice_bytes,
                        1024);
  return WINO_OK;
}
}  // namespace

int wino_wgrad_workspace(const wino_layer_t* layer, int prec, size_t workspace_limit,
                         size_t* bytes) {
  g_err.clear();
  if (!bytes) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  WgPlan w;
  const int rc = wgrad_plan(layer, prec, workspace_limit, &w);
  if (rc != WINO_OK) return rc;
  *bytes = w.u_bytes + w.v_bytes + w.m_bytes;
  return WINO_OK;
}

int wino_direct_forward(const wino_layer_t* layer, int in_prec, int acc_prec, const void* d,
                        const void* g, void* y, void* stream) {
  g_err.clear();
  if (!layer || !d || !g || !y) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  const wino_layer_t& L = *layer;
  if (L.N < 1 || L.C < 1 || L.H < 1 || L.W < 1 || L.K < 1 || L.R < 1 || L.S < 1 || L.pad < 0) {
    set_error("N, C, H, W, K, R, S must be >= 1 and pad >= 0");
    return WINO_EINVAL;
  }
  if ((in_prec != kFP32 && in_prec != kFP64) || (acc_prec != kFP32 && acc_prec != kFP64)) {
    set_error("accumulator precision must be fp32 or fp64");  // direct.py:76-79
    return WINO_EINVAL;
  }
  const int oh = L.H + 2 * L.pad - L.R + 1, ow = L.W + 2 * L.pad - L.S + 1;
  if (oh < 1 || ow < 1) {
    set_error("output dimensions must be >= 1");
    return WINO_EINVAL;
  }
  cudaError_t e = launch_direct(in_prec, acc_prec, d, g, y, L.N, L.C, L.H, L.W, L.K, L.R, L.S,
                                L.pad, oh, ow, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? WINO_OK : cuda_fail(e, "direct convolution");
}

int wino_grad_weights(const wino_layer_t* layer, int prec, const void* d, const void* dy,
                      void* dg, void* workspace, size_t workspace_bytes, size_t workspace_limit,
                      void* stream) {
  g_err.clear();
  if (!d || !dy || !dg || !workspace) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  WgPlan w;
  int rc = wgrad_plan(layer, prec, workspace_limit, &w);
  if (rc != WINO_OK) return rc;
  if (workspace_bytes < w.u_bytes + w.v_bytes + w.m_bytes) {
    set_error("workspace too small: %zu < %zu bytes", workspace_bytes,
              w.u_bytes + w.v_bytes + w.m_bytes);
    return WINO_EINVAL;
  }
  const wino_layer_t& L = *layer;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  void* Uw = ws;
  void* Vw = ws + w.u_bytes;
  unsigned char* Mb = ws + w.u_bytes + w.v_bytes;
  const size_t slice = w.slice_bytes;
  if (w.smallc) {
    unsigned char* summed = Mb + static_cast<size_t>(w.nblk) * slice;
    cudaError_t e = launch_wgrad_smallc(prec, d, dy, Mb, summed, L.K, L.C, L.H, L.W, L.pad, w.oh,
                                        w.ow, w.gh, w.gw, w.B, w.m_ld, w.nblk, s);
    if (e != cudaSuccess) return cuda_fail(e, "small-C weight gradient");
    e = launch_wgrad_inverse(prec, summed, dg, L.K, L.C, w.m_ld, 1, s);
    if (e != cudaSuccess) return cuda_fail(e, "weight-gradient inverse transform");
    return WINO_OK;
  }
  unsigned char* acc = Mb;  // running sum (fold mode)
  int slot = 0;             // keep_all: next free slice
  for (int ch = 0; ch < w.nchunks; ++ch) {
    const long long b0 = static_cast<long long>(ch) * w.nb;
    const long long nb = (b0 + w.nb <= w.B) ? w.nb : w.B - b0;
    const int sp = wgrad_effective_splits(prec, nb, w.splits);
    unsigned char* parts = w.keep_all ? Mb + static_cast<size_t>(slot) * slice : Mb + slice;
    cudaError_t e = launch_wgrad_transforms(prec, d, dy, Uw, Vw, L.K, L.C, L.H, L.W, L.pad, w.oh,
                                            w.ow, w.gh, w.gw, b0, nb, w.b_pad, s);
    if (e != cudaSuccess) return cuda_fail(e, "weight-gradient transforms");
    // M[comp][k][c] = sum_b Uw[comp][k][b] Vw[comp][c][b]: the forward GEMM with
    // (rows = C, reduction = tiles), partial sums in `sp` slices
    GemmArgs ga{Vw, Uw, parts, 16, L.K, static_cast<int>(nb), static_cast<int>(w.b_pad), L.C,
                w.bn, sp, w.m_ld};
    e = launch_batched_gemm(prec, ga, s);
    if (e != cudaSuccess) {
      if (g_err.empty()) return cuda_fail(e, "weight-gradient gemm");
      return WINO_ECUDA;
    }
    slot += sp;
    if (!w.keep_all) {
      e = launch_wgrad_accumulate(prec, acc, parts, static_cast<long long>(16) * L.K * w.m_ld, sp,
                                  ch == 0 ? 1 : 0, s);
      if (e != cudaSuccess) return cuda_fail(e, "weight-gradient accumulate");
    }
  }
  cudaError_t e = launch_wgrad_inverse(prec, Mb, dg, L.K, L.C, w.m_ld,
                                       w.keep_all ? w.total_slices : 1, s);
  if (e != cudaSuccess) return cuda_fail(e, "weight-gradient inverse transform");
  return WINO_OK;
}

}  // extern "C"
