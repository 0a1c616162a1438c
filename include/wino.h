/*
 * wino.h -- C ABI of the B200 Winograd fast-convolution path (libwino.so).
 *
 * This is the drop-in boundary for the reference's hot path
 *   winoconv.engine.winograd_forward(d, g, cfg, alg, cache_filters, counter, cache)
 *   (/root/reference/pkg/src/winoconv/engine.py:198-254)
 * and its helpers.  Plain C: opaque plan handle, caller-owned DEVICE pointers
 * (except wino_forward_host), int status codes, a thread-local error string.
 * No CUDA or torch types appear in the signatures; streams are passed as
 * `void*` (a cudaStream_t / CUstream, NULL = legacy default stream).
 *
 * Status codes map onto the reference's exception types:
 *   WINO_OK           0
 *   WINO_EINVAL       1  -> ValueError   (shape/cfg mismatch, engine.py:211-218;
 *                                         LayerConfig validation, direct.py:48-55)
 *   WINO_EUNSUPPORTED 2  -> KeyError / ValueError (no builtin F(m,r), winograd.py:227-231;
 *                                         R != alg.r, engine.py:217-218)
 *   WINO_ENOMEM       3  -> MemoryError  (cmd_bench skips the row, commands.py:169-171)
 *   WINO_ECUDA        4  -> RuntimeError
 *
 * Thread-safety: plans are immutable after creation; every call is reentrant
 * across host threads and streams.  Global state: the thread-local error
 * string, a once-initialised driver entry point, and per-(kernel, device)
 * "attributes set" flags and SM counts (atomics; setting them is idempotent),
 * so one process may drive several GPUs (cudaSetDevice before each call).
 */
#ifndef WINO_H_
#define WINO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WINO_OK 0
#define WINO_EINVAL 1
#define WINO_EUNSUPPORTED 2
#define WINO_ENOMEM 3
#define WINO_ECUDA 4

/* Arithmetic of the alpha^2 transform-space GEMMs.  Transforms always run in
 * the data type (fp32, or fp64 for WINO_PREC_FP64); accumulation is fp32
 * (fp64 for WINO_PREC_FP64). */
#define WINO_PREC_FP32 0 /* 3xTF32 split operands on tcgen05: fp32-accurate   */
#define WINO_PREC_TF32 1 /* single-pass TF32 on tcgen05                        */
#define WINO_PREC_BF16 2 /* bf16 operands on tcgen05 kind::f16; M staged as bf16 */
#define WINO_PREC_FP16 3 /* fp16 operands on tcgen05 kind::f16; M staged as fp16
                            of M * 2^-4 (|M| < 2^20); both keep fp32 M on
                            split-C plans and the transposed (K > P) GEMM       */
#define WINO_PREC_FP64 4 /* fp64 data and GEMM on CUDA cores (reference FP64)  */

/* One convolution layer; mirrors winoconv.direct.LayerConfig (direct.py:32-66).
 * Output is (N, K, H+2*pad-R+1, W+2*pad-S+1). */
typedef struct {
  int N, C, H, W, K, R, S, pad;
} wino_layer_t;

typedef struct wino_plan_s* wino_plan_t;

typedef struct {
  int m, r, alpha;            /* F(m x m, r x r)                                 */
  int out_h, out_w;
  int tiles_h, tiles_w;       /* ceil(out/m)  (engine.py:57-61)                  */
  long long P;                /* N * tiles_h * tiles_w  (engine.py:67-69)        */
  int prec, c_pad, op_bytes, op_splits;
  int gemm_bn;                /* filters per GEMM CTA (tcgen05 N)                */
  int gemm_splits;            /* split-C factor of the GEMM (small-P layers)     */
  int rows_per_chunk;         /* tile rows per workspace chunk                   */
  int num_chunks;
  long long chunk_tiles;      /* tiles per full chunk                            */
  size_t u_bytes;             /* transformed-filter stack U                      */
  size_t workspace_bytes;     /* V + M for one chunk (+ U when g is passed)      */
  int launches_per_forward;   /* kernels launched by one wino_forward (U given)  */
  int fused_small_c;          /* 1: C <= 8, whole layer in one fused kernel      */
  long long multiplies;       /* P*C*K*alpha^2: the reference "mul" counter      */
  int fused;                  /* 1: fused Winograd-GEMM kernel (no V/M staging)  */
  int fused_splits;           /* split-C factor of the fused kernel              */
  int m_bytes_per_elem;       /* staged M element: 4 (fp32), 2 (bf16 GEMM), 8   */
  int combined_transforms;    /* non-FX forwards launch filter+input together   */
  size_t staging_bytes;       /* transform-space staging (V + M of the chunks in
                                 flight): all an FX forward (U passed) needs;
                                 <= workspace_limit when one is given            */
} wino_plan_info_t;

/* Create a plan.  m in {2,4} (F(2x2,3x3), F(4x4,3x3)); R == S == 3.
 * workspace_limit: hard cap in bytes on the transform-space staging (V + M of
 * the chunks in flight; see staging_bytes).  0 = default budget of 128 MiB,
 * sized to stay L2-resident.  The tile/workspace planner splits the tile grid
 * into row chunks that fit and reduces split-C when its partial sums would
 * not; 16 MiB is the paper's workspace bound.  A limit
 * smaller than one tile row's staging still plans one row per chunk. */
int wino_plan_create(const wino_layer_t* layer, int m, int prec, size_t workspace_limit,
                     wino_plan_t* out);
int wino_plan_destroy(wino_plan_t plan);
int wino_plan_get_info(wino_plan_t plan, wino_plan_info_t* info);

/* U[s][xi*alpha+nu][k][c] = (G g_kc G^T)[xi,nu] split into op_splits planes,
 * c padded to c_pad.  Replaces transform_filters (engine.py:104-114); the FX
 * cache (engine.py:117-160) stores this buffer.  g is (K,C,3,3) fp32/fp64. */
int wino_filter_transform(wino_plan_t plan, const void* g, void* U, void* stream);

/* Full layer forward, replaces winograd_forward (engine.py:198-254).
 * d: (N,C,H,W) fp32 (fp64 for WINO_PREC_FP64) device pointer.
 * U: precomputed wino_filter_transform output, or NULL to transform g here
 *    (g must then be non-NULL; the U stack lives in the workspace).
 * y: (N,K,out_h,out_w) output, fully written (every element).
 * workspace: >= info.workspace_bytes (U==NULL) or >= info.staging_bytes (U given). */
int wino_forward(wino_plan_t plan, const void* d, const void* U, const void* g, void* y,
                 void* workspace, size_t workspace_bytes, void* stream);

/* End-to-end variant with HOST data: copies d_host -> d_dev, runs
 * wino_forward, copies y_dev -> y_host, all on `stream` (pin the host buffers
 * for asynchronous copies).  Returns after enqueueing. */
int wino_forward_host(wino_plan_t plan, const void* d_host, const void* U, const void* g,
                      void* y_host, void* d_dev, void* y_dev, void* workspace,
                      size_t workspace_bytes, void* stream);

/* Stage timer (diagnostics / bench): wino_forward_timed enqueues the same
 * forward plus one CUDA event after every launch on `stream`, without any host
 * synchronisation.  wino_timer_read synchronises on the last event and ADDS
 * each stage's device time (ms) to stage_ms[0..3] = {filter transform, input
 * transform, GEMM, output transform} and its launch count to launches[0..3],
 * then resets the timer.  wino_timer_break marks a gap (e.g. an unrelated
 * kernel enqueued between two timed forwards) so it is not attributed. */
typedef struct wino_timer_s* wino_timer_t;
int wino_timer_create(wino_timer_t* out);
int wino_timer_destroy(wino_timer_t timer);
int wino_timer_break(wino_timer_t timer);
int wino_timer_read(wino_timer_t timer, float* stage_ms, int* launches);
int wino_forward_timed(wino_plan_t plan, const void* d, const void* U, const void* g, void* y,
                       void* workspace, size_t workspace_bytes, void* stream, wino_timer_t timer);

/* Last error message of the calling thread ("" if none). */
/* Weight gradient dL/dg by the F(3x3, 2x2) decomposition; replaces
 * winoconv.engine.winograd_grad_weights (engine.py:278-328).
 * d: (N,C,H,W), dy: (N,K,out_h,out_w), dg: (K,C,3,3) -- device pointers in the
 * data type (fp32, or fp64 for WINO_PREC_FP64).  R == S == 3 (else
 * WINO_EUNSUPPORTED, the reference's ValueError).  workspace_limit bounds the
 * tile-chunk staging (0 = default); wino_wgrad_workspace returns the bytes a
 * call with the same arguments needs.  Enqueued on `stream`. */
int wino_wgrad_workspace(const wino_layer_t* layer, int prec, size_t workspace_limit,
                         size_t* bytes);
int wino_grad_weights(const wino_layer_t* layer, int prec, const void* d, const void* dy,
                      void* dg, void* workspace, size_t workspace_bytes, size_t workspace_limit,
                      void* stream);

/* Direct correlation with zero padding (any R x S), the reference's `direct` /
 * `direct-fp32` algorithms and cmd_accuracy's fp64 oracle (direct.py:82-114):
 * accumulation order c, v, u with a rounded multiply then a rounded add in the
 * accumulator precision, so the output is bitwise the reference's.
 * in_prec / acc_prec: WINO_PREC_FP32 or WINO_PREC_FP64 (d, g in in_prec; y in
 * acc_prec).  Device pointers, enqueued on `stream`. */
int wino_direct_forward(const wino_layer_t* layer, int in_prec, int acc_prec, const void* d,
                        const void* g, void* y, void* stream);

/* FFT overlap-and-save correlation, the reference's `fft` comparison algorithm
 * (fftconv.py:206-275), fp64 arithmetic on hand-written kernels: tile 8 (the
 * only size run_layer uses; others -> WINO_EUNSUPPORTED).  prec: WINO_PREC_FP32
 * or WINO_PREC_FP64 for d / y; g is (K,C,R,S) fp64.  Device pointers. */
int wino_fft_workspace(const wino_layer_t* layer, int tile, size_t* bytes);
int wino_fft_forward(const wino_layer_t* layer, int prec, int tile, const void* d,
                     const double* g, void* y, void* workspace, size_t workspace_bytes,
                     void* stream);

/* wino_forward with an activation fused into the output transform's stores
 * (not on the reference's path; the chained VGG-E stack uses it):
 * WINO_ACT_NONE, WINO_ACT_RELU (y = max(conv, 0)), or WINO_ACT_RELU_POOL
 * (y = 2x2 / stride-2 max-pool of max(conv, 0): y is (N, K, out_h/2, out_w/2),
 * out_h and out_w even).  Staged path (and the small-C layer) only:
 * WINO_EUNSUPPORTED on the fused / hybrid paths. */
#define WINO_ACT_NONE 0
#define WINO_ACT_RELU 1
#define WINO_ACT_RELU_POOL 2
int wino_forward_act(wino_plan_t plan, const void* d, const void* U, const void* g, void* y,
                     void* workspace, size_t workspace_bytes, int act, void* stream);

/* Chaining glue for the VGG-E conv stack (network.py; not on the reference's
 * path): y = relu(x), or relu(maxpool2x2(x)) with pool != 0 (H, W even;
 * y is (N,C,H/2,W/2)).  fp32 device pointers, enqueued on `stream`. */
int wino_relu_pool(const float* x, float* y, int N, int C, int H, int W, int pool, void* stream);

/* Batch shards over several GPUs from one host thread (SURVEY.md §8(b)
 * `wino_forward_sharded`, §8(e); the one-process-per-GPU torch.distributed
 * driver is sharding.py).  Images are independent: shard s of n_shards holds
 * the contiguous images [start, start + count) of the plan's N -- the first
 * N % n_shards shards take one extra, as sharding.shard_bounds -- and runs on
 * devices[s].  No data crosses devices (outputs stay sharded, no collective). */
int wino_shard_bounds(int N, int n_shards, int shard, int* start, int* count);
/* Bytes shard s's workspace needs: with_filters != 0 for a forward that
 * transforms g itself, 0 when U is passed.  0 for a shard without images. */
int wino_shard_workspace(wino_plan_t plan, int n_shards, int shard, int with_filters,
                         size_t* bytes);
/* Enqueue every shard's forward of `plan` (the full layer).  Per shard s, on
 * devices[s] (several shards may share a device): d[s] (count, C, H, W),
 * y[s] (count, K, out_h, out_w), U[s] = wino_filter_transform(plan, ...) on that
 * device, or U == NULL and g[s] (K, C, 3, 3); workspace[s] of
 * workspace_bytes[s] >= wino_shard_workspace; streams[s] (streams == NULL:
 * each device's legacy stream).  Shards without images are skipped (their
 * pointers may be NULL).  The calling thread's current device is restored.
 * Returns after enqueueing; on error the message names the shard. */
int wino_forward_sharded(wino_plan_t plan, int n_shards, const int* devices,
                         const void* const* d, const void* const* U, const void* const* g,
                         void* const* y, void* const* workspace, const size_t* workspace_bytes,
                         void* const* streams);

const char* wino_last_error(void);
/* Library version string. */
const char* wino_version(void);

#ifdef __cplusplus
}
#endif

#endif /* WINO_H_ */
