// Tiled FFT overlap-and-save convolution: the reference's `fft` comparison
// algorithm (winoconv/fftconv.py:206-275, paper sec. 4.4) in fp64 on the GPU,
// with hand-written kernels (no cuFFT / cuBLAS):
//   fft_filter_kernel  : h = reversed g zero-padded to a x a, ghat = DFT2(h),
//                        Hermitian-unique half (a x (a/2+1)) -> U[q][k][c]
//   fft_data_kernel    : zero-filled a x a tiles at (mh*ty - pad, mw*tx - pad)
//                        (virtual padding), DFT2 -> V[q][c][p]
//   fft_cgemm_kernel   : M[q][k][p] = sum_c U[q][k][c] V[q][c][p]   (complex fp64)
//   fft_inverse_kernel : Hermitian completion, inverse DFT2, the wraparound-free
//                        [R-1, a) x [S-1, a) block, clipped scatter into y.
// The DFTs are evaluated directly with a twiddle table (a = 8 or 16: 3-5
// radix-2 stages would save little at these sizes).  Everything is fp64, like
// the reference (numpy complex128); the output is cast to the input type.
#include <cuda_runtime.h>

#include <cstdio>

#include "wino_internal.h"

namespace wino {

// exp(-2 pi i j / a), j < a (correctly rounded literals)
__constant__ double2 c_tw8[8] = {
    {1.0, 0.0},
    {0.7071067811865476, -0.7071067811865475},
    {0.0, -1.0},
    {-0.7071067811865475, -0.7071067811865476},
    {-1.0, 0.0},
    {-0.7071067811865477, 0.7071067811865475},
    {0.0, 1.0},
    {0.7071067811865474, 0.7071067811865477}};
__constant__ double2 c_tw16[16] = {
    {1.0, 0.0},
    {0.9238795325112867, -0.3826834323650898},
    {0.7071067811865476, -0.7071067811865475},
    {0.38268343236508984, -0.9238795325112867},
    {0.0, -1.0},
    {-0.3826834323650897, -0.9238795325112867},
    {-0.7071067811865475, -0.7071067811865476},
    {-0.9238795325112867, -0.3826834323650899},
    {-1.0, 0.0},
    {-0.9238795325112868, 0.38268343236508967},
    {-0.7071067811865477, 0.7071067811865475},
    {-0.38268343236509034, 0.9238795325112865},
    {0.0, 1.0},
    {0.38268343236509, 0.9238795325112866},
    {0.7071067811865474, 0.7071067811865477},
    {0.9238795325112865, 0.3826834323650904}};

template <int A>
__device__ __forceinline__ double2 tw(int j) {
  if constexpr (A == 8)
    return c_tw8[j & 7];
  else
    return c_tw16[j & 15];
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}

// Forward 2D DFT of a real a x a block, streamed one input row at a time:
// X[r][s] = sum_u w^(r u) F[u][s],  F[u][s] = sum_v x[u][v] w^(s v),  s <= a/2.
// `row(u, xr)` fills input row u.  Keeps only X (a x (a/2+1) complex) live.
template <int A, typename RowFn>
__device__ __forceinline__ void dft2_real_rows(RowFn row, double2 (&X)[A][A / 2 + 1]) {
  constexpr int H = A / 2 + 1;
#pragma unroll
  for (int r = 0; r < A; ++r)
#pragma unroll
    for (int s = 0; s < H; ++s) X[r][s] = make_double2(0.0, 0.0);
#pragma unroll
  for (int u = 0; u < A; ++u) {
    double xr[A];
    row(u, xr);
#pragma unroll
    for (int s = 0; s < H; ++s) {
      double2 f = make_double2(0.0, 0.0);
#pragma unroll
      for (int v = 0; v < A; ++v) {
        const double2 w = tw<A>(s * v);
        f.x = fma(xr[v], w.x, f.x);
        f.y = fma(xr[v], w.y, f.y);
      }
#pragma unroll
      for (int r = 0; r < A; ++r) X[r][s] = cadd(X[r][s], cmul(f, tw<A>(r * u)));
    }
  }
}

template <int A>
__global__ void __launch_bounds__(128) fft_filter_kernel(const double* __restrict__ g,
                                                         double2* __restrict__ U, int K, int C,
                                                         int R, int S) {
  constexpr int H = A / 2 + 1;
  griddep_launch();
  griddep_wait();
  const long long kc = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (kc >= static_cast<long long>(K) * C) return;
  const double* gk = g + kc * R * S;
  double2 X[A][H];
  // reversed filter zero-padded to a x a: cyclic convolution realises correlation
  dft2_real_rows<A>(
      [&](int u, double (&xr)[A]) {
#pragma unroll
        for (int v = 0; v < A; ++v)
          xr[v] = (u < R && v < S) ? gk[(R - 1 - u) * S + (S - 1 - v)] : 0.0;
      },
      X);
  const long long KC = static_cast<long long>(K) * C;
#pragma unroll
  for (int r = 0; r < A; ++r)
#pragma unroll
    for (int s = 0; s < H; ++s) U[(r * H + s) * KC + kc] = X[r][s];
}

template <int A, typename T>
__global__ void __launch_bounds__(128) fft_data_kernel(const T* __restrict__ d,
                                                       double2* __restrict__ V, int N, int C,
                                                       int Hh, int W, int pad, int mh, int mw,
                                                       int gh, int gw) {
  constexpr int H = A / 2 + 1;
  griddep_launch();
  griddep_wait();
  const long long P = static_cast<long long>(N) * gh * gw;
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P * C) return;
  const long long p = i % P;  // p fastest: a warp's stores are contiguous
  const int c = static_cast<int>(i / P);
  const int n = static_cast<int>(p / (static_cast<long long>(gh) * gw));
  const int t = static_cast<int>(p % (static_cast<long long>(gh) * gw));
  const int ty = t / gw, tx = t % gw;
  const int y0 = mh * ty - pad, x0 = mw * tx - pad;
  const T* plane = d + (static_cast<size_t>(n) * C + c) * Hh * W;
  double2 X[A][H];
  dft2_real_rows<A>(
      [&](int u, double (&xr)[A]) {
        const int yy = y0 + u;
        const bool rok = yy >= 0 && yy < Hh;
#pragma unroll
        for (int v = 0; v < A; ++v) {
          const int xx = x0 + v;
          xr[v] = (rok && xx >= 0 && xx < W)
                      ? static_cast<double>(plane[static_cast<size_t>(yy) * W + xx])
                      : 0.0;
        }
      },
      X);
  const long long CP = static_cast<long long>(C) * P;
#pragma unroll
  for (int r = 0; r < A; ++r)
#pragma unroll
    for (int s = 0; s < H; ++s) V[(r * H + s) * CP + static_cast<long long>(c) * P + p] = X[r][s];
}

// Complex fp64 GEMM per frequency q: 32 x 32 (k, p) block per 256 threads,
// each thread 2 x 2 outputs; channels staged 16 at a time in shared memory.
constexpr int kFB = 32, kFC = 16;
__global__ void __launch_bounds__(256) fft_cgemm_kernel(const double2* __restrict__ U,
                                                        const double2* __restrict__ V,
                                                        double2* __restrict__ M, int K, int C,
                                                        long long P) {
  griddep_launch();
  griddep_wait();
  __shared__ double2 su[kFC][kFB + 1];
  __shared__ double2 sv[kFC][kFB + 1];
  const int q = blockIdx.z;
  const int k0 = blockIdx.y * kFB;
  const long long p0 = static_cast<long long>(blockIdx.x) * kFB;
  const double2* Uq = U + static_cast<long long>(q) * K * C;
  const double2* Vq = V + static_cast<long long>(q) * C * P;
  const int tid = threadIdx.x, tk = tid / 16, tp = tid % 16;
  double2 acc[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b] = make_double2(0.0, 0.0);
  for (int c0 = 0; c0 < C; c0 += kFC) {
    for (int e = tid; e < kFC * kFB; e += 256) {
      const int cc = e / kFB, j = e % kFB;
      const int k = k0 + j, c = c0 + cc;
      su[cc][j] = (k < K && c < C) ? Uq[static_cast<long long>(k) * C + c] : make_double2(0, 0);
      const long long p = p0 + j;
      sv[cc][j] = (p < P && c < C) ? Vq[static_cast<long long>(c) * P + p] : make_double2(0, 0);
    }
    __syncthreads();
#pragma unroll
    for (int cc = 0; cc < kFC; ++cc) {
      const double2 u0 = su[cc][tk], u1 = su[cc][tk + 16];
      const double2 v0 = sv[cc][tp], v1 = sv[cc][tp + 16];
      acc[0][0] = cadd(acc[0][0], cmul(u0, v0));
      acc[0][1] = cadd(acc[0][1], cmul(u0, v1));
      acc[1][0] = cadd(acc[1][0], cmul(u1, v0));
      acc[1][1] = cadd(acc[1][1], cmul(u1, v1));
    }
    __syncthreads();
  }
  double2* Mq = M + static_cast<long long>(q) * K * P;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int k = k0 + tk + 16 * a;
      const long long p = p0 + tp + 16 * b;
      if (k < K && p < P) Mq[static_cast<long long>(k) * P + p] = acc[a][b];
    }
}

template <int A, typename T>
__global__ void __launch_bounds__(128) fft_inverse_kernel(const double2* __restrict__ M,
                                                          T* __restrict__ y, int N, int K, int R,
                                                          int S, int oh, int ow, int mh, int mw,
                                                          int gh, int gw) {
  constexpr int H = A / 2 + 1;
  griddep_launch();
  griddep_wait();
  const long long P = static_cast<long long>(N) * gh * gw;
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P * K) return;
  const long long p = i % P;
  const int k = static_cast<int>(i / P);
  const long long KP = static_cast<long long>(K) * P;
  // y[u][v] = 1/a^2 sum_r sum_{s <= a/2} c_s Re(X[r][s] w^-(r u + s v)), with
  // c_0 = c_{a/2} = 1 and 2 otherwise: the Hermitian-unique half already
  // determines the real inverse (the reference completes the conjugate half and
  // takes .real, fftconv.py:262-268).  Only the wraparound-free block
  // [R-1, a) x [S-1, a) is formed, one spectrum column s at a time.
  constexpr int MU = A;  // upper bound of valid rows/cols (R, S >= 1)
  double acc[MU][MU];
#pragma unroll
  for (int u = 0; u < MU; ++u)
#pragma unroll
    for (int v = 0; v < MU; ++v) acc[u][v] = 0.0;
#pragma unroll
  for (int s = 0; s < H; ++s) {
    double2 Z[A];  // Z[u] = sum_r X[r][s] w^(-r u)
#pragma unroll
    for (int u = 0; u < A; ++u) Z[u] = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < A; ++r) {
      const double2 x = M[(r * H + s) * KP + static_cast<long long>(k) * P + p];
#pragma unroll
      for (int u = 0; u < A; ++u) {
        const double2 w = tw<A>(r * u);
        Z[u] = cadd(Z[u], cmul(x, make_double2(w.x, -w.y)));
      }
    }
    const double cs = (s == 0 || s == A / 2) ? 1.0 : 2.0;
#pragma unroll
    for (int u = 0; u < A; ++u)
#pragma unroll
      for (int v = 0; v < A; ++v) {
        const double2 w = tw<A>(s * v);  // Re(Z w^-sv) = Z.x w.x + Z.y w.y
        acc[u][v] = fma(cs, Z[u].x * w.x + Z[u].y * w.y, acc[u][v]);
      }
  }
  const int n = static_cast<int>(p / (static_cast<long long>(gh) * gw));
  const int t = static_cast<int>(p % (static_cast<long long>(gh) * gw));
  const int ty = t / gw, tx = t % gw;
  const double scale = 1.0 / (A * A);
  T* yk = y + (static_cast<size_t>(n) * K + k) * oh * ow;
#pragma unroll
  for (int u = 0; u < A; ++u) {
    const int oy = mh * ty + (u - (R - 1));
    if (u < R - 1 || oy >= oh) continue;
#pragma unroll
    for (int v = 0; v < A; ++v) {
      const int ox = mw * tx + (v - (S - 1));
      if (v < S - 1 || ox >= ow) continue;
      yk[static_cast<size_t>(oy) * ow + ox] = static_cast<T>(acc[u][v] * scale);
    }
  }
}

}  // namespace wino

using namespace wino;

namespace {
struct FftGeo {
  int a, mh, mw, gh, gw, Q;
  long long P;
  size_t u_bytes, v_bytes, m_bytes;
};
int fft_geo(const wino_layer_t* L, int tile, FftGeo* f) {
  if (!L || !f) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  if (tile != 8) {  // fftconv.py:215-218 allows any power of two; run_layer uses 8
    set_error("the GPU fft path implements tile 8 (run_layer's), got %d", tile);
    return WINO_EUNSUPPORTED;
  }
  if (L->N < 1 || L->C < 1 || L->H < 1 || L->W < 1 || L->K < 1 || L->R < 1 || L->S < 1 ||
      L->pad < 0) {
    set_error("invalid layer");
    return WINO_EINVAL;
  }
  if (tile <= L->R - 1 || tile <= L->S - 1) {
    set_error("tile %d too small for a %dx%d filter", tile, L->R, L->S);
    return WINO_EINVAL;
  }
  const int oh = L->H + 2 * L->pad - L->R + 1, ow = L->W + 2 * L->pad - L->S + 1;
  if (oh < 1 || ow < 1) {
    set_error("output dimensions must be >= 1");
    return WINO_EINVAL;
  }
  f->a = tile;
  f->mh = tile - L->R + 1;
  f->mw = tile - L->S + 1;
  f->gh = (oh + f->mh - 1) / f->mh;
  f->gw = (ow + f->mw - 1) / f->mw;
  f->P = static_cast<long long>(L->N) * f->gh * f->gw;
  f->Q = tile * (tile / 2 + 1);
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  f->u_bytes = al(static_cast<size_t>(f->Q) * L->K * L->C * 16);
  f->v_bytes = al(static_cast<size_t>(f->Q) * L->C * f->P * 16);
  f->m_bytes = al(static_cast<size_t>(f->Q) * L->K * f->P * 16);
  return WINO_OK;
}

template <int A, typename T>
cudaError_t fft_run(const wino_layer_t& L, const FftGeo& f, const T* d, const double* g, T* y,
                    unsigned char* ws, cudaStream_t s) {
  double2* U = reinterpret_cast<double2*>(ws);
  double2* V = reinterpret_cast<double2*>(ws + f.u_bytes);
  double2* M = reinterpret_cast<double2*>(ws + f.u_bytes + f.v_bytes);
  const int oh = L.H + 2 * L.pad - L.R + 1, ow = L.W + 2 * L.pad - L.S + 1;
  const long long kc = static_cast<long long>(L.K) * L.C;
  launch_k(fft_filter_kernel<A>, dim3(static_cast<unsigned>((kc + 127) / 128)), dim3(128), 0, s,
           g, U, L.K, L.C, L.R, L.S);
  const long long pc = f.P * L.C;
  launch_k(fft_data_kernel<A, T>, dim3(static_cast<unsigned>((pc + 127) / 128)), dim3(128), 0, s,
           d, V, L.N, L.C, L.H, L.W, L.pad, f.mh, f.mw, f.gh, f.gw);
  const dim3 grid(static_cast<unsigned>((f.P + kFB - 1) / kFB), (L.K + kFB - 1) / kFB, f.Q);
  launch_k(fft_cgemm_kernel, grid, dim3(256), 0, s, static_cast<const double2*>(U),
           static_cast<const double2*>(V), M, L.K, L.C, f.P);
  const long long pk = f.P * L.K;
  launch_k(fft_inverse_kernel<A, T>, dim3(static_cast<unsigned>((pk + 127) / 128)), dim3(128),
           0, s, static_cast<const double2*>(M), y, L.N, L.K, L.R, L.S, oh, ow, f.mh, f.mw,
           f.gh, f.gw);
  return cudaGetLastError();
}
}  // namespace

extern "C" {

int wino_fft_workspace(const wino_layer_t* layer, int tile, size_t* bytes) {
  FftGeo f;
  const int rc = fft_geo(layer, tile, &f);
  if (rc != WINO_OK) return rc;
  if (!bytes) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  *bytes = f.u_bytes + f.v_bytes + f.m_bytes;
  return WINO_OK;
}

int wino_fft_forward(const wino_layer_t* layer, int prec, int tile, const void* d,
                     const double* g, void* y, void* workspace, size_t workspace_bytes,
                     void* stream) {
  FftGeo f;
  const int rc = fft_geo(layer, tile, &f);
  if (rc != WINO_OK) return rc;
  if (!d || !g || !y || !workspace) {
    set_error("null argument");
    return WINO_EINVAL;
  }
  if (workspace_bytes < f.u_bytes + f.v_bytes + f.m_bytes) {
    set_error("fft workspace too small: %zu < %zu bytes", workspace_bytes,
              f.u_bytes + f.v_bytes + f.m_bytes);
    return WINO_EINVAL;
  }
  if (prec != WINO_PREC_FP32 && prec != WINO_PREC_FP64) {
    set_error("fft data precision must be fp32 or fp64");
    return WINO_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  cudaError_t e;
  if (prec == WINO_PREC_FP64)
    e = fft_run<8>(*layer, f, static_cast<const double*>(d), g, static_cast<double*>(y), ws, s);
  else
    e = fft_run<8>(*layer, f, static_cast<const float*>(d), g, static_cast<float*>(y), ws, s);
  if (e != cudaSuccess) {
    set_error("fft forward: %s", cudaGetErrorString(e));
    return WINO_ECUDA;
  }
  return WINO_OK;
}

}  // extern "C"
