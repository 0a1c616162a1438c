// Builtin minimal-filtering matrices F(2,3) and F(4,3), as compile-time
// constants.  Entries are the exact rationals of the reference
// (winograd.py:151-168 for F(2,3), winograd.py:192-215 for F(4,3)) written as
// correctly-rounded doubles and rounded ONCE more to the data type at use,
// exactly like the reference's Fraction -> float -> dtype lowering
// (engine.py:98-101, rational.py:135-141).
//
// All transform loops are fully unrolled; coefficient tests fold at compile
// time, so zero entries cost nothing and +-1 entries become add/sub.
#pragma once

namespace wino {

template <int M>
struct Alg;

template <>
struct Alg<2> {
  static constexpr int m = 2, r = 3, alpha = 4;
  __host__ __device__ static constexpr double BT(int i, int j) {
    constexpr double t[4][4] = {{1, 0, -1, 0}, {0, 1, 1, 0}, {0, -1, 1, 0}, {0, 1, 0, -1}};
    return t[i][j];
  }
  __host__ __device__ static constexpr double G(int i, int j) {
    constexpr double t[4][3] = {{1, 0, 0}, {0.5, 0.5, 0.5}, {0.5, -0.5, 0.5}, {0, 0, 1}};
    return t[i][j];
  }
  __host__ __device__ static constexpr double AT(int i, int j) {
    constexpr double t[2][4] = {{1, 1, 1, 0}, {0, 1, -1, -1}};
    return t[i][j];
  }
};

template <>
struct Alg<4> {
  static constexpr int m = 4, r = 3, alpha = 6;
  __host__ __device__ static constexpr double BT(int i, int j) {
    constexpr double t[6][6] = {{4, 0, -5, 0, 1, 0},  {0, -4, -4, 1, 1, 0}, {0, 4, -4, -1, 1, 0},
                                {0, -2, -1, 2, 1, 0}, {0, 2, -1, -2, 1, 0}, {0, 4, 0, -5, 0, 1}};
    return t[i][j];
  }
  __host__ __device__ static constexpr double G(int i, int j) {
    constexpr double t[6][3] = {{1.0 / 4, 0, 0},
                                {-1.0 / 6, -1.0 / 6, -1.0 / 6},
                                {-1.0 / 6, 1.0 / 6, -1.0 / 6},
                                {1.0 / 24, 1.0 / 12, 1.0 / 6},
                                {1.0 / 24, -1.0 / 12, 1.0 / 6},
                                {0, 0, 1}};
    return t[i][j];
  }
  __host__ __device__ static constexpr double AT(int i, int j) {
    constexpr double t[4][6] = {
        {1, 1, 1, 1, 1, 0}, {0, 1, -1, 2, -2, 0}, {0, 1, 1, 4, 4, 0}, {0, 1, -1, 8, -8, 1}};
    return t[i][j];
  }
};

// F(3,2) (winograd.py:171-189): the weight-gradient algorithm F(3x3, 2x2)
// (engine.py:278-328).  BT is 4x4, G is 4x2 (applied to 2x2 dY tiles), AT 3x4.
struct Alg32 {
  static constexpr int m = 3, r = 2, alpha = 4;
  __host__ __device__ static constexpr double BT(int i, int j) {
    constexpr double t[4][4] = {{1, 0, -1, 0}, {0, 1, 1, 0}, {0, -1, 1, 0}, {0, -1, 0, 1}};
    return t[i][j];
  }
  __host__ __device__ static constexpr double G(int i, int j) {
    constexpr double t[4][2] = {{1, 0}, {0.5, 0.5}, {0.5, -0.5}, {0, 1}};
    return t[i][j];
  }
  __host__ __device__ static constexpr double AT(int i, int j) {
    constexpr double t[3][4] = {{1, 1, 1, 0}, {0, 1, -1, 0}, {0, 1, 1, 1}};
    return t[i][j];
  }
};

// acc + c*x with the coefficient folded at compile time.
template <typename T>
__device__ __forceinline__ T mac(T acc, double c, T x, bool first) {
  if (c == 0.0) return acc;
  if (first) {
    if (c == 1.0) return x;
    if (c == -1.0) return -x;
    return static_cast<T>(c) * x;
  }
  if (c == 1.0) return acc + x;
  if (c == -1.0) return acc - x;
  return acc + static_cast<T>(c) * x;
}

// out[i][j] = sum_u sum_v L(i,u) * in[u][v] * L(j,v)   (L is ROWS x COLS)
// i.e. out = L in L^T: used for B^T d B (L = BT), G g G^T (L = G), A^T M A (L = AT).
template <typename T, int ROWS, int COLS, typename LF>
__device__ __forceinline__ void sandwich(const T (&in)[COLS][COLS], T (&out)[ROWS][ROWS], LF L) {
  T tmp[ROWS][COLS];
#pragma unroll
  for (int i = 0; i < ROWS; ++i) {
#pragma unroll
    for (int v = 0; v < COLS; ++v) {
      T acc = T(0);
      bool first = true;
#pragma unroll
      for (int u = 0; u < COLS; ++u) {
        const double c = L(i, u);
        acc = mac(acc, c, in[u][v], first);
        if (c != 0.0) first = false;
      }
      tmp[i][v] = acc;
    }
  }
#pragma unroll
  for (int i = 0; i < ROWS; ++i) {
#pragma unroll
    for (int j = 0; j < ROWS; ++j) {
      T acc = T(0);
      bool first = true;
#pragma unroll
      for (int v = 0; v < COLS; ++v) {
        const double c = L(j, v);
        acc = mac(acc, c, tmp[i][v], first);
        if (c != 0.0) first = false;
      }
      out[i][j] = acc;
    }
  }
}

// F(4,3) data transform of one 6-vector, t = B^T x, with shared
// subexpressions (12 flops instead of 22):
//   t0 = 4x0 - 5x2 + x4            t5 = 4x1 - 5x3 + x5
//   p = x4 - 4x2, q = x3 - 4x1:    t1 = p + q,  t2 = p - q
//   r = x4 - x2,  u = x1 - x3:     t3 = r - 2u, t4 = r + 2u
// The coefficients are exact in every operand type; only the fp32 rounding
// order differs from the coefficient-by-coefficient sum.
template <typename T>
__device__ __forceinline__ void bt6(const T (&x)[6], T (&t)[6]) {
  t[0] = fma(T(4), x[0], fma(T(-5), x[2], x[4]));
  t[5] = fma(T(4), x[1], fma(T(-5), x[3], x[5]));
  const T p = fma(T(-4), x[2], x[4]), q = fma(T(-4), x[1], x[3]);
  t[1] = p + q;
  t[2] = p - q;
  const T r = x[4] - x[2], u = x[1] - x[3];
  t[3] = fma(T(-2), u, r);
  t[4] = fma(T(2), u, r);
}

// out = B^T in B for F(4,3): bt6 over the columns, then over the rows.
template <typename T>
__device__ __forceinline__ void bt6_2d(const T (&in)[6][6], T (&out)[6][6]) {
  T tmp[6][6];
#pragma unroll
  for (int v = 0; v < 6; ++v) {
    T col[6], tc[6];
#pragma unroll
    for (int u = 0; u < 6; ++u) col[u] = in[u][v];
    bt6(col, tc);
#pragma unroll
    for (int i = 0; i < 6; ++i) tmp[i][v] = tc[i];
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) bt6(tmp[i], out[i]);
}

}  // namespace wino
