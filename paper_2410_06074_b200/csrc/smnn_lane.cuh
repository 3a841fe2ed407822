// smnn_lane.cuh -- lane arithmetic for the fused kernels.
//
// A "lane" value S carries one (float, double) or two (float2, double2)
// independent instances.  float2 maps onto Blackwell's packed FP32 pipe
// (FFMA2 / FMUL2 / FADD2, sm_100a), so two instances advance per instruction;
// double2 gives two independent dependency chains (ILP) on the FP64 pipe.
// All S-MNN block algebra below is written once against these ops.
#pragma once

#include <cuda_runtime.h>

#include "smnn_device.cuh"

namespace smnn {

template <class S> struct LaneT;
template <> struct LaneT<float> { using T = float; static constexpr int P = 1; };
template <> struct LaneT<double> { using T = double; static constexpr int P = 1; };
template <> struct LaneT<float2> { using T = float; static constexpr int P = 2; };
template <> struct LaneT<double2> { using T = double; static constexpr int P = 2; };

// ---- scalar (plain operators: lets the compiler fold the +-1 / +-2 constants of
// Appendix A.1 into neighbouring FFMAs; rounding stays IEEE round-to-nearest)
__device__ __forceinline__ float fma_(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ float mul_(float a, float b) { return a * b; }
__device__ __forceinline__ float add_(float a, float b) { return a + b; }
// fp64 keeps the explicit round-to-nearest intrinsics: with plain operators the
// fp64 checkpoint kernels measured 1.8x slower on B200 (different scheduling)
__device__ __forceinline__ double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float neg_(float a) { return -a; }
__device__ __forceinline__ double neg_(double a) { return -a; }
// MUFU.RSQ without the denormal-input fix-up sequence of rsqrtf (a pivot below
// FLT_MIN is a breakdown anyway and is reported through `bad_`).
__device__ __forceinline__ float rsq_(float a) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ double rsq_(double a) { return rsqrt(a); }
__device__ __forceinline__ int bad_(float a) { return a >= 1.17549435e-38f ? 0 : 1; }   // NaN, <= 0, denormal -> bad
__device__ __forceinline__ int bad_(double a) { return a > 0.0 ? 0 : 1; }

// ---- packed fp32 (FFMA2 / FMUL2 / FADD2)
__device__ __forceinline__ float2 fma_(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul_(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add_(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 neg_(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 rsq_(float2 a) { return make_float2(rsq_(a.x), rsq_(a.y)); }
__device__ __forceinline__ int bad_(float2 a) { return bad_(a.x) | (bad_(a.y) << 1); }

// ---- two fp64 chains
__device__ __forceinline__ double2 fma_(double2 a, double2 b, double2 c) {
  return make_double2(__fma_rn(a.x, b.x, c.x), __fma_rn(a.y, b.y, c.y));
}
__device__ __forceinline__ double2 mul_(double2 a, double2 b) { return make_double2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ double2 add_(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 neg_(double2 a) { return make_double2(-a.x, -a.y); }
__device__ __forceinline__ double2 rsq_(double2 a) { return make_double2(rsqrt(a.x), rsqrt(a.y)); }
__device__ __forceinline__ int bad_(double2 a) { return (a.x > 0.0 ? 0 : 1) | (a.y > 0.0 ? 0 : 2); }

template <class S> __device__ __forceinline__ S sub_(S a, S b) { return add_(a, neg_(b)); }
template <class S> __device__ __forceinline__ S fnma_(S a, S b, S c) { return fma_(neg_(a), b, c); }  // c - a b

template <class S> __device__ __forceinline__ S splat(double v);
template <> __device__ __forceinline__ float splat<float>(double v) { return float(v); }
template <> __device__ __forceinline__ double splat<double>(double v) { return v; }
template <> __device__ __forceinline__ float2 splat<float2>(double v) { return make_float2(float(v), float(v)); }
template <> __device__ __forceinline__ double2 splat<double2>(double v) { return make_double2(v, v); }

// Lane p of S (p < P).
__device__ __forceinline__ float lane(float a, int) { return a; }
__device__ __forceinline__ double lane(double a, int) { return a; }
__device__ __forceinline__ float lane(float2 a, int p) { return p ? a.y : a.x; }
__device__ __forceinline__ double lane(double2 a, int p) { return p ? a.y : a.x; }

// Build a lane value from per-instance scalars.
template <class S> struct Make;
template <> struct Make<float> { template <class T> __device__ static float f(const T* v) { return float(v[0]); } };
template <> struct Make<double> { template <class T> __device__ static double f(const T* v) { return double(v[0]); } };
template <> struct Make<float2> {
  template <class T> __device__ static float2 f(const T* v) { return make_float2(float(v[0]), float(v[1])); }
};
template <> struct Make<double2> {
  template <class T> __device__ static double2 f(const T* v) { return make_double2(double(v[0]), double(v[1])); }
};

// ============================================ block algebra on lanes ======
// Lower-triangular factors keep the INVERSE diagonal: Lf[i][i] = 1/L_ii.

template <int B, class S>
__device__ __forceinline__ void zero(S (&a)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) a[i] = splat<S>(0.0);
}
template <int B, class S>
__device__ __forceinline__ void zero(S (&a)[B][B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) zero<B, S>(a[i]);
}

// Scaled step powers a_m = ws2 * s^m, m = 0..2B-2 (zero vector: no interval).
template <int B, class S>
__device__ __forceinline__ void spow(S s, S ws2, S (&a)[2 * B - 1]) {
  a[0] = ws2;
#pragma unroll
  for (int m = 1; m < 2 * B - 1; ++m) a[m] = mul_(a[m - 1], s);
}

// M_j = wg2 c c^T + SP(a_next) + SM(a_prev)  (Appendix A.1);
// also returns wc = wg2 c for the rhs.
template <int B, class S>
__device__ __forceinline__ void lassemble(const S (&c)[B], S wg2, const S (&ap)[2 * B - 1],
                                          const S (&an)[2 * B - 1], S (&M)[B][B], S (&wc)[B]) {
  S e[2 * B - 1];
#pragma unroll
  for (int m = 0; m < 2 * B - 1; ++m) e[m] = (m & 1) ? sub_(an[m], ap[m]) : add_(an[m], ap[m]);
#pragma unroll
  for (int i = 0; i < B; ++i) wc[i] = mul_(wg2, c[i]);
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k <= i; ++k) {
      const double g = Gc(i, k) + (i == k ? 1.0 : 0.0);
      M[i][k] = fma_(splat<S>(g), e[i + k], mul_(wc[i], c[k]));
    }
}

// N = M_{t+1,t} = -H o a  (w_smooth^2 S**), full B x B.
template <int B, class S>
__device__ __forceinline__ void lN(const S (&a)[2 * B - 1], S (&N)[B][B]) {
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k < B; ++k) N[i][k] = mul_(splat<S>(-Hc(i, k)), a[i + k]);
}

// Cholesky of the lower triangle of D (in place allowed).  Returns bad-lane mask.
template <int B, class S>
__device__ __forceinline__ int lchol(const S (&D)[B][B], S (&Lf)[B][B]) {
  int bad = 0;
#pragma unroll
  for (int i = 0; i < B; ++i) {
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      S acc = D[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) acc = fnma_(Lf[i][k], Lf[j][k], acc);
      if (i == j) {
        bad |= bad_(acc);
        Lf[i][i] = rsq_(acc);
      } else {
        Lf[i][j] = mul_(acc, Lf[j][j]);
      }
    }
  }
  return bad;
}

template <int B, class S>
__device__ __forceinline__ void llsolve(const S (&Lf)[B][B], const S (&v)[B], S (&x)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) {
    S acc = v[i];
#pragma unroll
    for (int k = 0; k < i; ++k) acc = fnma_(Lf[i][k], x[k], acc);
    x[i] = mul_(acc, Lf[i][i]);
  }
}

template <int B, class S>
__device__ __forceinline__ void lltsolve(const S (&Lf)[B][B], const S (&v)[B], S (&x)[B]) {
#pragma unroll
  for (int i = B - 1; i >= 0; --i) {
    S acc = v[i];
#pragma unroll
    for (int k = i + 1; k < B; ++k) acc = fnma_(Lf[k][i], x[k], acc);
    x[i] = mul_(acc, Lf[i][i]);
  }
}

// X = L^{-1} Y column-wise
template <int B, class S>
__device__ __forceinline__ void lleft(const S (&Lf)[B][B], const S (&Y)[B][B], S (&X)[B][B]) {
#pragma unroll
  for (int c = 0; c < B; ++c)
#pragma unroll
    for (int i = 0; i < B; ++i) {
      S acc = Y[i][c];
#pragma unroll
      for (int k = 0; k < i; ++k) acc = fnma_(Lf[i][k], X[k][c], acc);
      X[i][c] = mul_(acc, Lf[i][i]);
    }
}

// P = N L^{-T} with N = -H o a  (rows of P = L^{-1} rows of N)
template <int B, class S>
__device__ __forceinline__ void lPfromN(const S (&a)[2 * B - 1], const S (&Lf)[B][B], S (&P)[B][B]) {
  S N[B][B];
  lN<B, S>(a, N);
#pragma unroll
  for (int r = 0; r < B; ++r) llsolve<B, S>(Lf, N[r], P[r]);
}

// One coupled elimination step: D = M - P P^T (lower), rhs -= P w.
template <int B, class S>
__device__ __forceinline__ void lcouple(const S (&P)[B][B], const S (&w)[B], S (&M)[B][B], S (&rhs)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) {
#pragma unroll
    for (int k = 0; k <= i; ++k) {
      S acc = M[i][k];
#pragma unroll
      for (int j = 0; j < B; ++j) acc = fnma_(P[i][j], P[k][j], acc);
      M[i][k] = acc;
    }
    S acc = rhs[i];
#pragma unroll
    for (int j = 0; j < B; ++j) acc = fnma_(P[i][j], w[j], acc);
    rhs[i] = acc;
  }
}

// y = A^T x
template <int B, class S>
__device__ __forceinline__ void lmatTvec(const S (&A)[B][B], const S (&x)[B], S (&y)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) {
    S acc = mul_(A[0][i], x[0]);
#pragma unroll
    for (int k = 1; k < B; ++k) acc = fma_(A[k][i], x[k], acc);
    y[i] = acc;
  }
}

}  // namespace smnn
