// smnn_device.cuh -- register-resident block algebra for the S-MNN kernels.
//
// Block size B = R + 1 <= 4 is a compile-time constant, so every b x b block
// lives in registers and every loop below is fully unrolled.  Tc is the
// arithmetic type (float or double).
//
// Notation follows PAPER.md Appendix A.1 (lines 560-634):
//   F_ik  = 1/(k-i)!  (k >= i), 0 otherwise
//   G     = F^T F                                    (appears in S*_t)
//   H_ik  = F_ik + (-1)^{i+k} F_ki                   (S**_t = -S+ H S+)
// so that for one interval of span s
//   S+^T F^T F S+ + S^2  has entries  G_ik s^{i+k} + [i=k] s^{2i}     ("SP")
//   S-^T F^T F S- + S^2  has entries  (-1)^{i+k} G_ik s^{i+k} + [i=k] s^{2i} ("SM")
//   S**              has entries  -H_ik s^{i+k}.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace smnn {

// ------------------------------------------------------------ constants ----
// Non-recursive constexpr tables (B <= 4 needs factorials up to 3! and powers
// up to 2B-2 = 6); indexed with compile-time indices after unrolling, so they
// fold into FFMA immediates.
__host__ __device__ constexpr double invfact(int k) {
  return k == 0 ? 1.0 : k == 1 ? 1.0 : k == 2 ? 0.5 : k == 3 ? 1.0 / 6.0 : k == 4 ? 1.0 / 24.0
       : k == 5 ? 1.0 / 120.0 : k == 6 ? 1.0 / 720.0 : 1.0 / 5040.0;
}
__host__ __device__ constexpr double Fc(int i, int k) { return k >= i ? invfact(k - i) : 0.0; }
__host__ __device__ constexpr double Gc(int i, int k) {
  // sum_{j <= min(i,k)} F_ji F_jk, unrolled for B <= 4
  return Fc(0, i) * Fc(0, k) + (i >= 1 && k >= 1 ? Fc(1, i) * Fc(1, k) : 0.0) +
         (i >= 2 && k >= 2 ? Fc(2, i) * Fc(2, k) : 0.0) + (i >= 3 && k >= 3 ? Fc(3, i) * Fc(3, k) : 0.0);
}
__host__ __device__ constexpr double sgn(int e) { return (e & 1) ? -1.0 : 1.0; }
__host__ __device__ constexpr double Hc(int i, int k) { return Fc(i, k) + sgn(i + k) * Fc(k, i); }

template <class T> __device__ __forceinline__ T rsqrt_(T x);
template <> __device__ __forceinline__ float rsqrt_<float>(float x) { return rsqrtf(x); }
template <> __device__ __forceinline__ double rsqrt_<double>(double x) { return rsqrt(x); }

// Powers s^0 .. s^{2B-2}.
template <int B, class T>
__device__ __forceinline__ void powers(T s, T (&p)[2 * B - 1]) {
  p[0] = T(1);
#pragma unroll
  for (int k = 1; k < 2 * B - 1; ++k) p[k] = p[k - 1] * s;
}

// --------------------------------------------------- Appendix A.1 blocks ---
// Smoothness part of M_t = M_{t,t}: SP(s_t) if t < T-1, SM(s_{t-1}) if t > 0.
// hn / hp are 0/1 masks for the existence of the next / previous interval.
template <int B, class T>
__device__ __forceinline__ void assemble_M(T (&M)[B][B], const T (&c)[B], const T (&pp)[2 * B - 1],
                                           T hp, const T (&pn)[2 * B - 1], T hn, T wg2, T ws2) {
#pragma unroll
  for (int i = 0; i < B; ++i) {
#pragma unroll
    for (int k = 0; k <= i; ++k) {
      T sm = T(Gc(i, k)) * (hn * pn[i + k] + T(sgn(i + k)) * hp * pp[i + k]);
      if (i == k) sm += hn * pn[2 * i] + hp * pp[2 * i];
      T m = wg2 * c[i] * c[k] + ws2 * sm;
      M[i][k] = m;
      M[k][i] = m;
    }
  }
}

// N_t = M_{t+1,t} = w_smooth^2 S**_t.
template <int B, class T>
__device__ __forceinline__ void assemble_N(T (&N)[B][B], const T (&p)[2 * B - 1], T ws2) {
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k < B; ++k) N[i][k] = -ws2 * T(Hc(i, k)) * p[i + k];
}

// ------------------------------------------------ small dense algebra -----
// Lower-triangular factors are stored with the INVERSE of the diagonal on the
// diagonal: Lf[i][i] = 1 / L_ii, Lf[i][k] = L_ik (k < i).

// Cholesky D = L L^T.  Returns false on a non-positive / non-finite pivot.
template <int B, class T>
__device__ __forceinline__ bool chol(const T (&D)[B][B], T (&Lf)[B][B]) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < B; ++i) {
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      T acc = D[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) acc -= Lf[i][k] * Lf[j][k];
      if (i == j) {
        ok = ok && (acc > T(0));  // NaN fails too
        Lf[i][i] = rsqrt_(acc);
      } else {
        Lf[i][j] = acc * Lf[j][j];
      }
    }
  }
  return ok;
}

// x = L^{-1} v
template <int B, class T>
__device__ __forceinline__ void lsolve(const T (&Lf)[B][B], const T (&v)[B], T (&x)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) {
    T acc = v[i];
#pragma unroll
    for (int k = 0; k < i; ++k) acc -= Lf[i][k] * x[k];
    x[i] = acc * Lf[i][i];
  }
}

// x = L^{-T} v
template <int B, class T>
__device__ __forceinline__ void ltsolve(const T (&Lf)[B][B], const T (&v)[B], T (&x)[B]) {
#pragma unroll
  for (int i = B - 1; i >= 0; --i) {
    T acc = v[i];
#pragma unroll
    for (int k = i + 1; k < B; ++k) acc -= Lf[k][i] * x[k];
    x[i] = acc * Lf[i][i];
  }
}

// P = N L^{-T}  (row r of P = L^{-1} applied to row r of N)
template <int B, class T>
__device__ __forceinline__ void right_ltsolve(const T (&N)[B][B], const T (&Lf)[B][B], T (&P)[B][B]) {
#pragma unroll
  for (int r = 0; r < B; ++r) lsolve<B, T>(Lf, N[r], P[r]);
}

// X = L^{-1} Y  (column-wise)
template <int B, class T>
__device__ __forceinline__ void left_lsolve(const T (&Lf)[B][B], const T (&Y)[B][B], T (&X)[B][B]) {
#pragma unroll
  for (int c = 0; c < B; ++c) {
#pragma unroll
    for (int i = 0; i < B; ++i) {
      T acc = Y[i][c];
#pragma unroll
      for (int k = 0; k < i; ++k) acc -= Lf[i][k] * X[k][c];
      X[i][c] = acc * Lf[i][i];
    }
  }
}

// D = M - P P^T
template <int B, class T>
__device__ __forceinline__ void sub_ppt(const T (&M)[B][B], const T (&P)[B][B], T (&D)[B][B]) {
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k <= i; ++k) {
      T acc = M[i][k];
#pragma unroll
      for (int j = 0; j < B; ++j) acc -= P[i][j] * P[k][j];
      D[i][k] = acc;
      D[k][i] = acc;
    }
}

// y = v - A x
template <int B, class T>
__device__ __forceinline__ void sub_matvec(const T (&v)[B], const T (&A)[B][B], const T (&x)[B], T (&y)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) {
    T acc = v[i];
#pragma unroll
    for (int k = 0; k < B; ++k) acc -= A[i][k] * x[k];
    y[i] = acc;
  }
}

// y = A^T x
template <int B, class T>
__device__ __forceinline__ void matTvec(const T (&A)[B][B], const T (&x)[B], T (&y)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) {
    T acc = T(0);
#pragma unroll
    for (int k = 0; k < B; ++k) acc += A[k][i] * x[k];
    y[i] = acc;
  }
}

// C = A B
template <int B, class T>
__device__ __forceinline__ void matmul(const T (&A)[B][B], const T (&Bm)[B][B], T (&C)[B][B]) {
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int j = 0; j < B; ++j) {
      T acc = T(0);
#pragma unroll
      for (int k = 0; k < B; ++k) acc += A[i][k] * Bm[k][j];
      C[i][j] = acc;
    }
}

}  // namespace smnn
