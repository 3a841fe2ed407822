// smnn_kernels.cu -- S-MNN hot path for sm_100a (B200).
//
// Kernels (one CUDA thread block per instance unless noted):
//   assemble_kernel   Appendix A.1 blocks M_t, N_t, beta_t -> HBM (inspection)
//   fused_kernel<FWD> Algorithm 1: assemble + block Cholesky + substitution,
//                     time-parallel (see "Time-parallel partition solver" in
//                     DESIGN.md); M never leaves registers/shared memory.
//   fused_kernel<BWD> Algorithm 2 + chain rule through Appendix A.1.
//   factor_kernel     Algorithm 3, one thread per instance, L/P -> HBM.
//   substitute_kernel Algorithm 4, one thread per instance.
//
// Time-parallel partition solver (per instance, K chunks = K threads):
//   chunk k covers [a_k, a_{k+1}); its last point sigma_k is a separator, the
//   points before it are the chunk interior I_k.  Interiors are coupled only
//   through separators, so
//   pass 1  each thread factors its interior (block Cholesky, Alg. 3 loop)
//           and carries a "spike" X_j = (G^{-1})_{j,f} N_L to obtain the Schur
//           complement of its interior onto (sigma_{k-1}, sigma_k);
//   BCR     the K x K block-tridiagonal separator system is solved in shared
//           memory by block cyclic reduction (log2 K levels);
//   pass 2  each thread re-factors its interior in G-step register segments
//           (resuming from pass-1 checkpoints) and back-substitutes with both
//           separator values known.
//   The result equals the sequential Algorithm 1 up to rounding.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstring>
#include <string>

#include "smnn.h"
#include "smnn_device.cuh"

#ifndef SMNN_MAX_THREADS
#define SMNN_MAX_THREADS 256
#endif

namespace smnn {

// Register-segment length of pass 2 (steps whose factors stay in registers).
template <int B, class Tc>
struct SegLen {
  static constexpr int value = (sizeof(Tc) == 8) ? (B <= 2 ? 8 : 4) : (B <= 3 ? 8 : 4);
};

// ------------------------------------------------------------------ args ----
template <class Tio>
struct Args {
  const Tio* coeffs;
  const Tio* rhs;
  const Tio* iv;
  const Tio* steps;
  const Tio* y_in;     // BWD: forward solution
  const Tio* grad_y;   // BWD: dl/dy
  Tio* y_out;          // FWD: solution
  Tio* g_coeffs;       // BWD outputs (nullable)
  Tio* g_rhs;
  Tio* g_iv;
  Tio* g_steps;
  int32_t* info;       // nullable
  void* ckpt;          // workspace (Tc elements), one slot per block
  int64_t n_inst;
  int T;
  int n_iv;
  int K;               // chunks per instance (<= blockDim.x)
  int nseg_ck;         // checkpoint segments per chunk (slot stride)
  double wg2, wi2, ws2;
};

template <int B>
struct Ck {  // checkpoint element counts
  static constexpr int L = B * B;  // Lf stored densely (simple indexing)
  static constexpr int W = B;
  static constexpr int X = B * B;
  static constexpr int N = L + W + X;
};

// Load helpers ---------------------------------------------------------------
template <int B, class Tio, class Tc>
__device__ __forceinline__ void ld_vec(const Tio* p, Tc (&v)[B]) {
#pragma unroll
  for (int r = 0; r < B; ++r) v[r] = Tc(__ldg(p + r));
}

template <class Tio, class Tc>
__device__ __forceinline__ Tc ld1(const Tio* p) { return Tc(__ldg(p)); }

__device__ __forceinline__ int chunk_begin(int k, int T, int K) {
  return int((int64_t(k) * T) / K);
}

// Per-instance base pointers (all further indexing is 32-bit).
template <class Tio>
struct View {
  const Tio *c, *d, *u, *s, *yin, *gy;
  Tio *yout, *gc, *gd, *gu, *gs;
  int T, n_iv;
  float dummy;
  __device__ View(const Args<Tio>& a, int64_t inst, int B) {
    T = a.T;
    n_iv = a.n_iv;
    const int64_t tb = inst * int64_t(a.T) * B, t1 = inst * int64_t(a.T), ts = inst * int64_t(a.T - 1);
    c = a.coeffs + tb;
    d = a.rhs + t1;
    u = a.iv + inst * a.n_iv;
    s = a.steps + ts;
    yin = a.y_in ? a.y_in + tb : nullptr;
    gy = a.grad_y ? a.grad_y + tb : nullptr;
    yout = a.y_out ? a.y_out + tb : nullptr;
    gc = a.g_coeffs ? a.g_coeffs + tb : nullptr;
    gd = a.g_rhs ? a.g_rhs + t1 : nullptr;
    gu = a.g_iv ? a.g_iv + inst * a.n_iv : nullptr;
    gs = a.g_steps ? a.g_steps + ts : nullptr;
  }
};

struct W3 {  // squared importance weights in the arithmetic type
  double g, i, s;
};

// RHS at point j: beta_j = wg2 c_j d_j (+ wi2 u at j = 0) in the forward pass,
// dl/dy_j in the backward pass.
template <int B, class Tio, class Tc, bool BWD>
__device__ __forceinline__ void load_rhs(const View<Tio>& v, const W3& w, int j, const Tc (&c)[B], Tc (&r)[B]) {
  if (BWD) {
    ld_vec<B, Tio, Tc>(v.gy + j * B, r);
  } else {
    const Tc d = ld1<Tio, Tc>(v.d + j);
#pragma unroll
    for (int i = 0; i < B; ++i) r[i] = Tc(w.g) * c[i] * d;
    if (j == 0) {
#pragma unroll
      for (int i = 0; i < B; ++i)
        if (i < v.n_iv) r[i] += Tc(w.i) * ld1<Tio, Tc>(v.u + i);
    }
  }
}

// M_j with its neighbours' step powers (pp = s_{j-1}^k, pn = s_j^k).
template <int B, class Tio, class Tc>
__device__ __forceinline__ void load_M(const View<Tio>& v, const W3& w, int j, const Tc (&c)[B],
                                       const Tc (&pp)[2 * B - 1], Tc hp, const Tc (&pn)[2 * B - 1], Tc hn,
                                       Tc (&M)[B][B]) {
  assemble_M<B, Tc>(M, c, pp, hp, pn, hn, Tc(w.g), Tc(w.s));
  if (j == 0) {
#pragma unroll
    for (int i = 0; i < B; ++i)
      if (i < v.n_iv) M[i][i] += Tc(w.i);
  }
}

// dl/ds_j contribution of interval (j, j+1), PAPER.md:618-634 differentiated:
//   -ws2 [ lj^T J+ yj + ln^T J- yn + ln^T K yj + yn^T K lj ]
template <int B, class Tc>
__device__ __forceinline__ Tc ds_interval(Tc s, Tc ws2, const Tc (&lj)[B], const Tc (&yj)[B], const Tc (&ln)[B],
                                          const Tc (&yn)[B]) {
  Tc q[2 * B - 1];  // q[m] = d/ds s^m = m s^{m-1}
  Tc p[2 * B - 1];
  powers<B, Tc>(s, p);
  q[0] = Tc(0);
#pragma unroll
  for (int m = 1; m < 2 * B - 1; ++m) q[m] = Tc(m) * p[m - 1];
  Tc acc = Tc(0);
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const Tc g = Tc(Gc(i, k)) * q[i + k];
      const Tc jp = g + (i == k ? q[2 * i] : Tc(0));
      const Tc jm = Tc(sgn(i + k)) * g + (i == k ? q[2 * i] : Tc(0));
      const Tc kd = -Tc(Hc(i, k)) * q[i + k];
      acc += lj[i] * jp * yj[k] + ln[i] * (jm * yn[k] + kd * yj[k]) + yn[i] * kd * lj[k];
    }
  return -ws2 * acc;
}

// Gradients at point j (PAPER.md:626-634 differentiated, Eq. 13):
//   dd_j = wg2 c.l ;  dc_j = wg2 ( d_j l - l (y.c) - y (l.c) ) ;  du = wi2 l_0.
template <int B, class Tio, class Tc>
__device__ __forceinline__ void point_grads(const View<Tio>& v, const W3& w, int j, const Tc (&lam)[B],
                                            const Tc (&yj)[B]) {
  Tc c[B];
  ld_vec<B, Tio, Tc>(v.c + j * B, c);
  Tc lc = Tc(0), yc = Tc(0);
#pragma unroll
  for (int i = 0; i < B; ++i) {
    lc += lam[i] * c[i];
    yc += yj[i] * c[i];
  }
  const Tc wg2 = Tc(w.g);
  if (v.gd) v.gd[j] = Tio(wg2 * lc);
  if (v.gc) {
    const Tc d = ld1<Tio, Tc>(v.d + j);
#pragma unroll
    for (int i = 0; i < B; ++i) v.gc[j * B + i] = Tio(wg2 * (d * lam[i] - lam[i] * yc - yj[i] * lc));
  }
  if (j == 0 && v.gu) {
    for (int i = 0; i < v.n_iv; ++i) v.gu[i] = Tio(Tc(w.i) * lam[i]);
  }
}

// Shared-memory separator system, structure of arrays over the K separators.
template <int B, class Tc>
struct Sep {
  Tc* D;   // [B*B][K]  diagonal block; holds the factor after elimination
  Tc* Bc;  // [B*B][K]  coupling block(i, i-h); holds Y1 after elimination
  Tc* Y2;  // [B*B][K]
  Tc* R;   // [B][K]    rhs; holds v after elimination
  Tc* Y;   // [B][K]    solution
  int* time;  // [K]     time index of separator i (for info)
  int* fail;  // [1]
  int K;
  __device__ void ld(const Tc* arr, int i, Tc (&m)[B][B]) const {
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) m[r][c] = arr[(r * B + c) * K + i];
  }
  __device__ void st(Tc* arr, int i, const Tc (&m)[B][B]) const {
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) arr[(r * B + c) * K + i] = m[r][c];
  }
  __device__ void ldv(const Tc* arr, int i, Tc (&v)[B]) const {
#pragma unroll
    for (int r = 0; r < B; ++r) v[r] = arr[r * K + i];
  }
  __device__ void stv(Tc* arr, int i, const Tc (&v)[B]) const {
#pragma unroll
    for (int r = 0; r < B; ++r) arr[r * K + i] = v[r];
  }
};

// Block cyclic reduction of the separator system (SPD block tridiagonal).
// All threads of the block must call it.
template <int B, class Tc>
__device__ __noinline__ void bcr_solve(Sep<B, Tc> S, int k) {
  const int K = S.K;
  int hmax = 0;
#pragma unroll 1
  for (int h = 1; h < K; h <<= 1) {
    hmax = h;
    if (k < K && (k % (2 * h)) == h) {
      Tc D[B][B], Lf[B][B], Bk[B][B], Y1[B][B], Y2[B][B], r[B], v[B];
      S.ld(S.D, k, D);
      if (!chol<B, Tc>(D, Lf)) atomicMin(S.fail, S.time[k] + 1);
      S.ld(S.Bc, k, Bk);
      left_lsolve<B, Tc>(Lf, Bk, Y1);
      if (k + h < K) {
        Tc Bn[B][B], BnT[B][B];
        S.ld(S.Bc, k + h, Bn);
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int j = 0; j < B; ++j) BnT[i][j] = Bn[j][i];
        left_lsolve<B, Tc>(Lf, BnT, Y2);
      } else {
        zero<B, Tc>(Y2);
      }
      S.ldv(S.R, k, r);
      lsolve<B, Tc>(Lf, r, v);
      S.st(S.D, k, Lf);
      S.st(S.Bc, k, Y1);
      S.st(S.Y2, k, Y2);
      S.stv(S.R, k, v);
    }
    __syncthreads();
    if (k < K && (k % (2 * h)) == 0) {
      Tc D[B][B], r[B];
      S.ld(S.D, k, D);
      S.ldv(S.R, k, r);
      if (k - h >= 0) {
        const int o = k - h;
        Tc Y2o[B][B], Y1o[B][B], vo[B], nb[B][B];
        S.ld(S.Y2, o, Y2o);
        S.ld(S.Bc, o, Y1o);
        S.ldv(S.R, o, vo);
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int j = 0; j < B; ++j) {
            Tc accD = Tc(0), accB = Tc(0);
#pragma unroll
            for (int m = 0; m < B; ++m) {
              accD += Y2o[m][i] * Y2o[m][j];
              accB += Y2o[m][i] * Y1o[m][j];
            }
            D[i][j] -= accD;
            nb[i][j] = (k - 2 * h >= 0) ? -accB : Tc(0);
          }
#pragma unroll
        for (int i = 0; i < B; ++i) {
          Tc acc = Tc(0);
#pragma unroll
          for (int m = 0; m < B; ++m) acc += Y2o[m][i] * vo[m];
          r[i] -= acc;
        }
        S.st(S.Bc, k, nb);
      }
      if (k + h < K) {
        const int o = k + h;
        Tc Y1o[B][B], vo[B];
        S.ld(S.Bc, o, Y1o);
        S.ldv(S.R, o, vo);
#pragma unroll
        for (int i = 0; i < B; ++i) {
#pragma unroll
          for (int j = 0; j < B; ++j) {
            Tc acc = Tc(0);
#pragma unroll
            for (int m = 0; m < B; ++m) acc += Y1o[m][i] * Y1o[m][j];
            D[i][j] -= acc;
          }
          Tc acc = Tc(0);
#pragma unroll
          for (int m = 0; m < B; ++m) acc += Y1o[m][i] * vo[m];
          r[i] -= acc;
        }
      }
      S.st(S.D, k, D);
      S.stv(S.R, k, r);
    }
    __syncthreads();
  }
  if (k == 0) {
    Tc D[B][B], Lf[B][B], r[B], t[B], y[B];
    S.ld(S.D, 0, D);
    if (!chol<B, Tc>(D, Lf)) atomicMin(S.fail, S.time[0] + 1);
    S.ldv(S.R, 0, r);
    lsolve<B, Tc>(Lf, r, t);
    ltsolve<B, Tc>(Lf, t, y);
    S.stv(S.Y, 0, y);
  }
  __syncthreads();
#pragma unroll 1
  for (int h = hmax; h >= 1; h >>= 1) {
    if (k < K && (k % (2 * h)) == h) {
      Tc Lf[B][B], Y1[B][B], v[B], yl[B], t[B], y[B];
      S.ld(S.D, k, Lf);
      S.ld(S.Bc, k, Y1);
      S.ldv(S.R, k, v);
      S.ldv(S.Y, k - h, yl);
      sub_matvec<B, Tc>(v, Y1, yl, t);
      if (k + h < K) {
        Tc Y2[B][B], yr[B], t2[B];
        S.ld(S.Y2, k, Y2);
        S.ldv(S.Y, k + h, yr);
        sub_matvec<B, Tc>(t, Y2, yr, t2);
#pragma unroll
        for (int i = 0; i < B; ++i) t[i] = t2[i];
      }
      ltsolve<B, Tc>(Lf, t, y);
      S.stv(S.Y, k, y);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- pass 1 ----
// Factor the interior [f, l] of chunk k (l = sigma - 1), carry the spike and
// write the Schur complement onto (sigma_{k-1}, sigma) plus the separator's
// own block into shared memory (D, R, Bc) and the left-neighbour terms into
// the temporaries (Y2 = A_ll, Y = r_l).
template <int B, class Tio, class Tc, bool BWD, int G>
__device__ __noinline__ void pass1(const View<Tio> v, const W3 w, Sep<B, Tc> S, Tc* ck, int k, int f, int sig) {
  const int T = v.T;
  const int K = S.K;
  const int l = sig - 1;
  const Tc ws2 = Tc(w.s);
  Tc Arr[B][B], Arl[B][B], All[B][B], rr[B], rl[B];
  zero<B, Tc>(Arr); zero<B, Tc>(Arl); zero<B, Tc>(All); zero<B, Tc>(rr); zero<B, Tc>(rl);
  Tc pprev[2 * B - 1];
  if (f < sig) {
    Tc Lf[B][B], wv[B], X[B][B];
    zero<B, Tc>(X);
    zero<B, Tc>(Lf);
    zero<B, Tc>(wv);
    powers<B, Tc>((f > 0) ? ld1<Tio, Tc>(v.s + f - 1) : Tc(0), pprev);
    Tc hp = (f > 0) ? Tc(1) : Tc(0);
#pragma unroll 1
    for (int j = f; j <= l; ++j) {
      Tc c[B], pn[2 * B - 1], M[B][B], rhs[B], D[B][B], P[B][B];
      ld_vec<B, Tio, Tc>(v.c + j * B, c);
      powers<B, Tc>(ld1<Tio, Tc>(v.s + j), pn);
      load_M<B, Tio, Tc>(v, w, j, c, pprev, hp, pn, Tc(1), M);
      load_rhs<B, Tio, Tc, BWD>(v, w, j, c, rhs);
      if (j > f) {
        Tc Np[B][B], t[B];
        assemble_N<B, Tc>(Np, pprev, ws2);
        right_ltsolve<B, Tc>(Np, Lf, P);
        sub_ppt<B, Tc>(M, P, D);
        sub_matvec<B, Tc>(rhs, P, wv, t);
#pragma unroll
        for (int i = 0; i < B; ++i) rhs[i] = t[i];
      } else {
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int q = 0; q < B; ++q) D[i][q] = M[i][q];
      }
      if (!chol<B, Tc>(D, Lf)) atomicMin(S.fail, j + 1);
      lsolve<B, Tc>(Lf, rhs, wv);
      if (k > 0) {
        Tc Y[B][B];
        if (j == f) {
          assemble_N<B, Tc>(Y, pprev, ws2);  // N_L = N_{f-1}
          left_lsolve<B, Tc>(Lf, Y, X);
        } else {
          matmul<B, Tc>(P, X, Y);
          left_lsolve<B, Tc>(Lf, Y, X);
#pragma unroll
          for (int i = 0; i < B; ++i)
#pragma unroll
            for (int q = 0; q < B; ++q) X[i][q] = -X[i][q];
        }
#pragma unroll
        for (int i = 0; i < B; ++i) {
#pragma unroll
          for (int q = 0; q <= i; ++q) {
            Tc acc = Tc(0);
#pragma unroll
            for (int m = 0; m < B; ++m) acc += X[m][i] * X[m][q];
            All[i][q] -= acc;
          }
          Tc acc = Tc(0);
#pragma unroll
          for (int m = 0; m < B; ++m) acc += X[m][i] * wv[m];
          rl[i] -= acc;
        }
      }
      // checkpoint at the end of every full G-step segment (pass-2 resume point)
      const int done = j - f + 1;
      if ((done % G) == 0 && j < l) {
        Tc* cp = ck + (done / G - 1) * Ck<B>::N * K + k;
        int e = 0;
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int q = 0; q < B; ++q) cp[(e++) * K] = Lf[i][q];
#pragma unroll
        for (int i = 0; i < B; ++i) cp[(e++) * K] = wv[i];
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int q = 0; q < B; ++q) cp[(e++) * K] = X[i][q];
      }
#pragma unroll
      for (int m = 0; m < 2 * B - 1; ++m) pprev[m] = pn[m];
      hp = Tc(1);
    }
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
      for (int q = i + 1; q < B; ++q) All[i][q] = All[q][i];
    // Schur complement of the interior onto the separators.
    Tc NR[B][B], Pl[B][B];
    assemble_N<B, Tc>(NR, pprev, ws2);  // N_l
    right_ltsolve<B, Tc>(NR, Lf, Pl);
#pragma unroll
    for (int i = 0; i < B; ++i) {
#pragma unroll
      for (int q = 0; q < B; ++q) {
        Tc acc = Tc(0), acc2 = Tc(0);
#pragma unroll
        for (int m = 0; m < B; ++m) {
          acc += Pl[i][m] * Pl[q][m];
          acc2 += Pl[i][m] * X[m][q];
        }
        Arr[i][q] = -acc;
        Arl[i][q] = -acc2;
      }
      Tc acc = Tc(0);
#pragma unroll
      for (int m = 0; m < B; ++m) acc += Pl[i][m] * wv[m];
      rr[i] = -acc;
    }
  } else {
    // chunk of one point: direct coupling sigma_{k-1} -> sigma_k
    powers<B, Tc>((sig > 0) ? ld1<Tio, Tc>(v.s + sig - 1) : Tc(0), pprev);
    if (k > 0) assemble_N<B, Tc>(Arl, pprev, ws2);
  }
  // separator's own block and rhs
  Tc c[B], pn[2 * B - 1], M[B][B], rhs[B];
  ld_vec<B, Tio, Tc>(v.c + sig * B, c);
  const bool hn = sig < T - 1;
  powers<B, Tc>(hn ? ld1<Tio, Tc>(v.s + sig) : Tc(0), pn);
  load_M<B, Tio, Tc>(v, w, sig, c, pprev, sig > 0 ? Tc(1) : Tc(0), pn, hn ? Tc(1) : Tc(0), M);
  load_rhs<B, Tio, Tc, BWD>(v, w, sig, c, rhs);
#pragma unroll
  for (int i = 0; i < B; ++i) {
    rhs[i] += rr[i];
#pragma unroll
    for (int q = 0; q < B; ++q) M[i][q] += Arr[i][q];
  }
  S.st(S.D, k, M);
  S.stv(S.R, k, rhs);
  S.st(S.Bc, k, Arl);
  S.st(S.Y2, k, All);  // temporaries, consumed by the left neighbour
  S.stv(S.Y, k, rl);
}

// ---------------------------------------------------------------- pass 2 ----
// Interior solve of chunk k with both separator values known, in G-step
// register segments processed last-to-first; FWD writes y, BWD writes the
// gradients (lam = dl/dbeta is the solution here, y comes from the forward).
template <int B, class Tio, class Tc, bool BWD, int G>
__device__ __noinline__ void pass2(const View<Tio> v, const W3 w, Sep<B, Tc> S, const Tc* ck, int k, int f,
                                   int sig) {
  const int K = S.K;
  const int l = sig - 1;
  const Tc ws2 = Tc(w.s);
  Tc yR[B], yL[B], ysR[B];
  S.ldv(S.Y, k, yR);
  if (k > 0) S.ldv(S.Y, k - 1, yL); else zero<B, Tc>(yL);
  zero<B, Tc>(ysR);
  if (!BWD) {
#pragma unroll
    for (int i = 0; i < B; ++i) v.yout[sig * B + i] = Tio(yR[i]);
  } else {
    ld_vec<B, Tio, Tc>(v.yin + sig * B, ysR);
    point_grads<B, Tio, Tc>(v, w, sig, yR, ysR);
  }
  Tc ynext[B], yfn[B];  // solution / forward y of the point after the current one
#pragma unroll
  for (int i = 0; i < B; ++i) { ynext[i] = yR[i]; yfn[i] = ysR[i]; }
  if (f < sig) {
    const int nint = l - f + 1;
    const int nseg = (nint + G - 1) / G;
#pragma unroll 1
    for (int seg = nseg - 1; seg >= 0; --seg) {
      const int j0 = f + seg * G;
      const int len = min(G, l + 1 - j0);
      Tc Lp[B][B], wp[B], pprev[2 * B - 1];
      Tc hp;
      if (seg > 0) {
        const Tc* cp = ck + (seg - 1) * Ck<B>::N * K + k;
        int e = 0;
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int q = 0; q < B; ++q) Lp[i][q] = cp[(e++) * K];
#pragma unroll
        for (int i = 0; i < B; ++i) wp[i] = cp[(e++) * K];
        if (k > 0) {  // w' = w - X y_L  (left-separator correction)
#pragma unroll
          for (int i = 0; i < B; ++i)
#pragma unroll
            for (int q = 0; q < B; ++q) wp[i] -= cp[(B * B + B + i * B + q) * K] * yL[q];
        }
        powers<B, Tc>(ld1<Tio, Tc>(v.s + j0 - 1), pprev);
        hp = Tc(1);
      } else {
        zero<B, Tc>(Lp);
        zero<B, Tc>(wp);
        powers<B, Tc>((f > 0) ? ld1<Tio, Tc>(v.s + f - 1) : Tc(0), pprev);
        hp = (f > 0) ? Tc(1) : Tc(0);
      }
      Tc Lr[G][B][B], Wr[G][B];
#pragma unroll
      for (int i = 0; i < G; ++i) {
        if (i < len) {
          const int j = j0 + i;
          Tc c[B], pn[2 * B - 1], M[B][B], rhs[B], D[B][B];
          ld_vec<B, Tio, Tc>(v.c + j * B, c);
          powers<B, Tc>(ld1<Tio, Tc>(v.s + j), pn);
          load_M<B, Tio, Tc>(v, w, j, c, pprev, hp, pn, Tc(1), M);
          load_rhs<B, Tio, Tc, BWD>(v, w, j, c, rhs);
          if (j == f && k > 0) {  // left separator: rhs -= N_{f-1} y_L
            Tc NL[B][B], t[B];
            assemble_N<B, Tc>(NL, pprev, ws2);
            sub_matvec<B, Tc>(rhs, NL, yL, t);
#pragma unroll
            for (int q = 0; q < B; ++q) rhs[q] = t[q];
          }
          if (j > f) {
            Tc Np[B][B], P[B][B], t[B];
            assemble_N<B, Tc>(Np, pprev, ws2);
            right_ltsolve<B, Tc>(Np, Lp, P);
            sub_ppt<B, Tc>(M, P, D);
            sub_matvec<B, Tc>(rhs, P, wp, t);
#pragma unroll
            for (int q = 0; q < B; ++q) rhs[q] = t[q];
          } else {
#pragma unroll
            for (int q = 0; q < B; ++q)
#pragma unroll
              for (int r = 0; r < B; ++r) D[q][r] = M[q][r];
          }
          if (j == l) {  // right separator: rhs -= N_l^T y_R
            Tc NR[B][B], t[B];
            assemble_N<B, Tc>(NR, pn, ws2);
            matTvec<B, Tc>(NR, yR, t);
#pragma unroll
            for (int q = 0; q < B; ++q) rhs[q] -= t[q];
          }
          chol<B, Tc>(D, Lr[i]);
          lsolve<B, Tc>(Lr[i], rhs, Wr[i]);
#pragma unroll
          for (int q = 0; q < B; ++q) {
            wp[q] = Wr[i][q];
#pragma unroll
            for (int r = 0; r <= q; ++r) Lp[q][r] = Lr[i][q][r];
          }
#pragma unroll
          for (int m = 0; m < 2 * B - 1; ++m) pprev[m] = pn[m];
          hp = Tc(1);
        }
      }
#pragma unroll
      for (int i = G - 1; i >= 0; --i) {
        if (i < len) {
          const int j = j0 + i;
          Tc yv[B];
          const Tc sj = ld1<Tio, Tc>(v.s + j);
          if (j == l) {
            ltsolve<B, Tc>(Lr[i], Wr[i], yv);
          } else {
            Tc pw[2 * B - 1], Nj[B][B], vv[B], u[B], t[B];
            powers<B, Tc>(sj, pw);
            assemble_N<B, Tc>(Nj, pw, ws2);
            matTvec<B, Tc>(Nj, ynext, vv);
            lsolve<B, Tc>(Lr[i], vv, u);
#pragma unroll
            for (int q = 0; q < B; ++q) t[q] = Wr[i][q] - u[q];
            ltsolve<B, Tc>(Lr[i], t, yv);
          }
          if (!BWD) {
#pragma unroll
            for (int q = 0; q < B; ++q) v.yout[j * B + q] = Tio(yv[q]);
          } else {
            Tc yf[B];
            ld_vec<B, Tio, Tc>(v.yin + j * B, yf);
            point_grads<B, Tio, Tc>(v, w, j, yv, yf);
            if (v.gs) v.gs[j] = Tio(ds_interval<B, Tc>(sj, ws2, yv, yf, ynext, yfn));
#pragma unroll
            for (int q = 0; q < B; ++q) yfn[q] = yf[q];
          }
#pragma unroll
          for (int q = 0; q < B; ++q) ynext[q] = yv[q];
        }
      }
    }
  }
  // BWD: interval (sigma_{k-1}, first point of the chunk)
  if (BWD && k > 0 && v.gs) {
    const int jm = f - 1;
    Tc yfm[B];
    ld_vec<B, Tio, Tc>(v.yin + jm * B, yfm);
    v.gs[jm] = Tio(ds_interval<B, Tc>(ld1<Tio, Tc>(v.s + jm), ws2, yL, yfm, ynext, yfn));
  }
}

// ------------------------------------------------------ the fused kernel ----
template <int B, class Tio, class Tc, bool BWD, int G>
__global__ void __launch_bounds__(SMNN_MAX_THREADS) fused_kernel(Args<Tio> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = a.K;
  Tc* base = reinterpret_cast<Tc*>(smem_raw);
  Sep<B, Tc> S;
  S.D = base;
  S.Bc = S.D + B * B * K;
  S.Y2 = S.Bc + B * B * K;
  S.R = S.Y2 + B * B * K;
  S.Y = S.R + B * K;
  S.time = reinterpret_cast<int*>(S.Y + B * K);
  S.fail = S.time + K;
  S.K = K;
  const W3 w{a.wg2, a.wi2, a.ws2};
  const int k = threadIdx.x;
  const int T = a.T;
  Tc* ck = reinterpret_cast<Tc*>(a.ckpt) + size_t(blockIdx.x) * size_t(a.nseg_ck) * Ck<B>::N * K;

  for (int64_t inst = blockIdx.x; inst < a.n_inst; inst += gridDim.x) {
    if (k == 0) *S.fail = INT_MAX;
    const View<Tio> v(a, inst, B);
    const int f = (k < K) ? chunk_begin(k, T, K) : 0;
    const int sig = (k < K) ? chunk_begin(k + 1, T, K) - 1 : 0;
    if (k < K) {
      S.time[k] = sig;
      pass1<B, Tio, Tc, BWD, G>(v, w, S, ck, k, f, sig);
    }
    __syncthreads();
    if (k + 1 < K) {  // add the right neighbour's Schur terms A_ll, r_l
      Tc D[B][B], Al[B][B], r[B], rl[B];
      S.ld(S.D, k, D);
      S.ld(S.Y2, k + 1, Al);
      S.ldv(S.R, k, r);
      S.ldv(S.Y, k + 1, rl);
#pragma unroll
      for (int i = 0; i < B; ++i) {
        r[i] += rl[i];
#pragma unroll
        for (int q = 0; q < B; ++q) D[i][q] += Al[i][q];
      }
      S.st(S.D, k, D);
      S.stv(S.R, k, r);
    }
    __syncthreads();
    bcr_solve<B, Tc>(S, k);
    if (k < K) pass2<B, Tio, Tc, BWD, G>(v, w, S, ck, k, f, sig);
    __syncthreads();
    if (k == 0 && a.info) a.info[inst] = (*S.fail == INT_MAX) ? 0 : *S.fail;
    __syncthreads();
  }
}

// ------------------------------------------------------- assemble kernel ----
template <int B, class Tio, class Tc>
__global__ void assemble_kernel(Args<Tio> a, Tio* Mo, Tio* No, Tio* bo) {
  const int T = a.T;
  const W3 w{a.wg2, a.wi2, a.ws2};
  const int64_t total = a.n_inst * T;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t inst = idx / T;
    const int t = int(idx % T);
    const View<Tio> v(a, inst, B);
    Tc c[B], pp[2 * B - 1], pn[2 * B - 1], M[B][B], r[B];
    ld_vec<B, Tio, Tc>(v.c + t * B, c);
    const bool hp = t > 0, hn = t < T - 1;
    powers<B, Tc>(hp ? ld1<Tio, Tc>(v.s + t - 1) : Tc(0), pp);
    powers<B, Tc>(hn ? ld1<Tio, Tc>(v.s + t) : Tc(0), pn);
    load_M<B, Tio, Tc>(v, w, t, c, pp, hp ? Tc(1) : Tc(0), pn, hn ? Tc(1) : Tc(0), M);
    load_rhs<B, Tio, Tc, false>(v, w, t, c, r);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      bo[idx * B + i] = Tio(r[i]);
#pragma unroll
      for (int q = 0; q < B; ++q) Mo[(idx * B + i) * B + q] = Tio(M[i][q]);
    }
    if (hn && No) {
      Tc N[B][B];
      assemble_N<B, Tc>(N, pn, Tc(w.s));
      const int64_t o = inst * (T - 1) + t;
#pragma unroll
      for (int i = 0; i < B; ++i)
#pragma unroll
        for (int q = 0; q < B; ++q) No[(o * B + i) * B + q] = Tio(N[i][q]);
    }
  }
}

// --------------------------------------------- Algorithm 3, sequential -----
template <int B, class Tio, class Tc>
__global__ void factor_kernel(Args<Tio> a, Tio* Lo, Tio* Po) {
  const int64_t inst = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (inst >= a.n_inst) return;
  const int T = a.T;
  const W3 w{a.wg2, a.wi2, a.ws2};
  const View<Tio> v(a, inst, B);
  const Tc ws2 = Tc(w.s);
  int fail = 0;
  Tc Lf[B][B], pp[2 * B - 1];
  zero<B, Tc>(Lf);
  powers<B, Tc>(Tc(0), pp);
  for (int t = 0; t < T; ++t) {
    Tc c[B], pn[2 * B - 1], M[B][B], D[B][B];
    ld_vec<B, Tio, Tc>(v.c + t * B, c);
    const bool hn = t < T - 1;
    powers<B, Tc>(hn ? ld1<Tio, Tc>(v.s + t) : Tc(0), pn);
    load_M<B, Tio, Tc>(v, w, t, c, pp, t > 0 ? Tc(1) : Tc(0), pn, hn ? Tc(1) : Tc(0), M);
    if (t > 0) {
      // P_{t-1} <- N_{t-1} L_{t-1}^{-T};  L_t <- M_t - P P^T   (Alg. 3)
      Tc N[B][B], P[B][B], Pl[B][B];
      assemble_N<B, Tc>(N, pp, ws2);
      right_ltsolve<B, Tc>(N, Lf, P);
      sub_ppt<B, Tc>(M, P, D);
      // to blockwise LDL: P_{t-1} <- P_{t-1} L_{t-1}^{-1}   (Alg. 3)
#pragma unroll
      for (int r = 0; r < B; ++r) ltsolve<B, Tc>(Lf, P[r], Pl[r]);
      if (Po) {
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int q = 0; q < B; ++q) Po[((inst * (T - 1) + t - 1) * B + i) * B + q] = Tio(Pl[i][q]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < B; ++i)
#pragma unroll
        for (int q = 0; q < B; ++q) D[i][q] = M[i][q];
    }
    if (!chol<B, Tc>(D, Lf) && fail == 0) fail = t + 1;  // standard Cholesky (line 255)
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
      for (int q = 0; q < B; ++q)
        Lo[((inst * T + t) * B + i) * B + q] =
            Tio(q < i ? Lf[i][q] : (q == i ? Tc(1) / Lf[i][i] : Tc(0)));
#pragma unroll
    for (int m = 0; m < 2 * B - 1; ++m) pp[m] = pn[m];
  }
  if (a.info) a.info[inst] = fail;
}

// --------------------------------------------- Algorithm 4, sequential -----
template <int B, class Tio, class Tc>
__global__ void substitute_kernel(int64_t n_inst, int T, const Tio* Lg, const Tio* Pg, const Tio* alpha, Tio* out) {
  const int64_t inst = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (inst >= n_inst) return;
  Tc prev[B];
  for (int t = 0; t < T; ++t) {
    Tc al[B], Lf[B][B], x[B], z[B];
    ld_vec<B, Tio, Tc>(alpha + (inst * T + t) * B, al);
    if (t > 0) {  // forward substitute: a_t -= P_{t-1} a_{t-1}  (Alg. 4)
#pragma unroll
      for (int i = 0; i < B; ++i) {
        Tc acc = Tc(0);
#pragma unroll
        for (int q = 0; q < B; ++q) acc += Tc(Pg[((inst * (T - 1) + t - 1) * B + i) * B + q]) * prev[q];
        al[i] -= acc;
      }
    }
#pragma unroll
    for (int i = 0; i < B; ++i) prev[i] = al[i];
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
      for (int q = 0; q < B; ++q) {
        Tc v = Tc(Lg[((inst * T + t) * B + i) * B + q]);
        Lf[i][q] = (i == q) ? Tc(1) / v : v;
      }
    lsolve<B, Tc>(Lf, al, x);  // a_t <- L_t^{-T} L_t^{-1} a_t  (line 307)
    ltsolve<B, Tc>(Lf, x, z);
#pragma unroll
    for (int i = 0; i < B; ++i) out[(inst * T + t) * B + i] = Tio(z[i]);
  }
  for (int t = T - 2; t >= 0; --t) {  // backward substitute (line 312)
    Tc nx[B], cur[B];
    ld_vec<B, Tio, Tc>(out + (inst * T + t + 1) * B, nx);
    ld_vec<B, Tio, Tc>(out + (inst * T + t) * B, cur);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      Tc acc = Tc(0);
#pragma unroll
      for (int q = 0; q < B; ++q) acc += Tc(Pg[((inst * (T - 1) + t) * B + q) * B + i]) * nx[q];
      out[(inst * T + t) * B + i] = Tio(cur[i] - acc);
    }
  }
}

}  // namespace smnn

// ============================================================ host side =====
namespace {

thread_local std::string g_err;

int fail_arg(const std::string& m) { g_err = m; return SMNN_ERR_ARG; }

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SMNN_OK;
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return SMNN_ERR_CUDA;
}

int validate(const smnn_problem* p) {
  if (!p) return fail_arg("problem is NULL");
  if (p->n_inst < 1) return fail_arg("n_inst must be >= 1");
  if (p->T < 1) return fail_arg("T must be >= 1");
  if (p->order < 0) return fail_arg("order must be >= 0");
  if (p->order > SMNN_MAX_ORDER) { g_err = "order > 3 is not supported"; return SMNN_ERR_UNSUPPORTED; }
  if (p->n_iv < 1 || p->n_iv > p->order + 1) return fail_arg("n_iv must be in 1..order+1");
  if (p->dtype != SMNN_F32 && p->dtype != SMNN_F64 && p->dtype != SMNN_F32_C64) {
    g_err = "unknown dtype"; return SMNN_ERR_UNSUPPORTED;
  }
  if (!(p->w_gov > 0) || !(p->w_init > 0) || !(p->w_smooth > 0)) return fail_arg("weights must be > 0");
  if (p->threads_per_inst < 0 || p->threads_per_inst > SMNN_MAX_THREADS || (p->threads_per_inst % 32) != 0)
    return fail_arg("threads_per_inst must be 0 (auto) or a multiple of 32 in 32..SMNN_MAX_THREADS");
  if (p->reserved != 0) return fail_arg("reserved must be 0");
  return SMNN_OK;
}

size_t tc_size(const smnn_problem* p) { return p->dtype == SMNN_F32 ? 4 : 8; }

int pass2_G(const smnn_problem* p) {
  const int B = p->order + 1;
  if (tc_size(p) == 8) return B <= 2 ? 8 : 4;
  return B <= 3 ? 8 : 4;  // == smnn::SegLen<B, Tc>::value
}

// Chunks (threads) per instance.
int threads_per_inst(const smnn_problem* p) {
  int nt = p->threads_per_inst;
  if (nt == 0) {
    const int target = 16;  // interior steps per chunk
    nt = (p->T + target - 1) / target;
    nt = ((nt + 31) / 32) * 32;
    nt = std::max(32, std::min(nt, SMNN_MAX_THREADS));
  }
  const int B = p->order + 1;
  const size_t per = size_t(3 * B * B + 2 * B) * tc_size(p) + 8;
  while (nt > 32 && per * nt > 160 * 1024) nt -= 32;
  return nt;
}

int chunks(const smnn_problem* p) { return std::min(threads_per_inst(p), p->T); }

size_t fused_smem(const smnn_problem* p) {
  const int B = p->order + 1;
  const int K = chunks(p);
  return size_t(3 * B * B + 2 * B) * K * tc_size(p) + size_t(K + 1) * sizeof(int) + 16;
}

int nseg_ck(const smnn_problem* p) {
  const int K = chunks(p);
  const int maxlen = (p->T + K - 1) / K;  // chunk length incl. separator
  const int nint = std::max(0, maxlen - 1);
  const int G = pass2_G(p);
  return std::max(0, (nint + G - 1) / G - 1);
}

size_t ck_elems(const smnn_problem* p) {
  const int B = p->order + 1;
  return size_t(2 * B * B + B);
}

int device_sms() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// Persistent grid: resident blocks, capped by the number of instances.
template <class K>
int fused_grid(K kernel, const smnn_problem* p) {
  int occ = 1;
  const int nt = threads_per_inst(p);
  const size_t smem = fused_smem(p);
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, nt, smem);
  occ = std::max(occ, 1);
  const int64_t g = std::min<int64_t>(p->n_inst, int64_t(occ) * device_sms());
  return int(std::max<int64_t>(g, 1));
}

template <int B, class Tio, class Tc>
int fused_grid_any(const smnn_problem* p) {
  using namespace smnn;
  constexpr int G = SegLen<B, Tc>::value;
  const int g1 = fused_grid(fused_kernel<B, Tio, Tc, false, G>, p);
  const int g2 = fused_grid(fused_kernel<B, Tio, Tc, true, G>, p);
  return std::max(g1, g2);
}

template <class Tio, class Tc>
int grid_for(const smnn_problem* p) {
  switch (p->order) {
    case 0: return fused_grid_any<1, Tio, Tc>(p);
    case 1: return fused_grid_any<2, Tio, Tc>(p);
    case 2: return fused_grid_any<3, Tio, Tc>(p);
    default: return fused_grid_any<4, Tio, Tc>(p);
  }
}

int grid_blocks(const smnn_problem* p) {
  if (p->dtype == SMNN_F32) return grid_for<float, float>(p);
  if (p->dtype == SMNN_F64) return grid_for<double, double>(p);
  return grid_for<float, double>(p);
}

size_t workspace_bytes(const smnn_problem* p) {
  const size_t per = size_t(nseg_ck(p)) * ck_elems(p) * chunks(p) * tc_size(p);
  return std::max<size_t>(per * grid_blocks(p), 256);
}

template <class Tio>
smnn::Args<Tio> make_args(const smnn_problem* p) {
  smnn::Args<Tio> a;
  std::memset(&a, 0, sizeof(a));
  a.n_inst = p->n_inst;
  a.T = p->T;
  a.n_iv = p->n_iv;
  a.K = chunks(p);
  a.nseg_ck = nseg_ck(p);
  a.wg2 = p->w_gov * p->w_gov;
  a.wi2 = p->w_init * p->w_init;
  a.ws2 = p->w_smooth * p->w_smooth;
  return a;
}

template <int B, class Tio, class Tc, bool BWD>
int launch_fused(const smnn_problem* p, smnn::Args<Tio> a, cudaStream_t st) {
  const int nt = threads_per_inst(p);
  const size_t smem = fused_smem(p);
  const int grid = grid_blocks(p);
  auto k = smnn::fused_kernel<B, Tio, Tc, BWD, smnn::SegLen<B, Tc>::value>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k<<<grid, nt, smem, st>>>(a);
  return check_cuda(cudaGetLastError(), "fused kernel launch");
}

template <class Tio, class Tc, bool BWD>
int dispatch_fused(const smnn_problem* p, const smnn::Args<Tio>& a, cudaStream_t st) {
  switch (p->order) {
    case 0: return launch_fused<1, Tio, Tc, BWD>(p, a, st);
    case 1: return launch_fused<2, Tio, Tc, BWD>(p, a, st);
    case 2: return launch_fused<3, Tio, Tc, BWD>(p, a, st);
    default: return launch_fused<4, Tio, Tc, BWD>(p, a, st);
  }
}

template <class Tio, class Tc>
int dispatch_assemble(const smnn_problem* p, const smnn::Args<Tio>& a, Tio* M, Tio* N, Tio* b, cudaStream_t st) {
  const int64_t total = p->n_inst * p->T;
  const int threads = 256;
  const int blocks = int(std::min<int64_t>((total + threads - 1) / threads, 148 * 32));
  switch (p->order) {
    case 0: smnn::assemble_kernel<1, Tio, Tc><<<blocks, threads, 0, st>>>(a, M, N, b); break;
    case 1: smnn::assemble_kernel<2, Tio, Tc><<<blocks, threads, 0, st>>>(a, M, N, b); break;
    case 2: smnn::assemble_kernel<3, Tio, Tc><<<blocks, threads, 0, st>>>(a, M, N, b); break;
    default: smnn::assemble_kernel<4, Tio, Tc><<<blocks, threads, 0, st>>>(a, M, N, b); break;
  }
  return check_cuda(cudaGetLastError(), "assemble launch");
}

template <class Tio, class Tc>
int dispatch_factor(const smnn_problem* p, const smnn::Args<Tio>& a, Tio* L, Tio* P, cudaStream_t st) {
  const int threads = 128;
  const int blocks = int((p->n_inst + threads - 1) / threads);
  switch (p->order) {
    case 0: smnn::factor_kernel<1, Tio, Tc><<<blocks, threads, 0, st>>>(a, L, P); break;
    case 1: smnn::factor_kernel<2, Tio, Tc><<<blocks, threads, 0, st>>>(a, L, P); break;
    case 2: smnn::factor_kernel<3, Tio, Tc><<<blocks, threads, 0, st>>>(a, L, P); break;
    default: smnn::factor_kernel<4, Tio, Tc><<<blocks, threads, 0, st>>>(a, L, P); break;
  }
  return check_cuda(cudaGetLastError(), "factor launch");
}

template <class Tio, class Tc>
int dispatch_substitute(const smnn_problem* p, const Tio* L, const Tio* P, const Tio* al, Tio* out, cudaStream_t st) {
  const int threads = 128;
  const int blocks = int((p->n_inst + threads - 1) / threads);
  switch (p->order) {
    case 0: smnn::substitute_kernel<1, Tio, Tc><<<blocks, threads, 0, st>>>(p->n_inst, p->T, L, P, al, out); break;
    case 1: smnn::substitute_kernel<2, Tio, Tc><<<blocks, threads, 0, st>>>(p->n_inst, p->T, L, P, al, out); break;
    case 2: smnn::substitute_kernel<3, Tio, Tc><<<blocks, threads, 0, st>>>(p->n_inst, p->T, L, P, al, out); break;
    default: smnn::substitute_kernel<4, Tio, Tc><<<blocks, threads, 0, st>>>(p->n_inst, p->T, L, P, al, out); break;
  }
  return check_cuda(cudaGetLastError(), "substitute launch");
}

template <class Tio>
void set_inputs(smnn::Args<Tio>& a, const void* c, const void* d, const void* u, const void* s) {
  a.coeffs = static_cast<const Tio*>(c);
  a.rhs = static_cast<const Tio*>(d);
  a.iv = static_cast<const Tio*>(u);
  a.steps = static_cast<const Tio*>(s);
}

int need(const void* ptr, const char* name) {
  if (ptr) return SMNN_OK;
  return fail_arg(std::string(name) + " is NULL");
}

int need_steps(const smnn_problem* p, const void* s) { return p->T > 1 ? need(s, "steps") : SMNN_OK; }

}  // namespace

struct smnn_plan {
  smnn_problem p;
  void* buf = nullptr;   // one allocation
  void *c, *d, *u, *s, *gy, *y, *gc, *gd, *gu, *gs, *ws;
  int32_t* info;
  size_t ws_bytes = 0;
};

extern "C" {

const char* smnn_version(void) { return "smnn-b200 0.1 (sm_100a)"; }
const char* smnn_last_error(void) { return g_err.c_str(); }

size_t smnn_workspace_bytes(const smnn_problem* p) {
  if (validate(p) != SMNN_OK) return 0;
  return workspace_bytes(p);
}

int smnn_assemble(const smnn_problem* p, const void* coeffs, const void* rhs, const void* iv, const void* steps,
                  void* M_diag, void* N_sub, void* beta, void* stream) {
  int e;
  if ((e = validate(p)) || (e = need(coeffs, "coeffs")) || (e = need(rhs, "rhs")) || (e = need(iv, "iv")) ||
      (e = need_steps(p, steps)) || (e = need(M_diag, "M_diag")) || (e = need(beta, "beta")) ||
      (p->T > 1 && (e = need(N_sub, "N_sub"))))
    return e;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->dtype == SMNN_F64) {
    auto a = make_args<double>(p);
    set_inputs(a, coeffs, rhs, iv, steps);
    return dispatch_assemble<double, double>(p, a, (double*)M_diag, (double*)N_sub, (double*)beta, st);
  }
  auto a = make_args<float>(p);
  set_inputs(a, coeffs, rhs, iv, steps);
  if (p->dtype == SMNN_F32) return dispatch_assemble<float, float>(p, a, (float*)M_diag, (float*)N_sub, (float*)beta, st);
  return dispatch_assemble<float, double>(p, a, (float*)M_diag, (float*)N_sub, (float*)beta, st);
}

int smnn_factor_solve_fwd(const smnn_problem* p, const void* coeffs, const void* rhs, const void* iv,
                          const void* steps, void* y, int32_t* info, void* workspace, size_t workspace_bytes_,
                          void* stream) {
  int e;
  if ((e = validate(p)) || (e = need(coeffs, "coeffs")) || (e = need(rhs, "rhs")) || (e = need(iv, "iv")) ||
      (e = need_steps(p, steps)) || (e = need(y, "y")))
    return e;
  const size_t wsn = workspace_bytes(p);
  if (workspace_bytes_ < wsn || (!workspace && wsn > 0)) {
    g_err = "workspace too small: need " + std::to_string(wsn) + " bytes";
    return SMNN_ERR_WORKSPACE;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->dtype == SMNN_F64) {
    auto a = make_args<double>(p);
    set_inputs(a, coeffs, rhs, iv, steps);
    a.y_out = (double*)y; a.info = info; a.ckpt = workspace;
    return dispatch_fused<double, double, false>(p, a, st);
  }
  auto a = make_args<float>(p);
  set_inputs(a, coeffs, rhs, iv, steps);
  a.y_out = (float*)y; a.info = info; a.ckpt = workspace;
  if (p->dtype == SMNN_F32) return dispatch_fused<float, float, false>(p, a, st);
  return dispatch_fused<float, double, false>(p, a, st);
}

int smnn_solve_bwd(const smnn_problem* p, const void* coeffs, const void* rhs, const void* iv, const void* steps,
                   const void* y, const void* grad_y, void* grad_coeffs, void* grad_rhs, void* grad_iv,
                   void* grad_steps, int32_t* info, void* workspace, size_t workspace_bytes_, void* stream) {
  int e;
  if ((e = validate(p)) || (e = need(coeffs, "coeffs")) || (e = need(rhs, "rhs")) || (e = need(iv, "iv")) ||
      (e = need_steps(p, steps)) || (e = need(y, "y")) || (e = need(grad_y, "grad_y")))
    return e;
  const size_t wsn = workspace_bytes(p);
  if (workspace_bytes_ < wsn || (!workspace && wsn > 0)) {
    g_err = "workspace too small: need " + std::to_string(wsn) + " bytes";
    return SMNN_ERR_WORKSPACE;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->dtype == SMNN_F64) {
    auto a = make_args<double>(p);
    set_inputs(a, coeffs, rhs, iv, steps);
    a.y_in = (const double*)y; a.grad_y = (const double*)grad_y;
    a.g_coeffs = (double*)grad_coeffs; a.g_rhs = (double*)grad_rhs; a.g_iv = (double*)grad_iv;
    a.g_steps = p->T > 1 ? (double*)grad_steps : nullptr; a.info = info; a.ckpt = workspace;
    return dispatch_fused<double, double, true>(p, a, st);
  }
  auto a = make_args<float>(p);
  set_inputs(a, coeffs, rhs, iv, steps);
  a.y_in = (const float*)y; a.grad_y = (const float*)grad_y;
  a.g_coeffs = (float*)grad_coeffs; a.g_rhs = (float*)grad_rhs; a.g_iv = (float*)grad_iv;
  a.g_steps = p->T > 1 ? (float*)grad_steps : nullptr; a.info = info; a.ckpt = workspace;
  if (p->dtype == SMNN_F32) return dispatch_fused<float, float, true>(p, a, st);
  return dispatch_fused<float, double, true>(p, a, st);
}

int smnn_factor(const smnn_problem* p, const void* coeffs, const void* steps, void* L, void* P, int32_t* info,
                void* stream) {
  int e;
  if ((e = validate(p)) || (e = need(coeffs, "coeffs")) || (e = need_steps(p, steps)) || (e = need(L, "L")) ||
      (p->T > 1 && (e = need(P, "P"))))
    return e;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->dtype == SMNN_F64) {
    auto a = make_args<double>(p);
    set_inputs(a, coeffs, nullptr, nullptr, steps);
    a.info = info;
    return dispatch_factor<double, double>(p, a, (double*)L, (double*)P, st);
  }
  auto a = make_args<float>(p);
  set_inputs(a, coeffs, nullptr, nullptr, steps);
  a.info = info;
  if (p->dtype == SMNN_F32) return dispatch_factor<float, float>(p, a, (float*)L, (float*)P, st);
  return dispatch_factor<float, double>(p, a, (float*)L, (float*)P, st);
}

int smnn_substitute(const smnn_problem* p, const void* L, const void* P, const void* alpha, void* out,
                    void* stream) {
  int e;
  if ((e = validate(p)) || (e = need(L, "L")) || (p->T > 1 && (e = need(P, "P"))) || (e = need(alpha, "alpha")) ||
      (e = need(out, "out")))
    return e;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->dtype == SMNN_F64)
    return dispatch_substitute<double, double>(p, (const double*)L, (const double*)P, (const double*)alpha,
                                               (double*)out, st);
  if (p->dtype == SMNN_F32)
    return dispatch_substitute<float, float>(p, (const float*)L, (const float*)P, (const float*)alpha, (float*)out, st);
  return dispatch_substitute<float, double>(p, (const float*)L, (const float*)P, (const float*)alpha, (float*)out, st);
}

int smnn_plan_create(smnn_plan** plan, const smnn_problem* p) {
  int e;
  if (!plan) return fail_arg("plan is NULL");
  if ((e = validate(p))) return e;
  smnn_plan* q = new smnn_plan();
  q->p = *p;
  const size_t es = p->dtype == SMNN_F64 ? 8 : 4;
  const size_t n = size_t(p->n_inst), T = size_t(p->T), b = size_t(p->order + 1);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t sz_c = al(n * T * b * es), sz_d = al(n * T * es), sz_u = al(n * p->n_iv * es),
               sz_s = al(n * std::max<size_t>(T - 1, 1) * es), sz_info = al(n * 4);
  q->ws_bytes = al(workspace_bytes(p));
  const size_t total = 4 * sz_c + 2 * sz_d + 2 * sz_u + 2 * sz_s + sz_info + q->ws_bytes;
  if ((e = check_cuda(cudaMalloc(&q->buf, total), "cudaMalloc(plan)"))) { delete q; return e; }
  char* ptr = static_cast<char*>(q->buf);
  auto take = [&](size_t s) { void* r = ptr; ptr += s; return r; };
  q->c = take(sz_c); q->gy = take(sz_c); q->y = take(sz_c); q->gc = take(sz_c);
  q->d = take(sz_d); q->gd = take(sz_d);
  q->u = take(sz_u); q->gu = take(sz_u);
  q->s = take(sz_s); q->gs = take(sz_s);
  q->info = static_cast<int32_t*>(take(sz_info));
  q->ws = take(q->ws_bytes);
  *plan = q;
  return SMNN_OK;
}

int smnn_plan_destroy(smnn_plan* plan) {
  if (!plan) return SMNN_OK;
  int e = check_cuda(cudaFree(plan->buf), "cudaFree(plan)");
  delete plan;
  return e;
}

int smnn_plan_fwd_bwd_host(smnn_plan* q, const void* coeffs, const void* rhs, const void* iv, const void* steps,
                           const void* grad_y, void* y, void* grad_coeffs, void* grad_rhs, void* grad_iv,
                           void* grad_steps, int32_t* info, void* stream) {
  int e;
  if (!q) return fail_arg("plan is NULL");
  const smnn_problem* p = &q->p;
  if ((e = need(coeffs, "coeffs")) || (e = need(rhs, "rhs")) || (e = need(iv, "iv")) || (e = need_steps(p, steps)) ||
      (e = need(grad_y, "grad_y")) || (e = need(y, "y")))
    return e;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t es = p->dtype == SMNN_F64 ? 8 : 4;
  const size_t n = size_t(p->n_inst), T = size_t(p->T), b = size_t(p->order + 1);
  const size_t bc = n * T * b * es, bd = n * T * es, bu = n * p->n_iv * es, bs = n * (T - 1) * es;
  const cudaMemcpyKind h2d = cudaMemcpyHostToDevice, d2h = cudaMemcpyDeviceToHost;
  if ((e = check_cuda(cudaMemcpyAsync(q->c, coeffs, bc, h2d, st), "H2D coeffs")) ||
      (e = check_cuda(cudaMemcpyAsync(q->d, rhs, bd, h2d, st), "H2D rhs")) ||
      (e = check_cuda(cudaMemcpyAsync(q->u, iv, bu, h2d, st), "H2D iv")) ||
      (bs && (e = check_cuda(cudaMemcpyAsync(q->s, steps, bs, h2d, st), "H2D steps"))) ||
      (e = check_cuda(cudaMemcpyAsync(q->gy, grad_y, bc, h2d, st), "H2D grad_y")))
    return e;
  if ((e = smnn_factor_solve_fwd(p, q->c, q->d, q->u, q->s, q->y, nullptr, q->ws, q->ws_bytes, stream))) return e;
  if ((e = smnn_solve_bwd(p, q->c, q->d, q->u, q->s, q->y, q->gy, q->gc, q->gd, q->gu, q->gs, q->info, q->ws,
                          q->ws_bytes, stream)))
    return e;
  if ((e = check_cuda(cudaMemcpyAsync(y, q->y, bc, d2h, st), "D2H y"))) return e;
  if (grad_coeffs && (e = check_cuda(cudaMemcpyAsync(grad_coeffs, q->gc, bc, d2h, st), "D2H grad_coeffs"))) return e;
  if (grad_rhs && (e = check_cuda(cudaMemcpyAsync(grad_rhs, q->gd, bd, d2h, st), "D2H grad_rhs"))) return e;
  if (grad_iv && (e = check_cuda(cudaMemcpyAsync(grad_iv, q->gu, bu, d2h, st), "D2H grad_iv"))) return e;
  if (grad_steps && bs && (e = check_cuda(cudaMemcpyAsync(grad_steps, q->gs, bs, d2h, st), "D2H grad_steps")))
    return e;
  if (info && (e = check_cuda(cudaMemcpyAsync(info, q->info, n * 4, d2h, st), "D2H info"))) return e;
  return SMNN_OK;
}

}  // extern "C"
