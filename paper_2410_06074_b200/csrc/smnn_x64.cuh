// smnn_x64.cuh -- cluster-resident S-MNN solve in fp64 arithmetic ("x64" path).
//
// The accurate path of the library: SMNN_F32_C64 (fp32 storage, fp64
// arithmetic) and SMNN_F64.  An fp32 normal-equations solve cannot meet the
// 1e-4 parity bar (R7: rounding M alone to fp32 costs 1e-4..1e-3 at
// the bench's conditioning), and the gradients' residual terms amplify even the
// fp32 ROUNDING of y by up to 1e4 (dl/ds: 1e-3), so the backward pass solves
// for y again, in fp64, beside dl/dbeta -- it never reads y from storage.
//
// One thread-block CLUSTER of NC CTAs solves one instance (PAPER.md:68-80 with
// V = Q = 1); CTA r of the cluster owns time chunks k = r NT .. r NT + NT - 1
// (NT threads, one chunk each, K = NC NT chunks, chunk k = [f_k, f_{k+1}),
// f_k = floor(k T / K), at most C points).  The chunk's last point sigma_k is a
// separator, the points before it its interior (0 .. C-1 points).
//
//   staging  c, d, s (+ dl/dy) of the CTA's time range: TMA bulk copies into
//            shared memory (cp.async.bulk + mbarrier); HBM is read once.
//   pass 1   block Cholesky of the chunk interior (Algorithm 3's loop,
//            PAPER.md:249-256), factors L_j kept in REGISTERS until pass 2,
//            with the spike X_j = (G^{-1})_{j,f} N_{f-1} giving the Schur
//            complement of the interior onto its two separators.
//   local    block cyclic reduction of the CTA's NT separators onto the two
//            CTA boundaries (the previous CTA's last separator, "position 0",
//            and its own last one, "position NT"), records in shared memory.
//   cluster  one barrier.cluster; every CTA reads the NC boundary Schur blocks
//            of its cluster through distributed shared memory and solves the
//            NC-block tridiagonal boundary system itself (block Cholesky +
//            substitution, Algorithms 3/4 on the reduced system).
//   back     the local reduction's back substitution: y at every separator.
//   pass 2   forward substitution of the interior with y(sigma_{k-1}) known,
//            back substitution from y(sigma_k) (Algorithm 4)
//            on the register-resident factors; FWD writes y, BWD the
//            Appendix A.1 gradient chain from lambda =
//            M^{-1} dl/dy (Eq. 13) and y.
//   store    outputs overwrite their inputs in shared memory and leave by TMA
//            bulk stores.
//
// NR right-hand sides share one factorisation: forward NR = 1 (beta), backward
// NR = 2 (dl/dy -> lambda, beta -> y).  Nothing but the inputs and outputs
// touches HBM: M, the factors, the separator systems and y (backward) live in
// registers and shared memory.
#pragma once

#include <cooperative_groups.h>

#include <climits>

#include "smnn_device.cuh"
#include "smnn_tma.cuh"

namespace smnn {
namespace x64 {

// ------------------------------------------------------------ parameters --
template <class Tio>
struct XArgs {
  const Tio* coeffs;
  const Tio* rhs;
  const Tio* iv;
  const Tio* steps;
  const Tio* grad_y;  // BWD
  Tio* y_out;         // FWD
  Tio* g_coeffs;      // BWD outputs (nullable)
  Tio* g_rhs;
  Tio* g_iv;
  Tio* g_steps;
  int32_t* info;      // nullable
  int T, n_iv;
  double wg2, wi2, ws2;
};

struct XL {
  int NC, NT, K;                                           // CTAs per cluster, threads per CTA, chunks
  int off_c, off_d, off_s, off_g, off_rec, off_pub, off_bar;  // shared-memory byte offsets (16-aligned)
};

template <int B, int NR>
struct Rec {  // separator record of the local reduction (odd stride: no bank conflicts at odd h)
  static constexpr int LT = B * (B + 1) / 2;
  static constexpr int L = 0, F = LT, E = LT + B * B, G = LT + 2 * B * B, Y = LT + 2 * B * B + NR * B;
  static constexpr int N = (LT + 2 * B * B + 2 * NR * B) | 1;
  // pass-1 hand-over, aliased on the records before the reduction starts
  static constexpr int HA = 0, HR = LT, HB = LT + NR * B;
};

template <int B, int NR>
struct Pub {  // a CTA's reduced boundary blocks, read by the cluster through DSMEM
  static constexpr int LT = B * (B + 1) / 2;
  static constexpr int DN = 0, BN = LT, RN = LT + B * B, D0 = LT + B * B + NR * B, R0 = 2 * LT + B * B + NR * B;
  static constexpr int N = 2 * LT + B * B + 2 * NR * B;
};

// ------------------------------------------------------------- algebra ----
// Lower-triangular factors keep the INVERSE diagonal: Lf[i][i] = 1 / L_ii.

// 1/sqrt(a) in fp64: the MUFU double-precision approximation x0 (about 2^-17
// relative) refined by one third-order step x0 (1 + e/2 + 3e^2/8), e = 1 - a x0^2
// (relative error ~2^-51, five DFMA-pipe ops; rsqrt(double) costs a longer
// sequence).  a <= 0 or NaN gives NaN or inf, which the recurrences carry to
// the pivot check.
__device__ __forceinline__ double rsq(double a) {
  double x;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(x) : "d"(a));
  const double e = fma(-a * x, x, 1.0);
  return fma(x * e, fma(0.375, e, 0.5), x);
}

// a_m = ws2 s^m, m = 0 .. 2B-2 (Appendix A.1 weights of one interval).
template <int B>
__device__ __forceinline__ void spow(double s, double ws2, double (&a)[2 * B - 1]) {
  a[0] = ws2;
#pragma unroll
  for (int m = 1; m < 2 * B - 1; ++m) a[m] = a[m - 1] * s;
}
template <int B>
__device__ __forceinline__ void zpow(double (&a)[2 * B - 1]) {
#pragma unroll
  for (int m = 0; m < 2 * B - 1; ++m) a[m] = 0.0;
}

// M_j (lower triangle) = wg2 c c^T + SP(an) + SM(ap)  (Appendix A.1):
// entries G_ik (an_{i+k} + (-1)^{i+k} ap_{i+k}) + [i=k] (an_{2i} + ap_{2i}).
template <int B>
__device__ __forceinline__ void assemble(const double (&c)[B], double wg2, const double (&ap)[2 * B - 1],
                                         const double (&an)[2 * B - 1], double (&M)[B][B], double (&wc)[B]) {
  double e[2 * B - 1];
#pragma unroll
  for (int m = 0; m < 2 * B - 1; ++m) e[m] = (m & 1) ? an[m] - ap[m] : an[m] + ap[m];
#pragma unroll
  for (int i = 0; i < B; ++i) wc[i] = wg2 * c[i];
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k <= i; ++k) M[i][k] = fma(wc[i], c[k], (Gc(i, k) + (i == k ? 1.0 : 0.0)) * e[i + k]);
}

// N = M_{t+1,t} = w_s^2 S** = -H o a.
template <int B>
__device__ __forceinline__ void nmat(const double (&a)[2 * B - 1], double (&N)[B][B]) {
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k < B; ++k) N[i][k] = (-Hc(i, k)) * a[i + k];
}

// In-place Cholesky of the lower triangle of S: S = L L^T, Lf with inverse diagonal.
template <int B>
__device__ __forceinline__ void chol(double (&S)[B][B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) {
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      double acc = S[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) acc = fma(-S[i][k], S[j][k], acc);
      S[i][j] = (i == j) ? rsq(acc) : acc * S[j][j];
    }
  }
}

// x = L^{-1} v (x may alias v)
template <int B>
__device__ __forceinline__ void lsolve(const double (&Lf)[B][B], const double (&v)[B], double (&x)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) {
    double acc = v[i];
#pragma unroll
    for (int k = 0; k < i; ++k) acc = fma(-Lf[i][k], x[k], acc);
    x[i] = acc * Lf[i][i];
  }
}
// x = L^{-T} v (x may alias v)
template <int B>
__device__ __forceinline__ void ltsolve(const double (&Lf)[B][B], const double (&v)[B], double (&x)[B]) {
#pragma unroll
  for (int i = B - 1; i >= 0; --i) {
    double acc = v[i];
#pragma unroll
    for (int k = i + 1; k < B; ++k) acc = fma(-Lf[k][i], x[k], acc);
    x[i] = acc * Lf[i][i];
  }
}
// X = L^{-1} Y column-wise (X may alias Y)
template <int B>
__device__ __forceinline__ void lleft(const double (&Lf)[B][B], const double (&Y)[B][B], double (&X)[B][B]) {
#pragma unroll
  for (int c = 0; c < B; ++c)
#pragma unroll
    for (int i = 0; i < B; ++i) {
      double acc = Y[i][c];
#pragma unroll
      for (int k = 0; k < i; ++k) acc = fma(-Lf[i][k], X[k][c], acc);
      X[i][c] = acc * Lf[i][i];
    }
}
// o = v - A x ; o = v - A^T x
template <int B>
__device__ __forceinline__ void vsub_ax(double (&v)[B], const double (&A)[B][B], const double (&x)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k < B; ++k) v[i] = fma(-A[i][k], x[k], v[i]);
}
template <int B>
__device__ __forceinline__ void vsub_atx(double (&v)[B], const double (&A)[B][B], const double (&x)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k < B; ++k) v[i] = fma(-A[k][i], x[k], v[i]);
}

// ---- records in shared memory
template <int B>
__device__ __forceinline__ void st_tri(double* p, const double (&m)[B][B]) {
  int e = 0;
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k <= i; ++k) p[e++] = m[i][k];
}
template <int B>
__device__ __forceinline__ void ld_tri(const double* p, double (&m)[B][B]) {
  int e = 0;
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k <= i; ++k) m[i][k] = p[e++];
}
template <int B>
__device__ __forceinline__ void st_full(double* p, const double (&m)[B][B]) {
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k < B; ++k) p[i * B + k] = m[i][k];
}
template <int B>
__device__ __forceinline__ void ld_full(const double* p, double (&m)[B][B]) {
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k < B; ++k) m[i][k] = p[i * B + k];
}
template <int B, int NR>
__device__ __forceinline__ void st_v(double* p, const double (&v)[NR][B]) {
#pragma unroll
  for (int q = 0; q < NR; ++q)
#pragma unroll
    for (int i = 0; i < B; ++i) p[q * B + i] = v[q][i];
}
template <int B, int NR>
__device__ __forceinline__ void ld_v(const double* p, double (&v)[NR][B]) {
#pragma unroll
  for (int q = 0; q < NR; ++q)
#pragma unroll
    for (int i = 0; i < B; ++i) v[q][i] = p[q * B + i];
}

// ------------------------------------------------- the staged time range ---
// Shared-memory views of the CTA's inputs (and, in place, outputs): element j
// of stream X at xs[(j - base) ...].
template <class Tio>
struct Stage {
  Tio* c;  // c_j at c[j * B] (pointer pre-offset by -ta * B)
  Tio* d;  // d_j at d[j]
  Tio* s;  // s_j at s[j]
  Tio* g;  // dl/dy_j at g[j * B]
};

// Right-hand sides at point j: rho 0 = dl/dy (BWD) or beta, rho 1 = beta (BWD):
// beta_j = wg2 c_j d_j (+ wi2 u at t = 0).
template <int B, int NR, class Tio, bool BWD>
__device__ __forceinline__ void rhs_at(const Stage<Tio>& st, const XArgs<Tio>& a, const double* u, int j,
                                       const double (&wc)[B], double (&r)[NR][B]) {
  const double d = double(st.d[j]);
  constexpr int qb = BWD ? 1 : 0;
  if (BWD) {
#pragma unroll
    for (int i = 0; i < B; ++i) r[0][i] = double(st.g[j * B + i]);
  }
#pragma unroll
  for (int i = 0; i < B; ++i) r[qb][i] = wc[i] * d;
  if (j == 0) {
#pragma unroll
    for (int i = 0; i < B; ++i)
      if (i < a.n_iv) r[qb][i] = fma(a.wi2, u[i], r[qb][i]);
  }
}

template <int B, class Tio>
__device__ __forceinline__ void load_c(const Stage<Tio>& st, int j, double (&c)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) c[i] = double(st.c[j * B + i]);
}

// dl/ds_j of interval (j, j+1), a_m = ws2 s_j^m (Appendix A.1 differentiated in s, R5):
//   -[ lj^T J+ yj + ln^T J- yn + ln^T K yj + yn^T K lj ],  J+/J-/K = d/ds of SP, SM, -H o s^{i+k}.
template <int B>
__device__ __forceinline__ double dsds(const double (&a)[2 * B - 1], const double (&lj)[B], const double (&yj)[B],
                                       const double (&ln)[B], const double (&yn)[B]) {
  double acc[2 * B - 1];
#pragma unroll
  for (int m = 0; m < 2 * B - 1; ++m) acc[m] = 0.0;
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int m = i + k;
      if (m == 0) continue;
      const double cp = Gc(i, k) * m + (i == k ? 2.0 * i : 0.0);
      const double cm = sgn(m) * Gc(i, k) * m + (i == k ? 2.0 * i : 0.0);
      const double ck = -Hc(i, k) * m;
      double t = fma(cp * lj[i], yj[k], acc[m]);
      t = fma(cm * ln[i], yn[k], t);
      acc[m] = fma(ck, fma(ln[i], yj[k], yn[i] * lj[k]), t);
    }
  double r = 0.0;
#pragma unroll
  for (int m = 1; m < 2 * B - 1; ++m) r = fma(a[m - 1], acc[m], r);
  return -r;
}

// Point gradients (Appendix A.1 with dM = -lambda y^T, dbeta = lambda; Eq. 13):
//   dd_j = wg2 c.lambda ; dc_j = wg2 (d_j lambda - lambda (y.c) - y (lambda.c))
template <int B, class Tio>
__device__ __forceinline__ void point_grads(const Stage<Tio>& st, double wg2, int j, const double (&lam)[B],
                                            const double (&y)[B], bool gc, bool gd) {
  double c[B];
  load_c<B, Tio>(st, j, c);
  double lc = lam[0] * c[0], yc = y[0] * c[0];
#pragma unroll
  for (int i = 1; i < B; ++i) {
    lc = fma(lam[i], c[i], lc);
    yc = fma(y[i], c[i], yc);
  }
  const double wl = wg2 * lc, wy = wg2 * yc, wd = wg2 * double(st.d[j]);
  if (gd) st.d[j] = Tio(wl);
  if (gc) {
#pragma unroll
    for (int i = 0; i < B; ++i) st.c[j * B + i] = Tio(fma(-y[i], wl, fma(-lam[i], wy, wd * lam[i])));
  }
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ============================================================ the kernel ==
template <int B, class Tio, bool BWD, int C>
__global__ void __launch_bounds__(128, 2) x64_kernel(XArgs<Tio> a, XL L) {
  constexpr int NR = BWD ? 2 : 1;
  constexpr int LT = B * (B + 1) / 2;
  using RC = Rec<B, NR>;
  using PB = Pub<B, NR>;
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  unsigned char* sm = smnn_dyn_smem;
  const int T = a.T, NT = L.NT, NC = L.NC, K = L.K;
  const int t = threadIdx.x, rank = int(cluster.block_rank());
  const int64_t g = blockIdx.x / NC;
  const int k = rank * NT + t;
  const int ta = chunk_begin(rank * NT, T, K), tb = chunk_begin((rank + 1) * NT, T, K);
  const int slo = max(ta - 1, 0), shi = min(tb, T - 1);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.off_bar);
  int* fail = reinterpret_cast<int*>(bar + 1);
  double* rec = reinterpret_cast<double*>(sm + L.off_rec);
  double* pub = reinterpret_cast<double*>(sm + L.off_pub);
  int* pubfail = reinterpret_cast<int*>(pub + PB::N);

  // ---- staging (TMA bulk copies of the CTA's time range)
  const int64_t tbB = g * int64_t(T) * B, t1 = g * int64_t(T), ts = g * int64_t(T - 1);
  const Span<Tio> pc(a.coeffs + tbB + int64_t(ta) * B, (tb - ta) * B);
  const Span<Tio> pd(a.rhs + t1 + ta, tb - ta);
  const Span<Tio> ps(a.steps + ts + slo, shi - slo);
  const Span<Tio> pg(BWD ? a.grad_y + tbB + int64_t(ta) * B : a.coeffs, BWD ? (tb - ta) * B : 0);
  if (t == 0) {
    fail[0] = INT_MAX;
    mbar_init(bar, 1);
    mbar_expect_tx(bar, pc.bytes + pd.bytes + ps.bytes + pg.bytes);
    bulk_g2s(sm + L.off_c, pc.lo, pc.bytes, bar);
    bulk_g2s(sm + L.off_d, pd.lo, pd.bytes, bar);
    if (ps.bytes) bulk_g2s(sm + L.off_s, ps.lo, ps.bytes, bar);
    if (BWD) bulk_g2s(sm + L.off_g, pg.lo, pg.bytes, bar);
  }
  Stage<Tio> st;
  st.c = reinterpret_cast<Tio*>(sm + L.off_c) + pc.pre - int64_t(ta) * B;
  st.d = reinterpret_cast<Tio*>(sm + L.off_d) + pd.pre - ta;
  st.s = reinterpret_cast<Tio*>(sm + L.off_s) + ps.pre - slo;
  st.g = BWD ? reinterpret_cast<Tio*>(sm + L.off_g) + pg.pre - int64_t(ta) * B : nullptr;
  double u[B];
#pragma unroll
  for (int i = 0; i < B; ++i) u[i] = (i < a.n_iv) ? double(a.iv[g * a.n_iv + i]) : 0.0;
  const int f = chunk_begin(k, T, K), sig = chunk_begin(k + 1, T, K) - 1, nint = sig - f;
  const double wg2 = a.wg2;
  __syncthreads();  // barrier initialised
  mbar_wait(bar, 0);

  // =========================================================== pass 1 ====
  double Lr[C - 1][B][B];  // interior factors (lower, inverse diagonal)
  double Lc[B][B], w[NR][B], X[B][B], All[B][B], rl[NR][B];
  double ap[2 * B - 1];
  if (k > 0) spow<B>(double(st.s[f - 1]), a.ws2, ap); else zpow<B>(ap);
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int q = 0; q < B; ++q) { X[i][q] = 0.0; All[i][q] = 0.0; Lc[i][q] = 0.0; }
#pragma unroll
  for (int q = 0; q < NR; ++q)
#pragma unroll
    for (int i = 0; i < B; ++i) { w[q][i] = 0.0; rl[q][i] = 0.0; }
#pragma unroll
  for (int i = 0; i < C - 1; ++i) {
    if (i < nint) {
      const int j = f + i;
      double c[B], an[2 * B - 1], M[B][B], wc[B], r[NR][B];
      load_c<B, Tio>(st, j, c);
      spow<B>(double(st.s[j]), a.ws2, an);
      assemble<B>(c, wg2, ap, an, M, wc);
      if (j == 0) {
#pragma unroll
        for (int q = 0; q < B; ++q)
          if (q < a.n_iv) M[q][q] += a.wi2;
      }
      rhs_at<B, NR, Tio, BWD>(st, a, u, j, wc, r);
      double N[B][B];
      nmat<B>(ap, N);  // N_{j-1} = M_{j, j-1}
      if (i == 0) {
        chol<B>(M);
#pragma unroll
        for (int q = 0; q < NR; ++q) lsolve<B>(M, r[q], w[q]);
        lleft<B>(M, N, X);  // X_f = L_f^{-1} N_{f-1} (zero for k = 0)
#pragma unroll
        for (int p = 0; p < B; ++p) {
#pragma unroll
          for (int q = 0; q <= p; ++q) {
            double acc = X[0][p] * X[0][q];
#pragma unroll
            for (int m = 1; m < B; ++m) acc = fma(X[m][p], X[m][q], acc);
            All[p][q] = acc;
          }
#pragma unroll
          for (int q = 0; q < NR; ++q) {
            double acc = X[0][p] * w[q][0];
#pragma unroll
            for (int m = 1; m < B; ++m) acc = fma(X[m][p], w[q][m], acc);
            rl[q][p] = acc;
          }
        }
      } else {
        double P[B][B];  // P_{j-1} = N_{j-1} L_{j-1}^{-T}
#pragma unroll
        for (int p = 0; p < B; ++p) lsolve<B>(Lc, N[p], P[p]);
#pragma unroll
        for (int p = 0; p < B; ++p)
#pragma unroll
          for (int q = 0; q <= p; ++q) {
            double acc = M[p][q];
#pragma unroll
            for (int m = 0; m < B; ++m) acc = fma(-P[p][m], P[q][m], acc);
            M[p][q] = acc;
          }
#pragma unroll
        for (int q = 0; q < NR; ++q) vsub_ax<B>(r[q], P, w[q]);
        chol<B>(M);
#pragma unroll
        for (int q = 0; q < NR; ++q) lsolve<B>(M, r[q], w[q]);
        double Y[B][B];  // X_j = -L_j^{-1} P_{j-1} X_{j-1}
#pragma unroll
        for (int p = 0; p < B; ++p)
#pragma unroll
          for (int q = 0; q < B; ++q) {
            double acc = -P[p][0] * X[0][q];
#pragma unroll
            for (int m = 1; m < B; ++m) acc = fma(-P[p][m], X[m][q], acc);
            Y[p][q] = acc;
          }
        lleft<B>(M, Y, X);
#pragma unroll
        for (int p = 0; p < B; ++p) {
#pragma unroll
          for (int q = 0; q <= p; ++q) {
            double acc = All[p][q];
#pragma unroll
            for (int m = 0; m < B; ++m) acc = fma(X[m][p], X[m][q], acc);
            All[p][q] = acc;
          }
#pragma unroll
          for (int q = 0; q < NR; ++q) {
            double acc = rl[q][p];
#pragma unroll
            for (int m = 0; m < B; ++m) acc = fma(X[m][p], w[q][m], acc);
            rl[q][p] = acc;
          }
        }
      }
#pragma unroll
      for (int p = 0; p < B; ++p)
#pragma unroll
        for (int q = 0; q <= p; ++q) { Lc[p][q] = M[p][q]; Lr[i][p][q] = M[p][q]; }
#pragma unroll
      for (int m = 0; m < 2 * B - 1; ++m) ap[m] = an[m];
    }
  }
  // pivot check once per chunk: a breakdown leaves a non-finite last factor
  bool bad = nint > 0 && !isfinite(Lc[B - 1][B - 1]);
  // the separator sigma: own block minus the interior's Schur terms
  double Dsep[B][B], Rsep[NR][B], Arl[B][B];
  {
    double c[B], an[2 * B - 1], wc[B];
    load_c<B, Tio>(st, sig, c);
    if (sig < T - 1) spow<B>(double(st.s[sig]), a.ws2, an); else zpow<B>(an);
    assemble<B>(c, wg2, ap, an, Dsep, wc);  // ap = a(s_{sig-1}) (zero when sig = 0)
    if (sig == 0) {
#pragma unroll
      for (int q = 0; q < B; ++q)
        if (q < a.n_iv) Dsep[q][q] += a.wi2;
    }
    rhs_at<B, NR, Tio, BWD>(st, a, u, sig, wc, Rsep);
    double N[B][B];
    nmat<B>(ap, N);  // N_{sig-1} = M_{sig, sig-1}
    if (nint > 0) {
      double P[B][B];
#pragma unroll
      for (int p = 0; p < B; ++p) lsolve<B>(Lc, N[p], P[p]);
#pragma unroll
      for (int p = 0; p < B; ++p)
#pragma unroll
        for (int q = 0; q <= p; ++q) {
          double acc = Dsep[p][q];
#pragma unroll
          for (int m = 0; m < B; ++m) acc = fma(-P[p][m], P[q][m], acc);
          Dsep[p][q] = acc;
        }
#pragma unroll
      for (int q = 0; q < NR; ++q) vsub_ax<B>(Rsep[q], P, w[q]);
#pragma unroll
      for (int p = 0; p < B; ++p)  // A_rl = -P_l X_l : coupling (sigma_k, sigma_{k-1})
#pragma unroll
        for (int q = 0; q < B; ++q) {
          double acc = -P[p][0] * X[0][q];
#pragma unroll
          for (int m = 1; m < B; ++m) acc = fma(-P[p][m], X[m][q], acc);
          Arl[p][q] = acc;
        }
    } else {
#pragma unroll
      for (int p = 0; p < B; ++p)
#pragma unroll
        for (int q = 0; q < B; ++q) Arl[p][q] = N[p][q];  // direct coupling (zero for k = 0)
    }
  }
  if (bad) atomicMin(fail, f + 1);

  // ================================================ local reduction =====
  // hand-over: A_ll = -sum X^T X and r_l = -sum X^T w belong to separator
  // k - 1 (thread t - 1, or position 0 for t = 0); A_rl^T is thread t - 1's
  // coupling to the right.
  {
    double* h = rec + t * RC::N;
    int e = 0;
#pragma unroll
    for (int p = 0; p < B; ++p)
#pragma unroll
      for (int q = 0; q <= p; ++q) h[RC::HA + e++] = -All[p][q];
#pragma unroll
    for (int q = 0; q < NR; ++q)
#pragma unroll
      for (int p = 0; p < B; ++p) h[RC::HR + q * B + p] = -rl[q][p];
    st_full<B>(h + RC::HB, Arl);
  }
  __syncthreads();
  // position p = t + 1 (separator k); thread 0 also carries position 0
  double Bl[B][B], Cr[B][B], D0[B][B], r0[NR][B];
  {
#pragma unroll
    for (int p = 0; p < B; ++p)
#pragma unroll
      for (int q = 0; q < B; ++q) { Bl[p][q] = Arl[p][q]; Cr[p][q] = 0.0; D0[p][q] = 0.0; }
#pragma unroll
    for (int q = 0; q < NR; ++q)
#pragma unroll
      for (int p = 0; p < B; ++p) r0[q][p] = 0.0;
    if (t + 1 < NT) {
      const double* h = rec + (t + 1) * RC::N;
      int e = 0;
#pragma unroll
      for (int p = 0; p < B; ++p)
#pragma unroll
        for (int q = 0; q <= p; ++q) Dsep[p][q] += h[RC::HA + e++];
#pragma unroll
      for (int q = 0; q < NR; ++q)
#pragma unroll
        for (int p = 0; p < B; ++p) Rsep[q][p] += h[RC::HR + q * B + p];
#pragma unroll
      for (int p = 0; p < B; ++p)
#pragma unroll
        for (int q = 0; q < B; ++q) Cr[p][q] = h[RC::HB + q * B + p];
    }
    if (t == 0) {
      const double* h = rec;
      int e = 0;
#pragma unroll
      for (int p = 0; p < B; ++p)
#pragma unroll
        for (int q = 0; q <= p; ++q) D0[p][q] = h[RC::HA + e++];
#pragma unroll
      for (int q = 0; q < NR; ++q)
#pragma unroll
        for (int p = 0; p < B; ++p) r0[q][p] = h[RC::HR + q * B + p];
    }
  }
  __syncthreads();  // hand-over read before the records are written
  const int pos = t + 1;
  int badsep = 0;
#pragma unroll 1
  for (int h = 1; h < NT; h <<= 1) {
    const int m = pos & (2 * h - 1);
    if (m == h) {  // eliminate: publish L, F = L^{-1} Bl, E = L^{-1} Cr, g = L^{-1} r
      chol<B>(Dsep);
      double F[B][B], E[B][B];
      lleft<B>(Dsep, Bl, F);
      lleft<B>(Dsep, Cr, E);
#pragma unroll
      for (int q = 0; q < NR; ++q) lsolve<B>(Dsep, Rsep[q], Rsep[q]);
      if (!isfinite(Dsep[B - 1][B - 1])) badsep = 1;
      double* pk = rec + pos * RC::N;
      st_tri<B>(pk + RC::L, Dsep);
      st_full<B>(pk + RC::F, F);
      st_full<B>(pk + RC::E, E);
      st_v<B, NR>(pk + RC::G, Rsep);
    }
    __syncthreads();
    if (m == 0) {  // survivor: absorb the eliminated neighbours pos - h (and pos + h)
      {
        const double* pl = rec + (pos - h) * RC::N;
        double El[B][B], Fl[B][B], gl[NR][B];
        ld_full<B>(pl + RC::E, El);
        ld_full<B>(pl + RC::F, Fl);
        ld_v<B, NR>(pl + RC::G, gl);
#pragma unroll
        for (int p = 0; p < B; ++p) {
#pragma unroll
          for (int q = 0; q <= p; ++q) {
            double acc = Dsep[p][q];
#pragma unroll
            for (int x = 0; x < B; ++x) acc = fma(-El[x][p], El[x][q], acc);
            Dsep[p][q] = acc;
          }
#pragma unroll
          for (int q = 0; q < B; ++q) {
            double acc = -El[0][p] * Fl[0][q];
#pragma unroll
            for (int x = 1; x < B; ++x) acc = fma(-El[x][p], Fl[x][q], acc);
            Bl[p][q] = acc;
          }
        }
#pragma unroll
        for (int q = 0; q < NR; ++q) vsub_atx<B>(Rsep[q], El, gl[q]);
      }
      if (pos < NT) {
        const double* pr = rec + (pos + h) * RC::N;
        double Fr[B][B], Er[B][B], gr[NR][B];
        ld_full<B>(pr + RC::F, Fr);
        ld_full<B>(pr + RC::E, Er);
        ld_v<B, NR>(pr + RC::G, gr);
#pragma unroll
        for (int p = 0; p < B; ++p) {
#pragma unroll
          for (int q = 0; q <= p; ++q) {
            double acc = Dsep[p][q];
#pragma unroll
            for (int x = 0; x < B; ++x) acc = fma(-Fr[x][p], Fr[x][q], acc);
            Dsep[p][q] = acc;
          }
#pragma unroll
          for (int q = 0; q < B; ++q) {
            double acc = -Fr[0][p] * Er[0][q];
#pragma unroll
            for (int x = 1; x < B; ++x) acc = fma(-Fr[x][p], Er[x][q], acc);
            Cr[p][q] = acc;
          }
        }
#pragma unroll
        for (int q = 0; q < NR; ++q) vsub_atx<B>(Rsep[q], Fr, gr[q]);
      }
    }
    if (t == 0) {  // position 0 absorbs position h (eliminated at this level)
      const double* pr = rec + h * RC::N;
      double Fr[B][B], gr[NR][B];
      ld_full<B>(pr + RC::F, Fr);
      ld_v<B, NR>(pr + RC::G, gr);
#pragma unroll
      for (int p = 0; p < B; ++p)
#pragma unroll
        for (int q = 0; q <= p; ++q) {
          double acc = D0[p][q];
#pragma unroll
          for (int x = 0; x < B; ++x) acc = fma(-Fr[x][p], Fr[x][q], acc);
          D0[p][q] = acc;
        }
#pragma unroll
      for (int q = 0; q < NR; ++q) vsub_atx<B>(r0[q], Fr, gr[q]);
    }
  }
  if (badsep) atomicMin(fail, sig + 1);
  // publish the CTA's boundary blocks: position NT (own last separator) and position 0
  if (t == NT - 1) {
    st_tri<B>(pub + PB::DN, Dsep);
    st_full<B>(pub + PB::BN, Bl);
    st_v<B, NR>(pub + PB::RN, Rsep);
  }
  if (t == 0) {
    st_tri<B>(pub + PB::D0, D0);
    st_v<B, NR>(pub + PB::R0, r0);
  }
  __syncthreads();
  if (t == 0) pubfail[0] = fail[0];
  cluster.sync();  // every CTA's boundary blocks are published

  // ================================== boundary system (every CTA, thread 0)
  if (t == 0) {
    // block tridiagonal over the NC CTA boundaries q: diagonal DN(q) + D0(q+1),
    // rhs RN(q) + R0(q+1), coupling (q, q-1) = BN(q).  Block Cholesky forward,
    // then back substitution down to q = rank - 1.
    double Lq[16][LT], Pq[16][B * B], wq[16][NR * B];
    int bfail = INT_MAX;
    double Lp[B][B];
    double wp[NR][B];
    for (int q = 0; q < NC; ++q) {
      const double* pq = cluster.map_shared_rank(pub, q);
      double Dq[B][B], Rq[NR][B];
      ld_tri<B>(pq + PB::DN, Dq);
      ld_v<B, NR>(pq + PB::RN, Rq);
      if (q + 1 < NC) {
        const double* pn = cluster.map_shared_rank(pub, q + 1);
        double D1[B][B], R1[NR][B];
        ld_tri<B>(pn + PB::D0, D1);
        ld_v<B, NR>(pn + PB::R0, R1);
#pragma unroll
        for (int p = 0; p < B; ++p)
#pragma unroll
          for (int x = 0; x <= p; ++x) Dq[p][x] += D1[p][x];
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
          for (int p = 0; p < B; ++p) Rq[r][p] += R1[r][p];
      }
      if (q > 0) {
        double Bq[B][B], P[B][B];
        ld_full<B>(pq + PB::BN, Bq);
#pragma unroll
        for (int p = 0; p < B; ++p) lsolve<B>(Lp, Bq[p], P[p]);
#pragma unroll
        for (int p = 0; p < B; ++p)
#pragma unroll
          for (int x = 0; x <= p; ++x) {
            double acc = Dq[p][x];
#pragma unroll
            for (int m = 0; m < B; ++m) acc = fma(-P[p][m], P[x][m], acc);
            Dq[p][x] = acc;
          }
#pragma unroll
        for (int r = 0; r < NR; ++r) vsub_ax<B>(Rq[r], P, wp[r]);
#pragma unroll
        for (int p = 0; p < B; ++p)
#pragma unroll
          for (int x = 0; x < B; ++x) Pq[q][p * B + x] = P[p][x];
      }
      chol<B>(Dq);
      if (!isfinite(Dq[B - 1][B - 1]) && bfail == INT_MAX) bfail = chunk_begin((q + 1) * NT, T, K);  // 1 + time
#pragma unroll
      for (int r = 0; r < NR; ++r) lsolve<B>(Dq, Rq[r], wp[r]);
      int e = 0;
#pragma unroll
      for (int p = 0; p < B; ++p)
#pragma unroll
        for (int x = 0; x <= p; ++x) { Lq[q][e++] = Dq[p][x]; Lp[p][x] = Dq[p][x]; }
#pragma unroll
      for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int p = 0; p < B; ++p) wq[q][r * B + p] = wp[r][p];
    }
    double yn[NR][B], yown[NR][B], yleft[NR][B];
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int p = 0; p < B; ++p) { yn[r][p] = 0.0; yown[r][p] = 0.0; yleft[r][p] = 0.0; }
    for (int q = NC - 1; q >= max(rank - 1, 0); --q) {
      double Lf[B][B];
      int e = 0;
#pragma unroll
      for (int p = 0; p < B; ++p)
#pragma unroll
        for (int x = 0; x <= p; ++x) Lf[p][x] = Lq[q][e++];
      double tv[NR][B];
#pragma unroll
      for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int p = 0; p < B; ++p) tv[r][p] = wq[q][r * B + p];
      if (q + 1 < NC) {
        double P[B][B];
#pragma unroll
        for (int p = 0; p < B; ++p)
#pragma unroll
          for (int x = 0; x < B; ++x) P[p][x] = Pq[q + 1][p * B + x];
#pragma unroll
        for (int r = 0; r < NR; ++r) vsub_atx<B>(tv[r], P, yn[r]);
      }
#pragma unroll
      for (int r = 0; r < NR; ++r) ltsolve<B>(Lf, tv[r], yn[r]);
      if (q == rank) {
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
          for (int p = 0; p < B; ++p) yown[r][p] = yn[r][p];
      }
      if (q == rank - 1) {
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
          for (int p = 0; p < B; ++p) yleft[r][p] = yn[r][p];
      }
    }
    st_v<B, NR>(rec + 0 * RC::N + RC::Y, yleft);
    st_v<B, NR>(rec + NT * RC::N + RC::Y, yown);
    if (rank == 0) {
      int fm = bfail;
      for (int q = 0; q < NC; ++q) fm = min(fm, *reinterpret_cast<const int*>(
                                                    cluster.map_shared_rank(pub, q) + PB::N));
      if (a.info) a.info[g] = (fm == INT_MAX) ? 0 : fm;
    }
  }
  __syncthreads();   // thread 0's remote reads are done
  cluster_arrive();  // ... so this CTA's published blocks may go once all have arrived (wait before exit)

  // ====================================== back substitution of the local reduction
  {
    int hmax = 1;
    while (hmax < NT) hmax <<= 1;
#pragma unroll 1
    for (int h = hmax >> 1; h >= 1; h >>= 1) {
      if ((pos & (2 * h - 1)) == h) {
        const double* pk = rec + pos * RC::N;
        double Lf[B][B], F[B][B], E[B][B], gv[NR][B], yl[NR][B], yr[NR][B];
        ld_tri<B>(pk + RC::L, Lf);
        ld_full<B>(pk + RC::F, F);
        ld_full<B>(pk + RC::E, E);
        ld_v<B, NR>(pk + RC::G, gv);
        ld_v<B, NR>(rec + (pos - h) * RC::N + RC::Y, yl);
        ld_v<B, NR>(rec + (pos + h) * RC::N + RC::Y, yr);
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          vsub_ax<B>(gv[q], F, yl[q]);
          vsub_ax<B>(gv[q], E, yr[q]);
          ltsolve<B>(Lf, gv[q], gv[q]);
        }
        st_v<B, NR>(rec + pos * RC::N + RC::Y, gv);
      }
      __syncthreads();
    }
  }

  // =========================================================== pass 2 ====
  double yL[NR][B], yR[NR][B];
  ld_v<B, NR>(rec + t * RC::N + RC::Y, yL);
  ld_v<B, NR>(rec + pos * RC::N + RC::Y, yR);
  __syncthreads();  // the staged inputs are overwritten below only after every thread's reads ... (none cross chunks)
  const bool gc = BWD && a.g_coeffs, gd = BWD && a.g_rhs, gs = BWD && a.g_steps;
  {
    double Wr[C - 1][NR][B];
    double vprev[NR][B];  // L_{j-1}^{-T} w'_{j-1}, or y_L at the chunk start
#pragma unroll
    for (int q = 0; q < NR; ++q)
#pragma unroll
      for (int p = 0; p < B; ++p) vprev[q][p] = yL[q][p];
    if (k > 0) spow<B>(double(st.s[f - 1]), a.ws2, ap); else zpow<B>(ap);
#pragma unroll
    for (int i = 0; i < C - 1; ++i) {
      if (i < nint) {
        const int j = f + i;
        double c[B], wc[B], r[NR][B], N[B][B], an[2 * B - 1];
        load_c<B, Tio>(st, j, c);
#pragma unroll
        for (int p = 0; p < B; ++p) wc[p] = wg2 * c[p];
        rhs_at<B, NR, Tio, BWD>(st, a, u, j, wc, r);
        nmat<B>(ap, N);  // rhs -= N_{j-1} (L_{j-1}^{-T} w'_{j-1})  resp.  N_{f-1} y_L
#pragma unroll
        for (int q = 0; q < NR; ++q) vsub_ax<B>(r[q], N, vprev[q]);
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          lsolve<B>(Lr[i], r[q], Wr[i][q]);
          ltsolve<B>(Lr[i], Wr[i][q], vprev[q]);
        }
        spow<B>(double(st.s[j]), a.ws2, an);
#pragma unroll
        for (int m = 0; m < 2 * B - 1; ++m) ap[m] = an[m];
      }
    }
    // the separator: y known
    if constexpr (BWD) {
      point_grads<B, Tio>(st, wg2, sig, yR[0], yR[1], gc, gd);
    } else {
#pragma unroll
      for (int p = 0; p < B; ++p) st.c[sig * B + p] = Tio(yR[0][p]);
    }
    double yn[NR][B];
#pragma unroll
    for (int q = 0; q < NR; ++q)
#pragma unroll
      for (int p = 0; p < B; ++p) yn[q][p] = yR[q][p];
#pragma unroll
    for (int i = C - 2; i >= 0; --i) {
      if (i < nint) {
        const int j = f + i;
        double an[2 * B - 1], N[B][B], yv[NR][B];
        spow<B>(double(st.s[j]), a.ws2, an);
        nmat<B>(an, N);  // N_j = M_{j+1, j}
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          double v[B];
#pragma unroll
          for (int p = 0; p < B; ++p) {
            double acc = N[0][p] * yn[q][0];
#pragma unroll
            for (int x = 1; x < B; ++x) acc = fma(N[x][p], yn[q][x], acc);
            v[p] = acc;
          }
          lsolve<B>(Lr[i], v, v);
#pragma unroll
          for (int p = 0; p < B; ++p) v[p] = Wr[i][q][p] - v[p];
          ltsolve<B>(Lr[i], v, yv[q]);
        }
        if constexpr (BWD) {
          point_grads<B, Tio>(st, wg2, j, yv[0], yv[1], gc, gd);
          if (gs) st.s[j] = Tio(dsds<B>(an, yv[0], yv[1], yn[0], yn[1]));
        } else {
#pragma unroll
          for (int p = 0; p < B; ++p) st.c[j * B + p] = Tio(yv[0][p]);
        }
#pragma unroll
        for (int q = 0; q < NR; ++q)
#pragma unroll
          for (int p = 0; p < B; ++p) yn[q][p] = yv[q][p];
      }
    }
    if constexpr (BWD) {
      if (k > 0 && gs) {  // interval (sigma_{k-1}, f) belongs to this chunk
        double am[2 * B - 1];
        spow<B>(double(st.s[f - 1]), a.ws2, am);
        st.s[f - 1] = Tio(dsds<B>(am, yL[0], yL[1], yn[0], yn[1]));
      }
      if (k == 0 && a.g_iv) {  // dl/du = wi2 lambda_0 (point 0 = f)
        for (int p = 0; p < a.n_iv; ++p) a.g_iv[g * a.n_iv + p] = Tio(a.wi2 * yn[0][p]);
      }
    }
  }

  // ---- outputs: TMA bulk store of the aligned body, plain stores at the ends
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  Tio* cb = st.c + int64_t(ta) * B;
  if (!BWD) {
    rf_store_out(a.y_out + tbB + int64_t(ta) * B, cb, (tb - ta) * B, t, NT);
  } else {
    if (a.g_coeffs) rf_store_out(a.g_coeffs + tbB + int64_t(ta) * B, cb, (tb - ta) * B, t, NT);
    if (a.g_rhs) rf_store_out(a.g_rhs + t1 + ta, st.d + ta, tb - ta, t, NT);
    if (a.g_steps && tb - 1 > slo) rf_store_out(a.g_steps + ts + slo, st.s + slo, tb - 1 - slo, t, NT);
  }
  if (t == 0) {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  cluster_wait();  // no CTA leaves while another may still read its published blocks
}

}  // namespace x64
}  // namespace smnn
