// smnn_rf.cuh -- register-factor (RF) resident kernel of the S-MNN solve.
//
// One CTA solves one instance whose inputs fit in shared memory (bulk-copied
// there by TMA, as in resident_kernel).  Thread k owns time chunk
// [f_k, f_{k+1}), f_k = floor(k T / K), K = blockDim.x chunks of at most CM
// points (CM compile-time); the chunk's last point sigma_k is a separator, the
// points before it its interior (>= 1 point).  Compared with resident_kernel:
//
//  * the interior Cholesky factors L_j (Algorithm 3's loop)
//    stay in REGISTERS between pass 1 and pass 2 (the chunk loop is fully
//    unrolled over CM, so every factor has a compile-time register home):
//    pass 2 is substitution only (Algorithm 4), with no
//    re-factorisation and no checkpoints;
//  * pass 2 forward-substitutes the right-hand side with both separator
//    values known (w'_j = L_j^{-1}(beta_j - N_{j-1} L_{j-1}^{-T} w'_{j-1}),
//    w'_f = L_f^{-1}(beta_f - N_{f-1} y_L)) and back-substitutes
//    y_j = L_j^{-T}(w'_j - L_j^{-1} N_j^T y_{j+1}) from y_{sigma_k};
//  * the separator block-cyclic reduction is inlined (no call boundary, so
//    the factor registers are not spilled around it).
// Everything else (Appendix A.1 assembly, the spike / Schur complement onto
// the separators, the BCR, the Appendix A.1 gradient chain) is the algebra of
// smnn_fused.cuh, shared with the other fused kernels.
#pragma once

#include "smnn_chunk.cuh"

namespace smnn {

#ifndef SMNN_RF_CM3
#define SMNN_RF_CM3 8  // fp32, order 2 (b = 3)
#endif
// Chunk capacity: factors of CM - 1 interior points live in registers
// ((CM-1) * B(B+1)/2 values of S).
template <int B, class S>
struct RfCM {
  static constexpr int value = sizeof(S) >= 8 ? (B == 1 ? 8 : B == 2 ? 6 : B == 3 ? 3 : 2)
                                              : (B == 1 ? 16 : B == 2 ? 12 : B == 3 ? SMNN_RF_CM3 : 5);
};

// Identity the compiler cannot see through (no rematerialisation from constants).
__device__ __forceinline__ int opaque(int v) { asm volatile("" : "+r"(v)); return v; }
__device__ __forceinline__ float opaque(float v) { asm volatile("" : "+f"(v)); return v; }
__device__ __forceinline__ double opaque(double v) { asm volatile("" : "+d"(v)); return v; }

// Backward: stage the forward solution y only after the separator reduction,
// into the reduction's record region (free by then), overlapped with the
// pass-2 forward sweep -- one staging buffer less (44 -> 32 B per time point),
// so one more CTA per SM.
#ifndef RF_LATE_Y
#define RF_LATE_Y 1
#endif

// Phase timestamps (debug builds only): per CTA, globaltimer at the phase boundaries.
#ifdef SMNN_RF_TIMING
__device__ unsigned long long rf_timing[6 * 65536];
__device__ __forceinline__ unsigned long long rf_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define RF_STAMP(i) do { if (threadIdx.x == 0 && blockIdx.x < 65536) rf_timing[6 * blockIdx.x + (i)] = rf_now(); } while (0)
#else
#define RF_STAMP(i) do { } while (0)
#endif

#ifndef SMNN_RF_MIN_BLOCKS
#define SMNN_RF_MIN_BLOCKS 1
#endif

#ifndef SMNN_RF_MAX_THREADS
#define SMNN_RF_MAX_THREADS 512
#endif

template <int B, class S>
__device__ __forceinline__ void rld_low(const S* p, S (&m)[B][B]) {
#pragma unroll
  for (int r = 0; r < B; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) m[r][c] = p[r * B + c];
}
template <int B, class S>
__device__ __forceinline__ void rst_low(S* p, const S (&m)[B][B]) {
#pragma unroll
  for (int r = 0; r < B; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) p[r * B + c] = m[r][c];
}
template <int B, class S>
__device__ __forceinline__ void rld_full(const S* p, S (&m)[B][B]) {
#pragma unroll
  for (int r = 0; r < B; ++r)
#pragma unroll
    for (int c = 0; c < B; ++c) m[r][c] = p[r * B + c];
}
template <int B, class S>
__device__ __forceinline__ void rst_full(S* p, const S (&m)[B][B]) {
#pragma unroll
  for (int r = 0; r < B; ++r)
#pragma unroll
    for (int c = 0; c < B; ++c) p[r * B + c] = m[r][c];
}
template <int B, class S>
__device__ __forceinline__ void rld_v(const S* p, S (&v)[B]) {
#pragma unroll
  for (int r = 0; r < B; ++r) v[r] = p[r];
}
template <int B, class S>
__device__ __forceinline__ void rst_v(S* p, const S (&v)[B]) {
#pragma unroll
  for (int r = 0; r < B; ++r) p[r] = v[r];
}

// Block cyclic reduction of the K separators (SPD block tridiagonal), the
// algebra of lbcr_body on the record layout: level h eliminates o = h (mod 2h)
// (Cholesky of D_o, Y1 = L^{-1} B_o, Y2 = L^{-1} B_{o+h}^T, v = L^{-1} r_o) and
// updates the survivors e = 0 (mod 2h); back substitution
// y_o = L_o^{-T}(v_o - Y1 y_{o-h} - Y2 y_{o+h}).  All K threads call it.
// ------------------------------------------------- BCR, registers resident ---
// Block cyclic reduction with every separator's blocks in its thread's
// registers (D, Bl = block (i, i-h), Cr = block (i, i+h), r).  At level h the
// threads i = h (mod 2h) eliminate their separator -- D = L L^T, publish
// L, F = L^{-1} Bl, E = L^{-1} Cr, g = L^{-1} r -- and after one barrier the
// survivors i = 0 (mod 2h) update from their neighbours i -+ h:
//   D -= E_{i-h}^T E_{i-h} + F_{i+h}^T F_{i+h},  r -= E_{i-h}^T g_{i-h} + F_{i+h}^T g_{i+h},
//   Bl = -E_{i-h}^T F_{i-h},  Cr = -F_{i+h}^T E_{i+h}.
// A separator publishes exactly once (when eliminated), so no buffer is
// overwritten and a level costs one barrier.  Back substitution, one barrier
// per level: y_i = L_i^{-T}(g_i - F_i y_{i-h} - E_i y_{i+h}).  This is the block
// Cholesky factorisation of the odd-even permuted separator system (backward
// stable), unlike PCR.  Record (BRec<B>::N values): L, F, E, g, y, then the
// pass-1 hand-over (A_ll lower, A_rl, r_l) in slots of its own.
template <int B, int NR = 1>
struct BRecN {  // NR right-hand sides share the reduction of the blocks
  static constexpr int LT = B * (B + 1) / 2;  // packed lower triangle
  static constexpr int L = 0, F = LT, E = LT + B * B, G = LT + 2 * B * B, Y = LT + 2 * B * B + NR * B;
  // pass-1 hand-over (A_ll packed lower, A_rl, r_l) shares the F / E / g slots:
  // read before the first reduction level publishes (one extra barrier)
  static constexpr int HA = F, HB = F + LT, HR = F + LT + B * B;
  static constexpr int N = (LT + 2 * B * B + 2 * NR * B) | 1;
  static constexpr bool shared_handover = true;
};
template <int B>
using BRec = BRecN<B, 1>;

template <int B, class S>
__device__ __forceinline__ void rld_tri(const S* p, S (&m)[B][B]) {
#pragma unroll
  for (int r = 0; r < B; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) m[r][c] = p[r * (r + 1) / 2 + c];
}
template <int B, class S>
__device__ __forceinline__ void rst_tri(S* p, const S (&m)[B][B]) {
#pragma unroll
  for (int r = 0; r < B; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) p[r * (r + 1) / 2 + c] = m[r][c];
}

template <int B, class S, int NR>
__device__ __forceinline__ void rbcr2n(S* rec, int K, int k, const int* stime, int* sfail, S (&D)[B][B],
                                       S (&Bl)[B][B], S (&Cr)[B][B], S (&r)[NR][B]) {
  using Q = BRecN<B, NR>;
  int bad = 0;
  int hmax = 1;
  while (hmax < K) hmax <<= 1;
  hmax >>= 1;  // largest level h < K (K >= 2)
#pragma unroll 1
  for (int h = 1; h < K; h <<= 1) {
    const int m = k & (2 * h - 1);
    if (m == h) {  // eliminate
      S Lf[B][B], F[B][B], E[B][B];
      bad |= lchol<B, S>(D, Lf);
      lleft<B, S>(Lf, Bl, F);
      lleft<B, S>(Lf, Cr, E);
      S* pk = rec + k * Q::N;
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        S gv[B];
        llsolve<B, S>(Lf, r[q], gv);
        rst_v<B, S>(pk + Q::G + q * B, gv);
      }
      rst_tri<B, S>(pk + Q::L, Lf);
      rst_full<B, S>(pk + Q::F, F);
      rst_full<B, S>(pk + Q::E, E);
    }
    __syncthreads();
    if (m == 0) {  // survivor: absorb the eliminated neighbours
      if (k - h >= 0) {
        const S* pl = rec + (k - h) * Q::N;
        S El[B][B], Fl[B][B];
        rld_full<B, S>(pl + Q::E, El);
        rld_full<B, S>(pl + Q::F, Fl);
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          S gl[B];
          rld_v<B, S>(pl + Q::G + q * B, gl);
#pragma unroll
          for (int i = 0; i < B; ++i) {
            S ar = r[q][i];
#pragma unroll
            for (int x = 0; x < B; ++x) ar = fnma_(El[x][i], gl[x], ar);
            r[q][i] = ar;
          }
        }
#pragma unroll
        for (int i = 0; i < B; ++i) {
#pragma unroll
          for (int j = 0; j <= i; ++j) {
            S a = D[i][j];
#pragma unroll
            for (int q = 0; q < B; ++q) a = fnma_(El[q][i], El[q][j], a);
            D[i][j] = a;
          }
#pragma unroll
          for (int j = 0; j < B; ++j) {
            S a = mul_(El[0][i], Fl[0][j]);
#pragma unroll
            for (int q = 1; q < B; ++q) a = fma_(El[q][i], Fl[q][j], a);
            Bl[i][j] = neg_(a);
          }
        }
      }
      if (k + h < K) {
        const S* pr = rec + (k + h) * Q::N;
        S Fr[B][B], Er[B][B];
        rld_full<B, S>(pr + Q::F, Fr);
        rld_full<B, S>(pr + Q::E, Er);
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          S gr[B];
          rld_v<B, S>(pr + Q::G + q * B, gr);
#pragma unroll
          for (int i = 0; i < B; ++i) {
            S ar = r[q][i];
#pragma unroll
            for (int x = 0; x < B; ++x) ar = fnma_(Fr[x][i], gr[x], ar);
            r[q][i] = ar;
          }
        }
#pragma unroll
        for (int i = 0; i < B; ++i) {
#pragma unroll
          for (int j = 0; j <= i; ++j) {
            S a = D[i][j];
#pragma unroll
            for (int q = 0; q < B; ++q) a = fnma_(Fr[q][i], Fr[q][j], a);
            D[i][j] = a;
          }
#pragma unroll
          for (int j = 0; j < B; ++j) {
            S a = mul_(Fr[0][i], Er[0][j]);
#pragma unroll
            for (int q = 1; q < B; ++q) a = fma_(Fr[q][i], Er[q][j], a);
            Cr[i][j] = neg_(a);
          }
        }
      } else {
        zero<B, S>(Cr);
      }
    }
  }
  if (k == 0) {  // the last survivor
    S Lf[B][B];
    bad |= lchol<B, S>(D, Lf);
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      S t[B], y[B];
      llsolve<B, S>(Lf, r[q], t);
      lltsolve<B, S>(Lf, t, y);
      rst_v<B, S>(rec + Q::Y + q * B, y);
    }
  }
  if (bad) report<1>(sfail, bad, stime[k]);
#pragma unroll 1
  for (int h = hmax; h >= 1; h >>= 1) {
    __syncthreads();
    if ((k & (2 * h - 1)) == h) {
      const S* pk = rec + k * Q::N;
      S Lf[B][B], F[B][B], E[B][B];
      rld_tri<B, S>(pk + Q::L, Lf);
      rld_full<B, S>(pk + Q::F, F);
      const bool right = k + h < K;
      if (right) rld_full<B, S>(pk + Q::E, E);
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        S yl[B], t[B], y[B];
        rld_v<B, S>(pk + Q::G + q * B, t);
        rld_v<B, S>(rec + (k - h) * Q::N + Q::Y + q * B, yl);
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int x = 0; x < B; ++x) t[i] = fnma_(F[i][x], yl[x], t[i]);
        if (right) {
          S yr[B];
          rld_v<B, S>(rec + (k + h) * Q::N + Q::Y + q * B, yr);
#pragma unroll
          for (int i = 0; i < B; ++i)
#pragma unroll
            for (int x = 0; x < B; ++x) t[i] = fnma_(E[i][x], yr[x], t[i]);
        }
        lltsolve<B, S>(Lf, t, y);
        rst_v<B, S>(rec + k * Q::N + Q::Y + q * B, y);
      }
    }
  }
  __syncthreads();
}

// One right-hand side (the rf kernel and the forward pipeline).
template <int B, class S>
__device__ __forceinline__ void rbcr2(S* rec, int K, int k, const int* stime, int* sfail, S (&D)[B][B],
                                      S (&Bl)[B][B], S (&Cr)[B][B], S (&r)[B]) {
  rbcr2n<B, S, 1>(rec, K, k, stime, sfail, D, Bl, Cr, *reinterpret_cast<S(*)[1][B]>(&r));
}


// The interior factors stay in registers from pass 1 to pass 2 (chunks of
// <= CM points; CM = RfCM, or RfCMW for the wide variant).
template <int B, class Tio, class S, bool BWD, int CM>
__global__ void __launch_bounds__(SMNN_RF_MAX_THREADS, SMNN_RF_MIN_BLOCKS) rf_kernel(Args<Tio> a, RLayout L) {
  unsigned char* sm = smnn_dyn_smem;
  Tio* smT = reinterpret_cast<Tio*>(sm);
  const int nt = blockDim.x, K = nt;
  const int k = int(threadIdx.x);
  const int T = a.T;
  using R2 = BRec<B>;
  S* sep = reinterpret_cast<S*>(sm + L.off_sep);  // K separator records
  int* stime = reinterpret_cast<int*>(sm + L.off_ck);  // after the record region
  int* sfail = stime + nt;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.off_bar);
  const Wts<S> w{opaque(splat<S>(a.wg2)), opaque(splat<S>(a.wi2)), opaque(splat<S>(a.ws2))};
  if (k == 0) mbar_init(bar, 1);
  __syncthreads();
  uint32_t parity = 0;
  const int f = chunk_begin(k, T, K), sig = chunk_begin(k + 1, T, K) - 1;
  const int nint = sig - f;  // interior points, 1 <= nint <= CM - 1 (host guarantees)
  constexpr int E = int(sizeof(Tio));

  for (int64_t g = blockIdx.x; g < a.n_inst; g += gridDim.x) {
    RF_STAMP(0);
    // ---- stage the instance (TMA bulk copies into shared memory)
    const int64_t tb = g * int64_t(T) * B, t1b = g * int64_t(T), tsb = g * int64_t(T - 1);
    const Span<Tio> pc(a.coeffs + tb, T * B);
    const Span<Tio> pd(a.rhs + t1b, T);
    const Span<Tio> ps(a.steps + tsb, T - 1);
    const Span<Tio> pg(BWD ? a.grad_y + tb : a.coeffs, BWD ? T * B : 0);
    const Span<Tio> py(BWD ? a.y_in + tb : a.coeffs, BWD ? T * B : 0);
    constexpr bool LATE_Y = BWD && RF_LATE_Y;
    if (k == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, pc.bytes + pd.bytes + ps.bytes + pg.bytes + (LATE_Y ? 0u : py.bytes));
      bulk_g2s(sm + L.off_c, pc.lo, pc.bytes, bar);
      bulk_g2s(sm + L.off_d, pd.lo, pd.bytes, bar);
      if (ps.bytes) bulk_g2s(sm + L.off_s, ps.lo, ps.bytes, bar);
      if (BWD) {
        bulk_g2s(sm + L.off_g, pg.lo, pg.bytes, bar);
        if (!LATE_Y) bulk_g2s(sm + L.off_y, py.lo, py.bytes, bar);
      }
    }
    Grp<Tio, 1> x;  // streams as element offsets into shared memory
    x.T = T;
    x.n_iv = a.n_iv;
    x.nv = 1;
    const int oc = L.off_c / E + pc.pre, od = L.off_d / E + pd.pre, os = L.off_s / E + ps.pre;
    const int og = BWD ? L.off_g / E + pg.pre : 0, oy = BWD ? L.off_y / E + py.pre : 0;
    x.c.o[0] = oc; x.d.o[0] = od; x.s.o[0] = os;
    x.gy.o[0] = og; x.yin.o[0] = oy;
    x.yout.o[0] = oc; x.gc.o[0] = oc; x.gd.o[0] = od; x.gs.o[0] = os;
    x.u[0] = a.iv + g * a.n_iv;
    x.gu[0] = (BWD && a.g_iv) ? a.g_iv + g * a.n_iv : nullptr;
    x.c.on = x.d.on = x.s.on = true;
    x.gy.on = x.yin.on = BWD;
    x.yout.on = !BWD;
    x.gc.on = BWD && a.g_coeffs;
    x.gd.on = BWD && a.g_rhs;
    x.gs.on = BWD && a.g_steps;
    x.gu_on = BWD && a.g_iv;
    // per-thread chunk views (immediate offsets from one base register each)
    // opaque() keeps these offsets in registers: otherwise the compiler
    // re-derives them from the kernel parameters at every unrolled step
    const Tio* cS = smT + opaque(oc + f * B);
    const Tio* dS = smT + opaque(od + f);
    const Tio* sS = smT + opaque(os + f);  // sS[-1] = s_{f-1}
    const Tio* gS = smT + opaque(og + f * B);
    if (k < 1) sfail[0] = INT_MAX;
    stime[k] = sig;
    mbar_wait(bar, parity);
    parity ^= 1u;
    __syncthreads();
    RF_STAMP(1);

    // ================================================================ pass 1
    S Lr[CM - 1][B][B];
    S Dsep[B][B], Rsep[B];
    S Bsep[B][B], Csep[B][B];
    {
      S All[B][B], rl[B], Arl[B][B];
      int bad = 0, badj = INT_MAX;
      S ap[2 * B - 1];
      if (k > 0) spow<B, S>(S(sS[-1]), w.s2, ap); else zero<2 * B - 1, S>(ap);
      S Lc[B][B], wv[B], X[B][B];
      zero<B, S>(Lc); zero<B, S>(wv); zero<B, S>(X); zero<B, S>(All); zero<B, S>(rl);
      S sg = splat<S>(1.0);
#pragma unroll
      for (int i = 0; i < CM - 1; ++i) {
        if (i < nint) {
          S c[B], an[2 * B - 1], M[B][B], wc[B], rhs[B];
#pragma unroll
          for (int r = 0; r < B; ++r) c[r] = S(cS[i * B + r]);
          spow<B, S>(S(sS[i]), w.s2, an);
          lassemble<B, S>(c, w.g2, ap, an, M, wc);
          if (BWD) {
#pragma unroll
            for (int r = 0; r < B; ++r) rhs[r] = S(gS[i * B + r]);
          } else {
            const S d = S(dS[i]);
#pragma unroll
            for (int r = 0; r < B; ++r) rhs[r] = mul_(wc[r], d);
          }
          if (i == 0 && k == 0) {  // initial-value rows at t = 0
#pragma unroll
            for (int r = 0; r < B; ++r)
              if (r < x.n_iv) {
                if (!BWD) rhs[r] = fma_(w.i2, S(x.u[0][r]), rhs[r]);
                M[r][r] = add_(M[r][r], w.i2);
              }
          }
          int b;
          if (i == 0) {
            b = lchol<B, S>(M, Lc);
            llsolve<B, S>(Lc, rhs, wv);
            S NL[B][B];  // spike X_f = L_f^{-1} N_{f-1} (zero for k = 0: ap = 0)
            lN<B, S>(ap, NL);
            lleft<B, S>(Lc, NL, X);
#pragma unroll
            for (int r = 0; r < B; ++r) {
#pragma unroll
              for (int q = 0; q <= r; ++q) {
                S acc = mul_(X[0][r], X[0][q]);
#pragma unroll
                for (int m = 1; m < B; ++m) acc = fma_(X[m][r], X[m][q], acc);
                All[r][q] = acc;
              }
              S acc = mul_(X[0][r], wv[0]);
#pragma unroll
              for (int m = 1; m < B; ++m) acc = fma_(X[m][r], wv[m], acc);
              rl[r] = acc;
            }
          } else {
            S Pm[B][B];
            lPfromN<B, S>(ap, Lc, Pm);  // P_{j-1} = N_{j-1} L_{j-1}^{-T}
            lcouple<B, S>(Pm, wv, M, rhs);
            b = lchol<B, S>(M, Lc);
            llsolve<B, S>(Lc, rhs, wv);
            S Y[B][B];  // spike X_j = -L_j^{-1} P_{j-1} X_{j-1}, carried with sign sg
#pragma unroll
            for (int r = 0; r < B; ++r)
#pragma unroll
              for (int q = 0; q < B; ++q) {
                S acc = mul_(Pm[r][0], X[0][q]);
#pragma unroll
                for (int m = 1; m < B; ++m) acc = fma_(Pm[r][m], X[m][q], acc);
                Y[r][q] = acc;
              }
            lleft<B, S>(Lc, Y, X);
            sg = neg_(sg);
#pragma unroll
            for (int r = 0; r < B; ++r) {
#pragma unroll
              for (int q = 0; q <= r; ++q) {
                S acc = All[r][q];
#pragma unroll
                for (int m = 0; m < B; ++m) acc = fma_(X[m][r], X[m][q], acc);
                All[r][q] = acc;
              }
              S acc = mul_(X[0][r], wv[0]);
#pragma unroll
              for (int m = 1; m < B; ++m) acc = fma_(X[m][r], wv[m], acc);
              rl[r] = fma_(sg, acc, rl[r]);
            }
          }
          (void)b;  // pivots are checked once per chunk, below
          rcopyL<B, S>(Lc, Lr[i]);
#pragma unroll
          for (int m = 0; m < 2 * B - 1; ++m) ap[m] = an[m];
        }
      }
      // A non-positive / non-finite pivot anywhere in the chunk leaves a
      // non-finite value in the last factor (rsqrt of it is NaN / inf and the
      // recurrence carries it forward): one check per chunk instead of per pivot.
      if (bad_(splat<S>(1.0) / Lc[B - 1][B - 1])) { bad = 1; badj = f; }
      // Schur complement of the interior onto (sigma_{k-1}, sigma_k); ap = a(s_l).
      S Pl[B][B];
      lPfromN<B, S>(ap, Lc, Pl);
#pragma unroll
      for (int r = 0; r < B; ++r) {
#pragma unroll
        for (int q = 0; q < B; ++q) {
          S a2 = mul_(Pl[r][0], X[0][q]);
#pragma unroll
          for (int m = 1; m < B; ++m) a2 = fma_(Pl[r][m], X[m][q], a2);
          Arl[r][q] = mul_(neg_(sg), a2);
        }
      }
      // separator's own block and rhs (Appendix A.1) plus A_rr = -P_l P_l^T, r_r = -P_l w_l
      {
        S c[B], an[2 * B - 1], wc[B];
#pragma unroll
        for (int r = 0; r < B; ++r) c[r] = S(cS[nint * B + r]);
        if (k + 1 < K) spow<B, S>(S(sS[nint]), w.s2, an); else zero<2 * B - 1, S>(an);
        lassemble<B, S>(c, w.g2, ap, an, Dsep, wc);
        if (BWD) {
#pragma unroll
          for (int r = 0; r < B; ++r) Rsep[r] = S(gS[nint * B + r]);
        } else {
          const S d = S(dS[nint]);
#pragma unroll
          for (int r = 0; r < B; ++r) Rsep[r] = mul_(wc[r], d);
        }
        lcouple<B, S>(Pl, wv, Dsep, Rsep);
      }
      // A_ll = -sum X^T X and r_l = -sum X^T w belong to sigma_{k-1}: hand them over.
#pragma unroll
      for (int r = 0; r < B; ++r) {
        rl[r] = neg_(rl[r]);
#pragma unroll
        for (int q = 0; q <= r; ++q) {
          All[r][q] = neg_(All[r][q]);
          All[q][r] = All[r][q];
        }
      }
      S* pk = sep + k * R2::N;  // hand-over to separator k-1
      rst_tri<B, S>(pk + R2::HA, All);
      rst_full<B, S>(pk + R2::HB, Arl);
      rst_v<B, S>(pk + R2::HR, rl);
      if (bad) report<1>(sfail, bad, badj);
#pragma unroll
      for (int r = 0; r < B; ++r)
#pragma unroll
        for (int q = 0; q < B; ++q) Bsep[r][q] = Arl[r][q];
    }
    __syncthreads();
    RF_STAMP(2);
    S yL[B], yR[B];
    if (k + 1 < K) {  // the right chunk's A_ll, r_l and the coupling to sigma_{k+1}
      S Al[B][B], An[B][B], rr[B];
      const S* pn = sep + (k + 1) * R2::N;
      rld_tri<B, S>(pn + R2::HA, Al);
      rld_full<B, S>(pn + R2::HB, An);
      rld_v<B, S>(pn + R2::HR, rr);
#pragma unroll
      for (int r = 0; r < B; ++r) {
        Rsep[r] = add_(Rsep[r], rr[r]);
#pragma unroll
        for (int q = 0; q <= r; ++q) Dsep[r][q] = add_(Dsep[r][q], Al[r][q]);
#pragma unroll
        for (int q = 0; q < B; ++q) Csep[r][q] = An[q][r];
      }
    } else {
      zero<B, S>(Csep);
    }
    if (R2::shared_handover) __syncthreads();  // hand-over read before level 1 publishes
    rbcr2<B, S>(sep, K, k, stime, sfail, Dsep, Bsep, Csep, Rsep);
    rld_v<B, S>(sep + k * R2::N + R2::Y, yR);
    if (k > 0) rld_v<B, S>(sep + (k - 1) * R2::N + R2::Y, yL); else zero<B, S>(yL);

    if (LATE_Y) {  // every thread has read its separator values: the records may go
      __syncthreads();
      if (k == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar, py.bytes);
        bulk_g2s(sm + L.off_y, py.lo, py.bytes, bar);
      }
    }
    RF_STAMP(3);
    // ================================================================ pass 2
    // forward substitution with both separator values known
    // w'_i goes to shared memory, in place over the step's consumed right-hand
    // side input (c_i forward -- y_i overwrites it afterwards; dl/dy_i backward)
    // when the storage type can hold it exactly, else to registers
    constexpr bool WSM = sizeof(S) == sizeof(Tio);
    S Wp[WSM ? 1 : CM - 1][B];
    Tio* wS = const_cast<Tio*>(BWD ? gS : cS);
    auto wput = [&](int i, const S (&v)[B]) {
#pragma unroll
      for (int r = 0; r < B; ++r) {
        if (WSM) wS[i * B + r] = Tio(v[r]); else Wp[WSM ? 0 : i][r] = v[r];
      }
    };
    auto wget = [&](int i, S (&v)[B]) {
#pragma unroll
      for (int r = 0; r < B; ++r) v[r] = WSM ? S(wS[i * B + r]) : Wp[WSM ? 0 : i][r];
    };
    {
      S ap[2 * B - 1];
      if (k > 0) spow<B, S>(S(sS[-1]), w.s2, ap); else zero<2 * B - 1, S>(ap);
      S wprev[B];
      zero<B, S>(wprev);
#pragma unroll
      for (int i = 0; i < CM - 1; ++i) {
        if (i < nint) {
          S an[2 * B - 1], rhs[B], t[B], Nt[B], wi[B];
          spow<B, S>(S(sS[i]), w.s2, an);
          if (BWD) {
#pragma unroll
            for (int r = 0; r < B; ++r) rhs[r] = S(gS[i * B + r]);
          } else {
            const S d = S(dS[i]);
#pragma unroll
            for (int r = 0; r < B; ++r) rhs[r] = mul_(mul_(w.g2, S(cS[i * B + r])), d);
            if (i == 0 && k == 0) {
#pragma unroll
              for (int r = 0; r < B; ++r)
                if (r < x.n_iv) rhs[r] = fma_(w.i2, S(x.u[0][r]), rhs[r]);
            }
          }
          if (i == 0) {
#pragma unroll
            for (int r = 0; r < B; ++r) t[r] = yL[r];
          } else {
            lltsolve<B, S>(Lr[i - 1], wprev, t);
          }
          rNv<B, S>(ap, t, Nt);
#pragma unroll
          for (int r = 0; r < B; ++r) rhs[r] = sub_(rhs[r], Nt[r]);
          llsolve<B, S>(Lr[i], rhs, wi);
          wput(i, wi);
#pragma unroll
          for (int r = 0; r < B; ++r) wprev[r] = wi[r];
#pragma unroll
          for (int m = 0; m < 2 * B - 1; ++m) ap[m] = an[m];
        }
      }
    }
    if (LATE_Y) {
      mbar_wait(bar, parity);
      parity ^= 1u;
    }
    // back substitution from y_{sigma_k}
    {
      S yn[B], yfn[B];
#pragma unroll
      for (int r = 0; r < B; ++r) yn[r] = yR[r];
      zero<B, S>(yfn);
      if (!BWD) {
#pragma unroll
        for (int r = 0; r < B; ++r) stl<S, Tio, 1, true>(x.yout, 1, sig * B + r, yR[r]);
      } else {
        ldlv<B, S, Tio, 1, true>(x.yin, sig * B, yfn);
        lpoint_grads<B, S, Tio, 1, true>(x, w, sig, yR, yfn);
      }
#pragma unroll
      for (int i = CM - 2; i >= 0; --i) {
        if (i < nint) {
          const int j = f + i;
          S an[2 * B - 1], v[B], u[B], t[B], yv[B];
          spow<B, S>(S(sS[i]), w.s2, an);
          rNtv<B, S>(an, yn, v);
          llsolve<B, S>(Lr[i], v, u);
          S wi[B];
          wget(i, wi);
#pragma unroll
          for (int r = 0; r < B; ++r) t[r] = sub_(wi[r], u[r]);
          lltsolve<B, S>(Lr[i], t, yv);
          if (!BWD) {
#pragma unroll
            for (int r = 0; r < B; ++r) stl<S, Tio, 1, true>(x.yout, 1, j * B + r, yv[r]);
          } else {
            S yf[B];
            ldlv<B, S, Tio, 1, true>(x.yin, j * B, yf);
            lpoint_grads<B, S, Tio, 1, true>(x, w, j, yv, yf);
            if (x.gs.on) stl<S, Tio, 1, true>(x.gs, 1, j, lds<B, S>(an, yv, yf, yn, yfn));
#pragma unroll
            for (int r = 0; r < B; ++r) yfn[r] = yf[r];
          }
#pragma unroll
          for (int r = 0; r < B; ++r) yn[r] = yv[r];
        }
      }
      if (BWD && k > 0 && x.gs.on) {  // interval (sigma_{k-1}, f)
        S yfm[B], am[2 * B - 1];
        ldlv<B, S, Tio, 1, true>(x.yin, (f - 1) * B, yfm);
        spow<B, S>(S(sS[-1]), w.s2, am);
        stl<S, Tio, 1, true>(x.gs, 1, f - 1, lds<B, S>(am, yL, yfm, yn, yfn));
      }
    }
    RF_STAMP(4);
    // ---- write the outputs back: TMA bulk store of the 16-byte aligned body,
    //      plain stores for the unaligned head / tail elements
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    {
      if (!BWD) {
        rf_store_out(a.y_out + tb, smT + oc, T * B, k, nt);
      } else {
        if (a.g_coeffs) rf_store_out(a.g_coeffs + tb, smT + oc, T * B, k, nt);
        if (a.g_rhs) rf_store_out(a.g_rhs + t1b, smT + od, T, k, nt);
        if (a.g_steps) rf_store_out(a.g_steps + tsb, smT + os, T - 1, k, nt);
      }
      if (k == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (k == 0 && a.info) a.info[g] = (sfail[0] == INT_MAX) ? 0 : sfail[0];
      // shared memory is reused (next instance) or released (exit) only after
      // the bulk stores have read it
      if (k == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
    RF_STAMP(5);
  }
}

}  // namespace smnn
