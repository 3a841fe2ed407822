// smnn_chunk.cuh -- per-chunk passes of the time-parallel S-MNN solver, shared
// by the resident kernels (smnn_rf.cuh) and the pipeline (smnn_pipe.cuh).
//
//   p1_chunk  pass 1 of one chunk: block Cholesky of the interior (Algorithm
//             3's loop) with the spike, Schur complement
//             onto the two separators;
//   p2_chunk  pass 2: re-factorisation in register segments and substitution
//             (Algorithm 4) with both separator values known;
//             forward writes y, backward the Appendix A.1 gradient chain.
#pragma once

#include <type_traits>

#include "smnn_fused.cuh"

namespace smnn {

// o = N(a) v and o = N(a)^T v with N_ik = -H_ik a_{i+k} (w_s^2 S**).
template <int B, class S>
__device__ __forceinline__ void rNv(const S (&a)[2 * B - 1], const S (&v)[B], S (&o)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) {
    S acc = mul_(splat<S>(-Hc(i, 0)), mul_(a[i], v[0]));
#pragma unroll
    for (int q = 1; q < B; ++q) acc = fma_(splat<S>(-Hc(i, q)), mul_(a[i + q], v[q]), acc);
    o[i] = acc;
  }
}
template <int B, class S>
__device__ __forceinline__ void rNtv(const S (&a)[2 * B - 1], const S (&v)[B], S (&o)[B]) {
#pragma unroll
  for (int q = 0; q < B; ++q) {
    S acc = mul_(splat<S>(-Hc(0, q)), mul_(a[q], v[0]));
#pragma unroll
    for (int i = 1; i < B; ++i) acc = fma_(splat<S>(-Hc(i, q)), mul_(a[i + q], v[i]), acc);
    o[q] = acc;
  }
}

template <int B, class S>
__device__ __forceinline__ void rcopyL(const S (&src)[B][B], S (&dst)[B][B]) {
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int q = 0; q <= i; ++q) dst[i][q] = src[i][q];
}

#ifndef SMNN_PIPE_HM4D
#define SMNN_PIPE_HM4D 4  // fp64 arithmetic, order 3 (b = 4)
#endif
#ifndef SMNN_P2_SEG_RT
#define SMNN_P2_SEG_RT 0  // 1: keep P2's run-through of the first segment for callers without P1's state
#endif
// P2 register segment: the factors of up to HM interior points stay in registers.
template <int B, class S, int NR = 1>
struct PipeHM {
  static constexpr int value = sizeof(S) >= 8 ? (B == 1 ? 12 : B == 2 ? 8 : B == 3 ? 5 : SMNN_PIPE_HM4D)
                                              : (B == 1 ? 23 : B == 2 ? 13 : B == 3 ? 9 : 6);
};
// Chunk capacity (points).  fp32: one segment (HM + 1 points; measured best --
// splitting costs a second factorisation of the first segment, more than the
// shorter separator system saves); fp64: two segments (2 HM points: fewer
// separators; measured +7..26 % on Lorenz / target / KdV).
template <int B, class S>
struct PipeCM {
  static constexpr int value = sizeof(S) >= 8 ? 2 * PipeHM<B, S>::value : PipeHM<B, S>::value + 1;
};

// Right-hand sides of point i of a chunk (NR of them): rhs 0 = dl/dy (BWD) or
// beta, rhs 1 = beta (BWD with NR = 2: y re-solved in the arithmetic type);
// beta_j = wg2 c_j d_j (+ wi2 u at t = 0).
template <int B, class Tio, class S, bool BWD, int NR>
__device__ __forceinline__ void chunk_rhs(const Wts<S>& w, int n_iv, const Tio* u, bool t0, const S (&wc)[B],
                                          const Tio* dS, const Tio* gS, int i, S (&rhs)[NR][B]) {
  static_assert(NR == 1 || (NR == 2 && BWD), "two right-hand sides only in the backward pass");
  constexpr int qb = BWD ? 1 : 0;  // index of beta
  if (BWD) {
#pragma unroll
    for (int r = 0; r < B; ++r) rhs[0][r] = S(gS[i * B + r]);
  }
  if (qb < NR) {
    const S d = S(dS[i]);
#pragma unroll
    for (int r = 0; r < B; ++r) rhs[qb < NR ? qb : 0][r] = mul_(wc[r], d);
    if (t0) {
#pragma unroll
      for (int r = 0; r < B; ++r)
        if (r < n_iv) rhs[qb < NR ? qb : 0][r] = fma_(w.i2, S(u[r]), rhs[qb < NR ? qb : 0][r]);
    }
  }
}

// rhs -= P w (the Schur coupling of the right-hand side only)
template <int B, class S>
__device__ __forceinline__ void lcouple_v(const S (&P)[B][B], const S (&w)[B], S (&rhs)[B]) {
#pragma unroll
  for (int i = 0; i < B; ++i) {
    S acc = rhs[i];
#pragma unroll
    for (int j = 0; j < B; ++j) acc = fnma_(P[i][j], w[j], acc);
    rhs[i] = acc;
  }
}

// Pass 1 of one chunk (interior nint >= 1 points, then the separator): block
// Cholesky of the interior with the spike (Algorithm 3's loop), the Schur
// complement onto the two separators, the separator's own block.  Returns the
// separator block Dsep (lower), rhs Rsep, coupling A_rl, and sum X^T X /
// sum X^T w (to be negated into A_ll / r_l of separator k-1); true on a
// pivot breakdown.  NR right-hand sides share the factorisation.
//
// seg (nullable, field stride K): a chunk P2 handles in two segments (nint >
// HM) gets its factorisation state at point h - 1 = nint - HM - 1 stored
// there (PSegState: L_{h-1}, w'_{h-1} with y_L = 0, and the spike sg X_{h-1},
// so that P2 forms w'_{h-1}(y_L) = w'_{h-1}(0) - sg X_{h-1} y_L and starts the
// second segment without re-factoring the first).
template <int B, int NR>
struct PSegState {
  static constexpr int LT = B * (B + 1) / 2;
  static constexpr int L = 0, W = LT, X = LT + NR * B, N = LT + NR * B + B * B;
};

template <int B, class Tio, class S, bool BWD, int CM, int NR = 1>
__device__ __forceinline__ bool p1_chunk(const Wts<S>& w, int n_iv, const Tio* u, int k, int K, int nint,
                                         const Tio* cS, const Tio* dS, const Tio* sS, const Tio* gS,
                                         S (&Dsep)[B][B], S (&Rsep)[NR][B], S (&Arl)[B][B], S (&All)[B][B],
                                         S (&rl)[NR][B], S* seg = nullptr) {
  using SS = PSegState<B, NR>;
  constexpr bool SEG = CM - 1 > PipeHM<B, S, NR>::value;  // chunks P2 may split in two segments
  const int hcap = (SEG && seg) ? nint - PipeHM<B, S, NR>::value - 1 : -1;  // < 0: nothing stored
  S ap[2 * B - 1];
  if (k > 0) spow<B, S>(S(sS[-1]), w.s2, ap); else zero<2 * B - 1, S>(ap);
  S Lc[B][B], wv[NR][B], X[B][B];
  zero<B, S>(Lc); zero<B, S>(X); zero<B, S>(All);
#pragma unroll
  for (int q = 0; q < NR; ++q) { zero<B, S>(wv[q]); zero<B, S>(rl[q]); }
  S sg = splat<S>(1.0);
  // The chunk loop stays rolled (nothing is kept per step): the unrolled body
  // of fp64 chunks overflowed the instruction cache (ncu: 43 % of the warp
  // stalls "no instruction" in P1).  Step 0 (no coupling to a previous
  // interior point) is peeled.
  auto step = [&](int i, auto first) {
    constexpr bool FIRST = decltype(first)::value;
    S c[B], an[2 * B - 1], M[B][B], wc[B], rhs[NR][B];
#pragma unroll
    for (int r = 0; r < B; ++r) c[r] = S(cS[i * B + r]);
    spow<B, S>(S(sS[i]), w.s2, an);
    lassemble<B, S>(c, w.g2, ap, an, M, wc);
    const bool t0 = FIRST && k == 0;
    chunk_rhs<B, Tio, S, BWD, NR>(w, n_iv, u, t0, wc, dS, gS, i, rhs);
    if (t0) {  // initial-value rows at t = 0
#pragma unroll
      for (int r = 0; r < B; ++r)
        if (r < n_iv) M[r][r] = add_(M[r][r], w.i2);
    }
    if constexpr (FIRST) {
      lchol<B, S>(M, Lc);
#pragma unroll
      for (int q = 0; q < NR; ++q) llsolve<B, S>(Lc, rhs[q], wv[q]);
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
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          S acc = mul_(X[0][r], wv[q][0]);
#pragma unroll
          for (int m = 1; m < B; ++m) acc = fma_(X[m][r], wv[q][m], acc);
          rl[q][r] = acc;
        }
      }
    } else {
      S Pm[B][B];
      lPfromN<B, S>(ap, Lc, Pm);  // P_{j-1} = N_{j-1} L_{j-1}^{-T}
      lcouple<B, S>(Pm, wv[0], M, rhs[0]);
#pragma unroll
      for (int q = 1; q < NR; ++q) lcouple_v<B, S>(Pm, wv[q], rhs[q]);
      lchol<B, S>(M, Lc);
#pragma unroll
      for (int q = 0; q < NR; ++q) llsolve<B, S>(Lc, rhs[q], wv[q]);
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
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          S acc = mul_(X[0][r], wv[q][0]);
#pragma unroll
          for (int m = 1; m < B; ++m) acc = fma_(X[m][r], wv[q][m], acc);
          rl[q][r] = fma_(sg, acc, rl[q][r]);
        }
      }
    }
    if (SEG && i == hcap) {  // P2's state at the end of its first segment (see PSegState)
      int e = 0;
#pragma unroll
      for (int r = 0; r < B; ++r)
#pragma unroll
        for (int q = 0; q <= r; ++q) seg[int64_t(SS::L + e++) * K] = Lc[r][q];
#pragma unroll
      for (int p = 0; p < NR; ++p)
#pragma unroll
        for (int r = 0; r < B; ++r) seg[int64_t(SS::W + p * B + r) * K] = wv[p][r];
#pragma unroll
      for (int r = 0; r < B; ++r)
#pragma unroll
        for (int q = 0; q < B; ++q) seg[int64_t(SS::X + r * B + q) * K] = mul_(sg, X[r][q]);
    }
#pragma unroll
    for (int m = 0; m < 2 * B - 1; ++m) ap[m] = an[m];
  };
  step(0, std::true_type{});
#pragma unroll 1
  for (int i = 1; i < nint; ++i) step(i, std::false_type{});

  // one pivot check per chunk: a breakdown leaves a non-finite last factor
  const bool bad = bad_(splat<S>(1.0) / Lc[B - 1][B - 1]) != 0;
  {  // Schur complement of the interior onto (sigma_{k-1}, sigma_k); ap = a(s_l)
    S Pl[B][B];
    lPfromN<B, S>(ap, Lc, Pl);
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int q = 0; q < B; ++q) {
        S a2 = mul_(Pl[r][0], X[0][q]);
#pragma unroll
        for (int m = 1; m < B; ++m) a2 = fma_(Pl[r][m], X[m][q], a2);
        Arl[r][q] = mul_(neg_(sg), a2);
      }
    S c[B], an[2 * B - 1], wc[B];
#pragma unroll
    for (int r = 0; r < B; ++r) c[r] = S(cS[nint * B + r]);
    if (k + 1 < K) spow<B, S>(S(sS[nint]), w.s2, an); else zero<2 * B - 1, S>(an);
    lassemble<B, S>(c, w.g2, ap, an, Dsep, wc);
    chunk_rhs<B, Tio, S, BWD, NR>(w, n_iv, u, false, wc, dS, gS, nint, Rsep);
    lcouple<B, S>(Pl, wv[0], Dsep, Rsep[0]);
#pragma unroll
    for (int q = 1; q < NR; ++q) lcouple_v<B, S>(Pl, wv[q], Rsep[q]);
  }
  return bad;
}

// y at point j for the backward gradient chain: the staged fp32 (or fp64) y,
// plus, in the SMNN_F32_C64 pipeline, the forward's fp32 remainder y_lo (staged)
// so that y_hi + y_lo carries the fp64 solution (include/smnn.h smnn_solve_bwd_ex).
template <int B, class S, class Tio>
__device__ __forceinline__ void ld_yfwd(const Grp<Tio, 1>& x, int j, S (&yf)[B]) {
  ldlv<B, S, Tio, 1, true>(x.yin, j * B, yf);
  if constexpr (sizeof(S) > sizeof(Tio)) {
    if (x.ylo_in) {
#pragma unroll
      for (int r = 0; r < B; ++r) yf[r] = add_(yf[r], S(smem_as<const Tio>()[x.ylo_off + j * B + r]));
    }
  }
}
// y at point j in the forward: rounded to storage, and its fp32 remainder when requested.
template <int B, class S, class Tio>
__device__ __forceinline__ void st_yout(const Grp<Tio, 1>& x, int j, const S (&y)[B]) {
#pragma unroll
  for (int r = 0; r < B; ++r) stl<S, Tio, 1, true>(x.yout, 1, j * B + r, y[r]);
  if constexpr (sizeof(S) > sizeof(Tio)) {
    if (x.ylo_out) {
#pragma unroll
      for (int r = 0; r < B; ++r) smem_as<Tio>()[x.ylo_off + j * B + r] = Tio(sub_(y[r], S(Tio(y[r]))));
    }
  }
}

// One segment [i0, i0 + len) of a chunk interior (len <= HM) in pass 2: forward
// sweep re-factoring M from the state (Ls, ws) = (L, w') at step i0 - 1 (from
// the chunk start -- initial-value rows, rhs -= N_{f-1} y_L -- when i0 == 0),
// then, if STORE, back substitution from yn = y at step i0 + len (NR = 2
// backward: yn[0] = lambda, yn[1] = y re-solved; NR = 1 backward: y_fwd read
// from storage into yfn), writing the outputs and returning yn at step i0.
// Without STORE the sweep only runs through and returns the state at the last step.
template <int B, class Tio, class S, bool BWD, int HM, bool STORE, int NR>
__device__ __forceinline__ void p2_seg(const Grp<Tio, 1>& x, const Wts<S>& w, int k, int f, int i0, int len,
                                       const Tio* cS, const Tio* dS, const Tio* sS, const Tio* gS, Tio* wS,
                                       const S (&yL)[NR][B], S (&Ls)[B][B], S (&ws)[NR][B], S (&yn)[NR][B],
                                       S (&yfn)[B]) {
  constexpr bool WSM = sizeof(S) == sizeof(Tio) && NR == 1;
  S Lr[STORE ? HM : 1][B][B];
  S Wp[(STORE && !WSM) ? HM : 1][NR][B];
  S ap[2 * B - 1];
  if (i0 > 0 || k > 0) spow<B, S>(S(sS[i0 - 1]), w.s2, ap); else zero<2 * B - 1, S>(ap);
  // forward sweep step q (point i = i0 + q); STORE keeps factor and w' per
  // step in registers (fully unrolled), the run-through keeps only the last
  // (rolled loop: small code, see p1_chunk)
  auto fstep = [&](int q) {
    const int i = i0 + q;
    S c[B], an[2 * B - 1], M[B][B], wc[B], rhs[NR][B];
#pragma unroll
    for (int r = 0; r < B; ++r) c[r] = S(cS[i * B + r]);
    spow<B, S>(S(sS[i]), w.s2, an);
    lassemble<B, S>(c, w.g2, ap, an, M, wc);
    const bool t0 = i == 0 && k == 0;
    chunk_rhs<B, Tio, S, BWD, NR>(w, x.n_iv, x.u[0], t0, wc, dS, gS, i, rhs);
    if (i == 0) {  // chunk start (q == 0, i0 == 0)
      if (t0) {
#pragma unroll
        for (int r = 0; r < B; ++r)
          if (r < x.n_iv) M[r][r] = add_(M[r][r], w.i2);
      }
#pragma unroll
      for (int p = 0; p < NR; ++p) {  // rhs -= N_{f-1} y_L
        S Nt[B];
        rNv<B, S>(ap, yL[p], Nt);
#pragma unroll
        for (int r = 0; r < B; ++r) rhs[p][r] = sub_(rhs[p][r], Nt[r]);
      }
    } else {
      S Pm[B][B];
      lPfromN<B, S>(ap, (STORE && q > 0) ? Lr[STORE ? (q > 0 ? q - 1 : 0) : 0] : Ls, Pm);
      lcouple<B, S>(Pm, ws[0], M, rhs[0]);
#pragma unroll
      for (int p = 1; p < NR; ++p) lcouple_v<B, S>(Pm, ws[p], rhs[p]);
    }
    S Lc[B][B];
    lchol<B, S>(M, Lc);
#pragma unroll
    for (int p = 0; p < NR; ++p) llsolve<B, S>(Lc, rhs[p], ws[p]);
    if (STORE) {
      rcopyL<B, S>(Lc, Lr[STORE ? q : 0]);
#pragma unroll
      for (int p = 0; p < NR; ++p)
#pragma unroll
        for (int r = 0; r < B; ++r) {
          if (WSM) wS[i * B + r] = Tio(ws[p][r]); else Wp[(STORE && !WSM) ? q : 0][p][r] = ws[p][r];
        }
    } else {
      rcopyL<B, S>(Lc, Ls);
    }
#pragma unroll
    for (int m = 0; m < 2 * B - 1; ++m) ap[m] = an[m];
  };
  if constexpr (STORE) {
#pragma unroll
    for (int q = 0; q < HM; ++q)
      if (q < len) fstep(q);
  } else {
#pragma unroll 1
    for (int q = 0; q < len; ++q) fstep(q);
  }
  if (!STORE) return;
#pragma unroll
  for (int q = HM - 1; q >= 0; --q) {
    if (q < len) {
      const int i = i0 + q, j = f + i;
      S an[2 * B - 1], yv[NR][B];
      spow<B, S>(S(sS[i]), w.s2, an);
#pragma unroll
      for (int p = 0; p < NR; ++p) {
        S v[B], uu[B], t[B];
        rNtv<B, S>(an, yn[p], v);
        llsolve<B, S>(Lr[STORE ? q : 0], v, uu);
#pragma unroll
        for (int r = 0; r < B; ++r)
          t[r] = sub_(WSM ? S(wS[i * B + r]) : Wp[(STORE && !WSM) ? q : 0][p][r], uu[r]);
        lltsolve<B, S>(Lr[STORE ? q : 0], t, yv[p]);
      }
      if (!BWD) {
        st_yout<B, S, Tio>(x, j, yv[0]);
      } else {
        S yf[B];  // y at j: re-solved (NR = 2) or read from storage
        if (NR == 2) {
#pragma unroll
          for (int r = 0; r < B; ++r) yf[r] = yv[NR - 1][r];
        } else {
          ld_yfwd<B, S, Tio>(x, j, yf);
        }
        lpoint_grads<B, S, Tio, 1, true>(x, w, j, yv[0], yf);
        if (x.gs.on) stl<S, Tio, 1, true>(x.gs, 1, j, lds<B, S>(an, yv[0], yf, yn[0], yfn));
#pragma unroll
        for (int r = 0; r < B; ++r) yfn[r] = yf[r];
      }
#pragma unroll
      for (int p = 0; p < NR; ++p)
#pragma unroll
        for (int r = 0; r < B; ++r) yn[p][r] = yv[p][r];
    }
  }
}

// Pass 2 of one chunk with y_L = y(sigma_{k-1}) and y_R = y(sigma_k) known
// (NR right-hand sides): outputs at the separator, then the interior in (at
// most) two register segments (p2_seg).
template <int B, class Tio, class S, bool BWD, int CM, int NR = 1>
__device__ __forceinline__ void p2_chunk(const Grp<Tio, 1>& x, const Wts<S>& w, int k, int f, int sig, int nint,
                                         const Tio* cS, const Tio* dS, const Tio* sS, const Tio* gS,
                                         const S (&yL)[NR][B], const S (&yR)[NR][B], const S* seg = nullptr,
                                         int K = 0) {
  // a chunk longer than HM is split as [0, h) + [h, nint) with the second
  // segment HM long; [0, h) is factored twice (run-through to reach the state
  // at h - 1, then stored for its back substitution).
  constexpr int HM = PipeHM<B, S, NR>::value;
  static_assert(CM - 1 <= 2 * HM, "two segments must cover a chunk");
  Tio* wS = const_cast<Tio*>(BWD ? gS : cS);
  S yn[NR][B], yfn[B], Ls[B][B], ws[NR][B];
#pragma unroll
  for (int p = 0; p < NR; ++p) {
#pragma unroll
    for (int r = 0; r < B; ++r) yn[p][r] = yR[p][r];
    zero<B, S>(ws[p]);
  }
  zero<B, S>(yfn);
  zero<B, S>(Ls);
  if (!BWD) {
    st_yout<B, S, Tio>(x, sig, yR[0]);
  } else {
    if (NR == 2) {
#pragma unroll
      for (int r = 0; r < B; ++r) yfn[r] = yR[NR - 1][r];
    } else {
      ld_yfwd<B, S, Tio>(x, sig, yfn);
    }
    lpoint_grads<B, S, Tio, 1, true>(x, w, sig, yR[0], yfn);
  }
  if (CM - 1 <= HM || nint <= HM) {
    p2_seg<B, Tio, S, BWD, HM, true, NR>(x, w, k, f, 0, nint, cS, dS, sS, gS, wS, yL, Ls, ws, yn, yfn);
  } else {
    // (measured: calling one stored-segment copy twice from a rolled loop
    // shrinks the code but costs more instructions than the icache saves)
    const int h = nint - HM;
    if (SMNN_P2_SEG_RT == 0 || seg) {  // P1 stored the state at h - 1 (PSegState): no run-through of [0, h)
      using SS = PSegState<B, NR>;
      int e = 0;
#pragma unroll
      for (int r = 0; r < B; ++r)
#pragma unroll
        for (int q = 0; q <= r; ++q) Ls[r][q] = seg[int64_t(SS::L + e++) * K];
      S Xs[B][B];
#pragma unroll
      for (int r = 0; r < B; ++r)
#pragma unroll
        for (int q = 0; q < B; ++q) Xs[r][q] = seg[int64_t(SS::X + r * B + q) * K];
#pragma unroll
      for (int p = 0; p < NR; ++p)
#pragma unroll
        for (int r = 0; r < B; ++r) {
          S acc = seg[int64_t(SS::W + p * B + r) * K];
#pragma unroll
          for (int q = 0; q < B; ++q) acc = fnma_(Xs[r][q], yL[p][q], acc);
          ws[p][r] = acc;
        }
    } else {
      p2_seg<B, Tio, S, BWD, HM, false, NR>(x, w, k, f, 0, h, cS, dS, sS, gS, wS, yL, Ls, ws, yn, yfn);
    }
    // (measured again with the y_lo backward: one rolled stored-segment copy called
    // twice is no faster at T = 1e4 and 8 % slower at T = 1e3 than two inlined copies;
    // with the P1 state, one rolled copy for one or two segments spills: 5-7 % slower)
    p2_seg<B, Tio, S, BWD, HM, true, NR>(x, w, k, f, h, HM, cS, dS, sS, gS, wS, yL, Ls, ws, yn, yfn);
    zero<B, S>(Ls);
#pragma unroll
    for (int p = 0; p < NR; ++p) zero<B, S>(ws[p]);
    p2_seg<B, Tio, S, BWD, HM, true, NR>(x, w, k, f, 0, h, cS, dS, sS, gS, wS, yL, Ls, ws, yn, yfn);
  }
  if (BWD && k > 0 && x.gs.on) {  // interval (sigma_{k-1}, f)
    S yfm[B], am[2 * B - 1];
    if (NR == 2) {
#pragma unroll
      for (int r = 0; r < B; ++r) yfm[r] = yL[NR - 1][r];
    } else {
      ld_yfwd<B, S, Tio>(x, f - 1, yfm);
    }
    spow<B, S>(S(sS[-1]), w.s2, am);
    stl<S, Tio, 1, true>(x.gs, 1, f - 1, lds<B, S>(am, yL[0], yfm, yn[0], yfn));
  }
}

template <int B, int NR = 1>
struct PSep {  // workspace record of one separator (field-major over the separators)
  static constexpr int LT = B * (B + 1) / 2;
  static constexpr int D = 0, R = LT, BL = LT + NR * B, AL = LT + NR * B + B * B, RL = 2 * LT + NR * B + B * B;
  static constexpr int N = 2 * LT + 2 * NR * B + B * B;
};

template <int B, class S, int NR = 1>
__device__ __forceinline__ void psep_ld(const S* in, int K, int NT, int j, S (&D)[B][B], S (&r)[NR][B],
                                        S (&Bl)[B][B]) {
  using Q = PSep<B, NR>;
  int e = 0;
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int q = 0; q <= i; ++q) D[i][q] = in[int64_t(Q::D + e++) * K + j];
#pragma unroll
  for (int p = 0; p < NR; ++p)
#pragma unroll
    for (int i = 0; i < B; ++i) r[p][i] = in[int64_t(Q::R + p * B + i) * K + j];
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int q = 0; q < B; ++q) Bl[i][q] = in[int64_t(Q::BL + i * B + q) * K + j];
  if (j + 1 < K && (j + 1) % NT == 0) {
    e = 0;
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
      for (int q = 0; q <= i; ++q) D[i][q] = add_(D[i][q], in[int64_t(Q::AL + e++) * K + j + 1]);
#pragma unroll
    for (int p = 0; p < NR; ++p)
#pragma unroll
      for (int i = 0; i < B; ++i) r[p][i] = add_(r[p][i], in[int64_t(Q::RL + p * B + i) * K + j + 1]);
  }
}

template <int B, class S, int NR = 1>
__device__ __forceinline__ void psep_ld_rb(const S* in, int K, int NT, int j, S (&r)[NR][B], S (&Bl)[B][B]) {
  using Q = PSep<B, NR>;
#pragma unroll
  for (int p = 0; p < NR; ++p)
#pragma unroll
    for (int i = 0; i < B; ++i) r[p][i] = in[int64_t(Q::R + p * B + i) * K + j];
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int q = 0; q < B; ++q) Bl[i][q] = in[int64_t(Q::BL + i * B + q) * K + j];
  if (j + 1 < K && (j + 1) % NT == 0) {
#pragma unroll
    for (int p = 0; p < NR; ++p)
#pragma unroll
      for (int i = 0; i < B; ++i) r[p][i] = add_(r[p][i], in[int64_t(Q::RL + p * B + i) * K + j + 1]);
  }
}
template <int B, class S, int NR = 1>
__device__ __forceinline__ void psep_ld_b(const S* in, int K, int j, S (&Bl)[B][B]) {
  using Q = PSep<B, NR>;
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int q = 0; q < B; ++q) Bl[i][q] = in[int64_t(Q::BL + i * B + q) * K + j];
}

}  // namespace smnn
