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
// P2 register segment: the factors of up to HM interior points stay in registers.
template <int B, class S>
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

// Pass 1 of one chunk (interior nint >= 1 points, then the separator): block
// Cholesky of the interior with the spike (Algorithm 3's loop), the Schur
// complement onto the two separators, the separator's own block.  Returns the
// separator block Dsep (lower), rhs Rsep, coupling A_rl, and sum X^T X /
// sum X^T w (to be negated into A_ll / r_l of separator k-1); true on a
// pivot breakdown.  Shared by the pipeline's P1 and the fused rf2 kernel.
template <int B, class Tio, class S, bool BWD, int CM>
__device__ __forceinline__ bool p1_chunk(const Wts<S>& w, int n_iv, const Tio* u, int k, int K, int nint,
                                         const Tio* cS, const Tio* dS, const Tio* sS, const Tio* gS,
                                         S (&Dsep)[B][B], S (&Rsep)[B], S (&Arl)[B][B], S (&All)[B][B],
                                         S (&rl)[B]) {
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
          if (r < n_iv) {
            if (!BWD) rhs[r] = fma_(w.i2, S(u[r]), rhs[r]);
            M[r][r] = add_(M[r][r], w.i2);
          }
      }
      if (i == 0) {
        lchol<B, S>(M, Lc);
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
        lchol<B, S>(M, Lc);
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
#pragma unroll
      for (int m = 0; m < 2 * B - 1; ++m) ap[m] = an[m];
    }
  }
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
  return bad;
}

// One segment [i0, i0 + len) of a chunk interior (len <= HM) in pass 2: forward
// sweep re-factoring M from the state (Ls, ws) = (L, w') at step i0 - 1 (from
// the chunk start -- initial-value rows, rhs -= N_{f-1} y_L -- when i0 == 0),
// then, if STORE, back substitution from (yn, yfn) = (y, y_fwd) at step
// i0 + len, writing the outputs and returning (yn, yfn) at step i0.  Without
// STORE the sweep only runs through and returns the state at the last step.
template <int B, class Tio, class S, bool BWD, int HM, bool STORE>
__device__ __forceinline__ void p2_seg(const Grp<Tio, 1>& x, const Wts<S>& w, int k, int f, int i0, int len,
                                       const Tio* cS, const Tio* dS, const Tio* sS, const Tio* gS, Tio* wS,
                                       const S (&yL)[B], S (&Ls)[B][B], S (&ws)[B], S (&yn)[B], S (&yfn)[B]) {
  constexpr bool WSM = sizeof(S) == sizeof(Tio);
  S Lr[STORE ? HM : 1][B][B];
  S Wp[(STORE && !WSM) ? HM : 1][B];
  S ap[2 * B - 1];
  if (i0 > 0 || k > 0) spow<B, S>(S(sS[i0 - 1]), w.s2, ap); else zero<2 * B - 1, S>(ap);
#pragma unroll
  for (int q = 0; q < HM; ++q) {
    if (q < len) {
      const int i = i0 + q;
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
      if (i == 0) {  // chunk start (q == 0, i0 == 0)
        if (k == 0) {
#pragma unroll
          for (int r = 0; r < B; ++r)
            if (r < x.n_iv) {
              if (!BWD) rhs[r] = fma_(w.i2, S(x.u[0][r]), rhs[r]);
              M[r][r] = add_(M[r][r], w.i2);
            }
        }
        S Nt[B];  // rhs -= N_{f-1} y_L
        rNv<B, S>(ap, yL, Nt);
#pragma unroll
        for (int r = 0; r < B; ++r) rhs[r] = sub_(rhs[r], Nt[r]);
      } else {
        S Pm[B][B];
        lPfromN<B, S>(ap, (STORE && q > 0) ? Lr[STORE ? (q > 0 ? q - 1 : 0) : 0] : Ls, Pm);
        lcouple<B, S>(Pm, ws, M, rhs);
      }
      S Lc[B][B];
      lchol<B, S>(M, Lc);
      llsolve<B, S>(Lc, rhs, ws);
      if (STORE) {
        rcopyL<B, S>(Lc, Lr[STORE ? q : 0]);
#pragma unroll
        for (int r = 0; r < B; ++r) {
          if (WSM) wS[i * B + r] = Tio(ws[r]); else Wp[(STORE && !WSM) ? q : 0][r] = ws[r];
        }
      } else {
        rcopyL<B, S>(Lc, Ls);
      }
#pragma unroll
      for (int m = 0; m < 2 * B - 1; ++m) ap[m] = an[m];
    }
  }
  if (!STORE) return;
#pragma unroll
  for (int q = HM - 1; q >= 0; --q) {
    if (q < len) {
      const int i = i0 + q, j = f + i;
      S an[2 * B - 1], v[B], uu[B], t[B], yv[B];
      spow<B, S>(S(sS[i]), w.s2, an);
      rNtv<B, S>(an, yn, v);
      llsolve<B, S>(Lr[STORE ? q : 0], v, uu);
#pragma unroll
      for (int r = 0; r < B; ++r) t[r] = sub_(WSM ? S(wS[i * B + r]) : Wp[(STORE && !WSM) ? q : 0][r], uu[r]);
      lltsolve<B, S>(Lr[STORE ? q : 0], t, yv);
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
}

// Pass 2 of one chunk with y_L = y(sigma_{k-1}) and y_R = y(sigma_k) known:
// outputs at the separator, then the interior in (at most) two register
// segments (p2_seg).  Shared by the pipeline's P2 and the fused rf2 kernel.
template <int B, class Tio, class S, bool BWD, int CM>
__device__ __forceinline__ void p2_chunk(const Grp<Tio, 1>& x, const Wts<S>& w, int k, int f, int sig, int nint,
                                         const Tio* cS, const Tio* dS, const Tio* sS, const Tio* gS,
                                         const S (&yL)[B], const S (&yR)[B]) {
    // outputs at the separator, then the interior in (at most) two register
  // segments: a chunk longer than HM is split as [0, h) + [h, nint) with the
  // second segment HM long; [0, h) is factored twice (run-through to reach
  // the state at h - 1, then stored for its back substitution).
  constexpr int HM = PipeHM<B, S>::value;
  static_assert(CM - 1 <= 2 * HM, "two segments must cover a chunk");
  Tio* wS = const_cast<Tio*>(BWD ? gS : cS);
  S yn[B], yfn[B], Ls[B][B], ws[B];
#pragma unroll
  for (int r = 0; r < B; ++r) yn[r] = yR[r];
  zero<B, S>(yfn);
  zero<B, S>(Ls);
  zero<B, S>(ws);
  if (!BWD) {
#pragma unroll
    for (int r = 0; r < B; ++r) stl<S, Tio, 1, true>(x.yout, 1, sig * B + r, yR[r]);
  } else {
    ldlv<B, S, Tio, 1, true>(x.yin, sig * B, yfn);
    lpoint_grads<B, S, Tio, 1, true>(x, w, sig, yR, yfn);
  }
  if (CM - 1 <= HM || nint <= HM) {
    p2_seg<B, Tio, S, BWD, HM, true>(x, w, k, f, 0, nint, cS, dS, sS, gS, wS, yL, Ls, ws, yn, yfn);
  } else {
    const int h = nint - HM;
    p2_seg<B, Tio, S, BWD, HM, false>(x, w, k, f, 0, h, cS, dS, sS, gS, wS, yL, Ls, ws, yn, yfn);
    p2_seg<B, Tio, S, BWD, HM, true>(x, w, k, f, h, HM, cS, dS, sS, gS, wS, yL, Ls, ws, yn, yfn);
    zero<B, S>(Ls);
    zero<B, S>(ws);
    p2_seg<B, Tio, S, BWD, HM, true>(x, w, k, f, 0, h, cS, dS, sS, gS, wS, yL, Ls, ws, yn, yfn);
  }
  if (BWD && k > 0 && x.gs.on) {  // interval (sigma_{k-1}, f)
    S yfm[B], am[2 * B - 1];
    ldlv<B, S, Tio, 1, true>(x.yin, (f - 1) * B, yfm);
    spow<B, S>(S(sS[-1]), w.s2, am);
    stl<S, Tio, 1, true>(x.gs, 1, f - 1, lds<B, S>(am, yL, yfm, yn, yfn));
  }
}

template <int B>
struct PSep {
  static constexpr int LT = B * (B + 1) / 2;
  static constexpr int D = 0, R = LT, BL = LT + B, AL = LT + B + B * B, RL = 2 * LT + B + B * B;
  static constexpr int N = 2 * LT + 2 * B + B * B;
};

template <int B, class S>
__device__ __forceinline__ void psep_ld(const S* in, int K, int NT, int j, S (&D)[B][B], S (&r)[B], S (&Bl)[B][B]) {
  using Q = PSep<B>;
  int e = 0;
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int q = 0; q <= i; ++q) D[i][q] = in[int64_t(Q::D + e++) * K + j];
#pragma unroll
  for (int i = 0; i < B; ++i) r[i] = in[int64_t(Q::R + i) * K + j];
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
    for (int i = 0; i < B; ++i) r[i] = add_(r[i], in[int64_t(Q::RL + i) * K + j + 1]);
  }
}

template <int B, class S>
__device__ __forceinline__ void psep_ld_rb(const S* in, int K, int NT, int j, S (&r)[B], S (&Bl)[B][B]) {
  using Q = PSep<B>;
#pragma unroll
  for (int i = 0; i < B; ++i) r[i] = in[int64_t(Q::R + i) * K + j];
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int q = 0; q < B; ++q) Bl[i][q] = in[int64_t(Q::BL + i * B + q) * K + j];
  if (j + 1 < K && (j + 1) % NT == 0) {
#pragma unroll
    for (int i = 0; i < B; ++i) r[i] = add_(r[i], in[int64_t(Q::RL + i) * K + j + 1]);
  }
}
template <int B, class S>
__device__ __forceinline__ void psep_ld_b(const S* in, int K, int j, S (&Bl)[B][B]) {
  using Q = PSep<B>;
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int q = 0; q < B; ++q) Bl[i][q] = in[int64_t(Q::BL + i * B + q) * K + j];
}

}  // namespace smnn
