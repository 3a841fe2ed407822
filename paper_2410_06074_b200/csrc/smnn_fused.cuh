// smnn_fused.cuh -- the fused, time-parallel S-MNN forward / backward kernel.
//
// One CUDA block solves a group of P = LaneT<S>::P instances (P = 2 packs two
// instances into every float2 / double2 register).  Thread k owns time chunk
// k = [a_k, a_{k+1}) of every instance of the group; the last point sigma_k of
// a chunk is a separator, the points before it the chunk interior.
//
//   pass 1  block Cholesky of the interior (Algorithm 3's loop)
//           with a spike X_j = (G^{-1})_{j,f} N_L carried along, giving the
//           Schur complement of the interior onto (sigma_{k-1}, sigma_k);
//           every G steps the state (L, w, X) is checkpointed;
//   BCR     block cyclic reduction of the K x K separator system in shared
//           memory (log2 K levels, the reduced system stays SPD);
//   pass 2  the interior is re-factored segment by segment (last segment
//           first, each resumed from its checkpoint, G steps in registers)
//           and back-substituted (Algorithm 4) with both
//           separator values known.  FWD writes y; BWD writes the gradients
//           of Algorithm 2 chained through Appendix A.1.
#pragma once

#include <cooperative_groups.h>

#include <climits>

#include "smnn_lane.cuh"
#include "smnn_tma.cuh"
#include "smnn_rf_host.h"

#ifndef SMNN_MAX_THREADS
#define SMNN_MAX_THREADS 256
#endif
#ifndef SMNN_MIN_BLOCKS
#define SMNN_MIN_BLOCKS 2
#endif

namespace smnn {


template <int B>
struct CkN {  // checkpoint: L lower (incl. inverse diagonal), w, X
  static constexpr int L = B * (B + 1) / 2;
  static constexpr int N = L + B + B * B;
};

// Separator system in shared memory, structure of arrays: element e of the
// separator with local index li sits at arr[e * nt + li].  Separators are
// numbered globally 0..K-1; separator i lives in CTA i / nt of the cluster
// (cs CTAs; cs == 1 outside the resident kernel) and is reached through
// distributed shared memory when that CTA is not this one.
template <int B, class S, bool CL = false>
struct SepL {
  S* D;   // [B*B][nt]  diagonal block; the factor after elimination
  S* Bc;  // [B*B][nt]  coupling block(i, i-h); Y1 after elimination
  S* Y2;  // [B*B][nt]
  S* R;   // [B][nt]    rhs; v after elimination
  S* Y;   // [B][nt]    solution
  int* time;  // [nt]   time index of each separator (for info)
  int* fail;  // [P]
  int K;      // separators in the whole cluster
  int nt;     // separators (= threads) per CTA
  int rank;   // this CTA's rank in the cluster
  int cs;     // cluster size
  __device__ __forceinline__ S* at(S* arr, int i) const {
    if (!CL) return arr + i;
    const int r = i / nt;
    S* p = arr + (i - r * nt);
    if (r != rank) p = cooperative_groups::this_cluster().map_shared_rank(p, r);
    return p;
  }
  __device__ __forceinline__ const S* at(const S* arr, int i) const { return at(const_cast<S*>(arr), i); }
  __device__ void ld(const S* a, int i, S (&m)[B][B]) const {
    const S* p = at(a, i);
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) m[r][c] = p[(r * B + c) * nt];
  }
  __device__ void st(S* a, int i, const S (&m)[B][B]) const {
    S* p = at(a, i);
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) p[(r * B + c) * nt] = m[r][c];
  }
  __device__ void ldv(const S* a, int i, S (&v)[B]) const {
    const S* p = at(a, i);
#pragma unroll
    for (int r = 0; r < B; ++r) v[r] = p[r * nt];
  }
  __device__ void stv(S* a, int i, const S (&v)[B]) const {
    S* p = at(a, i);
#pragma unroll
    for (int r = 0; r < B; ++r) p[r * nt] = v[r];
  }
  __device__ __forceinline__ int ltime(int i) const { return CL ? time[i - rank * nt] : time[i]; }
  __device__ __forceinline__ void sync() const {
    if (CL) cooperative_groups::this_cluster().sync(); else __syncthreads();
  }
};

template <int P>
__device__ __forceinline__ void report(int* fail, int bad, int t) {
#pragma unroll
  for (int q = 0; q < P; ++q)
    if (bad & (1 << q)) atomicMin(fail + q, t + 1);
}


template <class T>
__device__ __forceinline__ T* smem_as() { return reinterpret_cast<T*>(smnn_dyn_smem); }

// One data stream of the P instances of a group: global base pointers, or (in
// the resident kernel) element offsets into the dynamic shared memory, so the
// compiler emits LDS/STS with immediate offsets instead of generic LD/ST.
template <class Tio, int P>
struct Str {
  const Tio* p[P];
  int o[P];
  bool on;
};

// Per-group view of the P instances (invalid lanes alias lane 0).
template <class Tio, int P>
struct Grp {
  Str<Tio, P> c, d, s, yin, gy, yout, gc, gd, gs;
  const Tio* u[P];
  Tio* gu[P];
  // pipeline P2 only (smnn_chunk.cuh): y's fp32 remainder written (forward) / read (backward)
  // in shared memory at element offset ylo_off (relative to time index 0: may be negative)
  bool ylo_out = false, ylo_in = false;
  int ylo_off = 0;
  bool gu_on;
  int nv, T, n_iv;
  template <int B>
  __device__ void init(const Args<Tio>& a, int64_t inst0) {
    T = a.T;
    n_iv = a.n_iv;
    nv = (a.n_inst - inst0 < P) ? int(a.n_inst - inst0) : P;
    c.on = true; d.on = true; s.on = true;
    yin.on = a.y_in != nullptr; gy.on = a.grad_y != nullptr; yout.on = a.y_out != nullptr;
    gc.on = a.g_coeffs != nullptr; gd.on = a.g_rhs != nullptr; gs.on = a.g_steps != nullptr;
    gu_on = a.g_iv != nullptr;
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const int64_t i = inst0 + (q < nv ? q : 0);
      const int64_t tb = i * int64_t(T) * B, t1 = i * int64_t(T), ts = i * int64_t(T - 1);
      c.p[q] = a.coeffs + tb;
      d.p[q] = a.rhs + t1;
      u[q] = a.iv + i * a.n_iv;
      s.p[q] = a.steps + ts;
      yin.p[q] = a.y_in ? a.y_in + tb : nullptr;
      gy.p[q] = a.grad_y ? a.grad_y + tb : nullptr;
      yout.p[q] = a.y_out ? a.y_out + tb : nullptr;
      gc.p[q] = a.g_coeffs ? a.g_coeffs + tb : nullptr;
      gd.p[q] = a.g_rhs ? a.g_rhs + t1 : nullptr;
      gu[q] = a.g_iv ? a.g_iv + i * a.n_iv : nullptr;
      gs.p[q] = a.g_steps ? a.g_steps + ts : nullptr;
    }
  }
};

// SM = the stream lives in shared memory (resident kernel), else global (read-only path).
template <class S, class Tio, int P, bool SM>
__device__ __forceinline__ S ldl(const Str<Tio, P>& st, int off) {
  Tio v[P];
#pragma unroll
  for (int q = 0; q < P; ++q) v[q] = SM ? smem_as<const Tio>()[st.o[q] + off] : __ldg(st.p[q] + off);
  return Make<S>::f(v);
}
template <int B, class S, class Tio, int P, bool SM>
__device__ __forceinline__ void ldlv(const Str<Tio, P>& st, int off, S (&v)[B]) {
#pragma unroll
  for (int r = 0; r < B; ++r) v[r] = ldl<S, Tio, P, SM>(st, off + r);
}
template <class S, class Tio, int P, bool SM>
__device__ __forceinline__ void stl(const Str<Tio, P>& st, int nv, int off, S v) {
#pragma unroll
  for (int q = 0; q < P; ++q) {
    if (q < nv) {
      if (SM) smem_as<Tio>()[st.o[q] + off] = Tio(lane(v, q));
      else const_cast<Tio*>(st.p[q])[off] = Tio(lane(v, q));
    }
  }
}
template <class S, class Tio, int P>
__device__ __forceinline__ S ldg_l(const Tio* const (&p)[P], int off) {
  Tio v[P];
#pragma unroll
  for (int q = 0; q < P; ++q) v[q] = p[q][off];
  return Make<S>::f(v);
}

template <int B, class S>
struct Vec {
  S v[B];
};

template <class S>
struct Wts {
  S g2, i2, s2;
};

// Right-hand side at point j: beta_j = wg2 c_j d_j (+ wi2 u at t = 0) forward,
// dl/dy_j backward.  Also adds the initial-value diagonal to M at t = 0.
template <int B, class S, class Tio, int P, bool BWD, bool SM>
__device__ __forceinline__ void lrhs(const Grp<Tio, P>& x, const Wts<S>& w, int j, const S (&wc)[B], S (&M)[B][B],
                                     S (&r)[B]) {
  if (BWD) {
    ldlv<B, S, Tio, P, SM>(x.gy, j * B, r);
  } else {
    const S d = ldl<S, Tio, P, SM>(x.d, j);
#pragma unroll
    for (int i = 0; i < B; ++i) r[i] = mul_(wc[i], d);
  }
  if (j == 0) {
#pragma unroll
    for (int i = 0; i < B; ++i) {
      if (i < x.n_iv) {
        if (!BWD) r[i] = fma_(w.i2, ldg_l<S, Tio, P>(x.u, i), r[i]);
        M[i][i] = add_(M[i][i], w.i2);
      }
    }
  }
}

// ------------------------------------------------ gradients (BWD pass 2) ---
// Point terms (Appendix A.1 differentiated with dM = -lam y^T, Eq. 13):
//   dd_j = wg2 c.lam ; dc_j = wg2 (d_j lam - lam (y.c) - y (lam.c)) ; du = wi2 lam_0
template <int B, class S, class Tio, int P, bool SM>
__device__ __forceinline__ void lpoint_grads(const Grp<Tio, P>& x, const Wts<S>& w, int j, const S (&lam)[B],
                                             const S (&yj)[B]) {
  S c[B];
  ldlv<B, S, Tio, P, SM>(x.c, j * B, c);
  S lc = mul_(lam[0], c[0]), yc = mul_(yj[0], c[0]);
#pragma unroll
  for (int i = 1; i < B; ++i) {
    lc = fma_(lam[i], c[i], lc);
    yc = fma_(yj[i], c[i], yc);
  }
  const S d = ldl<S, Tio, P, SM>(x.d, j);  // read before dd_j may overwrite it in place
  if (x.gd.on) stl<S, Tio, P, SM>(x.gd, x.nv, j, mul_(w.g2, lc));
  if (x.gc.on) {
    const S wl = mul_(w.g2, lc), wy = mul_(w.g2, yc), wd = mul_(w.g2, d);
#pragma unroll
    for (int i = 0; i < B; ++i)
      stl<S, Tio, P, SM>(x.gc, x.nv, j * B + i, fnma_(yj[i], wl, fnma_(lam[i], wy, mul_(wd, lam[i]))));
  }
  if (j == 0 && x.gu_on) {
#pragma unroll
    for (int i = 0; i < B; ++i)
      if (i < x.n_iv) {
#pragma unroll
        for (int q = 0; q < P; ++q)
          if (q < x.nv) x.gu[q][i] = Tio(lane(mul_(w.i2, lam[i]), q));
      }
  }
}

// dl/ds_j of interval (j, j+1), a_m = ws2 s_j^m:
//   -[ lj^T J+ yj + ln^T J- yn + ln^T K yj + yn^T K lj ],  J+/J-/K = d/ds of SP, SM, -H o s^{i+k}
template <int B, class S>
__device__ __forceinline__ S lds(const S (&a)[2 * B - 1], const S (&lj)[B], const S (&yj)[B], const S (&ln)[B],
                                 const S (&yn)[B]) {
  S acc = splat<S>(0.0);
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int m = i + k;
      if (m == 0) continue;
      const double cp = Gc(i, k) * m + (i == k ? 2.0 * i : 0.0);
      const double cm = sgn(m) * Gc(i, k) * m + (i == k ? 2.0 * i : 0.0);
      const double ck = -Hc(i, k) * m;
      S t = mul_(splat<S>(cp), mul_(lj[i], yj[k]));
      t = fma_(splat<S>(cm), mul_(ln[i], yn[k]), t);
      t = fma_(splat<S>(ck), fma_(ln[i], yj[k], mul_(yn[i], lj[k])), t);
      acc = fma_(a[m - 1], t, acc);
    }
  return neg_(acc);
}

// ---------------------------------------------------------------- BCR ------
// Block cyclic reduction of the K separators (SPD block tridiagonal).  At
// level h the separators o = h (mod 2h) are eliminated and the survivors
// e = 0 (mod 2h) updated; the work of a level is packed onto the first
// threads (thread t handles o = h + 2h t, resp. e = 2h t) so that idle warps
// skip the level.  k is the caller's global thread index; all threads of the
// block (cluster) must call it.
template <int B, class S, int P, bool CL>
__device__ __forceinline__ void lbcr_body(const SepL<B, S, CL>& Sp, int k) {
  const int K = Sp.K;
  int hmax = 0;
#pragma unroll 1
  for (int h = 1; h < K; h <<= 1) {
    hmax = h;
    {
      const int o = h + 2 * h * k;
      if (o < K) {
        S D[B][B], Lf[B][B], Bk[B][B], Y1[B][B], Y2[B][B], r[B], v[B];
        Sp.ld(Sp.D, o, D);
        report<P>(Sp.fail, lchol<B, S>(D, Lf), Sp.ltime(o));
        Sp.ld(Sp.Bc, o, Bk);
        lleft<B, S>(Lf, Bk, Y1);
        if (o + h < K) {
          S Bn[B][B], BnT[B][B];
          Sp.ld(Sp.Bc, o + h, Bn);
#pragma unroll
          for (int i = 0; i < B; ++i)
#pragma unroll
            for (int j = 0; j < B; ++j) BnT[i][j] = Bn[j][i];
          lleft<B, S>(Lf, BnT, Y2);
        } else {
          zero<B, S>(Y2);
        }
        Sp.ldv(Sp.R, o, r);
        llsolve<B, S>(Lf, r, v);
        Sp.st(Sp.D, o, Lf);
        Sp.st(Sp.Bc, o, Y1);
        Sp.st(Sp.Y2, o, Y2);
        Sp.stv(Sp.R, o, v);
      }
    }
    Sp.sync();
    {
      const int e = 2 * h * k;
      if (e < K) {
        S D[B][B], r[B];
        Sp.ld(Sp.D, e, D);
        Sp.ldv(Sp.R, e, r);
        if (e - h >= 0) {
          const int o = e - h;
          S Y2o[B][B], Y1o[B][B], vo[B], nb[B][B];
          Sp.ld(Sp.Y2, o, Y2o);
          Sp.ld(Sp.Bc, o, Y1o);
          Sp.ldv(Sp.R, o, vo);
#pragma unroll
          for (int i = 0; i < B; ++i) {
#pragma unroll
            for (int j = 0; j < B; ++j) {
              S aD = D[i][j], aB = splat<S>(0.0);
#pragma unroll
              for (int m = 0; m < B; ++m) {
                aD = fnma_(Y2o[m][i], Y2o[m][j], aD);
                aB = fnma_(Y2o[m][i], Y1o[m][j], aB);
              }
              D[i][j] = aD;
              nb[i][j] = (e - 2 * h >= 0) ? aB : splat<S>(0.0);
            }
            S ar = r[i];
#pragma unroll
            for (int m = 0; m < B; ++m) ar = fnma_(Y2o[m][i], vo[m], ar);
            r[i] = ar;
          }
          Sp.st(Sp.Bc, e, nb);
        }
        if (e + h < K) {
          const int o = e + h;
          S Y1o[B][B], vo[B];
          Sp.ld(Sp.Bc, o, Y1o);
          Sp.ldv(Sp.R, o, vo);
#pragma unroll
          for (int i = 0; i < B; ++i) {
#pragma unroll
            for (int j = 0; j < B; ++j) {
              S aD = D[i][j];
#pragma unroll
              for (int m = 0; m < B; ++m) aD = fnma_(Y1o[m][i], Y1o[m][j], aD);
              D[i][j] = aD;
            }
            S ar = r[i];
#pragma unroll
            for (int m = 0; m < B; ++m) ar = fnma_(Y1o[m][i], vo[m], ar);
            r[i] = ar;
          }
        }
        Sp.st(Sp.D, e, D);
        Sp.stv(Sp.R, e, r);
      }
    }
    Sp.sync();
  }
  if (k == 0) {
    S D[B][B], Lf[B][B], r[B], t[B], y[B];
    Sp.ld(Sp.D, 0, D);
    report<P>(Sp.fail, lchol<B, S>(D, Lf), Sp.ltime(0));
    Sp.ldv(Sp.R, 0, r);
    llsolve<B, S>(Lf, r, t);
    lltsolve<B, S>(Lf, t, y);
    Sp.stv(Sp.Y, 0, y);
  }
  Sp.sync();
#pragma unroll 1
  for (int h = hmax; h >= 1; h >>= 1) {
    const int o = h + 2 * h * k;
    if (o < K) {
      S Lf[B][B], Y1[B][B], v[B], yl[B], t[B], y[B];
      Sp.ld(Sp.D, o, Lf);
      Sp.ld(Sp.Bc, o, Y1);
      Sp.ldv(Sp.R, o, v);
      Sp.ldv(Sp.Y, o - h, yl);
#pragma unroll
      for (int i = 0; i < B; ++i) {
        S acc = v[i];
#pragma unroll
        for (int m = 0; m < B; ++m) acc = fnma_(Y1[i][m], yl[m], acc);
        t[i] = acc;
      }
      if (o + h < K) {
        S Y2[B][B], yr[B];
        Sp.ld(Sp.Y2, o, Y2);
        Sp.ldv(Sp.Y, o + h, yr);
#pragma unroll
        for (int i = 0; i < B; ++i) {
          S acc = t[i];
#pragma unroll
          for (int m = 0; m < B; ++m) acc = fnma_(Y2[i][m], yr[m], acc);
          t[i] = acc;
        }
      }
      lltsolve<B, S>(Lf, t, y);
      Sp.stv(Sp.Y, o, y);
    }
    Sp.sync();
  }
}

template <int B, class S, int P, bool CL>
__device__ __noinline__ void lbcr(SepL<B, S, CL> Sp, int k) {
  lbcr_body<B, S, P, CL>(Sp, k);
}

// ---------------------------------------------------------------- pass 1 ---
// RING: store every interior factor L_j into a per-thread shared-memory ring
// (element e of step i at ring[(i * RE + e) * rnt + rtid]) so that pass 2
// only substitutes; otherwise checkpoint every G steps for re-factoring.
template <int B, class Tio, class S, int P, bool BWD, int G, bool SM, bool CL, bool RING = false>
__device__ __forceinline__ void lpass1_body(const Grp<Tio, P>& x, const Wts<S>& w, const SepL<B, S, CL>& Sp, S* ck, int k,
                                            int f, int sig, S* ring = nullptr, int rnt = 0, int rtid = 0) {
  constexpr int RE = B * (B + 1) / 2 + B;
  const int T = x.T, l = sig - 1;
  S ap[2 * B - 1];
  if (f > 0) spow<B, S>(ldl<S, Tio, P, SM>(x.s, f - 1), w.s2, ap); else zero<2 * B - 1, S>(ap);
  S Arr[B][B], Arl[B][B], All[B][B], rr[B], rl[B];
  zero<B, S>(Arr); zero<B, S>(Arl); zero<B, S>(All); zero<B, S>(rr); zero<B, S>(rl);
  int bad = 0, badj = INT_MAX;
  if (f < sig) {
    S Lf[B][B], wv[B], X[B][B];
    zero<B, S>(X);
    S sg = splat<S>(1.0);
    {  // first interior point: no coupling to the left inside the chunk
      S c[B], an[2 * B - 1], M[B][B], wc[B], rhs[B];
      ldlv<B, S, Tio, P, SM>(x.c, f * B, c);
      spow<B, S>(ldl<S, Tio, P, SM>(x.s, f), w.s2, an);
      lassemble<B, S>(c, w.g2, ap, an, M, wc);
      lrhs<B, S, Tio, P, BWD, SM>(x, w, f, wc, M, rhs);
      const int b = lchol<B, S>(M, Lf);
      if (b) { bad |= b; badj = min(badj, f); }
      llsolve<B, S>(Lf, rhs, wv);
      if (RING) {
        int e = 0;
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int q = 0; q <= i; ++q) ring[(e++) * rnt + rtid] = Lf[i][q];
      }
      if (k > 0) {  // X_f = L_f^{-1} N_{f-1}
        S NL[B][B];
        lN<B, S>(ap, NL);
        lleft<B, S>(Lf, NL, X);
#pragma unroll
        for (int i = 0; i < B; ++i) {
#pragma unroll
          for (int q = 0; q <= i; ++q) {
            S acc = All[i][q];
#pragma unroll
            for (int m = 0; m < B; ++m) acc = fma_(X[m][i], X[m][q], acc);
            All[i][q] = acc;
          }
          S acc = rl[i];
#pragma unroll
          for (int m = 0; m < B; ++m) acc = fma_(X[m][i], wv[m], acc);
          rl[i] = acc;
        }
      }
#pragma unroll
      for (int m = 0; m < 2 * B - 1; ++m) ap[m] = an[m];
    }
#pragma unroll 1
    for (int j = f + 1; j <= l; ++j) {
      S c[B], an[2 * B - 1], M[B][B], wc[B], rhs[B], Pm[B][B];
      ldlv<B, S, Tio, P, SM>(x.c, j * B, c);
      spow<B, S>(ldl<S, Tio, P, SM>(x.s, j), w.s2, an);
      lassemble<B, S>(c, w.g2, ap, an, M, wc);
      lrhs<B, S, Tio, P, BWD, SM>(x, w, j, wc, M, rhs);
      lPfromN<B, S>(ap, Lf, Pm);
      lcouple<B, S>(Pm, wv, M, rhs);
      const int b = lchol<B, S>(M, Lf);
      if (b) { bad |= b; badj = min(badj, j); }
      llsolve<B, S>(Lf, rhs, wv);
      if (RING) {
        S* rp = ring + (j - f) * RE * rnt + rtid;
        int e = 0;
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int q = 0; q <= i; ++q) rp[(e++) * rnt] = Lf[i][q];
      }
      if (k > 0) {  // spike X_j = -L_j^{-1} P X_{j-1}; carried with alternating sign sg
        S Y[B][B];
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int q = 0; q < B; ++q) {
            S acc = mul_(Pm[i][0], X[0][q]);
#pragma unroll
            for (int m = 1; m < B; ++m) acc = fma_(Pm[i][m], X[m][q], acc);
            Y[i][q] = acc;
          }
        lleft<B, S>(Lf, Y, X);
        sg = neg_(sg);
#pragma unroll
        for (int i = 0; i < B; ++i) {
#pragma unroll
          for (int q = 0; q <= i; ++q) {
            S acc = All[i][q];
#pragma unroll
            for (int m = 0; m < B; ++m) acc = fma_(X[m][i], X[m][q], acc);
            All[i][q] = acc;
          }
          S acc = mul_(X[0][i], wv[0]);
#pragma unroll
          for (int m = 1; m < B; ++m) acc = fma_(X[m][i], wv[m], acc);
          rl[i] = fma_(sg, acc, rl[i]);
        }
      }
      const int done = j - f + 1;
      if (!RING && (done % G) == 0 && j < l) {  // checkpoint: resume point of pass-2 segment done/G
        S* cp = ck + (done / G - 1) * CkN<B>::N * Sp.nt + (k - Sp.rank * Sp.nt);
        int e = 0;
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int q = 0; q <= i; ++q) cp[(e++) * Sp.nt] = Lf[i][q];
#pragma unroll
        for (int i = 0; i < B; ++i) cp[(e++) * Sp.nt] = wv[i];
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int q = 0; q < B; ++q) cp[(e++) * Sp.nt] = mul_(sg, X[i][q]);
      }
#pragma unroll
      for (int m = 0; m < 2 * B - 1; ++m) ap[m] = an[m];
    }
    // Schur complement of the interior onto the separators (ap = a(s_l)).
    S Pl[B][B];
    lPfromN<B, S>(ap, Lf, Pl);
#pragma unroll
    for (int i = 0; i < B; ++i) {
#pragma unroll
      for (int q = 0; q < B; ++q) {
        S a1 = mul_(Pl[i][0], Pl[q][0]), a2 = mul_(Pl[i][0], X[0][q]);
#pragma unroll
        for (int m = 1; m < B; ++m) {
          a1 = fma_(Pl[i][m], Pl[q][m], a1);
          a2 = fma_(Pl[i][m], X[m][q], a2);
        }
        Arr[i][q] = neg_(a1);
        Arl[i][q] = mul_(neg_(sg), a2);
      }
      S a3 = mul_(Pl[i][0], wv[0]);
#pragma unroll
      for (int m = 1; m < B; ++m) a3 = fma_(Pl[i][m], wv[m], a3);
      rr[i] = neg_(a3);
      rl[i] = neg_(rl[i]);
#pragma unroll
      for (int q = 0; q <= i; ++q) {
        All[i][q] = neg_(All[i][q]);
        All[q][i] = All[i][q];
      }
    }
  } else if (k > 0) {
    lN<B, S>(ap, Arl);  // chunk of one point: direct coupling sigma_{k-1} -> sigma_k
  }
  // the separator's own block and rhs (ap = a(s_{sig-1}))
  {
    S c[B], an[2 * B - 1], M[B][B], wc[B], rhs[B];
    ldlv<B, S, Tio, P, SM>(x.c, sig * B, c);
    if (sig < T - 1) spow<B, S>(ldl<S, Tio, P, SM>(x.s, sig), w.s2, an); else zero<2 * B - 1, S>(an);
    lassemble<B, S>(c, w.g2, ap, an, M, wc);
    lrhs<B, S, Tio, P, BWD, SM>(x, w, sig, wc, M, rhs);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      rhs[i] = add_(rhs[i], rr[i]);
#pragma unroll
      for (int q = 0; q <= i; ++q) {
        M[i][q] = add_(M[i][q], Arr[i][q]);
        M[q][i] = M[i][q];
      }
    }
    Sp.st(Sp.D, k, M);
    Sp.stv(Sp.R, k, rhs);
    Sp.st(Sp.Bc, k, Arl);
    Sp.st(Sp.Y2, k, All);  // temporaries consumed by the left neighbour
    Sp.stv(Sp.Y, k, rl);
  }
  if (bad) report<P>(Sp.fail, bad, badj);
}

// ---------------------------------------------------------------- pass 2 ---
template <int B, class Tio, class S, int P, bool BWD, int G, bool SM, bool CL>
__device__ __forceinline__ void lpass2_body(const Grp<Tio, P>& x, const Wts<S>& w, const SepL<B, S, CL>& Sp,
                                            const S* ck, int k, int f, int sig, const Vec<B, S>& yLv,
                                            const Vec<B, S>& yRv) {
  const int l = sig - 1;
  S yR[B], yL[B], yfR[B];
#pragma unroll
  for (int i = 0; i < B; ++i) { yR[i] = yRv.v[i]; yL[i] = yLv.v[i]; }
  zero<B, S>(yfR);
  if (!BWD) {
#pragma unroll
    for (int i = 0; i < B; ++i) stl<S, Tio, P, SM>(x.yout, x.nv, sig * B + i, yR[i]);
  } else {
    ldlv<B, S, Tio, P, SM>(x.yin, sig * B, yfR);
    lpoint_grads<B, S, Tio, P, SM>(x, w, sig, yR, yfR);
  }
  S yn[B], yfn[B];  // solution / forward y at the point after the current one
#pragma unroll
  for (int i = 0; i < B; ++i) { yn[i] = yR[i]; yfn[i] = yfR[i]; }
  if (f < sig) {
    const int nseg = (l - f + 1 + G - 1) / G;
#pragma unroll 1
    for (int seg = nseg - 1; seg >= 0; --seg) {
      const int j0 = f + seg * G;
      const int len = min(G, l + 1 - j0);
      S Lp[B][B], wp[B], ap[2 * B - 1];
      if (seg > 0) {
        const S* cp = ck + (seg - 1) * CkN<B>::N * Sp.nt + (k - Sp.rank * Sp.nt);
        int e = 0;
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int q = 0; q <= i; ++q) Lp[i][q] = cp[(e++) * Sp.nt];
#pragma unroll
        for (int i = 0; i < B; ++i) wp[i] = cp[(e++) * Sp.nt];
        if (k > 0) {  // w' = w - X y_L  (left-separator correction)
#pragma unroll
          for (int i = 0; i < B; ++i)
#pragma unroll
            for (int q = 0; q < B; ++q) wp[i] = fnma_(cp[(CkN<B>::L + B + i * B + q) * Sp.nt], yL[q], wp[i]);
        }
        spow<B, S>(ldl<S, Tio, P, SM>(x.s, j0 - 1), w.s2, ap);
      } else {
        zero<B, S>(Lp);
        zero<B, S>(wp);
        if (f > 0) spow<B, S>(ldl<S, Tio, P, SM>(x.s, f - 1), w.s2, ap); else zero<2 * B - 1, S>(ap);
      }
      S Lr[G][B][B], Wr[G][B], Sr[G];
#pragma unroll
      for (int i = 0; i < G; ++i) {
        if (i < len) {
          const int j = j0 + i;
          S c[B], an[2 * B - 1], M[B][B], wc[B], rhs[B];
          ldlv<B, S, Tio, P, SM>(x.c, j * B, c);
          Sr[i] = ldl<S, Tio, P, SM>(x.s, j);
          spow<B, S>(Sr[i], w.s2, an);
          lassemble<B, S>(c, w.g2, ap, an, M, wc);
          lrhs<B, S, Tio, P, BWD, SM>(x, w, j, wc, M, rhs);
          if (j == f) {
            if (k > 0) {  // rhs -= N_{f-1} y_L
              S NL[B][B];
              lN<B, S>(ap, NL);
#pragma unroll
              for (int q = 0; q < B; ++q)
#pragma unroll
                for (int r = 0; r < B; ++r) rhs[q] = fnma_(NL[q][r], yL[r], rhs[q]);
            }
          } else {
            S Pm[B][B];
            lPfromN<B, S>(ap, Lp, Pm);
            lcouple<B, S>(Pm, wp, M, rhs);
          }
          if (j == l) {  // rhs -= N_l^T y_R
            S NR[B][B], t[B];
            lN<B, S>(an, NR);
            lmatTvec<B, S>(NR, yR, t);
#pragma unroll
            for (int q = 0; q < B; ++q) rhs[q] = sub_(rhs[q], t[q]);
          }
          lchol<B, S>(M, Lr[i]);
          llsolve<B, S>(Lr[i], rhs, Wr[i]);
#pragma unroll
          for (int q = 0; q < B; ++q) {
            wp[q] = Wr[i][q];
#pragma unroll
            for (int r = 0; r <= q; ++r) Lp[q][r] = Lr[i][q][r];
          }
#pragma unroll
          for (int m = 0; m < 2 * B - 1; ++m) ap[m] = an[m];
        }
      }
#pragma unroll
      for (int i = G - 1; i >= 0; --i) {
        if (i < len) {
          const int j = j0 + i;
          S yv[B], an[2 * B - 1];
          spow<B, S>(Sr[i], w.s2, an);
          if (j == l) {
            lltsolve<B, S>(Lr[i], Wr[i], yv);
          } else {  // y_j = L^{-T} (w_j - L^{-1} N_j^T y_{j+1})
            S Nj[B][B], v[B], u[B], t[B];
            lN<B, S>(an, Nj);
            lmatTvec<B, S>(Nj, yn, v);
            llsolve<B, S>(Lr[i], v, u);
#pragma unroll
            for (int q = 0; q < B; ++q) t[q] = sub_(Wr[i][q], u[q]);
            lltsolve<B, S>(Lr[i], t, yv);
          }
          if (!BWD) {
#pragma unroll
            for (int q = 0; q < B; ++q) stl<S, Tio, P, SM>(x.yout, x.nv, j * B + q, yv[q]);
          } else {
            S yf[B];
            ldlv<B, S, Tio, P, SM>(x.yin, j * B, yf);
            lpoint_grads<B, S, Tio, P, SM>(x, w, j, yv, yf);
            if (x.gs.on) stl<S, Tio, P, SM>(x.gs, x.nv, j, lds<B, S>(an, yv, yf, yn, yfn));
#pragma unroll
            for (int q = 0; q < B; ++q) yfn[q] = yf[q];
          }
#pragma unroll
          for (int q = 0; q < B; ++q) yn[q] = yv[q];
        }
      }
    }
  }
  if (BWD && k > 0 && x.gs.on) {  // interval (sigma_{k-1}, first point of the chunk)
    const int jm = f - 1;
    S yfm[B], am[2 * B - 1];
    ldlv<B, S, Tio, P, SM>(x.yin, jm * B, yfm);
    spow<B, S>(ldl<S, Tio, P, SM>(x.s, jm), w.s2, am);
    stl<S, Tio, P, SM>(x.gs, x.nv, jm, lds<B, S>(am, yL, yfm, yn, yfn));
  }
}

// Pass 2 with the interior factors stored by pass 1 (RING): forward
// substitution with both separator corrections, then back substitution; no
// re-factorisation.  The ring's w slots receive the forward-substituted rhs.
template <int B, class Tio, class S, int P, bool BWD, bool SM, bool CL>
__device__ __forceinline__ void lpass2r_body(const Grp<Tio, P>& x, const Wts<S>& w, const SepL<B, S, CL>& Sp,
                                             S* ring, int rnt, int rtid, int k, int f, int sig, const Vec<B, S>& yLv,
                                             const Vec<B, S>& yRv) {
  constexpr int LN = B * (B + 1) / 2, RE = LN + B;
  const int l = sig - 1;
  S yR[B], yL[B], yfR[B];
#pragma unroll
  for (int i = 0; i < B; ++i) { yR[i] = yRv.v[i]; yL[i] = yLv.v[i]; }
  zero<B, S>(yfR);
  if (!BWD) {
#pragma unroll
    for (int i = 0; i < B; ++i) stl<S, Tio, P, SM>(x.yout, x.nv, sig * B + i, yR[i]);
  } else {
    ldlv<B, S, Tio, P, SM>(x.yin, sig * B, yfR);
    lpoint_grads<B, S, Tio, P, SM>(x, w, sig, yR, yfR);
  }
  S yn[B], yfn[B];
#pragma unroll
  for (int i = 0; i < B; ++i) { yn[i] = yR[i]; yfn[i] = yfR[i]; }
  if (f < sig) {
    S Lp[B][B], wp[B], ap[2 * B - 1];
    zero<B, S>(Lp);
    zero<B, S>(wp);
    if (f > 0) spow<B, S>(ldl<S, Tio, P, SM>(x.s, f - 1), w.s2, ap); else zero<2 * B - 1, S>(ap);
#pragma unroll 1
    for (int j = f; j <= l; ++j) {  // forward substitution
      S* rp = ring + (j - f) * RE * rnt + rtid;
      S Lf[B][B], rhs[B], an[2 * B - 1];
      int e = 0;
#pragma unroll
      for (int i = 0; i < B; ++i)
#pragma unroll
        for (int q = 0; q <= i; ++q) Lf[i][q] = rp[(e++) * rnt];
      if (BWD) {
        ldlv<B, S, Tio, P, SM>(x.gy, j * B, rhs);
      } else {
        S c[B];
        ldlv<B, S, Tio, P, SM>(x.c, j * B, c);
        const S wd = mul_(w.g2, ldl<S, Tio, P, SM>(x.d, j));
#pragma unroll
        for (int i = 0; i < B; ++i) rhs[i] = mul_(wd, c[i]);
        if (j == 0) {
#pragma unroll
          for (int i = 0; i < B; ++i)
            if (i < x.n_iv) rhs[i] = fma_(w.i2, ldg_l<S, Tio, P>(x.u, i), rhs[i]);
        }
      }
      spow<B, S>(ldl<S, Tio, P, SM>(x.s, j), w.s2, an);
      S N[B][B], t[B];
      lN<B, S>(ap, N);
      if (j == f) {
#pragma unroll
        for (int q = 0; q < B; ++q) t[q] = yL[q];  // rhs -= N_{f-1} y_L (zero for k = 0)
      } else {
        lltsolve<B, S>(Lp, wp, t);  // rhs -= P~_{j-1} w_{j-1} = N_{j-1} L_{j-1}^{-T} w_{j-1}
      }
#pragma unroll
      for (int q = 0; q < B; ++q)
#pragma unroll
        for (int r = 0; r < B; ++r) rhs[q] = fnma_(N[q][r], t[r], rhs[q]);
      if (j == l) {  // rhs -= N_l^T y_R
        S NR[B][B], u[B];
        lN<B, S>(an, NR);
        lmatTvec<B, S>(NR, yR, u);
#pragma unroll
        for (int q = 0; q < B; ++q) rhs[q] = sub_(rhs[q], u[q]);
      }
      llsolve<B, S>(Lf, rhs, wp);
#pragma unroll
      for (int q = 0; q < B; ++q) rp[(LN + q) * rnt] = wp[q];
#pragma unroll
      for (int q = 0; q < B; ++q)
#pragma unroll
        for (int r = 0; r <= q; ++r) Lp[q][r] = Lf[q][r];
#pragma unroll
      for (int m = 0; m < 2 * B - 1; ++m) ap[m] = an[m];
    }
#pragma unroll 1
    for (int j = l; j >= f; --j) {  // back substitution
      const S* rp = ring + (j - f) * RE * rnt + rtid;
      S Lf[B][B], wj[B], yv[B], an[2 * B - 1];
      int e = 0;
#pragma unroll
      for (int i = 0; i < B; ++i)
#pragma unroll
        for (int q = 0; q <= i; ++q) Lf[i][q] = rp[(e++) * rnt];
#pragma unroll
      for (int q = 0; q < B; ++q) wj[q] = rp[(LN + q) * rnt];
      const S sj = ldl<S, Tio, P, SM>(x.s, j);
      spow<B, S>(sj, w.s2, an);
      if (j == l) {
        lltsolve<B, S>(Lf, wj, yv);
      } else {  // y_j = L^{-T} (w_j - L^{-1} N_j^T y_{j+1})
        S Nj[B][B], v[B], u[B], t[B];
        lN<B, S>(an, Nj);
        lmatTvec<B, S>(Nj, yn, v);
        llsolve<B, S>(Lf, v, u);
#pragma unroll
        for (int q = 0; q < B; ++q) t[q] = sub_(wj[q], u[q]);
        lltsolve<B, S>(Lf, t, yv);
      }
      if (!BWD) {
#pragma unroll
        for (int q = 0; q < B; ++q) stl<S, Tio, P, SM>(x.yout, x.nv, j * B + q, yv[q]);
      } else {
        S yf[B];
        ldlv<B, S, Tio, P, SM>(x.yin, j * B, yf);
        lpoint_grads<B, S, Tio, P, SM>(x, w, j, yv, yf);
        if (x.gs.on) stl<S, Tio, P, SM>(x.gs, x.nv, j, lds<B, S>(an, yv, yf, yn, yfn));
#pragma unroll
        for (int q = 0; q < B; ++q) yfn[q] = yf[q];
      }
#pragma unroll
      for (int q = 0; q < B; ++q) yn[q] = yv[q];
    }
  }
  if (BWD && k > 0 && x.gs.on) {  // interval (sigma_{k-1}, first point of the chunk)
    const int jm = f - 1;
    S yfm[B], am[2 * B - 1];
    ldlv<B, S, Tio, P, SM>(x.yin, jm * B, yfm);
    spow<B, S>(ldl<S, Tio, P, SM>(x.s, jm), w.s2, am);
    stl<S, Tio, P, SM>(x.gs, x.nv, jm, lds<B, S>(am, yL, yfm, yn, yfn));
  }
}

// Out-of-line versions for the streaming kernel (keeps its register allocation per pass).
template <int B, class Tio, class S, int P, bool BWD, int G, bool SM>
__device__ __noinline__ void lpass1(const Grp<Tio, P> x, const Wts<S> w, SepL<B, S> Sp, S* ck, int k, int f,
                                    int sig) {
  lpass1_body<B, Tio, S, P, BWD, G, SM, false>(x, w, Sp, ck, k, f, sig);
}
template <int B, class Tio, class S, int P, bool BWD, int G, bool SM>
__device__ __noinline__ void lpass2(const Grp<Tio, P> x, const Wts<S> w, SepL<B, S> Sp, const S* ck, int k, int f,
                                    int sig, const Vec<B, S> yL, const Vec<B, S> yR) {
  lpass2_body<B, Tio, S, P, BWD, G, SM, false>(x, w, Sp, ck, k, f, sig, yL, yR);
}


// ------------------------------------------------------------ the kernel ---
template <int B, class S>
__device__ __forceinline__ void write_dummy_sep(const SepL<B, S, false>& Sp, int i) {
  S Id[B][B], Z[B][B], z[B];
  zero<B, S>(Z);
  zero<B, S>(z);
#pragma unroll
  for (int r = 0; r < B; ++r)
#pragma unroll
    for (int c = 0; c < B; ++c) Id[r][c] = splat<S>(r == c ? 1.0 : 0.0);
  Sp.st(Sp.D, i, Id);
  Sp.st(Sp.Bc, i, Z);
  Sp.st(Sp.Y2, i, Z);
  Sp.stv(Sp.R, i, z);
  Sp.stv(Sp.Y, i, z);
}

// Separator scratch after the five record fields: a reserved per-warp region
// of W (3 B^2 + 3 B) values (W = nt / 32; the host layouts keep it), then the
// separator times and failure flags.
template <int B, class S>
__device__ __forceinline__ int* sep_tail(S* y_end, int nt) {
  return reinterpret_cast<int*>(y_end + (nt >> 5) * (3 * B * B + 3 * B));
}

template <int B, class Tio, class S, bool BWD, int G>
__global__ void __launch_bounds__(SMNN_MAX_THREADS, SMNN_MIN_BLOCKS) fused_kernel(Args<Tio> a) {
  constexpr int P = LaneT<S>::P;
  unsigned char* smem_raw = smnn_dyn_smem;
  const int K = a.K;
  const int nt = blockDim.x;  // separator slots (K real + dummies)
  SepL<B, S> Sp;
  Sp.D = reinterpret_cast<S*>(smem_raw);
  Sp.Bc = Sp.D + B * B * nt;
  Sp.Y2 = Sp.Bc + B * B * nt;
  Sp.R = Sp.Y2 + B * B * nt;
  Sp.Y = Sp.R + B * nt;
  Sp.time = sep_tail<B, S>(Sp.Y + B * nt, nt);
  Sp.fail = Sp.time + nt;
  Sp.K = K;
  Sp.nt = nt;
  Sp.rank = 0;
  Sp.cs = 1;
  const Wts<S> w{splat<S>(a.wg2), splat<S>(a.wi2), splat<S>(a.ws2)};
  const int k = threadIdx.x;
  const int T = a.T;
  S* ck = reinterpret_cast<S*>(a.ckpt) + size_t(blockIdx.x) * size_t(a.nseg_ck) * CkN<B>::N * nt;
  const int64_t ngroups = (a.n_inst + P - 1) / P;
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    if (k < P) Sp.fail[k] = INT_MAX;
    Grp<Tio, P> x;
    x.template init<B>(a, g * P);
    const int f = (k < K) ? chunk_begin(k, T, K) : 0;
    const int sig = (k < K) ? chunk_begin(k + 1, T, K) - 1 : 0;
    __syncthreads();
    if (k < K) {
      Sp.time[k] = sig;
      lpass1<B, Tio, S, P, BWD, G, false>(x, w, Sp, ck, k, f, sig);
    } else {
      write_dummy_sep<B, S>(Sp, k);
    }
    __syncthreads();
    S Dk[B][B], rk[B];
    if (k + 1 < K) {  // add the right neighbour's Schur terms A_ll, r_l
      S Al[B][B], rl[B];
      Sp.ld(Sp.D, k, Dk);
      Sp.ld(Sp.Y2, k + 1, Al);
      Sp.ldv(Sp.R, k, rk);
      Sp.ldv(Sp.Y, k + 1, rl);
#pragma unroll
      for (int i = 0; i < B; ++i) {
        rk[i] = add_(rk[i], rl[i]);
#pragma unroll
        for (int q = 0; q < B; ++q) Dk[i][q] = add_(Dk[i][q], Al[i][q]);
      }
    }
    __syncthreads();
    if (k + 1 < K) {
      Sp.st(Sp.D, k, Dk);
      Sp.stv(Sp.R, k, rk);
    }
    __syncthreads();
    lbcr<B, S, P, false>(Sp, k);
    if (k < K) {
      Vec<B, S> yL, yR;
      Sp.ldv(Sp.Y, k, yR.v);
      if (k > 0) Sp.ldv(Sp.Y, k - 1, yL.v); else zero<B, S>(yL.v);
      lpass2<B, Tio, S, P, BWD, G, false>(x, w, Sp, ck, k, f, sig, yL, yR);
    }
    __syncthreads();
    if (k < x.nv && a.info) a.info[g * P + k] = (Sp.fail[k] == INT_MAX) ? 0 : Sp.fail[k];
  }
}

// ======================================================================
// Resident kernel: the instance's inputs are bulk-copied (TMA, cp.async.bulk)
// into shared memory, split over a thread-block cluster of cs CTAs when one
// SM cannot hold them; both passes read shared memory; outputs overwrite
// their inputs in place (y over c forward; dc, dd, ds over c, d, s backward)
// and are written back with coalesced stores; the separator BCR runs across
// the cluster through distributed shared memory.  HBM traffic is therefore
// the algorithmic bytes (inputs read once, outputs written once).
// ======================================================================

struct RLayout {
  int nt, cs;                              // threads per CTA, CTAs per cluster
  int off_c, off_d, off_s, off_g, off_y;   // data regions of lane 0 (bytes, 16-aligned)
  int lane;                                // byte stride between the lanes' data regions
  int off_sep, off_ck, off_bar;
};



template <int B, class Tio, class S, bool BWD, int G, bool CL>
__global__ void __launch_bounds__(SMNN_MAX_THREADS, (LaneT<S>::P == 1 ? SMNN_MIN_BLOCKS : 1))
    resident_kernel(Args<Tio> a, RLayout L) {
  constexpr int P = LaneT<S>::P;
  unsigned char* sm = smnn_dyn_smem;
  const int cs = L.cs, nt = L.nt, tid = threadIdx.x;
  const int rank = CL ? int(cooperative_groups::this_cluster().block_rank()) : 0;
  const int K = cs * nt;
  const int T = a.T;
  SepL<B, S, CL> Sp;
  Sp.D = reinterpret_cast<S*>(sm + L.off_sep);
  Sp.Bc = Sp.D + B * B * nt;
  Sp.Y2 = Sp.Bc + B * B * nt;
  Sp.R = Sp.Y2 + B * B * nt;
  Sp.Y = Sp.R + B * nt;
  Sp.time = sep_tail<B, S>(Sp.Y + B * nt, nt);
  Sp.fail = Sp.time + nt;
  Sp.K = K;
  Sp.nt = nt;
  Sp.rank = rank;
  Sp.cs = cs;
  S* ck = reinterpret_cast<S*>(sm + L.off_ck);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.off_bar);
  const Wts<S> w{splat<S>(a.wg2), splat<S>(a.wi2), splat<S>(a.ws2)};
  if (tid == 0) mbar_init(bar, 1);
  __syncthreads();
  uint32_t parity = 0;
  const int64_t nclusters = gridDim.x / cs;
  const int k = rank * nt + tid;  // global chunk index
  const int t0 = chunk_begin(rank * nt, T, K), t1 = chunk_begin((rank + 1) * nt, T, K);
  const int s0 = max(t0 - 1, 0), s1 = min(t1, T - 1);
  const int y0 = max(t0 - 1, 0);
  const int f = chunk_begin(k, T, K), sig = chunk_begin(k + 1, T, K) - 1;
  constexpr int E = int(sizeof(Tio));
  const int64_t ngroups = (a.n_inst + P - 1) / P;

  for (int64_t g = blockIdx.x / cs; g < ngroups; g += nclusters) {
    const int nv = (a.n_inst - g * P < P) ? int(a.n_inst - g * P) : P;
    Grp<Tio, P> x;  // streams as element offsets into shared memory
    x.T = T;
    x.n_iv = a.n_iv;
    x.nv = nv;
    int pre_c[P], pre_d[P], pre_s[P];
    const Tio* lo[P][5];
    uint32_t nb[P][5];
    uint32_t tx = 0;
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const int64_t inst = g * P + (q < nv ? q : 0);
      const int64_t tb = inst * int64_t(T) * B, t1b = inst * int64_t(T), tsb = inst * int64_t(T - 1);
      const int lb = q * L.lane;
      const Span<Tio> pc(a.coeffs + tb + t0 * B, (t1 - t0) * B);
      const Span<Tio> pd(a.rhs + t1b + t0, t1 - t0);
      const Span<Tio> ps(a.steps + tsb + s0, s1 - s0);
      const Span<Tio> pg(BWD ? a.grad_y + tb + t0 * B : a.coeffs, BWD ? (t1 - t0) * B : 0);
      const Span<Tio> py(BWD ? a.y_in + tb + y0 * B : a.coeffs, BWD ? (t1 - y0) * B : 0);
      lo[q][0] = pc.lo; nb[q][0] = pc.bytes;
      lo[q][1] = pd.lo; nb[q][1] = pd.bytes;
      lo[q][2] = ps.lo; nb[q][2] = ps.bytes;
      lo[q][3] = pg.lo; nb[q][3] = pg.bytes;
      lo[q][4] = py.lo; nb[q][4] = py.bytes;
      tx += pc.bytes + pd.bytes + ps.bytes + pg.bytes + py.bytes;
      pre_c[q] = pc.pre;
      pre_d[q] = pd.pre;
      pre_s[q] = ps.pre;
      const int oc = (L.off_c + lb) / E + pc.pre - t0 * B;
      const int od = (L.off_d + lb) / E + pd.pre - t0;
      const int os = (L.off_s + lb) / E + ps.pre - s0;
      x.c.o[q] = oc;
      x.d.o[q] = od;
      x.s.o[q] = os;
      x.u[q] = a.iv + inst * a.n_iv;
      x.gy.o[q] = BWD ? (L.off_g + lb) / E + pg.pre - t0 * B : 0;
      x.yin.o[q] = BWD ? (L.off_y + lb) / E + py.pre - y0 * B : 0;
      x.yout.o[q] = oc;
      x.gc.o[q] = oc;
      x.gd.o[q] = od;
      x.gs.o[q] = os;
      x.gu[q] = (BWD && a.g_iv) ? a.g_iv + inst * a.n_iv : nullptr;
    }
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, tx);
      const int offs[5] = {L.off_c, L.off_d, L.off_s, L.off_g, L.off_y};
#pragma unroll
      for (int q = 0; q < P; ++q)
#pragma unroll
        for (int r = 0; r < 5; ++r)
          if (nb[q][r]) bulk_g2s(sm + offs[r] + q * L.lane, lo[q][r], nb[q][r], bar);
    }
    x.c.on = x.d.on = x.s.on = true;
    x.gy.on = x.yin.on = BWD;
    x.yout.on = !BWD;
    x.gc.on = BWD && a.g_coeffs;
    x.gd.on = BWD && a.g_rhs;
    x.gs.on = BWD && a.g_steps;
    x.gu_on = BWD && a.g_iv;
    if (tid < P) Sp.fail[tid] = INT_MAX;
    Sp.time[tid] = sig;
    mbar_wait(bar, parity);
    parity ^= 1u;
    __syncthreads();

    lpass1_body<B, Tio, S, P, BWD, G, true, CL>(x, w, Sp, ck, k, f, sig);
    Sp.sync();
    S Dk[B][B], rk[B];
    const bool right = k + 1 < K;
    if (right) {  // add the right neighbour's Schur terms A_ll, r_l (maybe remote)
      S Al[B][B], rl[B];
      Sp.ld(Sp.D, k, Dk);
      Sp.ld(Sp.Y2, k + 1, Al);
      Sp.ldv(Sp.R, k, rk);
      Sp.ldv(Sp.Y, k + 1, rl);
#pragma unroll
      for (int i = 0; i < B; ++i) {
        rk[i] = add_(rk[i], rl[i]);
#pragma unroll
        for (int q = 0; q < B; ++q) Dk[i][q] = add_(Dk[i][q], Al[i][q]);
      }
    }
    Sp.sync();
    if (right) {
      Sp.st(Sp.D, k, Dk);
      Sp.stv(Sp.R, k, rk);
    }
    Sp.sync();
    lbcr<B, S, P, CL>(Sp, k);
    Vec<B, S> yL, yR;
    Sp.ldv(Sp.Y, k, yR.v);
    if (k > 0) Sp.ldv(Sp.Y, k - 1, yL.v); else zero<B, S>(yL.v);
    Sp.sync();
    lpass2_body<B, Tio, S, P, BWD, G, true, CL>(x, w, Sp, ck, k, f, sig, yL, yR);
    __syncthreads();
    // write the outputs back (coalesced)
#pragma unroll
    for (int q = 0; q < P; ++q) {
      if (q >= nv) break;
      const int64_t inst = g * P + q;
      const int64_t tb = inst * int64_t(T) * B, t1b = inst * int64_t(T), tsb = inst * int64_t(T - 1);
      const Tio* rc = reinterpret_cast<const Tio*>(sm + L.off_c + q * L.lane) + pre_c[q];
      const Tio* rd = reinterpret_cast<const Tio*>(sm + L.off_d + q * L.lane) + pre_d[q];
      const Tio* rs = reinterpret_cast<const Tio*>(sm + L.off_s + q * L.lane) + pre_s[q];
      if (!BWD) {
        Tio* dst = a.y_out + tb + t0 * B;
        for (int e = tid; e < (t1 - t0) * B; e += nt) dst[e] = rc[e];
      } else {
        if (a.g_coeffs) {
          Tio* dst = a.g_coeffs + tb + t0 * B;
          for (int e = tid; e < (t1 - t0) * B; e += nt) dst[e] = rc[e];
        }
        if (a.g_rhs) {
          Tio* dst = a.g_rhs + t1b + t0;
          for (int e = tid; e < t1 - t0; e += nt) dst[e] = rd[e];
        }
        if (a.g_steps) {  // this CTA owns intervals [s0, t1 - 1)
          Tio* dst = a.g_steps + tsb + s0;
          for (int e = tid; e < t1 - 1 - s0; e += nt) dst[e] = rs[e];
        }
      }
    }
    Sp.sync();
    if (rank == 0 && tid < nv && a.info) {
      int fv = Sp.fail[tid];
      if (CL)
        for (int r = 1; r < cs; ++r)
          fv = min(fv, *cooperative_groups::this_cluster().map_shared_rank(Sp.fail + tid, r));
      a.info[g * P + tid] = (fv == INT_MAX) ? 0 : fv;
    }
    Sp.sync();
  }
}

}  // namespace smnn
