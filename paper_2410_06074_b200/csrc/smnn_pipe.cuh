// smnn_pipe.cuh -- the S-MNN solve as a three-kernel pipeline.
//
// The time-parallel partition solver of smnn_rf.cuh split at its two
// synchronisation points, so that the register-heavy chunk sweeps and the
// latency-bound separator reduction no longer share one CTA's lifetime:
//
//   P1  chunk kernel: thread = time chunk [f_k, f_{k+1}); block Cholesky of the
//       chunk interior with the spike (Algorithm 3's loop),
//       Schur complement of the interior onto its two separators; writes the
//       separator blocks to the workspace.  No barrier after staging.
//   SEP separator kernel: CTA = instance, thread = separator; assembles the
//       K x K block-tridiagonal Schur system and solves it by block cyclic
//       reduction with the blocks in registers (rbcr2); writes y at the
//       separators and info.
//   P2  chunk kernel: re-factors the chunk interior in registers (forward
//       sweep, with both separator values known) and back-substitutes
//       (Algorithm 4); FWD writes y, BWD the Appendix A.1
//       gradient chain.  No barrier after staging.
//
// The chunk kernels stage their CTA's time range with TMA bulk copies
// (cp.async.bulk) and write outputs with TMA bulk stores, as the RF kernel.
// Workspace (S = arithmetic type), per instance g and chunk / separator k,
// field-major so that a warp's 32 consecutive chunks touch 128 contiguous
// bytes per field:
//   sep1 [g][PSep<B,NR>::N][K]  D_own (lower, packed), R_own, A_rl, A_ll (packed), r_l
//   ysep [g][NR B][K]           y at the separators (per right-hand side)
// NR = 2 in the SMNN_F32_C64 backward without the forward's y remainder: dl/dy
// and beta share the factorisation, so y is re-solved in fp64 beside lambda
// instead of read from fp32 storage.  With the remainder (Args::y_lo_in) the
// backward is NR = 1 and reads y_hi + y_lo (smnn_solve_bwd_ex).
//   cfail[g][K]              1 + first point of a chunk whose pivots broke down, else INT_MAX
#pragma once

#include "smnn_rf.cuh"

namespace smnn {

#ifndef SMNN_PIPE_NT
#define SMNN_PIPE_NT 128
#endif
// separator kernel residency (CTAs/SM the register budget is cut for): fp32
// arithmetic 3, fp64 2 (fewer spills; measured target f64 8.4e9 -> 9.4e9,
// while fp32 at 2 loses 3 %)
#ifndef SMNN_SEP2_MINB
#define SMNN_SEP2_MINB 3
#endif
#ifndef SMNN_SEP2_MINB64
#define SMNN_SEP2_MINB64 2
#endif
#ifndef SMNN_PIPE_P2_MINB
#define SMNN_PIPE_P2_MINB 4
#endif
// fp64 arithmetic: chunk kernels compiled for one CTA/SM fewer (P1 3, P2
// forward 4 / backward 3) -- fewer spills; measured KdV +6 %, target / SST /
// Lorenz f64 +3 %
#ifndef SMNN_PIPE_P2_MINB64
#define SMNN_PIPE_P2_MINB64 3
#endif
#ifndef SMNN_PIPE_P2_MINB64R  // backward with two right-hand sides (SMNN_F32_C64)
#define SMNN_PIPE_P2_MINB64R 3
#endif
#ifndef SMNN_PIPE_P2_MINB64F
#define SMNN_PIPE_P2_MINB64F 4
#endif
#ifndef SMNN_PIPE_P1_MINB64
#define SMNN_PIPE_P1_MINB64 3
#endif
#ifndef SMNN_PIPE_SEP_MAX
#define SMNN_PIPE_SEP_MAX 2048
#endif

// Programmatic dependent launch (sm_90+): the separator and P2 kernels are
// launched with programmatic stream serialisation (smnn_pipe.cu), so they may
// start while the previous kernel drains; griddepcontrol.wait blocks until the
// previous grid has completed and its memory is visible (a no-op when the
// kernel was launched normally), launch_dependents lets the next one start.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

struct PipeL {
  int K;          // chunks (= separators) per instance (at this level of the separator hierarchy)
  int K0;         // level-0 separators (time mapping for `info`)
  int sstride;    // level-0 separators per separator of this level (8^level)
  int NT;         // threads per CTA of the chunk kernels
  int parts;      // CTAs per instance of the chunk kernels
  int off_c, off_d, off_s, off_g, off_y, off_h, off_bar;  // shared-memory byte offsets (16-aligned)
  int off_yl;     // P2, SMNN_F32_C64: y's fp32 remainder (forward out / backward in), 0 = none
  void* sep1;
  void* ysep;
  int* cfail;
  void* seg;      // level 0, two-segment chunks: P1 -> P2 factorisation state (PSegState), else nullptr
};

// Time range of a chunk-kernel CTA: chunks [c0, c0 + nc), points [ta, tb),
// steps s staged from slo = max(ta - 1, 0) to shi = min(tb, T - 1).
struct PRange {
  int64_t g;
  int c0, nc, ta, tb, slo, shi;
  __device__ PRange(const PipeL& L, int T) {
    g = blockIdx.x / L.parts;
    const int part = int(blockIdx.x % L.parts);
    c0 = part * L.NT;
    nc = min(L.NT, L.K - c0);
    ta = chunk_begin(c0, T, L.K);
    tb = chunk_begin(c0 + nc, T, L.K);
    slo = max(ta - 1, 0);
    shi = min(tb, T - 1);
  }
};

// Time index of separator j of a level whose separators are every
// L.sstride-th level-0 separator (error reporting, include/smnn.h `info`).
__device__ __forceinline__ int sep_time(const PipeL& L, int j, int T) {
  return chunk_begin(int(int64_t(j + 1) * L.sstride), T, L.K0) - 1;
}

// ============================================================== P1 ========
template <int B, class Tio, class S, bool BWD, int CM, int NR>
__global__ void __launch_bounds__(SMNN_PIPE_NT, sizeof(S) >= 8 ? ((B == 3 && NR == 1) ? 4 : SMNN_PIPE_P1_MINB64) : 4)
    pipe_p1_kernel(Args<Tio> a, PipeL L) {  // fp64 order 2, one rhs: 4 CTAs/SM (<= 128 registers, no spills)
  using Q = PSep<B, NR>;
  unsigned char* sm = smnn_dyn_smem;
  Tio* smT = reinterpret_cast<Tio*>(sm);
  const int T = a.T, K = L.K, tid = threadIdx.x;
  const PRange R(L, T);
  const int64_t g = R.g;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.off_bar);
  const Wts<S> w{opaque(splat<S>(a.wg2)), opaque(splat<S>(a.wi2)), opaque(splat<S>(a.ws2))};
  const int64_t tb = g * int64_t(T) * B, t1b = g * int64_t(T), tsb = g * int64_t(T - 1);
  const Span<Tio> pc(a.coeffs + tb + R.ta * B, (R.tb - R.ta) * B);
  const Span<Tio> pd(a.rhs + t1b + R.ta, (BWD && NR == 1) ? 0 : R.tb - R.ta);
  const Span<Tio> ps(a.steps + tsb + R.slo, R.shi - R.slo);
  const Span<Tio> pg(BWD ? a.grad_y + tb + R.ta * B : a.coeffs, BWD ? (R.tb - R.ta) * B : 0);
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_expect_tx(bar, pc.bytes + pd.bytes + ps.bytes + pg.bytes);
    bulk_g2s(sm + L.off_c, pc.lo, pc.bytes, bar);
    if (pd.bytes) bulk_g2s(sm + L.off_d, pd.lo, pd.bytes, bar);
    if (ps.bytes) bulk_g2s(sm + L.off_s, ps.lo, ps.bytes, bar);
    if (pg.bytes) bulk_g2s(sm + L.off_g, pg.lo, pg.bytes, bar);
  }
  constexpr int E = int(sizeof(Tio));
  const int k = R.c0 + tid;
  const bool act = tid < R.nc;
  const int f = act ? chunk_begin(k, T, K) : R.ta;
  const int sig = act ? chunk_begin(k + 1, T, K) - 1 : R.ta + 1;
  const int nint = sig - f;
  const Tio* cS = smT + opaque(L.off_c / E + pc.pre + (f - R.ta) * B);
  const Tio* dS = smT + opaque(L.off_d / E + pd.pre + (f - R.ta));
  const Tio* sS = smT + opaque(L.off_s / E + ps.pre + (f - R.slo));  // sS[-1] = s_{f-1}
  const Tio* gS = smT + opaque(L.off_g / E + pg.pre + (f - R.ta) * B);
  const Tio* u = a.iv + g * a.n_iv;
  __syncthreads();  // barrier initialised
  mbar_wait(bar, 0);

  S Dsep[B][B], Rsep[NR][B], Arl[B][B], All[B][B], rl[NR][B];
  bool bad = false;
  S* seg = (L.seg && act) ? reinterpret_cast<S*>(L.seg) + g * int64_t(PSegState<B, NR>::N) * K + k : nullptr;
  if (act)
    bad = p1_chunk<B, Tio, S, BWD, CM, NR>(w, a.n_iv, u, k, K, nint, cS, dS, sS, gS, Dsep, Rsep, Arl, All, rl, seg);
  // A_ll = -sum X^T X, r_l = -sum X^T w belong to separator k - 1: hand them to
  // the left neighbour through shared memory (the staged inputs are still in
  // use, so a region of its own); a CTA's first chunk writes them to the
  // workspace for the previous CTA's last separator.
  S* ho = reinterpret_cast<S*>(sm + L.off_h);  // (LT + NR B) values per thread, field-major
  if (act) {
    int e = 0;
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int q = 0; q <= r; ++q) ho[(e++) * SMNN_PIPE_NT + tid] = neg_(All[r][q]);
#pragma unroll
    for (int p = 0; p < NR; ++p)
#pragma unroll
      for (int r = 0; r < B; ++r) ho[(Q::LT + p * B + r) * SMNN_PIPE_NT + tid] = neg_(rl[p][r]);
  }
  __syncthreads();
  if (!act) return;
  if (tid + 1 < R.nc) {
    int e = 0;
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int q = 0; q <= r; ++q) Dsep[r][q] = add_(Dsep[r][q], ho[(e++) * SMNN_PIPE_NT + tid + 1]);
#pragma unroll
    for (int p = 0; p < NR; ++p)
#pragma unroll
      for (int r = 0; r < B; ++r) Rsep[p][r] = add_(Rsep[p][r], ho[(Q::LT + p * B + r) * SMNN_PIPE_NT + tid + 1]);
  }
  // write the separator blocks (field-major: coalesced across the warp)
  S* o = reinterpret_cast<S*>(L.sep1) + g * int64_t(Q::N) * K + k;
  int e = 0;
#pragma unroll
  for (int r = 0; r < B; ++r)
#pragma unroll
    for (int q = 0; q <= r; ++q) o[int64_t(Q::D + e++) * K] = Dsep[r][q];
#pragma unroll
  for (int p = 0; p < NR; ++p)
#pragma unroll
    for (int r = 0; r < B; ++r) o[int64_t(Q::R + p * B + r) * K] = Rsep[p][r];
#pragma unroll
  for (int r = 0; r < B; ++r)
#pragma unroll
    for (int q = 0; q < B; ++q) o[int64_t(Q::BL + r * B + q) * K] = Arl[r][q];
  if (tid == 0 && k > 0) {  // the previous CTA's last separator adds these (psep_ld)
    e = 0;
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int q = 0; q <= r; ++q) o[int64_t(Q::AL + e++) * K] = neg_(All[r][q]);
#pragma unroll
    for (int p = 0; p < NR; ++p)
#pragma unroll
      for (int r = 0; r < B; ++r) o[int64_t(Q::RL + p * B + r) * K] = neg_(rl[p][r]);
  }
  L.cfail[g * K + k] = bad ? f + 1 : INT_MAX;  // 1 + first point of the chunk
  // (measured: solving the separator system in each instance's last P1 CTA to
  // finish -- atomic arrival count, sep2_body with 8 separators per thread on
  // L2-hot records -- is slower than the separate kernel on the target:
  // P1 + tail 1111 us vs P1 595 + SEP 456 us; the latency-bound tail holds a
  // CTA slot ~5x longer than a chunk CTA and spills at P1's 128 registers)
}

// ============================================================== SEP =======
// Separator system of instance g, one thread per separator (K <= 256 threads;
// every thread of the CTA is separator k).
template <int B, class S, int NR>
__device__ __forceinline__ void sep1_body(const PipeL& L, int T, int32_t* info, int64_t g, int k, unsigned char* sm) {
  using BR = BRecN<B, NR>;
  const int K = L.K;
  S* rec = reinterpret_cast<S*>(sm);
  int* stime = reinterpret_cast<int*>(rec + size_t(BR::N) * K);
  int* sfail = stime + K;
  if (k == 0) sfail[0] = INT_MAX;
  stime[k] = sep_time(L, k, T);
  const S* in = reinterpret_cast<const S*>(L.sep1) + g * int64_t(PSep<B, NR>::N) * K;
  S D[B][B], Bl[B][B], Cr[B][B], r[NR][B];
  psep_ld<B, S, NR>(in, K, L.NT, k, D, r, Bl);  // own block + A_ll, r_l across a P1 CTA boundary
  if (k + 1 < K) {  // the coupling to sigma_{k+1}
    S Bn[B][B];
    psep_ld_b<B, S, NR>(in, K, k + 1, Bn);
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
      for (int q = 0; q < B; ++q) Cr[i][q] = Bn[q][i];
  } else {
    zero<B, S>(Cr);
  }
  const int cf = L.cfail[g * K + k];
  __syncthreads();
  if (cf != INT_MAX) atomicMin(sfail, cf);
  rbcr2n<B, S, NR>(rec, K, k, stime, sfail, D, Bl, Cr, r);
  S* y = reinterpret_cast<S*>(L.ysep) + g * int64_t(NR * B) * K + k;
#pragma unroll
  for (int i = 0; i < NR * B; ++i) y[int64_t(i) * K] = rec[k * BR::N + BR::Y + i];
  if (k == 0 && info) info[g] = (sfail[0] == INT_MAX) ? 0 : sfail[0];
}

template <int B, class S, int NR>
__global__ void __launch_bounds__(256, 2) pipe_sep_kernel(PipeL L, int T, int32_t* info) {  // K <= 256 (larger K: sep2)
  pdl_trigger();  // P2 may launch (and stage its inputs) while this grid drains
  pdl_wait();     // P1's records complete and visible
  sep1_body<B, S, NR>(L, T, info, blockIdx.x, int(threadIdx.x), smnn_dyn_smem);
}


// ========================================================== SEP, large K ===
// The separator system is itself block tridiagonal with explicit blocks
// (D_j = D_own_j + A_ll,j+1, r_j = R_own_j + r_l,j+1, coupling (j, j-1) = A_rl,j).
// For large K the partition method is applied to it once more: thread t owns
// m consecutive separators j0 = t m .. j0 + m - 1, block-Cholesky-eliminates
// the first m - 1 (with the spike towards super-separator t - 1, factors kept
// in registers), the K/m super-separators j0 + m - 1 are solved by rbcr2, and
// the owned separators are recovered by forward + back substitution.
// Local elimination of the m separators j0 .. j0 + m - 1 one thread owns
// (m <= MS): block Cholesky of the first m - 1 with the spike towards the
// previous super-separator (factors Lr and forward-substituted rhs wv kept),
// then the super-separator js = j0 + m - 1: its block minus the interior's
// Schur terms (Ds, Rs), its coupling to the previous super-separator (Bs) and
// the hand-over sums (All = sum X^T X, rl = sum X^T w; negated by the caller).
// Returns true on a pivot breakdown.  Shared by pipe_sep2_kernel (one level)
// and the hierarchical separator kernels (pipe_sepl_kernel / pipe_sepr_kernel).
template <int B, class S, int MS, int NR>
__device__ __forceinline__ bool sep_local(const S* in, int K, int NTin, int j0, int m, S (&Lr)[MS - 1][B][B],
                                          S (&Ds)[B][B], S (&Rs)[NR][B], S (&Bs)[B][B], S (&All)[B][B],
                                          S (&rl)[NR][B]) {
  const int js = j0 + m - 1;
  S Lc[B][B], wv[NR][B], X[B][B], Pl[B][B];
  zero<B, S>(Lc); zero<B, S>(X); zero<B, S>(All);
#pragma unroll
  for (int p = 0; p < NR; ++p) { zero<B, S>(wv[p]); zero<B, S>(rl[p]); }
  S sg = splat<S>(1.0);
#pragma unroll
  for (int i = 0; i < MS - 1; ++i) {
    S D[B][B], r[NR][B], Bl[B][B];
    psep_ld<B, S, NR>(in, K, NTin, j0 + min(i, max(m - 2, 0)), D, r, Bl);  // unconditional: loads run ahead
    if (i < m - 1) {
      if (i == 0) {  // Bl couples to the previous super-separator (zero for the first)
        lchol<B, S>(D, Lc);
#pragma unroll
        for (int p = 0; p < NR; ++p) llsolve<B, S>(Lc, r[p], wv[p]);
        lleft<B, S>(Lc, Bl, X);
#pragma unroll
        for (int a = 0; a < B; ++a) {
#pragma unroll
          for (int q = 0; q <= a; ++q) {
            S acc = mul_(X[0][a], X[0][q]);
#pragma unroll
            for (int mm = 1; mm < B; ++mm) acc = fma_(X[mm][a], X[mm][q], acc);
            All[a][q] = acc;
          }
#pragma unroll
          for (int p = 0; p < NR; ++p) {
            S acc = mul_(X[0][a], wv[p][0]);
#pragma unroll
            for (int mm = 1; mm < B; ++mm) acc = fma_(X[mm][a], wv[p][mm], acc);
            rl[p][a] = acc;
          }
        }
      } else {
        S Pm[B][B];  // P = Bl_j L_{j-1}^{-T}
#pragma unroll
        for (int a = 0; a < B; ++a) llsolve<B, S>(Lc, Bl[a], Pm[a]);
        lcouple<B, S>(Pm, wv[0], D, r[0]);
#pragma unroll
        for (int p = 1; p < NR; ++p) lcouple_v<B, S>(Pm, wv[p], r[p]);
        lchol<B, S>(D, Lc);
#pragma unroll
        for (int p = 0; p < NR; ++p) llsolve<B, S>(Lc, r[p], wv[p]);
        S Y[B][B];
#pragma unroll
        for (int a = 0; a < B; ++a)
#pragma unroll
          for (int q = 0; q < B; ++q) {
            S acc = mul_(Pm[a][0], X[0][q]);
#pragma unroll
            for (int mm = 1; mm < B; ++mm) acc = fma_(Pm[a][mm], X[mm][q], acc);
            Y[a][q] = acc;
          }
        lleft<B, S>(Lc, Y, X);
        sg = neg_(sg);
#pragma unroll
        for (int a = 0; a < B; ++a) {
#pragma unroll
          for (int q = 0; q <= a; ++q) {
            S acc = All[a][q];
#pragma unroll
            for (int mm = 0; mm < B; ++mm) acc = fma_(X[mm][a], X[mm][q], acc);
            All[a][q] = acc;
          }
#pragma unroll
          for (int p = 0; p < NR; ++p) {
            S acc = mul_(X[0][a], wv[p][0]);
#pragma unroll
            for (int mm = 1; mm < B; ++mm) acc = fma_(X[mm][a], wv[p][mm], acc);
            rl[p][a] = fma_(sg, acc, rl[p][a]);
          }
        }
      }
      rcopyL<B, S>(Lc, Lr[i]);
    }
  }
  // ---- the super-separator js: own block minus the interior's Schur terms
  S Bl[B][B];
  psep_ld<B, S, NR>(in, K, NTin, js, Ds, Rs, Bl);
  if (m > 1) {
#pragma unroll
    for (int a = 0; a < B; ++a) llsolve<B, S>(Lc, Bl[a], Pl[a]);
    lcouple<B, S>(Pl, wv[0], Ds, Rs[0]);
#pragma unroll
    for (int p = 1; p < NR; ++p) lcouple_v<B, S>(Pl, wv[p], Rs[p]);
#pragma unroll
    for (int a = 0; a < B; ++a)
#pragma unroll
      for (int q = 0; q < B; ++q) {
        S acc = mul_(Pl[a][0], X[0][q]);
#pragma unroll
        for (int mm = 1; mm < B; ++mm) acc = fma_(Pl[a][mm], X[mm][q], acc);
        Bs[a][q] = mul_(neg_(sg), acc);
      }
  } else {
#pragma unroll
    for (int a = 0; a < B; ++a)
#pragma unroll
      for (int q = 0; q < B; ++q) Bs[a][q] = Bl[a][q];
  }
  return m > 1 && bad_(splat<S>(1.0) / Lc[B - 1][B - 1]) != 0;
}

// Recovery of the owned separators j0 .. j0 + m - 2 from the factors Lr of
// sep_local and the solutions at the neighbouring super-separators (yL: the
// previous one, yR: own, js): forward substitution with yL, back substitution
// from yR.  Writes y of all m owned separators to yo ([NR B][Kout] field-major).
template <int B, class S, int MS, int NR>
__device__ __forceinline__ void sep_recover(const S* in, int K, int NTin, int j0, int m,
                                            const S (&Lr)[MS - 1][B][B], const S (&yL)[NR][B],
                                            const S (&yR)[NR][B], S* yo, int64_t Kout) {
  const int js = j0 + m - 1;
#pragma unroll
  for (int p = 0; p < NR; ++p)
#pragma unroll
    for (int a = 0; a < B; ++a) yo[int64_t(p * B + a) * Kout + js] = yR[p][a];
  S Wp[MS - 1][NR][B];
#pragma unroll
  for (int i = 0; i < MS - 1; ++i) {
    S r[NR][B], Bl[B][B];
    psep_ld_rb<B, S, NR>(in, K, NTin, j0 + min(i, max(m - 2, 0)), r, Bl);
    if (i < m - 1) {
#pragma unroll
      for (int p = 0; p < NR; ++p) {
        S tv[B], u[B];
        if (i == 0) {
#pragma unroll
          for (int a = 0; a < B; ++a) tv[a] = yL[p][a];
        } else {
          lltsolve<B, S>(Lr[i - 1], Wp[i - 1][p], tv);
        }
#pragma unroll
        for (int a = 0; a < B; ++a) {
          S acc = r[p][a];
#pragma unroll
          for (int q = 0; q < B; ++q) acc = fnma_(Bl[a][q], tv[q], acc);
          u[a] = acc;
        }
        llsolve<B, S>(Lr[i], u, Wp[i][p]);
      }
    }
  }
  S yn[NR][B];
#pragma unroll
  for (int p = 0; p < NR; ++p)
#pragma unroll
    for (int a = 0; a < B; ++a) yn[p][a] = yR[p][a];
#pragma unroll
  for (int i = MS - 2; i >= 0; --i) {
    S Bn[B][B];
    psep_ld_b<B, S, NR>(in, K, j0 + min(i, max(m - 2, 0)) + 1, Bn);  // coupling (j+1, j)
    if (i < m - 1) {
#pragma unroll
      for (int p = 0; p < NR; ++p) {
        S v[B], u[B], tv[B], yv[B];
#pragma unroll
        for (int a = 0; a < B; ++a) {
          S acc = mul_(Bn[0][a], yn[p][0]);
#pragma unroll
          for (int q = 1; q < B; ++q) acc = fma_(Bn[q][a], yn[p][q], acc);
          v[a] = acc;
        }
        llsolve<B, S>(Lr[i], v, u);
#pragma unroll
        for (int a = 0; a < B; ++a) tv[a] = sub_(Wp[i][p][a], u[a]);
        lltsolve<B, S>(Lr[i], tv, yv);
#pragma unroll
        for (int a = 0; a < B; ++a) yo[int64_t(p * B + a) * Kout + j0 + i] = yv[a];
#pragma unroll
        for (int a = 0; a < B; ++a) yn[p][a] = yv[a];
      }
    }
  }
}

// Separator system of instance g, m = K / nt separators per thread (nt threads,
// thread t): the body of pipe_sep2_kernel.
template <int B, class S, int MS, int NR>
__device__ __forceinline__ void sep2_body(const PipeL& L, int T, int32_t* info, int64_t g, int t, int nt,
                                          unsigned char* sm) {
  using BR = BRecN<B, NR>;
  const int K = L.K;
  const int m = K / nt;  // separators per thread (host: K = m * nt, m <= MS)
  S* rec = reinterpret_cast<S*>(sm);
  int* stime = reinterpret_cast<int*>(rec + size_t(BR::N) * nt);
  int* sfail = stime + nt;
  const int j0 = t * m, js = j0 + m - 1;
  if (t == 0) sfail[0] = INT_MAX;
  stime[t] = sep_time(L, js, T);
  const S* in = reinterpret_cast<const S*>(L.sep1) + g * int64_t(PSep<B, NR>::N) * K;
  int cf = INT_MAX;
  for (int j = j0; j <= js; ++j) cf = min(cf, L.cfail[g * K + j]);
  S Lr[MS - 1][B][B], Ds[B][B], Rs[NR][B], Bs[B][B], All[B][B], rl[NR][B];
  if (sep_local<B, S, MS, NR>(in, K, L.NT, j0, m, Lr, Ds, Rs, Bs, All, rl)) cf = min(cf, 1 + sep_time(L, j0, T));
  // hand-over (A_ll, r_l, coupling) to super-separator t - 1
  S* pk = rec + t * BR::N;
#pragma unroll
  for (int a = 0; a < B; ++a) {
#pragma unroll
    for (int p = 0; p < NR; ++p) rl[p][a] = neg_(rl[p][a]);
#pragma unroll
    for (int q = 0; q <= a; ++q) All[a][q] = neg_(All[a][q]);
  }
  rst_tri<B, S>(pk + BR::HA, All);
  rst_full<B, S>(pk + BR::HB, Bs);
#pragma unroll
  for (int p = 0; p < NR; ++p) rst_v<B, S>(pk + BR::HR + p * B, rl[p]);
  __syncthreads();
  S Cs[B][B];
  if (t + 1 < nt) {
    S Al[B][B], An[B][B];
    const S* pn = rec + (t + 1) * BR::N;
    rld_tri<B, S>(pn + BR::HA, Al);
    rld_full<B, S>(pn + BR::HB, An);
#pragma unroll
    for (int p = 0; p < NR; ++p) {
      S rr[B];
      rld_v<B, S>(pn + BR::HR + p * B, rr);
#pragma unroll
      for (int a = 0; a < B; ++a) Rs[p][a] = add_(Rs[p][a], rr[a]);
    }
#pragma unroll
    for (int a = 0; a < B; ++a) {
#pragma unroll
      for (int q = 0; q <= a; ++q) Ds[a][q] = add_(Ds[a][q], Al[a][q]);
#pragma unroll
      for (int q = 0; q < B; ++q) Cs[a][q] = An[q][a];
    }
  } else {
    zero<B, S>(Cs);
  }
  if (cf != INT_MAX) atomicMin(sfail, cf);
  __syncthreads();  // hand-over slots are reused by the reduction
  rbcr2n<B, S, NR>(rec, nt, t, stime, sfail, Ds, Bs, Cs, Rs);
  S yR[NR][B], yL[NR][B];
#pragma unroll
  for (int p = 0; p < NR; ++p) {
    rld_v<B, S>(rec + t * BR::N + BR::Y + p * B, yR[p]);
    if (t > 0) rld_v<B, S>(rec + (t - 1) * BR::N + BR::Y + p * B, yL[p]); else zero<B, S>(yL[p]);
  }
  S* yo = reinterpret_cast<S*>(L.ysep) + g * int64_t(NR * B) * K;
  {  // the local factors again for the recovery: not held in registers through the
     // reduction (measured: no spills at 128 registers, target fwd 1.62 -> 1.60 ms)
    S Lq[MS - 1][B][B], D2[B][B], R2[NR][B], B2[B][B], A2[B][B], r2[NR][B];
    sep_local<B, S, MS, NR>(in, K, L.NT, j0, m, Lq, D2, R2, B2, A2, r2);
    sep_recover<B, S, MS, NR>(in, K, L.NT, j0, m, Lq, yL, yR, yo, K);
  }
  if (t == 0 && info) info[g] = (sfail[0] == INT_MAX) ? 0 : sfail[0];
}

template <int B, class S, int MS, int NR>
__global__ void __launch_bounds__(256, sizeof(S) >= 8 ? SMNN_SEP2_MINB64 : SMNN_SEP2_MINB) pipe_sep2_kernel(PipeL L, int T, int32_t* info) {
  pdl_trigger();
  pdl_wait();
  sep2_body<B, S, MS, NR>(L, T, info, blockIdx.x, int(threadIdx.x), int(blockDim.x), smnn_dyn_smem);
}

// ================================================ hierarchical separators ==
// More separators than one CTA's reduction takes (K > 2048, horizons beyond
// ~2e4 points): the partition method applied level by level.  Level l holds
// K_l separator records in the PSep format (P1 writes level 0); SEPL turns
// them into K_l / 8 super-separator records of level l + 1 (8 separators per
// thread, 128 threads = 1024 separators per CTA, the A_ll / r_l hand-over
// through shared memory inside a CTA and through the record's AL / RL fields
// across CTAs, exactly as P1 does); the top level (<= 2048) is solved by
// pipe_sep2_kernel; SEPR recovers level l's y from level l + 1's (re-doing the
// local elimination for its factors).  Every level's system is the Schur
// complement of the one below: the result equals the one-level solve up to
// rounding (block Cholesky of a permuted system).
constexpr int kSepLM = 8, kSepLNT = 128;

template <int B, class S, int NR>
__global__ void __launch_bounds__(kSepLNT, 2) pipe_sepl_kernel(PipeL L, PipeL U, int T) {
  using Q = PSep<B, NR>;
  constexpr int LT = B * (B + 1) / 2, HN = LT + NR * B;
  __shared__ S ho[HN * kSepLNT];
  const int K = L.K, Ku = U.K;  // Ku = K / 8
  const int parts = K / (kSepLM * kSepLNT);
  const int64_t g = blockIdx.x / parts;
  const int c = int(blockIdx.x % parts), t = int(threadIdx.x);
  const int su = c * kSepLNT + t;  // this thread's super-separator (level l + 1)
  const int j0 = su * kSepLM;
  const S* in = reinterpret_cast<const S*>(L.sep1) + g * int64_t(Q::N) * K;
  int cf = INT_MAX;
  for (int j = j0; j < j0 + kSepLM; ++j) cf = min(cf, L.cfail[g * K + j]);
  S Lr[kSepLM - 1][B][B], Ds[B][B], Rs[NR][B], Bs[B][B], All[B][B], rl[NR][B];
  if (sep_local<B, S, kSepLM, NR>(in, K, L.NT, j0, kSepLM, Lr, Ds, Rs, Bs, All, rl)) cf = min(cf, 1 + sep_time(L, j0, T));
  int e = 0;
#pragma unroll
  for (int a = 0; a < B; ++a)
#pragma unroll
    for (int q = 0; q <= a; ++q) ho[(e++) * kSepLNT + t] = neg_(All[a][q]);
#pragma unroll
  for (int p = 0; p < NR; ++p)
#pragma unroll
    for (int a = 0; a < B; ++a) ho[(LT + p * B + a) * kSepLNT + t] = neg_(rl[p][a]);
  __syncthreads();
  if (t + 1 < kSepLNT) {
    e = 0;
#pragma unroll
    for (int a = 0; a < B; ++a)
#pragma unroll
      for (int q = 0; q <= a; ++q) Ds[a][q] = add_(Ds[a][q], ho[(e++) * kSepLNT + t + 1]);
#pragma unroll
    for (int p = 0; p < NR; ++p)
#pragma unroll
      for (int a = 0; a < B; ++a) Rs[p][a] = add_(Rs[p][a], ho[(LT + p * B + a) * kSepLNT + t + 1]);
  }
  S* o = reinterpret_cast<S*>(U.sep1) + g * int64_t(Q::N) * Ku + su;
  e = 0;
#pragma unroll
  for (int a = 0; a < B; ++a)
#pragma unroll
    for (int q = 0; q <= a; ++q) o[int64_t(Q::D + e++) * Ku] = Ds[a][q];
#pragma unroll
  for (int p = 0; p < NR; ++p)
#pragma unroll
    for (int a = 0; a < B; ++a) o[int64_t(Q::R + p * B + a) * Ku] = Rs[p][a];
#pragma unroll
  for (int a = 0; a < B; ++a)
#pragma unroll
    for (int q = 0; q < B; ++q) o[int64_t(Q::BL + a * B + q) * Ku] = Bs[a][q];
  if (t == 0 && su > 0) {  // the previous CTA's last super-separator adds these (psep_ld, NT = 128)
    e = 0;
#pragma unroll
    for (int a = 0; a < B; ++a)
#pragma unroll
      for (int q = 0; q <= a; ++q) o[int64_t(Q::AL + e++) * Ku] = neg_(All[a][q]);
#pragma unroll
    for (int p = 0; p < NR; ++p)
#pragma unroll
      for (int a = 0; a < B; ++a) o[int64_t(Q::RL + p * B + a) * Ku] = neg_(rl[p][a]);
  }
  U.cfail[g * Ku + su] = cf;
}

template <int B, class S, int NR>
__global__ void __launch_bounds__(kSepLNT, 2) pipe_sepr_kernel(PipeL L, PipeL U) {
  using Q = PSep<B, NR>;
  const int K = L.K, Ku = U.K;
  const int parts = K / (kSepLM * kSepLNT);
  const int64_t g = blockIdx.x / parts;
  const int c = int(blockIdx.x % parts), t = int(threadIdx.x);
  const int su = c * kSepLNT + t;
  const int j0 = su * kSepLM;
  const S* in = reinterpret_cast<const S*>(L.sep1) + g * int64_t(Q::N) * K;
  S Lr[kSepLM - 1][B][B], Ds[B][B], Rs[NR][B], Bs[B][B], All[B][B], rl[NR][B];
  sep_local<B, S, kSepLM, NR>(in, K, L.NT, j0, kSepLM, Lr, Ds, Rs, Bs, All, rl);  // factors only
  const S* yu = reinterpret_cast<const S*>(U.ysep) + g * int64_t(NR * B) * Ku;
  S yL[NR][B], yR[NR][B];
#pragma unroll
  for (int p = 0; p < NR; ++p)
#pragma unroll
    for (int a = 0; a < B; ++a) {
      yR[p][a] = yu[int64_t(p * B + a) * Ku + su];
      yL[p][a] = su > 0 ? yu[int64_t(p * B + a) * Ku + su - 1] : splat<S>(0.0);
    }
  S* yo = reinterpret_cast<S*>(L.ysep) + g * int64_t(NR * B) * K;
  sep_recover<B, S, kSepLM, NR>(in, K, L.NT, j0, kSepLM, Lr, yL, yR, yo, K);
}


// ============================================================== P2 ========
template <int B, class Tio, class S, bool BWD, int CM, int NR>
__global__ void __launch_bounds__(SMNN_PIPE_NT, sizeof(S) >= 8 ? (BWD ? (NR == 2 ? SMNN_PIPE_P2_MINB64R : SMNN_PIPE_P2_MINB64)
                                                                        : SMNN_PIPE_P2_MINB64F)
                                                                 : (BWD ? SMNN_PIPE_P2_MINB : SMNN_PIPE_P2_MINB + 1))
    pipe_p2_kernel(Args<Tio> a, PipeL L) {  // forward: 5 CTAs/SM (measured +4 %), backward: 4 (spills at 5)
  unsigned char* sm = smnn_dyn_smem;
  Tio* smT = reinterpret_cast<Tio*>(sm);
  const int T = a.T, K = L.K, tid = threadIdx.x;
  const PRange R(L, T);
  const int64_t g = R.g;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.off_bar);
  const Wts<S> w{opaque(splat<S>(a.wg2)), opaque(splat<S>(a.wi2)), opaque(splat<S>(a.ws2))};
  const int64_t tb = g * int64_t(T) * B, t1b = g * int64_t(T), tsb = g * int64_t(T - 1);
  const int ylo = R.slo;  // BWD (NR = 1): y_fwd from max(ta - 1, 0)
  constexpr bool YIN = BWD && NR == 1;  // NR = 2 re-solves y instead of reading it
  const Span<Tio> pc(a.coeffs + tb + R.ta * B, (R.tb - R.ta) * B);
  const Span<Tio> pd(a.rhs + t1b + R.ta, R.tb - R.ta);
  const Span<Tio> ps(a.steps + tsb + R.slo, R.shi - R.slo);
  const Span<Tio> pg(BWD ? a.grad_y + tb + R.ta * B : a.coeffs, BWD ? (R.tb - R.ta) * B : 0);
  const Span<Tio> py(YIN ? a.y_in + tb + ylo * B : a.coeffs, YIN ? (R.tb - ylo) * B : 0);
  // SMNN_F32_C64 y remainder: staged in (backward) or stored out (forward) through its own region
  constexpr bool C64 = sizeof(S) > sizeof(Tio);
  const bool yl_in = C64 && YIN && a.y_lo_in && L.off_yl, yl_out = C64 && !BWD && a.y_lo_out && L.off_yl;
  const Span<Tio> pyl(yl_in ? a.y_lo_in + tb + ylo * B : a.coeffs, yl_in ? (R.tb - ylo) * B : 0);
  const Span<Tio> pyo(yl_out ? a.y_lo_out + tb + R.ta * B : a.coeffs, yl_out ? (R.tb - R.ta) * B : 0);
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_expect_tx(bar, pc.bytes + pd.bytes + ps.bytes + pg.bytes + py.bytes + pyl.bytes);
    bulk_g2s(sm + L.off_c, pc.lo, pc.bytes, bar);
    bulk_g2s(sm + L.off_d, pd.lo, pd.bytes, bar);
    if (ps.bytes) bulk_g2s(sm + L.off_s, ps.lo, ps.bytes, bar);
    if (BWD) bulk_g2s(sm + L.off_g, pg.lo, pg.bytes, bar);
    if (YIN) bulk_g2s(sm + L.off_y, py.lo, py.bytes, bar);
    if (pyl.bytes) bulk_g2s(sm + L.off_yl, pyl.lo, pyl.bytes, bar);
  }
  constexpr int E = int(sizeof(Tio));
  const int k = R.c0 + tid;
  const bool act = tid < R.nc;
  const int f = act ? chunk_begin(k, T, K) : R.ta;
  const int sig = act ? chunk_begin(k + 1, T, K) - 1 : R.ta + 1;
  const int nint = sig - f;
  // element offsets of the staged streams, relative to global time index 0
  const int oc = L.off_c / E + pc.pre - R.ta * B, od = L.off_d / E + pd.pre - R.ta;
  const int os = L.off_s / E + ps.pre - R.slo;
  const int og = BWD ? L.off_g / E + pg.pre - R.ta * B : 0, oy = YIN ? L.off_y / E + py.pre - ylo * B : 0;
  Grp<Tio, 1> x;
  x.T = T; x.n_iv = a.n_iv; x.nv = 1;
  x.c.o[0] = oc; x.d.o[0] = od; x.s.o[0] = os; x.gy.o[0] = og; x.yin.o[0] = oy;
  x.yout.o[0] = oc; x.gc.o[0] = oc; x.gd.o[0] = od; x.gs.o[0] = os;
  x.u[0] = a.iv + g * a.n_iv;
  x.gu[0] = (BWD && a.g_iv) ? a.g_iv + g * a.n_iv : nullptr;
  const int oyl = yl_in ? L.off_yl / E + pyl.pre - ylo * B : L.off_yl / E + pyo.pre - R.ta * B;
  x.ylo_out = yl_out;
  x.ylo_in = yl_in;
  x.ylo_off = oyl;
  x.c.on = x.d.on = x.s.on = true;
  x.gy.on = BWD;
  x.yin.on = YIN;
  x.yout.on = !BWD;
  x.gc.on = BWD && a.g_coeffs;
  x.gd.on = BWD && a.g_rhs;
  x.gs.on = BWD && a.g_steps;
  x.gu_on = BWD && a.g_iv;
  const Tio* cS = smT + opaque(oc + f * B);
  const Tio* dS = smT + opaque(od + f);
  const Tio* sS = smT + opaque(os + f);
  const Tio* gS = smT + opaque(og + f * B);
  S yL[NR][B], yR[NR][B];
  pdl_wait();  // the inputs are being staged; the separator solution (and P1's state) must be complete
  if (act) {
    const S* ys = reinterpret_cast<const S*>(L.ysep) + g * int64_t(NR * B) * K + k;
#pragma unroll
    for (int p = 0; p < NR; ++p) {
#pragma unroll
      for (int i = 0; i < B; ++i) yR[p][i] = ys[int64_t(p * B + i) * K];
      if (k > 0) {
#pragma unroll
        for (int i = 0; i < B; ++i) yL[p][i] = ys[int64_t(p * B + i) * K - 1];
      } else {
        zero<B, S>(yL[p]);
      }
    }
  }
  __syncthreads();  // barrier initialised
  mbar_wait(bar, 0);

  const S* seg = L.seg ? reinterpret_cast<const S*>(L.seg) + g * int64_t(PSegState<B, NR>::N) * K + k : nullptr;
  if (act) p2_chunk<B, Tio, S, BWD, CM, NR>(x, w, k, f, sig, nint, cS, dS, sS, gS, yL, yR, seg, K);
  // ---- outputs: TMA bulk store of the aligned body, plain stores at the ends
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int nt = blockDim.x;
  if (!BWD) {
    rf_store_out(a.y_out + tb + R.ta * B, smT + oc + R.ta * B, (R.tb - R.ta) * B, tid, nt);
    if (yl_out) rf_store_out(a.y_lo_out + tb + R.ta * B, smT + oyl + R.ta * B, (R.tb - R.ta) * B, tid, nt);
  } else {
    if (a.g_coeffs) rf_store_out(a.g_coeffs + tb + R.ta * B, smT + oc + R.ta * B, (R.tb - R.ta) * B, tid, nt);
    if (a.g_rhs) rf_store_out(a.g_rhs + t1b + R.ta, smT + od + R.ta, R.tb - R.ta, tid, nt);
    if (a.g_steps && R.tb - 1 > R.slo)  // this CTA owns intervals [slo, tb - 1)
      rf_store_out(a.g_steps + tsb + R.slo, smT + os + R.slo, R.tb - 1 - R.slo, tid, nt);
  }
  if (tid == 0) {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

}  // namespace smnn
