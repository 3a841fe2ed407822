// smnn_pipe.cu -- host side of the three-kernel pipeline (smnn_pipe.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <map>
#include <cstdlib>
#include <mutex>
#include <string>

#include "smnn.h"
#include "smnn_pipe.cuh"
#include "smnn_rf_host.h"

namespace smnn {
namespace {

size_t al16(size_t x) { return (x + 15) & ~size_t(15); }
size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// fp64 separator systems of SMNN_SEP2_SMALL..256 separators: sep2 with 4 per
// thread (K / 4 threads) instead of one thread per separator -- measured on the
// f32c64 pipeline at 4e7 instance-steps: T = 1000 8.98e9 -> 1.05e10, T = 1461
// 7.88e9 -> 9.02e9, T = 2000 8.19e9 -> 1.04e10 instance-steps/s (from K = 32,
// T = 300: 9.98e9 -> 9.0e9, so not below 64)
#ifndef SMNN_SEP2_SMALL
#define SMNN_SEP2_SMALL 64
#endif
#ifndef SMNN_SEP2_SMALL_M  // separators per thread there (measured 2 and 8: slower at T = 1000..2000)
#define SMNN_SEP2_SMALL_M 4
#endif
// fp64 separator kernel: 8 separators per thread (K/8 threads per instance,
// up to 4 instances per SM at the same 128 registers) from this K on (off:
// measured slower at K = 1024)
// programmatic dependent launch of the separator and P2 kernels (P1 stays a full
// stream barrier: it stages caller inputs that earlier kernels may have written).
// Measured: +0.3..0.6 % at 4e7 instance-steps, +3..4.5 % at the Lorenz / SST sizes
#ifndef SMNN_PIPE_PDL
#define SMNN_PIPE_PDL 1
#endif
#ifndef SMNN_PIPE_M8_64
#define SMNN_PIPE_M8_64 (1 << 30)
#endif

template <int B>
size_t nr_sep_fields(int nr) { return nr == 2 ? size_t(PSep<B, 2>::N) : size_t(PSep<B, 1>::N); }

constexpr int kMaxLevels = 3;  // separator hierarchy: up to 2048 * 8^3 level-0 separators

struct PipePlan {
  bool ok = false;
  int K = 0, NT = 0, parts = 0, CM = 0;
  bool sep2 = false;  // separator kernel: pipe_sep2_kernel (K/m2 threads, m2 separators each)
  int m2 = 4;
  size_t smem_p1 = 0, smem_p2 = 0, smem_sep = 0;
  size_t ws_sep1 = 0, ws_ysep = 0, ws_fail = 0;  // level 0
  PipeL L1{}, L2{};
  // hierarchical separators (K > 2048): levels 1..levels, K_l = K / 8^l, the
  // top level solved by the separator kernel
  int levels = 0;
  int Kl[kMaxLevels + 1] = {};
  size_t off_rec[kMaxLevels + 1] = {}, off_y[kMaxLevels + 1] = {}, off_fail[kMaxLevels + 1] = {};
  size_t off_seg = 0, ws_seg = 0;  // P1 -> P2 state of two-segment chunks (level 0; 0 bytes: none)
  size_t ws_total = 0;
};

// Right-hand sides of a pipeline call: 2 in the SMNN_F32_C64 backward (dl/dy and
// beta: y is re-solved in fp64 beside lambda; see include/smnn.h smnn_solve_bwd).
// With the forward's fp32 remainder of y (ylo: Args::y_lo_in) the backward reads
// y_hi + y_lo and needs one right-hand side.
int pipe_nr(const smnn_problem* p, bool bwd, bool ylo) {
  return (bwd && p->dtype == SMNN_F32_C64 && !ylo) ? 2 : 1;
}

template <int B, class S>
PipePlan plan_B(const smnn_problem* p, size_t es, bool bwd, bool ylo) {
  PipePlan q;
  const int nr = pipe_nr(p, bwd, ylo);
  const bool c64 = sizeof(S) > es;
  constexpr int CM = PipeCM<B, S>::value;
  const int T = p->T;
  if (p->threads_per_inst != 0 || T < 4) return q;
  // chunks: a multiple of 32 (no idle lanes in the chunk kernels), each of
  // 2..CM points (chunk_begin spreads the remainder)
  int K = std::min(((T + CM - 1) / CM + 31) / 32 * 32, T / 2);
  if (K > 256) {  // large K: sep2 with 4 (K <= 1024) or 8 separators per thread, K / m <= 256 threads
    const int q128 = K > 1024 ? 256 : 128;
    K = std::min((K + q128 - 1) / q128 * q128, T / 2);
  }
  int levels = 0, Ktop = K;
  // (measured: a forced hierarchy level at K = 1024 -- SEPL + a 128-separator top
  // solve + SEPR instead of sep2 -- is slower on the target, fwd 1.86 vs 1.71 ms)
  if (K > SMNN_PIPE_SEP_MAX) {  // separator hierarchy: 8 separators per thread and level
    const int64_t kmin = (int64_t(T) + CM - 1) / CM;
    for (levels = 1; levels <= kMaxLevels; ++levels) {
      int64_t f = 1;
      for (int l = 0; l < levels; ++l) f *= kSepLM;
      const int64_t unit = f * 256;  // top level: a multiple of 256 separators (sep2 divisibility)
      const int64_t K0 = (kmin + unit - 1) / unit * unit;
      if (K0 / f <= SMNN_PIPE_SEP_MAX) {
        K = K0 <= T / 2 && K0 < (int64_t(1) << 30) ? int(K0) : 0;
        Ktop = int(K0 / f);
        break;
      }
    }
    if (levels > kMaxLevels || K == 0) return q;
  }
  if (K < 1 || Ktop > SMNN_PIPE_SEP_MAX || (T + K - 1) / K > CM) return q;
  q.levels = levels;
  for (int l = 0, k = K; l <= levels; ++l, k /= kSepLM) q.Kl[l] = k;
  q.sep2 = Ktop > 256 && Ktop % 128 == 0;
  if (q.sep2) {  // separators per thread: 4, or 8 when K/4 would exceed 256 threads
    q.m2 = (Ktop / 4 > 256 || (sizeof(S) >= 8 && Ktop >= SMNN_PIPE_M8_64)) ? 8 : 4;
    if (Ktop % (32 * q.m2) != 0 || Ktop / q.m2 > 256) q.sep2 = false;
  } else if (sizeof(S) >= 8 && Ktop >= SMNN_SEP2_SMALL && Ktop % SMNN_SEP2_SMALL_M == 0) {
    q.sep2 = true;  // small K, fp64: 4 separators per thread, K / 4 threads (Lorenz, SST shapes)
    q.m2 = SMNN_SEP2_SMALL_M;
  }
  if (Ktop > 256 && !q.sep2) return q;
  const size_t ls = sizeof(S);
  q.K = K;
  q.CM = CM;
  {  // chunk-kernel CTAs of equal size (K = 160: 2 x 96 instead of 128 + 32)
    const int parts = (K + SMNN_PIPE_NT - 1) / SMNN_PIPE_NT;
    q.NT = std::min(SMNN_PIPE_NT, ((K + parts - 1) / parts + 31) / 32 * 32);
  }
  int steps = 0;
  auto layout = [&](PipeL& L, bool p2) {
    size_t off = 0;
    auto take = [&](size_t bytes) { const size_t o = off; off = al16(off + bytes); return int(o); };
    L.off_c = take(size_t(steps) * B * es + 32);
    L.off_d = (p2 || !bwd || nr == 2) ? take(size_t(steps) * es + 32) : 0;
    L.off_s = take(size_t(steps) * es + 32);
    L.off_g = bwd ? take(size_t(steps) * B * es + 32) : 0;
    L.off_y = (bwd && p2 && nr == 1) ? take(size_t(steps) * B * es + 32) : 0;
    // SMNN_F32_C64: y's fp32 remainder, forward out / backward (one right-hand side) in
    L.off_yl = (c64 && p2 && (!bwd || nr == 1)) ? take(size_t(steps) * B * es + 32) : 0;
    L.off_h = p2 ? 0 : take(size_t(PSep<B>::LT + nr * B) * SMNN_PIPE_NT * ls);
    L.off_bar = take(16);
    return off;
  };
  // chunk-kernel CTA: 128 chunks, fewer when its staged range would exceed
  // 75 KB (fp64 storage with long chunks: keep >= 3 CTAs per SM; measured
  // 1 CTA/SM and 5x slower at order 1, T = 1e4, f64 before; 3 x 75 KB fit)
  for (;;) {
    steps = q.NT * CM + 2;  // points of one CTA range (+ s_{ta-1}, y_{ta-1})
    q.smem_p1 = layout(q.L1, false);
    q.smem_p2 = layout(q.L2, true);
    if (q.NT <= 32 || std::max(q.smem_p1, q.smem_p2) <= 75 * 1024) break;
    q.NT /= 2;
  }
  q.parts = (K + q.NT - 1) / q.NT;
  const size_t recn = nr == 2 ? size_t(BRecN<B, 2>::N) : size_t(BRecN<B, 1>::N);
  q.smem_sep = recn * (q.sep2 ? Ktop / q.m2 : Ktop) * ls + size_t(2 * Ktop + 4) * 4;
  if (q.smem_p1 > 200 * 1024 || q.smem_p2 > 200 * 1024 || q.smem_sep > 220 * 1024) return q;
  const size_t nrec = nr == 2 ? PSep<B, 2>::N : PSep<B, 1>::N;
  size_t off = 0;
  for (int l = 0; l <= levels; ++l) {  // per level: records, y at the separators, failure flags
    q.off_rec[l] = off;
    off += al256(size_t(p->n_inst) * nrec * q.Kl[l] * ls);
    q.off_y[l] = off;
    off += al256(size_t(p->n_inst) * nr * B * q.Kl[l] * ls);
    q.off_fail[l] = off;
    off += al256(size_t(p->n_inst) * q.Kl[l] * 4);
  }
  if (CM - 1 > PipeHM<B, S>::value) {  // chunks P2 handles in two segments: P1 stores their state
    q.off_seg = off;
    q.ws_seg = al256(size_t(p->n_inst) * size_t(nr == 2 ? PSegState<B, 2>::N : PSegState<B, 1>::N) * K * ls);
    off += q.ws_seg;
  }
  q.ws_total = off;
  q.ws_sep1 = q.off_y[0];
  q.ws_ysep = q.off_fail[0] - q.off_y[0];
  q.ws_fail = (levels > 0 ? q.off_rec[1] : off) - q.off_fail[0];
  for (PipeL* L : {&q.L1, &q.L2}) {
    L->K = K;
    L->K0 = K;
    L->sstride = 1;
    L->NT = q.NT;
    L->parts = q.parts;
  }
  q.ok = true;
  return q;
}

template <class S>
PipePlan plan_S(const smnn_problem* p, size_t es, bool bwd, bool ylo) {
  switch (p->order) {
    case 0: return plan_B<1, S>(p, es, bwd, ylo);
    case 1: return plan_B<2, S>(p, es, bwd, ylo);
    case 2: return plan_B<3, S>(p, es, bwd, ylo);
    default: return plan_B<4, S>(p, es, bwd, ylo);
  }
}

PipePlan plan_of(const smnn_problem* p, bool bwd, bool ylo = false) {
  if (p->dtype == SMNN_F32) return plan_S<float>(p, 4, bwd, false);
  return plan_S<double>(p, p->dtype == SMNN_F64 ? 8 : 4, bwd, ylo && p->dtype == SMNN_F32_C64);
}

template <int B, class Tio, class S, bool BWD, int NR>
int launch_B(const smnn_problem* p, const Args<Tio>& a, cudaStream_t st, std::string& err) {
  constexpr int CM = PipeCM<B, S>::value;
  PipePlan q = plan_B<B, S>(p, sizeof(Tio), BWD, BWD && NR == 1 && sizeof(S) > sizeof(Tio));
  if (!q.ok) return 0;
  auto k1 = pipe_p1_kernel<B, Tio, S, BWD, CM, NR>;
  auto k2 = pipe_sep_kernel<B, S, NR>;
  auto k2b = q.m2 > 4 ? pipe_sep2_kernel<B, S, 8, NR> : pipe_sep2_kernel<B, S, 4, NR>;
  auto k3 = pipe_p2_kernel<B, Tio, S, BWD, CM, NR>;
  for (auto [kp, sm] : {std::make_pair(reinterpret_cast<const void*>(k1), q.smem_p1),
                         std::make_pair(reinterpret_cast<const void*>(k3), q.smem_p2),
                         std::make_pair(q.sep2 ? reinterpret_cast<const void*>(k2b) : reinterpret_cast<const void*>(k2),
                                        q.smem_sep)})
    if (const cudaError_t ea = ensure_smem(kp, sm); ea != cudaSuccess) {
      err = std::string("pipeline shared-memory attribute: ") + cudaGetErrorString(ea);
      cudaGetLastError();
      return SMNN_ERR_CUDA;
    }
  const int64_t n = p->n_inst;
  if (n <= 0) return 1;
  const int T = p->T, K = q.K;
  char* ws = static_cast<char*>(a.ckpt);
  auto level = [&](int l) {  // PipeL of separator level l (l = 0: the chunk kernels' view)
    PipeL L = q.L1;
    L.K = q.Kl[l];
    L.K0 = K;
    int st = 1;
    for (int i = 0; i < l; ++i) st *= kSepLM;
    L.sstride = st;
    L.NT = l == 0 ? q.NT : kSepLNT;  // CTA size of the kernel that wrote the level's records
    L.sep1 = ws + q.off_rec[l];
    L.ysep = ws + q.off_y[l];
    L.cfail = reinterpret_cast<int*>(ws + q.off_fail[l]);
    L.seg = (l == 0 && q.ws_seg) ? ws + q.off_seg : nullptr;
    return L;
  };
  auto chain = [&](cudaStream_t s) {
    PipeL L1 = level(0), L2 = level(0);
    L2.off_c = q.L2.off_c; L2.off_d = q.L2.off_d; L2.off_s = q.L2.off_s; L2.off_g = q.L2.off_g;
    L2.off_y = q.L2.off_y; L2.off_h = q.L2.off_h; L2.off_bar = q.L2.off_bar; L2.off_yl = q.L2.off_yl;
    k1<<<unsigned(n * q.parts), q.NT, q.smem_p1, s>>>(a, L1);
    for (int l = 0; l < q.levels; ++l)
      pipe_sepl_kernel<B, S, NR><<<unsigned(n * (q.Kl[l] / (kSepLM * kSepLNT))), kSepLNT, 0, s>>>(level(l), level(l + 1),
                                                                                                    T);
    const PipeL Lt = level(q.levels);
    // separator and P2 kernels: programmatic dependent launch (they wait for their
    // predecessor on the device: pdl_wait in smnn_pipe.cuh)
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = SMNN_PIPE_PDL;
    auto cfg = [&](unsigned grid, unsigned block, size_t smem) {
      cudaLaunchConfig_t c = {};
      c.gridDim = dim3(grid);
      c.blockDim = dim3(block);
      c.dynamicSmemBytes = smem;
      c.stream = s;
      c.attrs = pdl;
      c.numAttrs = 1;
      return c;
    };
    if (q.sep2) {
      const cudaLaunchConfig_t c = cfg(unsigned(n), unsigned(Lt.K / q.m2), q.smem_sep);
      cudaLaunchKernelEx(&c, k2b, Lt, T, a.info);
    } else {
      const cudaLaunchConfig_t c = cfg(unsigned(n), unsigned(Lt.K), q.smem_sep);
      cudaLaunchKernelEx(&c, k2, Lt, T, a.info);
    }
    for (int l = q.levels - 1; l >= 0; --l)
      pipe_sepr_kernel<B, S, NR><<<unsigned(n * (q.Kl[l] / (kSepLM * kSepLNT))), kSepLNT, 0, s>>>(level(l), level(l + 1));
    {
      const cudaLaunchConfig_t c = cfg(unsigned(n * q.parts), unsigned(q.NT), q.smem_p2);
      cudaLaunchKernelEx(&c, k3, a, L2);
    }
  };
  // (measured: splitting the instances into 2 groups on separate streams, so
  // one group's separator kernel overlaps the other's chunk kernels, gave no
  // gain on the f32c64 target -- 2.80 vs 2.68 ms backward)
  chain(st);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    err = std::string("pipeline launch: ") + cudaGetErrorString(e);
    return SMNN_ERR_CUDA;
  }
  return 1;
}

template <class Tio, class S, bool BWD, int NR>
int launch_order_nr(const smnn_problem* p, const Args<Tio>& a, cudaStream_t st, std::string& err) {
  switch (p->order) {
    case 0: return launch_B<1, Tio, S, BWD, NR>(p, a, st, err);
    case 1: return launch_B<2, Tio, S, BWD, NR>(p, a, st, err);
    case 2: return launch_B<3, Tio, S, BWD, NR>(p, a, st, err);
    default: return launch_B<4, Tio, S, BWD, NR>(p, a, st, err);
  }
}

template <class Tio, class S, bool BWD>
int launch_order(const smnn_problem* p, const Args<Tio>& a, cudaStream_t st, std::string& err) {
  if constexpr (BWD && sizeof(S) > sizeof(Tio)) {  // SMNN_F32_C64 backward: y_hi + y_lo read, or re-solved
    if (a.y_lo_in) return launch_order_nr<Tio, S, BWD, 1>(p, a, st, err);
    return launch_order_nr<Tio, S, BWD, 2>(p, a, st, err);
  } else {
    return launch_order_nr<Tio, S, BWD, 1>(p, a, st, err);
  }
}

}  // namespace

bool pipe_eligible(const smnn_problem* p, bool bwd) { return plan_of(p, bwd).ok; }

bool pipe_ylo_eligible(const smnn_problem* p) {
  if (p->dtype != SMNN_F32_C64) return false;
  const PipePlan f = plan_of(p, false), b = plan_of(p, true), r = plan_of(p, true, true);
  return f.ok && r.ok && b.ok && r.NT == b.NT;  // not where staging y_lo would shrink the CTAs
}

int pipe_launches(const smnn_problem* p, bool bwd) {
  const PipePlan q = plan_of(p, bwd);
  return q.ok ? 3 + 2 * q.levels : 0;
}

size_t pipe_workspace_bytes(const smnn_problem* p) {
  const PipePlan f = plan_of(p, false), b = plan_of(p, true);
  size_t n = 0;
  if (f.ok) n = std::max(n, f.ws_total);
  if (b.ok) n = std::max(n, b.ws_total);
  if (const PipePlan r = plan_of(p, true, true); r.ok) n = std::max(n, r.ws_total);
  return n;
}

template <class Tio, class Tc>
int pipe_launch(const smnn_problem* p, const Args<Tio>& a, bool bwd, cudaStream_t st, std::string& err) {
  return bwd ? launch_order<Tio, Tc, true>(p, a, st, err) : launch_order<Tio, Tc, false>(p, a, st, err);
}

template int pipe_launch<float, float>(const smnn_problem*, const Args<float>&, bool, cudaStream_t, std::string&);
template int pipe_launch<float, double>(const smnn_problem*, const Args<float>&, bool, cudaStream_t, std::string&);
template int pipe_launch<double, double>(const smnn_problem*, const Args<double>&, bool, cudaStream_t,
                                         std::string&);

}  // namespace smnn
