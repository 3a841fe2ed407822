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

struct PipePlan {
  bool ok = false;
  int K = 0, NT = 0, parts = 0, CM = 0;
  bool sep2 = false;  // separator kernel: pipe_sep2_kernel (K/m2 threads, m2 separators each)
  int m2 = 4;
  size_t smem_p1 = 0, smem_p2 = 0, smem_sep = 0;
  size_t ws_sep1 = 0, ws_ysep = 0, ws_fail = 0;
  PipeL L1{}, L2{};
};

template <int B, class S>
PipePlan plan_B(const smnn_problem* p, size_t es, bool bwd) {
  PipePlan q;
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
  if (K < 1 || K > SMNN_PIPE_SEP_MAX || (T + K - 1) / K > CM) return q;
  q.sep2 = K > 256 && K % 128 == 0;
  if (q.sep2) {  // separators per thread: 4, or 8 when K/4 would exceed 256 threads
    const char* e = std::getenv("SMNN_PIPE_M");
    q.m2 = e ? (std::atoi(e) > 4 ? 8 : 4) : (K / 4 > 256 ? 8 : 4);
    if (K % (32 * q.m2) != 0 || K / q.m2 > 256) q.sep2 = false;
  }
  if (K > 256 && !q.sep2) return q;
  const size_t ls = sizeof(S);
  q.K = K;
  q.CM = CM;
  q.NT = std::min(SMNN_PIPE_NT, ((K + 31) / 32) * 32);
  int steps = 0;
  auto layout = [&](PipeL& L, bool p2) {
    size_t off = 0;
    auto take = [&](size_t bytes) { const size_t o = off; off = al16(off + bytes); return int(o); };
    L.off_c = take(size_t(steps) * B * es + 32);
    L.off_d = (p2 || !bwd) ? take(size_t(steps) * es + 32) : 0;
    L.off_s = take(size_t(steps) * es + 32);
    L.off_g = bwd ? take(size_t(steps) * B * es + 32) : 0;
    L.off_y = (bwd && p2) ? take(size_t(steps) * B * es + 32) : 0;
    L.off_h = p2 ? 0 : take(size_t(PSep<B>::LT + B) * SMNN_PIPE_NT * ls);
    L.off_bar = take(16);
    return off;
  };
  // chunk-kernel CTA: 128 chunks, fewer when its staged range would exceed
  // 64 KB (fp64 storage with long chunks: keep >= 3 CTAs per SM; measured
  // 1 CTA/SM and 5x slower at order 1, T = 1e4, f64 before)
  for (;;) {
    steps = q.NT * CM + 2;  // points of one CTA range (+ s_{ta-1}, y_{ta-1})
    q.smem_p1 = layout(q.L1, false);
    q.smem_p2 = layout(q.L2, true);
    if (q.NT <= 32 || std::max(q.smem_p1, q.smem_p2) <= 64 * 1024) break;
    q.NT /= 2;
  }
  q.parts = (K + q.NT - 1) / q.NT;
  q.smem_sep = size_t(BRec<B>::N) * (q.sep2 ? K / q.m2 : K) * ls + size_t(2 * K + 4) * 4;
  if (q.smem_p1 > 200 * 1024 || q.smem_p2 > 200 * 1024 || q.smem_sep > 220 * 1024) return q;
  q.ws_sep1 = al256(size_t(p->n_inst) * PSep<B>::N * K * ls);
  q.ws_ysep = al256(size_t(p->n_inst) * B * K * ls);
  q.ws_fail = al256(size_t(p->n_inst) * K * 4);
  for (PipeL* L : {&q.L1, &q.L2}) {
    L->K = K;
    L->NT = q.NT;
    L->parts = q.parts;
    const char* e = std::getenv("SMNN_PIPE_SEPMAP");
    L->sepmap = e ? std::atoi(e) : 0;
  }
  q.ok = true;
  return q;
}

template <class S>
PipePlan plan_S(const smnn_problem* p, size_t es, bool bwd) {
  switch (p->order) {
    case 0: return plan_B<1, S>(p, es, bwd);
    case 1: return plan_B<2, S>(p, es, bwd);
    case 2: return plan_B<3, S>(p, es, bwd);
    default: return plan_B<4, S>(p, es, bwd);
  }
}

PipePlan plan_of(const smnn_problem* p, bool bwd) {
  if (p->dtype == SMNN_F32) return plan_S<float>(p, 4, bwd);
  return plan_S<double>(p, p->dtype == SMNN_F64 ? 8 : 4, bwd);
}

// The dynamic shared-memory attribute must cover the largest request made so
// far for each kernel (keyed by the kernel's address: instantiations share a type).
template <class Kern>
void set_smem(Kern k, size_t smem) {
  static std::mutex mu;
  static std::map<const void*, size_t> top;
  std::lock_guard<std::mutex> lk(mu);
  size_t& t = top[reinterpret_cast<const void*>(k)];
  if (smem > t) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    t = smem;
  }
}

// Fork-join streams of the pipeline: the batch is split into groups whose
// P1 -> SEP -> P2 chains run on different streams, so the latency-bound
// separator kernel of one group overlaps the throughput-bound chunk kernels of
// another.  One pool per device, created on first use.
struct ForkJoin {
  static constexpr int kMax = 4;
  cudaStream_t s[kMax] = {};
  cudaEvent_t fork = nullptr, join[kMax] = {};
};

ForkJoin* fork_join() {
  static std::mutex mu;
  static ForkJoin pools[64];
  static bool made[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  ForkJoin& f = pools[dev];
  if (!made[dev]) {
    for (int i = 0; i < ForkJoin::kMax; ++i) {
      if (cudaStreamCreateWithFlags(&f.s[i], cudaStreamNonBlocking) != cudaSuccess) return nullptr;
      if (cudaEventCreateWithFlags(&f.join[i], cudaEventDisableTiming) != cudaSuccess) return nullptr;
    }
    if (cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    made[dev] = true;
  }
  return &f;
}

int pipe_groups(int64_t n_inst) {
  const char* e = std::getenv("SMNN_PIPE_STREAMS");
  const int want = e ? std::max(1, std::min(ForkJoin::kMax, std::atoi(e))) : 1;  // measured: no gain on B200
  return int(std::max<int64_t>(1, std::min<int64_t>(want, n_inst / 512)));  // >= 512 instances per group
}

template <int B, class Tio, class S, bool BWD>
int launch_B(const smnn_problem* p, const Args<Tio>& a, cudaStream_t st, std::string& err) {
  constexpr int CM = PipeCM<B, S>::value;
  PipePlan q = plan_B<B, S>(p, sizeof(Tio), BWD);
  if (!q.ok) return 0;
  auto k1 = pipe_p1_kernel<B, Tio, S, BWD, CM>;
  auto k2 = pipe_sep_kernel<B, S>;
  auto k2b = q.m2 > 4 ? pipe_sep2_kernel<B, S, 8> : pipe_sep2_kernel<B, S, 4>;
  auto k3 = pipe_p2_kernel<B, Tio, S, BWD, CM>;
  set_smem(k1, q.smem_p1);
  set_smem(k3, q.smem_p2);
  set_smem(q.sep2 ? k2b : k2, q.smem_sep);
  const int G = pipe_groups(p->n_inst);
  ForkJoin* fj = G > 1 ? fork_join() : nullptr;
  const int groups = fj ? G : 1;
  if (fj && cudaEventRecord(fj->fork, st) != cudaSuccess) fj = nullptr;
  char* ws = static_cast<char*>(a.ckpt);
  const int T = p->T, K = q.K;
  const size_t ls = sizeof(S);
  // stage-major launch order (all groups' P1, then SEP, then P2): a group's
  // separator kernel becomes ready while the next group's P1 still runs
  struct Grp3 {
    Args<Tio> a;
    PipeL L1, L2;
    int32_t* info;
    int64_t ni;
    cudaStream_t s;
  } gr[ForkJoin::kMax];
  for (int gi = 0; gi < groups; ++gi) {
    const int64_t i0 = p->n_inst * gi / groups, i1 = p->n_inst * (gi + 1) / groups, ni = i1 - i0;
    Grp3& G3 = gr[gi];
    G3.ni = ni;
    G3.s = st;
    if (fj) {
      G3.s = fj->s[gi];
      cudaStreamWaitEvent(G3.s, fj->fork, 0);
    }
    Args<Tio>& ag = G3.a;  // the group's instances [i0, i1)
    ag = a;
    ag.n_inst = ni;
    ag.coeffs = a.coeffs + i0 * T * B;
    ag.rhs = a.rhs + i0 * T;
    ag.iv = a.iv + i0 * a.n_iv;
    ag.steps = a.steps + i0 * (T - 1);
    if (a.y_in) ag.y_in = a.y_in + i0 * T * B;
    if (a.grad_y) ag.grad_y = a.grad_y + i0 * T * B;
    if (a.y_out) ag.y_out = a.y_out + i0 * T * B;
    if (a.g_coeffs) ag.g_coeffs = a.g_coeffs + i0 * T * B;
    if (a.g_rhs) ag.g_rhs = a.g_rhs + i0 * T;
    if (a.g_iv) ag.g_iv = a.g_iv + i0 * a.n_iv;
    if (a.g_steps) ag.g_steps = a.g_steps + i0 * (T - 1);
    G3.info = a.info ? a.info + i0 : nullptr;
    G3.L1 = q.L1;
    G3.L2 = q.L2;
    for (PipeL* L : {&G3.L1, &G3.L2}) {
      L->sep1 = ws + size_t(i0) * PSep<B>::N * K * ls;
      L->ysep = ws + q.ws_sep1 + size_t(i0) * B * K * ls;
      L->cfail = reinterpret_cast<int*>(ws + q.ws_sep1 + q.ws_ysep) + i0 * K;
    }
  }
  for (int gi = 0; gi < groups; ++gi)
    if (gr[gi].ni > 0) k1<<<unsigned(gr[gi].ni * q.parts), q.NT, q.smem_p1, gr[gi].s>>>(gr[gi].a, gr[gi].L1);
  for (int gi = 0; gi < groups; ++gi) {
    if (gr[gi].ni <= 0) continue;
    if (q.sep2)
      k2b<<<unsigned(gr[gi].ni), q.K / q.m2, q.smem_sep, gr[gi].s>>>(gr[gi].L1, T, gr[gi].info);
    else
      k2<<<unsigned(gr[gi].ni), q.K, q.smem_sep, gr[gi].s>>>(gr[gi].L1, T, gr[gi].info);
  }
  for (int gi = 0; gi < groups; ++gi) {
    if (gr[gi].ni <= 0) continue;
    k3<<<unsigned(gr[gi].ni * q.parts), q.NT, q.smem_p2, gr[gi].s>>>(gr[gi].a, gr[gi].L2);
    if (fj) {
      cudaEventRecord(fj->join[gi], gr[gi].s);
      cudaStreamWaitEvent(st, fj->join[gi], 0);
    }
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    err = std::string("pipeline launch: ") + cudaGetErrorString(e);
    return SMNN_ERR_CUDA;
  }
  return 1;
}

template <class Tio, class S, bool BWD>
int launch_order(const smnn_problem* p, const Args<Tio>& a, cudaStream_t st, std::string& err) {
  switch (p->order) {
    case 0: return launch_B<1, Tio, S, BWD>(p, a, st, err);
    case 1: return launch_B<2, Tio, S, BWD>(p, a, st, err);
    case 2: return launch_B<3, Tio, S, BWD>(p, a, st, err);
    default: return launch_B<4, Tio, S, BWD>(p, a, st, err);
  }
}

}  // namespace

bool pipe_eligible(const smnn_problem* p, bool bwd) { return plan_of(p, bwd).ok; }

size_t pipe_workspace_bytes(const smnn_problem* p) {
  const PipePlan f = plan_of(p, false), b = plan_of(p, true);
  size_t n = 0;
  if (f.ok) n = std::max(n, f.ws_sep1 + f.ws_ysep + f.ws_fail);
  if (b.ok) n = std::max(n, b.ws_sep1 + b.ws_ysep + b.ws_fail);
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
