// smnn_rf.cu -- host side of the register-factor resident kernel (smnn_rf.cuh).
//
// Separate translation unit so the library's kernels compile in parallel;
// smnn_kernels.cu calls rf_launch<Tio, Tc>() first and falls back to the
// checkpointing kernels when the problem is not eligible.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "smnn.h"
#include "smnn_rf.cuh"
#include "smnn_rf_host.h"

namespace smnn {
namespace {

size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

// Chunks (= threads) per instance: the fewest multiple-of-32 count whose
// chunks hold at most CM points, with every chunk >= 2 points (an interior).
int rf_threads(const smnn_problem* p, int CM, int max_threads = SMNN_RF_MAX_THREADS) {
  int nt = p->threads_per_inst;
  if (nt == 0) {
    nt = (p->T + CM - 1) / CM;
    nt = ((nt + 31) / 32) * 32;
  }
  if (nt < 32 || nt > max_threads) return 0;
  if (2 * nt > p->T) return 0;                       // every chunk needs an interior point
  if ((p->T + nt - 1) / nt > CM) return 0;           // longest chunk must fit the registers
  return nt;
}

template <int B, class S>
size_t rf_smem(const smnn_problem* p, int nt, size_t es, bool bwd, RLayout& L) {
  const size_t ls = sizeof(S);
  const int T = p->T;
  L = RLayout{};
  L.nt = nt;
  L.cs = 1;
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t o = off; off = al16(off + bytes); return int(o); };
  L.off_c = take(size_t(T) * B * es + 32);
  L.off_d = take(size_t(T) * es + 32);
  L.off_s = take(size_t(T) * es + 32);
  L.off_g = bwd ? take(size_t(T) * B * es + 32) : 0;
  const bool late_y = bwd && RF_LATE_Y;
  L.off_y = (bwd && !late_y) ? take(size_t(T) * B * es + 32) : 0;
  L.lane = int(off);
  const size_t rec = size_t(BRec<B>::N) * nt * ls;  // separator records (rbcr2)
  L.off_sep = take(late_y ? std::max(rec, size_t(T) * B * es + 32) : rec);  // late y reuses the records
  if (late_y) L.off_y = L.off_sep;
  L.off_ck = take(size_t(nt + 4) * 4);  // separator times + failure flag
  L.off_bar = take(16);
  return off;
}

// Wide register-factor variant: chunks of up to 12 points (fp32, b = 3).
// Measured on B200: the rf kernel is fastest with ~128 chunks per instance
// (4 warps; fewer chunks = a shorter separator reduction, more = more
// parallel pass work) -- SST (T = 1461) 1.39e10 -> 1.73e10 with 12-point chunks
// (128 threads instead of 192), while Lorenz (T = 1000) stays fastest with the
// 8-point template at 128 threads (the wide template's extra registers cost
// 13 % there).  The host takes the variant whose thread count is the smallest
// one >= 128.
template <int B, class S>
struct RfCMW {
  static constexpr int value = (B == 3 && sizeof(S) == 4) ? 12 : RfCM<B, S>::value;
};

// 0: not eligible, 1: register-factor variant, 3: wide register-factor variant
template <int B, class S>
int variant_B(const smnn_problem* p, size_t es, bool bwd) {
  RLayout L;
  const int nt = rf_threads(p, RfCM<B, S>::value);
  const bool ok = nt != 0 && rf_smem<B, S>(p, nt, es, bwd, L) <= 200 * 1024;
  if (RfCMW<B, S>::value != RfCM<B, S>::value) {
    const int nw = rf_threads(p, RfCMW<B, S>::value);
    const bool okw = nw != 0 && rf_smem<B, S>(p, nw, es, bwd, L) <= 200 * 1024;
    // smallest thread count >= 128 (else the largest)
    auto score = [](int n) { return n >= 128 ? n : 100000 - n; };
    if (okw && (!ok || score(nw) < score(nt))) return 3;
  }
  return ok ? 1 : 0;
}

template <int B, class S>
bool eligible_B(const smnn_problem* p, size_t es, bool bwd) {
  return variant_B<B, S>(p, es, bwd) != 0;
}

template <int B, class Tio, class S, bool BWD>
int launch_B(const smnn_problem* p, const Args<Tio>& a, cudaStream_t st, std::string& err) {
  const int var = variant_B<B, S>(p, sizeof(Tio), BWD);
  if (var == 0) return 0;
  constexpr int CM = RfCM<B, S>::value, CMW = RfCMW<B, S>::value;
  const int nt = var == 3 ? rf_threads(p, CMW) : rf_threads(p, CM);
  RLayout L{};
  const size_t smem = rf_smem<B, S>(p, nt, sizeof(Tio), BWD, L);
  auto kern = var == 3 ? rf_kernel<B, Tio, S, BWD, CMW> : rf_kernel<B, Tio, S, BWD, CM>;
  if (const cudaError_t ea = ensure_smem_k(kern, smem); ea != cudaSuccess) {
    err = std::string("rf kernel shared-memory attribute: ") + cudaGetErrorString(ea);
    cudaGetLastError();
    return SMNN_ERR_CUDA;
  }
  // one CTA per instance up to 2^31 - 1 (the block scheduler balances the tail);
  // the kernel strides over instances beyond that
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(p->n_inst, int64_t(INT32_MAX)));
  Args<Tio> aa = a;
  aa.K = nt;
  kern<<<unsigned(grid), nt, smem, st>>>(aa, L);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    err = std::string("rf kernel launch: ") + cudaGetErrorString(e);
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

bool rf_eligible(const smnn_problem* p, bool bwd) {
  const size_t es = p->dtype == SMNN_F64 ? 8 : 4;
  const bool d = p->dtype != SMNN_F32;
  switch (p->order) {
    case 0: return d ? eligible_B<1, double>(p, es, bwd) : eligible_B<1, float>(p, es, bwd);
    case 1: return d ? eligible_B<2, double>(p, es, bwd) : eligible_B<2, float>(p, es, bwd);
    case 2: return d ? eligible_B<3, double>(p, es, bwd) : eligible_B<3, float>(p, es, bwd);
    default: return d ? eligible_B<4, double>(p, es, bwd) : eligible_B<4, float>(p, es, bwd);
  }
}

template <class Tio, class Tc>
int rf_launch(const smnn_problem* p, const Args<Tio>& a, bool bwd, cudaStream_t st, std::string& err) {
  return bwd ? launch_order<Tio, Tc, true>(p, a, st, err) : launch_order<Tio, Tc, false>(p, a, st, err);
}

template int rf_launch<float, float>(const smnn_problem*, const Args<float>&, bool, cudaStream_t, std::string&);
template int rf_launch<float, double>(const smnn_problem*, const Args<float>&, bool, cudaStream_t, std::string&);
template int rf_launch<double, double>(const smnn_problem*, const Args<double>&, bool, cudaStream_t, std::string&);

}  // namespace smnn

#ifdef SMNN_RF_TIMING
extern "C" int smnn_debug_rf_timing(unsigned long long* host, size_t n) {
  return int(cudaMemcpyFromSymbol(host, smnn::rf_timing, n * sizeof(unsigned long long)));
}
#endif
