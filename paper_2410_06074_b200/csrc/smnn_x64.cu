// smnn_x64.cu -- host side of the cluster-resident fp64-arithmetic path (smnn_x64.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "smnn.h"
#include "smnn_rf_host.h"
#include "smnn_x64.cuh"

namespace smnn {


namespace {

constexpr int kMaxNT = 128;   // x64_kernel's __launch_bounds__
constexpr int kMaxNC = 16;    // non-portable cluster limit on B200

// Chunk capacity C (points per chunk) by block size and direction: the
// interior factors (and pass-2 forward-substituted right-hand sides) of C - 1
// points stay in registers (kernel compiled for 2 CTAs x 128 threads per SM).
template <int B, bool BWD>
struct XC {
  static constexpr int value = B == 1 ? (BWD ? 12 : 16) : B == 2 ? (BWD ? 9 : 12) : B == 3 ? (BWD ? 7 : 9)
                                                                                          : (BWD ? 5 : 6);
};

int chunk_cap(int order, bool bwd) {
  switch (order) {
    case 0: return bwd ? XC<1, true>::value : XC<1, false>::value;
    case 1: return bwd ? XC<2, true>::value : XC<2, false>::value;
    case 2: return bwd ? XC<3, true>::value : XC<3, false>::value;
    default: return bwd ? XC<4, true>::value : XC<4, false>::value;
  }
}

int cb(int64_t k, int T, int K) { return int((k * T) / K); }
size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

struct XPlan {
  x64::XL L{};
  size_t smem = 0;
  bool ok = false;
};

// Threads per CTA NT (a power of two <= 128) and CTAs per cluster NC so that
// K = NC NT chunks of at most C points cover T; the shared-memory layout.
XPlan plan(const smnn_problem* p, bool bwd) {
  XPlan x;
  const int T = p->T, B = p->order + 1, C = chunk_cap(p->order, bwd);
  const size_t es = p->dtype == SMNN_F64 ? 8 : 4;
  const int NR = bwd ? 2 : 1;
  const int64_t kmin = (int64_t(T) + C - 1) / C;
  int NT = 1, NC = 1;
  if (kmin <= kMaxNT) {
    while (NT < kmin) NT <<= 1;
    while (NT > T) NT >>= 1;
  } else {
    NT = kMaxNT;
    const int64_t nc = (kmin + NT - 1) / NT;
    if (nc > kMaxNC) return x;
    NC = int(nc);
  }
  const int K = NC * NT;
  if (K > T || (T + K - 1) / K > C) return x;
  int nmax = 0;
  for (int r = 0; r < NC; ++r) nmax = std::max(nmax, cb(int64_t(r + 1) * NT, T, K) - cb(int64_t(r) * NT, T, K));
  const int LT = B * (B + 1) / 2;
  const int RN = (LT + 2 * B * B + 2 * NR * B) | 1;
  const int PN = 2 * LT + B * B + 2 * NR * B;
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t o = off; off = al16(off + bytes); return int(o); };
  x.L.NC = NC;
  x.L.NT = NT;
  x.L.K = K;
  x.L.off_c = take(size_t(nmax) * B * es + 32);
  x.L.off_d = take(size_t(nmax) * es + 32);
  x.L.off_s = take(size_t(nmax + 1) * es + 32);
  x.L.off_g = bwd ? take(size_t(nmax) * B * es + 32) : 0;
  x.L.off_rec = take(size_t(NT + 1) * RN * 8);
  x.L.off_pub = take(size_t(PN) * 8 + 16);
  x.L.off_bar = take(16);
  x.smem = off;
  x.ok = off <= 200 * 1024;
  return x;
}

int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// Dynamic shared-memory attribute: the largest request so far per (device,
// kernel) (ensure_smem).  Whether one cluster of the requested shape fits
// (cudaOccupancyMaxActiveClusters) is cached per (device, kernel, shape).
template <class K>
bool prepare(K kern, const XPlan& x, std::string& err) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int, int, size_t>, int> cache;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), x.smem);
  if (e == cudaSuccess && x.L.NC > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) {
    err = std::string("x64 kernel setup: ") + cudaGetErrorString(e);
    cudaGetLastError();
    return false;
  }
  const auto key = std::make_tuple(cur_device(), reinterpret_cast<const void*>(kern), x.L.NC, x.L.NT, x.smem);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second > 0;
  int ncl = 0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = x.L.NC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(x.L.NC);
  cfg.blockDim = dim3(x.L.NT);
  cfg.dynamicSmemBytes = x.smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
  if (e != cudaSuccess) {
    err = std::string("x64 kernel setup: ") + cudaGetErrorString(e);
    cudaGetLastError();
    ncl = 0;
  }
  cache[key] = ncl;
  return ncl > 0;
}

template <int B, class Tio, bool BWD>
int launch(const smnn_problem* p, const Args<Tio>& a, const XPlan& x, cudaStream_t st, std::string& err) {
  auto kern = x64::x64_kernel<B, Tio, BWD, XC<B, BWD>::value>;
  if (!prepare(kern, x, err)) return err.empty() ? 0 : SMNN_ERR_CUDA;
  x64::XArgs<Tio> xa;
  xa.coeffs = a.coeffs;
  xa.rhs = a.rhs;
  xa.iv = a.iv;
  xa.steps = a.steps;
  xa.grad_y = a.grad_y;
  xa.y_out = a.y_out;
  xa.g_coeffs = a.g_coeffs;
  xa.g_rhs = a.g_rhs;
  xa.g_iv = a.g_iv;
  xa.g_steps = a.g_steps;
  xa.info = a.info;
  xa.T = p->T;
  xa.n_iv = p->n_iv;
  xa.wg2 = a.wg2;
  xa.wi2 = a.wi2;
  xa.ws2 = a.ws2;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = x.L.NC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(unsigned(p->n_inst * x.L.NC));
  cfg.blockDim = dim3(x.L.NT);
  cfg.dynamicSmemBytes = x.smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, xa, x.L);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    err = std::string("x64 kernel launch: ") + cudaGetErrorString(e);
    cudaGetLastError();  // a launch-configuration error must not leak into the next call's check
    return SMNN_ERR_CUDA;
  }
  return 1;
}

template <class Tio, bool BWD>
int dispatch(const smnn_problem* p, const Args<Tio>& a, cudaStream_t st, std::string& err) {
  const XPlan x = plan(p, BWD);
  if (!x.ok) return 0;
  switch (p->order) {
    case 0: return launch<1, Tio, BWD>(p, a, x, st, err);
    case 1: return launch<2, Tio, BWD>(p, a, x, st, err);
    case 2: return launch<3, Tio, BWD>(p, a, x, st, err);
    default: return launch<4, Tio, BWD>(p, a, x, st, err);
  }
}

}  // namespace

bool x64_eligible(const smnn_problem* p, bool bwd) {
  return p->dtype != SMNN_F32 && p->n_inst * 16 < (int64_t(1) << 31) && plan(p, bwd).ok;
}

template <class Tio>
int x64_launch(const smnn_problem* p, const Args<Tio>& a, bool bwd, cudaStream_t st, std::string& err) {
  if (p->dtype == SMNN_F32) return 0;
  return bwd ? dispatch<Tio, true>(p, a, st, err) : dispatch<Tio, false>(p, a, st, err);
}

template int x64_launch<float>(const smnn_problem*, const Args<float>&, bool, cudaStream_t, std::string&);
template int x64_launch<double>(const smnn_problem*, const Args<double>&, bool, cudaStream_t, std::string&);

}  // namespace smnn
