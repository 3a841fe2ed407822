// smnn_kernels.cu -- S-MNN hot path for sm_100a (B200).
//
// Kernels (one CUDA thread block per instance unless noted):
//   assemble_kernel   Appendix A.1 blocks M_t, N_t, beta_t -> HBM (inspection)
//   fused_kernel<FWD> Algorithm 1: assemble + block Cholesky + substitution,
//                     time-parallel (see "Time-parallel partition solver" in
//                     DESIGN.md); M never leaves registers/shared memory.
//   fused_kernel<BWD> Algorithm 2 + chain rule through Appendix A.1.
//   factor_kernel     Algorithm 3, one thread per instance, L/P -> HBM.
//   substitute_kernel Algorithm 4, one thread per instance.
//
// Time-parallel partition solver (per instance, K chunks = K threads):
//   chunk k covers [a_k, a_{k+1}); its last point sigma_k is a separator, the
//   points before it are the chunk interior I_k.  Interiors are coupled only
//   through separators, so
//   pass 1  each thread factors its interior (block Cholesky, Alg. 3 loop)
//           and carries a "spike" X_j = (G^{-1})_{j,f} N_L to obtain the Schur
//           complement of its interior onto (sigma_{k-1}, sigma_k);
//   BCR     the K x K block-tridiagonal separator system is solved in shared
//           memory by block cyclic reduction (log2 K levels);
//   pass 2  each thread re-factors its interior in G-step register segments
//           (resuming from pass-1 checkpoints) and back-substitutes with both
//           separator values known.
//   The result equals the sequential Algorithm 1 up to rounding.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "smnn.h"
#include "smnn_device.cuh"
#include "smnn_fused.cuh"
#include "smnn_rf_host.h"

#ifndef SMNN_F32_LANE
#define SMNN_F32_LANE float
#endif
#ifndef SMNN_F64_LANE
#define SMNN_F64_LANE double
#endif

namespace smnn {

// Register-segment length of pass 2 (steps whose factors stay in registers).
template <int B, class S>
struct SegLen {
  static constexpr int value = (sizeof(S) >= 8) ? (B == 1 ? 8 : B == 2 ? 4 : 2) : (B <= 2 ? 8 : B == 3 ? 4 : 2);
};

// Lane type of the fused kernels for (storage, arithmetic).
template <class Tio, class Tc> struct LaneOf;
template <> struct LaneOf<float, float> { using S = SMNN_F32_LANE; };
template <> struct LaneOf<double, double> { using S = SMNN_F64_LANE; };
template <> struct LaneOf<float, double> { using S = SMNN_F64_LANE; };

// Load helpers (sequential kernels) ---------------------------------------
template <int B, class Tio, class Tc>
__device__ __forceinline__ void ld_vec(const Tio* p, Tc (&v)[B]) {
#pragma unroll
  for (int r = 0; r < B; ++r) v[r] = Tc(__ldg(p + r));
}

template <class Tio, class Tc>
__device__ __forceinline__ Tc ld1(const Tio* p) { return Tc(__ldg(p)); }

// Per-instance base pointers (all further indexing is 32-bit).
template <class Tio>
struct View {
  const Tio *c, *d, *u, *s, *yin, *gy;
  Tio *yout, *gc, *gd, *gu, *gs;
  int T, n_iv;
  float dummy;
  __device__ View(const Args<Tio>& a, int64_t inst, int B) {
    T = a.T;
    n_iv = a.n_iv;
    const int64_t tb = inst * int64_t(a.T) * B, t1 = inst * int64_t(a.T), ts = inst * int64_t(a.T - 1);
    c = a.coeffs + tb;
    d = a.rhs + t1;
    u = a.iv + inst * a.n_iv;
    s = a.steps + ts;
    yin = a.y_in ? a.y_in + tb : nullptr;
    gy = a.grad_y ? a.grad_y + tb : nullptr;
    yout = a.y_out ? a.y_out + tb : nullptr;
    gc = a.g_coeffs ? a.g_coeffs + tb : nullptr;
    gd = a.g_rhs ? a.g_rhs + t1 : nullptr;
    gu = a.g_iv ? a.g_iv + inst * a.n_iv : nullptr;
    gs = a.g_steps ? a.g_steps + ts : nullptr;
  }
};

struct W3 {  // squared importance weights in the arithmetic type
  double g, i, s;
};

// RHS at point j: beta_j = wg2 c_j d_j (+ wi2 u at j = 0) in the forward pass,
// dl/dy_j in the backward pass.
template <int B, class Tio, class Tc, bool BWD>
__device__ __forceinline__ void load_rhs(const View<Tio>& v, const W3& w, int j, const Tc (&c)[B], Tc (&r)[B]) {
  if (BWD) {
    ld_vec<B, Tio, Tc>(v.gy + j * B, r);
  } else {
    const Tc d = ld1<Tio, Tc>(v.d + j);
#pragma unroll
    for (int i = 0; i < B; ++i) r[i] = Tc(w.g) * c[i] * d;
    if (j == 0) {
#pragma unroll
      for (int i = 0; i < B; ++i)
        if (i < v.n_iv) r[i] += Tc(w.i) * ld1<Tio, Tc>(v.u + i);
    }
  }
}

// M_j with its neighbours' step powers (pp = s_{j-1}^k, pn = s_j^k).
template <int B, class Tio, class Tc>
__device__ __forceinline__ void load_M(const View<Tio>& v, const W3& w, int j, const Tc (&c)[B],
                                       const Tc (&pp)[2 * B - 1], Tc hp, const Tc (&pn)[2 * B - 1], Tc hn,
                                       Tc (&M)[B][B]) {
  assemble_M<B, Tc>(M, c, pp, hp, pn, hn, Tc(w.g), Tc(w.s));
  if (j == 0) {
#pragma unroll
    for (int i = 0; i < B; ++i)
      if (i < v.n_iv) M[i][i] += Tc(w.i);
  }
}

// ------------------------------------------------------- assemble kernel ----
template <int B, class Tio, class Tc>
__global__ void assemble_kernel(Args<Tio> a, Tio* Mo, Tio* No, Tio* bo) {
  const int T = a.T;
  const W3 w{a.wg2, a.wi2, a.ws2};
  const int64_t total = a.n_inst * T;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t inst = idx / T;
    const int t = int(idx % T);
    const View<Tio> v(a, inst, B);
    Tc c[B], pp[2 * B - 1], pn[2 * B - 1], M[B][B], r[B];
    ld_vec<B, Tio, Tc>(v.c + t * B, c);
    const bool hp = t > 0, hn = t < T - 1;
    powers<B, Tc>(hp ? ld1<Tio, Tc>(v.s + t - 1) : Tc(0), pp);
    powers<B, Tc>(hn ? ld1<Tio, Tc>(v.s + t) : Tc(0), pn);
    load_M<B, Tio, Tc>(v, w, t, c, pp, hp ? Tc(1) : Tc(0), pn, hn ? Tc(1) : Tc(0), M);
    load_rhs<B, Tio, Tc, false>(v, w, t, c, r);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      bo[idx * B + i] = Tio(r[i]);
#pragma unroll
      for (int q = 0; q < B; ++q) Mo[(idx * B + i) * B + q] = Tio(M[i][q]);
    }
    if (hn && No) {
      Tc N[B][B];
      assemble_N<B, Tc>(N, pn, Tc(w.s));
      const int64_t o = inst * (T - 1) + t;
#pragma unroll
      for (int i = 0; i < B; ++i)
#pragma unroll
        for (int q = 0; q < B; ++q) No[(o * B + i) * B + q] = Tio(N[i][q]);
    }
  }
}

// --------------------------------------------- Algorithm 3, sequential -----
template <int B, class Tio, class Tc>
__global__ void factor_kernel(Args<Tio> a, Tio* Lo, Tio* Po) {
  const int64_t inst = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (inst >= a.n_inst) return;
  const int T = a.T;
  const W3 w{a.wg2, a.wi2, a.ws2};
  const View<Tio> v(a, inst, B);
  const Tc ws2 = Tc(w.s);
  int fail = 0;
  Tc Lf[B][B], pp[2 * B - 1];
  zero<B, Tc>(Lf);
  powers<B, Tc>(Tc(0), pp);
  for (int t = 0; t < T; ++t) {
    Tc c[B], pn[2 * B - 1], M[B][B], D[B][B];
    ld_vec<B, Tio, Tc>(v.c + t * B, c);
    const bool hn = t < T - 1;
    powers<B, Tc>(hn ? ld1<Tio, Tc>(v.s + t) : Tc(0), pn);
    load_M<B, Tio, Tc>(v, w, t, c, pp, t > 0 ? Tc(1) : Tc(0), pn, hn ? Tc(1) : Tc(0), M);
    if (t > 0) {
      // P_{t-1} <- N_{t-1} L_{t-1}^{-T};  L_t <- M_t - P P^T   (Alg. 3)
      Tc N[B][B], P[B][B], Pl[B][B];
      assemble_N<B, Tc>(N, pp, ws2);
      right_ltsolve<B, Tc>(N, Lf, P);
      sub_ppt<B, Tc>(M, P, D);
      // to blockwise LDL: P_{t-1} <- P_{t-1} L_{t-1}^{-1}   (Alg. 3)
#pragma unroll
      for (int r = 0; r < B; ++r) ltsolve<B, Tc>(Lf, P[r], Pl[r]);
      if (Po) {
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int q = 0; q < B; ++q) Po[((inst * (T - 1) + t - 1) * B + i) * B + q] = Tio(Pl[i][q]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < B; ++i)
#pragma unroll
        for (int q = 0; q < B; ++q) D[i][q] = M[i][q];
    }
    if (!chol<B, Tc>(D, Lf) && fail == 0) fail = t + 1;  // standard Cholesky (line 255)
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
      for (int q = 0; q < B; ++q)
        Lo[((inst * T + t) * B + i) * B + q] =
            Tio(q < i ? Lf[i][q] : (q == i ? Tc(1) / Lf[i][i] : Tc(0)));
#pragma unroll
    for (int m = 0; m < 2 * B - 1; ++m) pp[m] = pn[m];
  }
  if (a.info) a.info[inst] = fail;
}

// --------------------------------------------- Algorithm 4, sequential -----
template <int B, class Tio, class Tc>
__global__ void substitute_kernel(int64_t n_inst, int T, const Tio* Lg, const Tio* Pg, const Tio* alpha, Tio* out) {
  const int64_t inst = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (inst >= n_inst) return;
  Tc prev[B];
  for (int t = 0; t < T; ++t) {
    Tc al[B], Lf[B][B], x[B], z[B];
    ld_vec<B, Tio, Tc>(alpha + (inst * T + t) * B, al);
    if (t > 0) {  // forward substitute: a_t -= P_{t-1} a_{t-1}  (Alg. 4)
#pragma unroll
      for (int i = 0; i < B; ++i) {
        Tc acc = Tc(0);
#pragma unroll
        for (int q = 0; q < B; ++q) acc += Tc(Pg[((inst * (T - 1) + t - 1) * B + i) * B + q]) * prev[q];
        al[i] -= acc;
      }
    }
#pragma unroll
    for (int i = 0; i < B; ++i) prev[i] = al[i];
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
      for (int q = 0; q < B; ++q) {
        Tc v = Tc(Lg[((inst * T + t) * B + i) * B + q]);
        Lf[i][q] = (i == q) ? Tc(1) / v : v;
      }
    lsolve<B, Tc>(Lf, al, x);  // a_t <- L_t^{-T} L_t^{-1} a_t  (line 307)
    ltsolve<B, Tc>(Lf, x, z);
#pragma unroll
    for (int i = 0; i < B; ++i) out[(inst * T + t) * B + i] = Tio(z[i]);
  }
  for (int t = T - 2; t >= 0; --t) {  // backward substitute (line 312)
    Tc nx[B], cur[B];
    ld_vec<B, Tio, Tc>(out + (inst * T + t + 1) * B, nx);
    ld_vec<B, Tio, Tc>(out + (inst * T + t) * B, cur);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      Tc acc = Tc(0);
#pragma unroll
      for (int q = 0; q < B; ++q) acc += Tc(Pg[((inst * (T - 1) + t) * B + q) * B + i]) * nx[q];
      out[(inst * T + t) * B + i] = Tio(cur[i] - acc);
    }
  }
}

}  // namespace smnn

// ============================================================ host side =====
namespace {

thread_local std::string g_err;

int fail_arg(const std::string& m) { g_err = m; return SMNN_ERR_ARG; }

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SMNN_OK;
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return SMNN_ERR_CUDA;
}

int validate(const smnn_problem* p) {
  if (!p) return fail_arg("problem is NULL");
  if (p->n_inst < 1) return fail_arg("n_inst must be >= 1");
  if (p->T < 1) return fail_arg("T must be >= 1");
  if (p->order < 0) return fail_arg("order must be >= 0");
  if (p->order > SMNN_MAX_ORDER) { g_err = "order > 3 is not supported"; return SMNN_ERR_UNSUPPORTED; }
  if (p->n_iv < 1 || p->n_iv > p->order + 1) return fail_arg("n_iv must be in 1..order+1");
  if (p->dtype != SMNN_F32 && p->dtype != SMNN_F64 && p->dtype != SMNN_F32_C64) {
    g_err = "unknown dtype"; return SMNN_ERR_UNSUPPORTED;
  }
  if (!(p->w_gov > 0) || !(p->w_init > 0) || !(p->w_smooth > 0)) return fail_arg("weights must be > 0");
  if (p->threads_per_inst < 0 || p->threads_per_inst > SMNN_MAX_THREADS || (p->threads_per_inst % 32) != 0)
    return fail_arg("threads_per_inst must be 0 (auto) or a multiple of 32 in 32..SMNN_MAX_THREADS");
  if (p->path < 0 || p->path > SMNN_PATH_STREAM) return fail_arg("path must be 0 (auto) or an SMNN_PATH_* code");
  return SMNN_OK;
}

size_t tc_size(const smnn_problem* p) { return p->dtype == SMNN_F32 ? 4 : 8; }

// Lane of the fused kernels: P instances per register, `bytes` per lane value.
struct LaneInfo {
  int P;
  size_t bytes;
};
LaneInfo lane_info(const smnn_problem* p) {
  if (p->dtype == SMNN_F32) return {smnn::LaneT<SMNN_F32_LANE>::P, sizeof(SMNN_F32_LANE)};
  return {smnn::LaneT<SMNN_F64_LANE>::P, sizeof(SMNN_F64_LANE)};
}

int pass2_G(const smnn_problem* p) {
  const int B = p->order + 1;
  return lane_info(p).bytes >= 8 ? (B == 1 ? 8 : B == 2 ? 4 : 2) : (B <= 2 ? 8 : B == 3 ? 4 : 2);  // == SegLen
}

size_t sep_bytes_per_chunk(const smnn_problem* p) {
  const int B = p->order + 1;
  return size_t(3 * B * B + 2 * B) * lane_info(p).bytes + sizeof(int);
}

// Target steps per time chunk of the checkpoint kernels.
constexpr int chunk_target() { return 8; }

// Chunks (threads) per instance.
int threads_per_inst(const smnn_problem* p) {
  int nt = p->threads_per_inst;
  if (nt == 0) {
    const int target = chunk_target();  // steps per chunk
    nt = (p->T + target - 1) / target;
    nt = ((nt + 31) / 32) * 32;
    nt = std::max(32, std::min(nt, SMNN_MAX_THREADS));
  }
  while (nt > 32 && sep_bytes_per_chunk(p) * nt > 160 * 1024) nt -= 32;
  return nt;
}

int chunks(const smnn_problem* p) { return std::min(threads_per_inst(p), p->T); }

size_t ports_bytes(const smnn_problem* p, int nt) {  // per-warp scratch of the warp-tiled BCR
  const int B = p->order + 1;
  return size_t(nt / 32) * (3 * B * B + 3 * B) * lane_info(p).bytes;
}

size_t fused_smem(const smnn_problem* p) {
  const int nt = threads_per_inst(p);
  return sep_bytes_per_chunk(p) * nt + ports_bytes(p, nt) + 4 * sizeof(int) + 16;
}

int nseg_ck(const smnn_problem* p) {
  const int K = chunks(p);
  const int maxlen = (p->T + K - 1) / K;  // chunk length incl. separator
  const int nint = std::max(0, maxlen - 1);
  const int G = pass2_G(p);
  return std::max(0, (nint + G - 1) / G - 1);
}

size_t ck_elems(const smnn_problem* p) {
  const int B = p->order + 1;
  return size_t(B * (B + 1) / 2 + B + B * B);  // == smnn::CkN<B>::N
}

int64_t n_groups(const smnn_problem* p) {
  const int P = lane_info(p).P;
  return (p->n_inst + P - 1) / P;
}

int device_sms() {  // of the current device
  int dev = 0, v = 148;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
    return v;
  cudaGetLastError();
  return 148;
}

// Occupancy of a kernel (cached per device / kernel / block / smem); raises
// the kernel's dynamic shared-memory limit on this device (ensure_smem).
std::mutex g_occ_mu;
std::map<std::tuple<int, const void*, int, size_t>, int> g_occ;

template <class Kern>
int occupancy(Kern kernel, int nt, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, reinterpret_cast<const void*>(kernel), nt, smem);
  smnn::ensure_smem(reinterpret_cast<const void*>(kernel), smem);
  {
    std::lock_guard<std::mutex> lk(g_occ_mu);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
  }
  int occ = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, nt, smem) != cudaSuccess) {
    cudaGetLastError();
    occ = 1;
  }
  occ = std::max(occ, 1);
  std::lock_guard<std::mutex> lk(g_occ_mu);
  g_occ[key] = occ;
  return occ;
}

template <int B, class Tio, class Tc>
int fused_grid_any(const smnn_problem* p) {
  using S = typename smnn::LaneOf<Tio, Tc>::S;
  constexpr int G = smnn::SegLen<B, S>::value;
  const int nt = threads_per_inst(p);
  const size_t smem = fused_smem(p);
  const int occ = std::max(occupancy(smnn::fused_kernel<B, Tio, S, false, G>, nt, smem),
                           occupancy(smnn::fused_kernel<B, Tio, S, true, G>, nt, smem));
  return int(std::max<int64_t>(1, std::min<int64_t>(n_groups(p), int64_t(occ) * device_sms())));
}

template <class Tio, class Tc>
int grid_for(const smnn_problem* p) {
  switch (p->order) {
    case 0: return fused_grid_any<1, Tio, Tc>(p);
    case 1: return fused_grid_any<2, Tio, Tc>(p);
    case 2: return fused_grid_any<3, Tio, Tc>(p);
    default: return fused_grid_any<4, Tio, Tc>(p);
  }
}

int grid_blocks(const smnn_problem* p) {
  if (p->dtype == SMNN_F32) return grid_for<float, float>(p);
  if (p->dtype == SMNN_F64) return grid_for<double, double>(p);
  return grid_for<float, double>(p);
}

size_t workspace_bytes_direct(const smnn_problem* p) {
  const size_t per = size_t(nseg_ck(p)) * ck_elems(p) * threads_per_inst(p) * lane_info(p).bytes;
  return std::max<size_t>({per * grid_blocks(p), smnn::pipe_workspace_bytes(p), size_t(256)});
}

int kernel_path(const smnn_problem* p, bool bwd);

// ---- SMNN_F32_C64 backward on the paths that read y from storage --------
// The gradients' residual terms (d - c.y, the Taylor-row residuals) amplify
// the fp32 rounding of y by up to ~1e4, so an fp32-stored y cannot give 1e-4
// gradients.  The x64 kernel and the pipeline re-solve y in fp64 beside
// dl/dbeta (two right-hand sides, one factorisation); the other paths run the backward as SMNN_F64 on promoted copies instead: inputs and
// dl/dy widened to fp64 in the workspace, the fp64 forward (y in fp64), the
// fp64 backward, gradients narrowed into the caller's fp32 outputs.
// SMNN_F32_C64 on the pipeline in both directions: the forward can hand the
// backward the fp32 remainder y_lo of its fp64 y (smnn_factor_solve_fwd_ex), so
// the backward reads y_hi + y_lo instead of re-solving y (one right-hand side).
bool ylo_used(const smnn_problem* p) {
  return p->dtype == SMNN_F32_C64 && kernel_path(p, false) == SMNN_PATH_PIPE &&
         kernel_path(p, true) == SMNN_PATH_PIPE && smnn::pipe_ylo_eligible(p);
}

bool promote_bwd(const smnn_problem* p) {
  if (p->dtype != SMNN_F32_C64) return false;
  const int path = kernel_path(p, true);
  return path != SMNN_PATH_X64 && path != SMNN_PATH_PIPE;  // both re-solve y in fp64 themselves
}

smnn_problem as_f64(const smnn_problem* p) {
  smnn_problem q = *p;
  q.dtype = SMNN_F64;
  return q;
}

struct Promo {  // element offsets (doubles) of the promoted buffers in the workspace
  size_t c, d, u, s, gy, y, gc, gd, gu, gs, info, end;
};
Promo promo_layout(const smnn_problem* p) {
  const size_t n = size_t(p->n_inst), T = size_t(p->T), b = size_t(p->order + 1), ni = size_t(p->n_iv);
  const size_t sT = n * T * b, s1 = n * T, su = n * ni, ss = n * (T > 0 ? T - 1 : 0);
  auto al = [](size_t x) { return (x + 31) & ~size_t(31); };  // 256-byte aligned
  Promo o{};
  size_t off = 0;
  auto take = [&](size_t k) { const size_t r = off; off += al(std::max<size_t>(k, 1)); return r; };
  o.c = take(sT); o.d = take(s1); o.u = take(su); o.s = take(ss); o.gy = take(sT); o.y = take(sT);
  o.gc = take(sT); o.gd = take(s1); o.gu = take(su); o.gs = take(ss);
  o.info = take((n + 1) / 2);  // int32 forward info
  o.end = off;
  return o;
}

size_t workspace_bytes(const smnn_problem* p) {
  size_t n = workspace_bytes_direct(p);
  if (promote_bwd(p)) {
    const smnn_problem q = as_f64(p);
    n = std::max(n, promo_layout(p).end * sizeof(double) + workspace_bytes_direct(&q));
  }
  return n;
}

template <class Tio>
smnn::Args<Tio> make_args(const smnn_problem* p) {
  smnn::Args<Tio> a;
  std::memset(&a, 0, sizeof(a));
  a.n_inst = p->n_inst;
  a.T = p->T;
  a.n_iv = p->n_iv;
  a.K = chunks(p);
  a.nseg_ck = nseg_ck(p);
  a.wg2 = p->w_gov * p->w_gov;
  a.wi2 = p->w_init * p->w_init;
  a.ws2 = p->w_smooth * p->w_smooth;
  return a;
}

// ---------------------------------------------------------------- resident --
struct RPlan {
  smnn::RLayout L;
  size_t smem = 0;
  bool ok = false;
};

size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

// Shared-memory layout of the resident kernel for (problem, direction): the
// smallest cluster whose CTAs each hold their time range of the instance.
template <int B, class Tio, class S>
RPlan resident_plan(const smnn_problem* p, bool bwd) {
  RPlan best;
  if (p->path == SMNN_PATH_STREAM) return best;  // forced streaming checkpoint kernel
  const size_t es = sizeof(Tio), ls = sizeof(S);
  constexpr int G = smnn::SegLen<B, S>::value;
  const int T = p->T;
  const size_t budgets[2] = {110 * 1024, 200 * 1024};
  for (size_t budget : budgets) {
    {
      const int cs = 1;  // one CTA per instance group (cluster variants measured slower on B200)
      int nt = p->threads_per_inst;
      if (nt == 0) {
        const int m = chunk_target();  // steps per chunk
        nt = (T + cs * m - 1) / (cs * m);
        nt = std::max(32, std::min(((nt + 31) / 32) * 32, SMNN_MAX_THREADS));
      }
      if (int64_t(cs) * nt > T) {
        nt = (T / cs / 32) * 32;
        if (nt < 32) continue;
      }
      const int K = cs * nt;
      const int maxchunk = (T + K - 1) / K;
      const int Lmax = nt * maxchunk;
      smnn::RLayout L{};
      L.nt = nt;
      L.cs = cs;
      constexpr int P = smnn::LaneT<S>::P;
      size_t off = 0;
      auto take = [&](size_t bytes) { const size_t o = off; off = al16(off + bytes); return int(o); };
      // per-lane data block: c, d, s (+ g, y backward); lanes repeat it P times
      L.off_c = take(size_t(Lmax) * B * es + 32);
      L.off_d = take(size_t(Lmax) * es + 32);
      L.off_s = take(size_t(Lmax + 1) * es + 32);
      L.off_g = bwd ? take(size_t(Lmax) * B * es + 32) : 0;
      L.off_y = bwd ? take(size_t(Lmax + 1) * B * es + 32) : 0;
      L.lane = int(off);
      off *= P;
      L.off_sep = take(size_t(3 * B * B + 2 * B) * nt * ls + size_t(nt / 32) * (3 * B * B + 3 * B) * ls +
                       size_t(nt + 4) * 4);
      const int nck = std::max(0, (maxchunk - 1 + G - 1) / G - 1);
      L.off_ck = take(size_t(nck) * smnn::CkN<B>::N * nt * ls + 16);
      L.off_bar = take(16);
      if (off <= budget) {
        best.L = L;
        best.smem = off;
        best.ok = true;
        return best;
      }
    }
  }
  return best;
}

template <int B, class Tio, class Tc, bool BWD>
int launch_resident(const smnn_problem* p, const smnn::Args<Tio>& a, const RPlan& rp, cudaStream_t st) {
  using S = typename smnn::LaneOf<Tio, Tc>::S;
  auto kern = rp.L.cs > 1 ? smnn::resident_kernel<B, Tio, S, BWD, smnn::SegLen<B, S>::value, true>
                          : smnn::resident_kernel<B, Tio, S, BWD, smnn::SegLen<B, S>::value, false>;
  if (const int e0 = check_cuda(smnn::ensure_smem(reinterpret_cast<const void*>(kern), rp.smem),
                                "resident kernel shared-memory attribute"))
    return e0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = rp.L.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(rp.L.nt);
  cfg.dynamicSmemBytes = rp.smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(rp.L.cs);
  int nclusters = 0;
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int, int, size_t>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, reinterpret_cast<const void*>(kern), rp.L.cs, rp.L.nt, rp.smem);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) nclusters = it->second;
  }
  if (nclusters == 0) {
    if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters < 1) {
      cudaGetLastError();
      nclusters = std::max(1, device_sms() / rp.L.cs);
    }
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = nclusters;
  }
  const int64_t nc = std::min<int64_t>(n_groups(p), nclusters);
  cfg.gridDim = dim3(unsigned(nc * rp.L.cs));
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, rp.L);
  return check_cuda(e == cudaSuccess ? cudaGetLastError() : e, "resident kernel launch");
}

template <int B, class Tio, class Tc, bool BWD>
int launch_fused(const smnn_problem* p, smnn::Args<Tio> a, cudaStream_t st) {
  using S = typename smnn::LaneOf<Tio, Tc>::S;
  const RPlan rp = resident_plan<B, Tio, S>(p, BWD);
  if (rp.ok) return launch_resident<B, Tio, Tc, BWD>(p, a, rp, st);
  const int nt = threads_per_inst(p);
  const size_t smem = fused_smem(p);
  const int grid = grid_blocks(p);
  auto k = smnn::fused_kernel<B, Tio, S, BWD, smnn::SegLen<B, S>::value>;
  occupancy(k, nt, smem);  // sets the dynamic smem attribute once
  k<<<grid, nt, smem, st>>>(a);
  return check_cuda(cudaGetLastError(), "fused kernel launch");
}

// Kernel path of the fused calls (SMNN_PATH_*; p->path forces one, the
// parity tests force every path).  Automatic order, measured on B200
// (profiles/r2/path_sweep_*.jsonl): fp64 arithmetic (SMNN_F64, SMNN_F32_C64)
// takes the pipeline (T = 500 .. 2e4 at 4e7 instance-steps: forward equal to or
// up to 1.8x faster than the x64 cluster kernel, backward 1.2-2.1x faster),
// then x64, then rf; fp32 arithmetic takes the resident rf kernel
// while one CTA holds the instance (T <~ 4k: Lorenz 9.3e9 -> 14.4e9
// instance-steps/s over the checkpoint kernel), then the pipeline (T = 1e4:
// 7.1e9 -> 22e9); the checkpointing kernels take what none of them fits.
int kernel_path(const smnn_problem* p, bool bwd) {
  const int want = p->path;  // 0 = auto; a forced path the problem does not fit falls back to auto
  const bool f32 = p->dtype == SMNN_F32;
  if (want == SMNN_PATH_X64 && smnn::x64_eligible(p, bwd)) return SMNN_PATH_X64;
  if (want == SMNN_PATH_RF && smnn::rf_eligible(p, bwd)) return SMNN_PATH_RF;
  if (want == SMNN_PATH_PIPE && smnn::pipe_eligible(p, bwd)) return SMNN_PATH_PIPE;
  if (want == SMNN_PATH_CHECKPOINT || want == SMNN_PATH_STREAM) return SMNN_PATH_CHECKPOINT;
  if (f32 && smnn::rf_eligible(p, bwd)) return SMNN_PATH_RF;
  if (smnn::pipe_eligible(p, bwd)) return SMNN_PATH_PIPE;
  if (!f32 && smnn::x64_eligible(p, bwd)) return SMNN_PATH_X64;
  if (!f32 && smnn::rf_eligible(p, bwd)) return SMNN_PATH_RF;
  return SMNN_PATH_CHECKPOINT;
}

template <class Tio, class Tc, bool BWD>
int dispatch_fused(const smnn_problem* p, const smnn::Args<Tio>& a, cudaStream_t st) {
  {
    const int path = kernel_path(p, BWD);
    std::string err;
    int r = 0;
    if (path == SMNN_PATH_X64) r = smnn::x64_launch<Tio>(p, a, BWD, st, err);
    if (path == SMNN_PATH_RF) r = smnn::rf_launch<Tio, Tc>(p, a, BWD, st, err);
    if (path == SMNN_PATH_PIPE) r = smnn::pipe_launch<Tio, Tc>(p, a, BWD, st, err);
    if (r < 0) { g_err = err; return r; }
    if (r == 1) return SMNN_OK;
  }
  switch (p->order) {
    case 0: return launch_fused<1, Tio, Tc, BWD>(p, a, st);
    case 1: return launch_fused<2, Tio, Tc, BWD>(p, a, st);
    case 2: return launch_fused<3, Tio, Tc, BWD>(p, a, st);
    default: return launch_fused<4, Tio, Tc, BWD>(p, a, st);
  }
}

template <class Tio, class Tc>
int dispatch_assemble(const smnn_problem* p, const smnn::Args<Tio>& a, Tio* M, Tio* N, Tio* b, cudaStream_t st) {
  const int64_t total = p->n_inst * p->T;
  const int threads = 256;
  const int blocks = int(std::min<int64_t>((total + threads - 1) / threads, 148 * 32));
  switch (p->order) {
    case 0: smnn::assemble_kernel<1, Tio, Tc><<<blocks, threads, 0, st>>>(a, M, N, b); break;
    case 1: smnn::assemble_kernel<2, Tio, Tc><<<blocks, threads, 0, st>>>(a, M, N, b); break;
    case 2: smnn::assemble_kernel<3, Tio, Tc><<<blocks, threads, 0, st>>>(a, M, N, b); break;
    default: smnn::assemble_kernel<4, Tio, Tc><<<blocks, threads, 0, st>>>(a, M, N, b); break;
  }
  return check_cuda(cudaGetLastError(), "assemble launch");
}

template <class Tio, class Tc>
int dispatch_factor(const smnn_problem* p, const smnn::Args<Tio>& a, Tio* L, Tio* P, cudaStream_t st) {
  const int threads = 128;
  const int blocks = int((p->n_inst + threads - 1) / threads);
  switch (p->order) {
    case 0: smnn::factor_kernel<1, Tio, Tc><<<blocks, threads, 0, st>>>(a, L, P); break;
    case 1: smnn::factor_kernel<2, Tio, Tc><<<blocks, threads, 0, st>>>(a, L, P); break;
    case 2: smnn::factor_kernel<3, Tio, Tc><<<blocks, threads, 0, st>>>(a, L, P); break;
    default: smnn::factor_kernel<4, Tio, Tc><<<blocks, threads, 0, st>>>(a, L, P); break;
  }
  return check_cuda(cudaGetLastError(), "factor launch");
}

template <class Tio, class Tc>
int dispatch_substitute(const smnn_problem* p, const Tio* L, const Tio* P, const Tio* al, Tio* out, cudaStream_t st) {
  const int threads = 128;
  const int blocks = int((p->n_inst + threads - 1) / threads);
  switch (p->order) {
    case 0: smnn::substitute_kernel<1, Tio, Tc><<<blocks, threads, 0, st>>>(p->n_inst, p->T, L, P, al, out); break;
    case 1: smnn::substitute_kernel<2, Tio, Tc><<<blocks, threads, 0, st>>>(p->n_inst, p->T, L, P, al, out); break;
    case 2: smnn::substitute_kernel<3, Tio, Tc><<<blocks, threads, 0, st>>>(p->n_inst, p->T, L, P, al, out); break;
    default: smnn::substitute_kernel<4, Tio, Tc><<<blocks, threads, 0, st>>>(p->n_inst, p->T, L, P, al, out); break;
  }
  return check_cuda(cudaGetLastError(), "substitute launch");
}

template <class Tio>
void set_inputs(smnn::Args<Tio>& a, const void* c, const void* d, const void* u, const void* s) {
  a.coeffs = static_cast<const Tio*>(c);
  a.rhs = static_cast<const Tio*>(d);
  a.iv = static_cast<const Tio*>(u);
  a.steps = static_cast<const Tio*>(s);
}

int need(const void* ptr, const char* name) {
  if (ptr) return SMNN_OK;
  return fail_arg(std::string(name) + " is NULL");
}

int need_steps(const smnn_problem* p, const void* s) { return p->T > 1 ? need(s, "steps") : SMNN_OK; }

}  // namespace

// info[i] = forward info if it reports a breakdown, else the backward one
__global__ void merge_info_kernel(int64_t n, const int32_t* fwd, int32_t* bwd) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && fwd[i] != 0) bwd[i] = fwd[i];
}

__global__ void widen_kernel(int64_t n, const float* __restrict__ in, double* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = double(in[i]);
}
__global__ void narrow_kernel(int64_t n, const double* __restrict__ in, float* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = float(in[i]);
}

namespace {
unsigned ew_grid(int64_t n) { return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16))); }
}  // namespace

extern "C" int smnn_factor_solve_fwd(const smnn_problem*, const void*, const void*, const void*, const void*, void*,
                                     int32_t*, void*, size_t, void*);
extern "C" int smnn_solve_bwd(const smnn_problem*, const void*, const void*, const void*, const void*, const void*,
                              const void*, void*, void*, void*, void*, int32_t*, void*, size_t, void*);

// SMNN_F32_C64 backward on a path that reads y from storage: the whole
// backward runs as SMNN_F64 on promoted copies (see promote_bwd).
static int bwd_promoted(const smnn_problem* p, const void* coeffs, const void* rhs, const void* iv, const void* steps,
                        const void* grad_y, void* gc, void* gd, void* gu, void* gs, int32_t* info, void* workspace,
                        size_t ws_bytes, cudaStream_t st) {
  const Promo o = promo_layout(p);
  double* W = static_cast<double*>(workspace);
  void* inner = W + o.end;
  const size_t inner_bytes = ws_bytes - o.end * sizeof(double);
  const int64_t n = p->n_inst, T = p->T, b = p->order + 1, ni = p->n_iv;
  const int64_t nT = n * T * b, n1 = n * T, nu = n * ni, ns = n * std::max<int64_t>(T - 1, 0);
  auto widen = [&](const void* src, size_t off, int64_t cnt) {
    if (cnt > 0) widen_kernel<<<ew_grid(cnt), 256, 0, st>>>(cnt, static_cast<const float*>(src), W + off);
  };
  widen(coeffs, o.c, nT);
  widen(rhs, o.d, n1);
  widen(iv, o.u, nu);
  if (T > 1) widen(steps, o.s, ns);
  widen(grad_y, o.gy, nT);
  int e;
  if ((e = check_cuda(cudaGetLastError(), "widen_kernel"))) return e;
  const smnn_problem q = as_f64(p);
  int32_t* info_f = reinterpret_cast<int32_t*>(W + o.info);
  if ((e = smnn_factor_solve_fwd(&q, W + o.c, W + o.d, W + o.u, W + o.s, W + o.y, info_f, inner, inner_bytes, st)))
    return e;
  if ((e = smnn_solve_bwd(&q, W + o.c, W + o.d, W + o.u, W + o.s, W + o.y, W + o.gy, gc ? W + o.gc : nullptr,
                          gd ? W + o.gd : nullptr, gu ? W + o.gu : nullptr, (gs && T > 1) ? W + o.gs : nullptr, info,
                          inner, inner_bytes, st)))
    return e;
  auto narrow = [&](void* dst, size_t off, int64_t cnt) {
    if (dst && cnt > 0) narrow_kernel<<<ew_grid(cnt), 256, 0, st>>>(cnt, W + off, static_cast<float*>(dst));
  };
  narrow(gc, o.gc, nT);
  narrow(gd, o.gd, n1);
  narrow(gu, o.gu, nu);
  if (T > 1) narrow(gs, o.gs, ns);
  if (info) merge_info_kernel<<<ew_grid(n), 256, 0, st>>>(n, info_f, info);
  return check_cuda(cudaGetLastError(), "narrow_kernel");
}

// most instance groups a host-plan call pipelines (<= smnn_plan::kMaxGroups);
// measured on the f32c64 target (tools/e2e_groups.py): 8 and 16 equal (32.0 /
// 31.7 ms per step, PCIe-bound), 32 slower (34.1 ms)
#ifndef SMNN_PLAN_GMAX
#define SMNN_PLAN_GMAX 8
#endif

struct smnn_plan {
  smnn_problem p;
  void* buf = nullptr;   // one allocation
  void *c, *d, *u, *s, *gy, *y, *gc, *gd, *gu, *gs, *ws;
  void* ylo = nullptr;  // SMNN_F32_C64: fp32 remainder of y, forward -> backward (smnn_solve_bwd_ex)
  int32_t* info;     // backward pass
  int32_t* info_f;   // forward pass (merged into info: the first breakdown wins)
  size_t ws_bytes = 0;
  // copy-in / compute / copy-out streams: instance groups are pipelined so that
  // H2D of group i+1, the kernels of group i and D2H of group i-1 overlap
  // (PCIe is full duplex; the copy engines run beside the SMs)
  cudaStream_t sin = nullptr, scomp = nullptr, sout = nullptr;
  static constexpr int kMaxGroups = 32;
  cudaEvent_t ev_start = nullptr, ev_in[kMaxGroups] = {}, ev_comp[kMaxGroups] = {}, ev_out = nullptr;
};

extern "C" {

const char* smnn_version(void) { return "smnn-b200 0.1 (sm_100a)"; }
const char* smnn_last_error(void) { return g_err.c_str(); }

int smnn_kernel_path(const smnn_problem* p, int bwd) {
  int e;
  if ((e = validate(p))) return e;
  return kernel_path(p, bwd != 0);
}

int smnn_launch_count(const smnn_problem* p, int bwd) {
  int e;
  if ((e = validate(p))) return e;
  if (bwd && promote_bwd(p)) {  // widen (c, d, u, s, dl/dy), fp64 fwd + bwd, narrow (4 gradients), merge info
    const smnn_problem q = as_f64(p);
    const int io = p->T > 1 ? 5 : 4;
    return io + smnn_launch_count(&q, 0) + smnn_launch_count(&q, 1) + (io - 1) + 1;
  }
  return kernel_path(p, bwd != 0) == SMNN_PATH_PIPE ? smnn::pipe_launches(p, bwd != 0) : 1;
}

size_t smnn_workspace_bytes(const smnn_problem* p) {
  if (validate(p) != SMNN_OK) return 0;
  return workspace_bytes(p);
}

int smnn_assemble(const smnn_problem* p, const void* coeffs, const void* rhs, const void* iv, const void* steps,
                  void* M_diag, void* N_sub, void* beta, void* stream) {
  int e;
  if ((e = validate(p)) || (e = need(coeffs, "coeffs")) || (e = need(rhs, "rhs")) || (e = need(iv, "iv")) ||
      (e = need_steps(p, steps)) || (e = need(M_diag, "M_diag")) || (e = need(beta, "beta")) ||
      (p->T > 1 && (e = need(N_sub, "N_sub"))))
    return e;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->dtype == SMNN_F64) {
    auto a = make_args<double>(p);
    set_inputs(a, coeffs, rhs, iv, steps);
    return dispatch_assemble<double, double>(p, a, (double*)M_diag, (double*)N_sub, (double*)beta, st);
  }
  auto a = make_args<float>(p);
  set_inputs(a, coeffs, rhs, iv, steps);
  if (p->dtype == SMNN_F32) return dispatch_assemble<float, float>(p, a, (float*)M_diag, (float*)N_sub, (float*)beta, st);
  return dispatch_assemble<float, double>(p, a, (float*)M_diag, (float*)N_sub, (float*)beta, st);
}

int smnn_ylo_used(const smnn_problem* p) {
  int e;
  if ((e = validate(p))) return e;
  return ylo_used(p) ? 1 : 0;
}

int smnn_factor_solve_fwd(const smnn_problem* p, const void* coeffs, const void* rhs, const void* iv,
                          const void* steps, void* y, int32_t* info, void* workspace, size_t workspace_bytes_,
                          void* stream) {
  return smnn_factor_solve_fwd_ex(p, coeffs, rhs, iv, steps, y, nullptr, info, workspace, workspace_bytes_, stream);
}

int smnn_factor_solve_fwd_ex(const smnn_problem* p, const void* coeffs, const void* rhs, const void* iv,
                             const void* steps, void* y, void* y_lo, int32_t* info, void* workspace,
                             size_t workspace_bytes_, void* stream) {
  int e;
  if ((e = validate(p)) || (e = need(coeffs, "coeffs")) || (e = need(rhs, "rhs")) || (e = need(iv, "iv")) ||
      (e = need_steps(p, steps)) || (e = need(y, "y")))
    return e;
  const size_t wsn = workspace_bytes(p);
  if (workspace_bytes_ < wsn || (!workspace && wsn > 0)) {
    g_err = "workspace too small: need " + std::to_string(wsn) + " bytes";
    return SMNN_ERR_WORKSPACE;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->dtype == SMNN_F64) {
    auto a = make_args<double>(p);
    set_inputs(a, coeffs, rhs, iv, steps);
    a.y_out = (double*)y; a.info = info; a.ckpt = workspace;
    return dispatch_fused<double, double, false>(p, a, st);
  }
  auto a = make_args<float>(p);
  set_inputs(a, coeffs, rhs, iv, steps);
  a.y_out = (float*)y; a.info = info; a.ckpt = workspace;
  if (p->dtype == SMNN_F32) return dispatch_fused<float, float, false>(p, a, st);
  if (y_lo && !ylo_used(p)) {  // not this path's: y_lo = 0 (y_hi + y_lo = y_hi stays a valid pair)
    const size_t nb = size_t(p->n_inst) * size_t(p->T) * size_t(p->order + 1) * sizeof(float);
    if ((e = check_cuda(cudaMemsetAsync(y_lo, 0, nb, st), "y_lo clear"))) return e;
  } else {
    a.y_lo_out = static_cast<float*>(y_lo);
  }
  return dispatch_fused<float, double, false>(p, a, st);
}

int smnn_solve_bwd(const smnn_problem* p, const void* coeffs, const void* rhs, const void* iv, const void* steps,
                   const void* y, const void* grad_y, void* grad_coeffs, void* grad_rhs, void* grad_iv,
                   void* grad_steps, int32_t* info, void* workspace, size_t workspace_bytes_, void* stream) {
  return smnn_solve_bwd_ex(p, coeffs, rhs, iv, steps, y, nullptr, grad_y, grad_coeffs, grad_rhs, grad_iv, grad_steps,
                           info, workspace, workspace_bytes_, stream);
}

int smnn_solve_bwd_ex(const smnn_problem* p, const void* coeffs, const void* rhs, const void* iv, const void* steps,
                      const void* y, const void* y_lo, const void* grad_y, void* grad_coeffs, void* grad_rhs,
                      void* grad_iv, void* grad_steps, int32_t* info, void* workspace, size_t workspace_bytes_,
                      void* stream) {
  int e;
  if ((e = validate(p)) || (e = need(coeffs, "coeffs")) || (e = need(rhs, "rhs")) || (e = need(iv, "iv")) ||
      (e = need_steps(p, steps)) || (e = need(y, "y")) || (e = need(grad_y, "grad_y")))
    return e;
  const size_t wsn = workspace_bytes(p);
  if (workspace_bytes_ < wsn || (!workspace && wsn > 0)) {
    g_err = "workspace too small: need " + std::to_string(wsn) + " bytes";
    return SMNN_ERR_WORKSPACE;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->dtype == SMNN_F64) {
    auto a = make_args<double>(p);
    set_inputs(a, coeffs, rhs, iv, steps);
    a.y_in = (const double*)y; a.grad_y = (const double*)grad_y;
    a.g_coeffs = (double*)grad_coeffs; a.g_rhs = (double*)grad_rhs; a.g_iv = (double*)grad_iv;
    a.g_steps = p->T > 1 ? (double*)grad_steps : nullptr; a.info = info; a.ckpt = workspace;
    return dispatch_fused<double, double, true>(p, a, st);
  }
  if (y_lo && ylo_used(p)) {  // one right-hand side: y = y_hi + y_lo read, not re-solved
    auto a = make_args<float>(p);
    set_inputs(a, coeffs, rhs, iv, steps);
    a.y_in = (const float*)y; a.y_lo_in = (const float*)y_lo; a.grad_y = (const float*)grad_y;
    a.g_coeffs = (float*)grad_coeffs; a.g_rhs = (float*)grad_rhs; a.g_iv = (float*)grad_iv;
    a.g_steps = p->T > 1 ? (float*)grad_steps : nullptr; a.info = info; a.ckpt = workspace;
    return dispatch_fused<float, double, true>(p, a, st);
  }
  if (promote_bwd(p))
    return bwd_promoted(p, coeffs, rhs, iv, steps, grad_y, grad_coeffs, grad_rhs, grad_iv, grad_steps, info, workspace,
                        workspace_bytes_, st);
  auto a = make_args<float>(p);
  set_inputs(a, coeffs, rhs, iv, steps);
  a.y_in = (const float*)y; a.grad_y = (const float*)grad_y;
  a.g_coeffs = (float*)grad_coeffs; a.g_rhs = (float*)grad_rhs; a.g_iv = (float*)grad_iv;
  a.g_steps = p->T > 1 ? (float*)grad_steps : nullptr; a.info = info; a.ckpt = workspace;
  if (p->dtype == SMNN_F32) return dispatch_fused<float, float, true>(p, a, st);
  return dispatch_fused<float, double, true>(p, a, st);
}

int smnn_factor(const smnn_problem* p, const void* coeffs, const void* steps, void* L, void* P, int32_t* info,
                void* stream) {
  int e;
  if ((e = validate(p)) || (e = need(coeffs, "coeffs")) || (e = need_steps(p, steps)) || (e = need(L, "L")) ||
      (p->T > 1 && (e = need(P, "P"))))
    return e;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->dtype == SMNN_F64) {
    auto a = make_args<double>(p);
    set_inputs(a, coeffs, nullptr, nullptr, steps);
    a.info = info;
    return dispatch_factor<double, double>(p, a, (double*)L, (double*)P, st);
  }
  auto a = make_args<float>(p);
  set_inputs(a, coeffs, nullptr, nullptr, steps);
  a.info = info;
  if (p->dtype == SMNN_F32) return dispatch_factor<float, float>(p, a, (float*)L, (float*)P, st);
  return dispatch_factor<float, double>(p, a, (float*)L, (float*)P, st);
}

int smnn_substitute(const smnn_problem* p, const void* L, const void* P, const void* alpha, void* out,
                    void* stream) {
  int e;
  if ((e = validate(p)) || (e = need(L, "L")) || (p->T > 1 && (e = need(P, "P"))) || (e = need(alpha, "alpha")) ||
      (e = need(out, "out")))
    return e;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->dtype == SMNN_F64)
    return dispatch_substitute<double, double>(p, (const double*)L, (const double*)P, (const double*)alpha,
                                               (double*)out, st);
  if (p->dtype == SMNN_F32)
    return dispatch_substitute<float, float>(p, (const float*)L, (const float*)P, (const float*)alpha, (float*)out, st);
  return dispatch_substitute<float, double>(p, (const float*)L, (const float*)P, (const float*)alpha, (float*)out, st);
}

int smnn_plan_create(smnn_plan** plan, const smnn_problem* p) {
  int e;
  if (!plan) return fail_arg("plan is NULL");
  if ((e = validate(p))) return e;
  smnn_plan* q = new smnn_plan();
  q->p = *p;
  const size_t es = p->dtype == SMNN_F64 ? 8 : 4;
  const size_t n = size_t(p->n_inst), T = size_t(p->T), b = size_t(p->order + 1);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t sz_c = al(n * T * b * es), sz_d = al(n * T * es), sz_u = al(n * p->n_iv * es),
               sz_s = al(n * std::max<size_t>(T - 1, 1) * es), sz_info = al(n * 4);
  q->ws_bytes = al(workspace_bytes(p));
  const bool c64 = p->dtype == SMNN_F32_C64;
  const size_t total = (c64 ? 5 : 4) * sz_c + 2 * sz_d + 2 * sz_u + 2 * sz_s + 2 * sz_info + q->ws_bytes;
  if ((e = check_cuda(cudaMalloc(&q->buf, total), "cudaMalloc(plan)"))) { delete q; return e; }
  char* ptr = static_cast<char*>(q->buf);
  auto take = [&](size_t s) { void* r = ptr; ptr += s; return r; };
  q->c = take(sz_c); q->gy = take(sz_c); q->y = take(sz_c); q->gc = take(sz_c);
  if (c64) q->ylo = take(sz_c);
  q->d = take(sz_d); q->gd = take(sz_d);
  q->u = take(sz_u); q->gu = take(sz_u);
  q->s = take(sz_s); q->gs = take(sz_s);
  q->info = static_cast<int32_t*>(take(sz_info));
  q->info_f = static_cast<int32_t*>(take(sz_info));
  q->ws = take(q->ws_bytes);
  const unsigned fl = cudaStreamNonBlocking;
  if ((e = check_cuda(cudaStreamCreateWithFlags(&q->sin, fl), "stream")) ||
      (e = check_cuda(cudaStreamCreateWithFlags(&q->scomp, fl), "stream")) ||
      (e = check_cuda(cudaStreamCreateWithFlags(&q->sout, fl), "stream")) ||
      (e = check_cuda(cudaEventCreateWithFlags(&q->ev_start, cudaEventDisableTiming), "event")) ||
      (e = check_cuda(cudaEventCreateWithFlags(&q->ev_out, cudaEventDisableTiming), "event"))) {
    smnn_plan_destroy(q);
    return e;
  }
  for (int i = 0; i < smnn_plan::kMaxGroups; ++i)
    if ((e = check_cuda(cudaEventCreateWithFlags(&q->ev_in[i], cudaEventDisableTiming), "event")) ||
        (e = check_cuda(cudaEventCreateWithFlags(&q->ev_comp[i], cudaEventDisableTiming), "event"))) {
      smnn_plan_destroy(q);
      return e;
    }
  *plan = q;
  return SMNN_OK;
}

int smnn_plan_destroy(smnn_plan* plan) {
  if (!plan) return SMNN_OK;
  for (cudaStream_t st : {plan->sin, plan->scomp, plan->sout})
    if (st) cudaStreamDestroy(st);
  for (cudaEvent_t ev : {plan->ev_start, plan->ev_out})
    if (ev) cudaEventDestroy(ev);
  for (int i = 0; i < smnn_plan::kMaxGroups; ++i) {
    if (plan->ev_in[i]) cudaEventDestroy(plan->ev_in[i]);
    if (plan->ev_comp[i]) cudaEventDestroy(plan->ev_comp[i]);
  }
  int e = check_cuda(cudaFree(plan->buf), "cudaFree(plan)");
  delete plan;
  return e;
}

int smnn_plan_fwd_bwd_host(smnn_plan* q, const void* coeffs, const void* rhs, const void* iv, const void* steps,
                           const void* grad_y, void* y, void* grad_coeffs, void* grad_rhs, void* grad_iv,
                           void* grad_steps, int32_t* info, void* stream) {
  int e;
  if (!q) return fail_arg("plan is NULL");
  const smnn_problem* p = &q->p;
  if ((e = need(coeffs, "coeffs")) || (e = need(rhs, "rhs")) || (e = need(iv, "iv")) || (e = need_steps(p, steps)) ||
      (e = need(grad_y, "grad_y")) || (e = need(y, "y")))
    return e;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t es = p->dtype == SMNN_F64 ? 8 : 4;
  const int64_t n = p->n_inst;
  const size_t T = size_t(p->T), b = size_t(p->order + 1), niv = size_t(p->n_iv);
  const cudaMemcpyKind h2d = cudaMemcpyHostToDevice, d2h = cudaMemcpyDeviceToHost;
  // groups of instances, each large enough to keep the GPU busy on its own
  // one group per ~16 MiB of input, 1..8 groups (measured on B200: Lorenz,
  // 49 MB in, best at 2 groups; the 1.3 GB target best at 8)
  const size_t in_bytes = size_t(n) * T * (2 * b + 2) * es;
  const int Gmax = int(std::max<size_t>(1, std::min<size_t>(SMNN_PLAN_GMAX, in_bytes >> 24)));
  const int G = int(std::max<int64_t>(1, std::min<int64_t>(Gmax, n / 64)));
  auto H = [](const void* base, size_t off) { return static_cast<const char*>(base) + off; };
  auto Hm = [](void* base, size_t off) { return static_cast<char*>(base) + off; };
  auto D = [](void* base, size_t off) { return static_cast<char*>(base) + off; };
  // Order after the caller's stream AND after this plan's previous call (which
  // may have run on another stream): its copies and kernels use the same
  // device buffers.  ev_out was recorded at the end of that call (waiting on a
  // never-recorded event is a no-op).
  if ((e = check_cuda(cudaEventRecord(q->ev_start, st), "event")) ||
      (e = check_cuda(cudaStreamWaitEvent(q->sin, q->ev_out, 0), "wait")) ||
      (e = check_cuda(cudaStreamWaitEvent(q->sin, q->ev_start, 0), "wait")) ||
      (e = check_cuda(cudaStreamWaitEvent(q->scomp, q->ev_start, 0), "wait")) ||
      (e = check_cuda(cudaStreamWaitEvent(q->sout, q->ev_start, 0), "wait")))
    return e;
  for (int gi = 0; gi < G; ++gi) {
    const int64_t i0 = n * gi / G, i1 = n * (gi + 1) / G, ni = i1 - i0;
    const size_t oc = size_t(i0) * T * b * es, od = size_t(i0) * T * es, ou = size_t(i0) * niv * es,
                 os = size_t(i0) * (T - 1) * es;
    const size_t bc = size_t(ni) * T * b * es, bd = size_t(ni) * T * es, bu = size_t(ni) * niv * es,
                 bs = size_t(ni) * (T - 1) * es;
    if ((e = check_cuda(cudaMemcpyAsync(D(q->c, oc), H(coeffs, oc), bc, h2d, q->sin), "H2D coeffs")) ||
        (e = check_cuda(cudaMemcpyAsync(D(q->d, od), H(rhs, od), bd, h2d, q->sin), "H2D rhs")) ||
        (e = check_cuda(cudaMemcpyAsync(D(q->u, ou), H(iv, ou), bu, h2d, q->sin), "H2D iv")) ||
        (bs && (e = check_cuda(cudaMemcpyAsync(D(q->s, os), H(steps, os), bs, h2d, q->sin), "H2D steps"))) ||
        (e = check_cuda(cudaMemcpyAsync(D(q->gy, oc), H(grad_y, oc), bc, h2d, q->sin), "H2D grad_y")) ||
        (e = check_cuda(cudaEventRecord(q->ev_in[gi], q->sin), "event")) ||
        (e = check_cuda(cudaStreamWaitEvent(q->scomp, q->ev_in[gi], 0), "wait")))
      return e;
    smnn_problem pg = *p;
    pg.n_inst = ni;
    void* ylo = q->ylo ? D(q->ylo, oc) : nullptr;
    if ((e = smnn_factor_solve_fwd_ex(&pg, D(q->c, oc), D(q->d, od), D(q->u, ou), D(q->s, os), D(q->y, oc), ylo,
                                      q->info_f + i0, q->ws, q->ws_bytes, q->scomp)))
      return e;
    if ((e = smnn_solve_bwd_ex(&pg, D(q->c, oc), D(q->d, od), D(q->u, ou), D(q->s, os), D(q->y, oc), ylo, D(q->gy, oc),
                            D(q->gc, oc), D(q->gd, od), D(q->gu, ou), D(q->gs, os),
                            q->info + i0, q->ws, q->ws_bytes, q->scomp)))
      return e;
    if (ni > 0) {
      merge_info_kernel<<<unsigned((ni + 255) / 256), 256, 0, q->scomp>>>(ni, q->info_f + i0, q->info + i0);
      if ((e = check_cuda(cudaGetLastError(), "merge_info_kernel"))) return e;
    }
    if ((e = check_cuda(cudaEventRecord(q->ev_comp[gi], q->scomp), "event")) ||
        (e = check_cuda(cudaStreamWaitEvent(q->sout, q->ev_comp[gi], 0), "wait")) ||
        (e = check_cuda(cudaMemcpyAsync(Hm(y, oc), D(q->y, oc), bc, d2h, q->sout), "D2H y")))
      return e;
    if (grad_coeffs && (e = check_cuda(cudaMemcpyAsync(Hm(grad_coeffs, oc), D(q->gc, oc), bc, d2h, q->sout), "D2H dc")))
      return e;
    if (grad_rhs && (e = check_cuda(cudaMemcpyAsync(Hm(grad_rhs, od), D(q->gd, od), bd, d2h, q->sout), "D2H dd")))
      return e;
    if (grad_iv && (e = check_cuda(cudaMemcpyAsync(Hm(grad_iv, ou), D(q->gu, ou), bu, d2h, q->sout), "D2H du")))
      return e;
    if (grad_steps && bs &&
        (e = check_cuda(cudaMemcpyAsync(Hm(grad_steps, os), D(q->gs, os), bs, d2h, q->sout), "D2H ds")))
      return e;
    if (info && (e = check_cuda(cudaMemcpyAsync(info + i0, q->info + i0, size_t(ni) * 4, d2h, q->sout), "D2H info")))
      return e;
  }
  // the caller's stream resumes after the last copy-out
  if ((e = check_cuda(cudaEventRecord(q->ev_out, q->sout), "event")) ||
      (e = check_cuda(cudaStreamWaitEvent(st, q->ev_out, 0), "wait")))
    return e;
  return SMNN_OK;
}

}  // extern "C"
