// smnn_rf_host.h -- entry of the register-factor resident kernel (smnn_rf.cu).
#pragma once

#include <cuda_runtime.h>

#include <stdint.h>

#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "smnn.h"

namespace smnn {

// Raise a kernel's dynamic shared-memory limit to at least `smem` on the
// CURRENT device (the attribute is per device; the cache is keyed by
// (device, kernel) and keeps the largest request made so far).
inline cudaError_t ensure_smem(const void* kern, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> top;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& t = top[std::make_pair(dev, kern)];
  if (smem <= t) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e == cudaSuccess) t = smem;
  return e;
}
template <class Kern>
cudaError_t ensure_smem_k(Kern* k, size_t smem) {
  return ensure_smem(reinterpret_cast<const void*>(k), smem);
}

// Arguments of the fused kernels (device pointers; see include/smnn.h).
template <class Tio>
struct Args {
  const Tio* coeffs;
  const Tio* rhs;
  const Tio* iv;
  const Tio* steps;
  const Tio* y_in;     // BWD: forward solution
  const Tio* grad_y;   // BWD: dl/dy
  Tio* y_out;          // FWD: solution
  Tio* y_lo_out;       // FWD, SMNN_F32_C64 pipeline: fp32 remainder y - (double)y_out (nullable)
  const Tio* y_lo_in;  // BWD, SMNN_F32_C64 pipeline: that remainder (nullable: y re-solved)
  Tio* g_coeffs;       // BWD outputs (nullable)
  Tio* g_rhs;
  Tio* g_iv;
  Tio* g_steps;
  int32_t* info;       // nullable
  void* ckpt;          // workspace, one slot per block
  int64_t n_inst;
  int T;
  int n_iv;
  int K;               // chunks per instance (<= blockDim.x)
  int nseg_ck;         // checkpoints per chunk (slot stride)
  double wg2, wi2, ws2;
};

// Launches the RF kernel for `p` (forward or backward) when the problem fits
// it (instance resident in shared memory, chunks within the register budget).
// Returns 1 when launched, 0 when not eligible (caller falls back), or a
// negative SMNN_ERR_* code with `err` set.
template <class Tio, class Tc>
int rf_launch(const smnn_problem* p, const Args<Tio>& a, bool bwd, cudaStream_t st, std::string& err);

// Three-kernel pipeline (smnn_pipe.cu): same contract as rf_launch; its
// workspace (separator blocks, separator solution, chunk failure flags) is
// carved from Args::ckpt, which must hold pipe_workspace_bytes(p).
template <class Tio, class Tc>
int pipe_launch(const smnn_problem* p, const Args<Tio>& a, bool bwd, cudaStream_t st, std::string& err);
size_t pipe_workspace_bytes(const smnn_problem* p);

// Whether rf_launch / pipe_launch would take the problem (no launch).
bool rf_eligible(const smnn_problem* p, bool bwd);
bool pipe_eligible(const smnn_problem* p, bool bwd);
bool pipe_ylo_eligible(const smnn_problem* p);  // SMNN_F32_C64: forward writes / backward reads y_lo
int pipe_launches(const smnn_problem* p, bool bwd);  // 3 + 2 per separator-hierarchy level

// Cluster-resident fp64-arithmetic path (smnn_x64.cu): SMNN_F32_C64 and
// SMNN_F64 while one cluster of <= 16 CTAs holds an instance.  Same contract
// as rf_launch; no workspace.
template <class Tio>
int x64_launch(const smnn_problem* p, const Args<Tio>& a, bool bwd, cudaStream_t st, std::string& err);
bool x64_eligible(const smnn_problem* p, bool bwd);

}  // namespace smnn
