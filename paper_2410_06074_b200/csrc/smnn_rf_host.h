// smnn_rf_host.h -- entry of the register-factor resident kernel (smnn_rf.cu).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "smnn.h"

namespace smnn {

template <class Tio>
struct Args;

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

}  // namespace smnn
