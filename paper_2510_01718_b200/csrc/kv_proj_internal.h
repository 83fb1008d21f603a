// kv_proj_internal.h — launchers shared between the kernels and the C ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "../../include/bd_kv_proj.h"

namespace bdk {

// Thread-local error text set by the launchers; returned by bd_last_error().
void set_error(const std::string& msg);

// Counts kernel launches for the bench's gpu_launches evidence.
void note_launch();

// Exact SIMT kernel (FP32/FP64): reference rounding sequence (attention.py:258-270).
cudaError_t launch_exact(const bd_kv_problem* probs, int count, int dtype, int* flag,
                         cudaStream_t stream);

// tcgen05 tensor-core kernel (FP16/BF16). Returns BD_* status; sets error text.
int launch_tc(const bd_kv_problem* probs, int count, int dtype, int* flag, cudaStream_t stream);

// SM count of the current device (cached).
int sm_count();

}  // namespace bdk
