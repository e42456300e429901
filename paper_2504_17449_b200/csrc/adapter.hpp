// SPDX-License-Identifier: Apache-2.0
// Adapter fold (adapter.cu): registration-time re-association of the down projection onto
// the attention context, ctx.(Wo.Wd) + (bo.Wd + bd).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "host_util.hpp"

namespace hmi_b200 {

// n_images slot images of slot_bytes each at `in` (device): image s is layer s % L of a task.
// Writes Wc^T [r_pad][d] 16-bit at offset 0 and bc [r_pad] f32 at off_bd of the matching
// image in `out` (other bytes of `out` untouched). wo: [L][d][d] f32 row-major [in][out]
// (the reference's Wo), bo: [L][d].
void launch_adapter_fold(const uint8_t* in, uint8_t* out, int n_images, const float* wo,
                         const float* bo, int L, int d, int r_pad, size_t slot_bytes,
                         size_t off_bd, int precision, cudaStream_t stream);

}  // namespace hmi_b200
