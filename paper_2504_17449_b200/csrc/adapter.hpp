// SPDX-License-Identifier: Apache-2.0
// Host interface of the fused per-tenant adapter kernel (adapter.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "host_util.hpp"

namespace hmi_b200 {

struct AdapterMaps {
  CUtensorMap a, h, out, wd, wu;
};

struct AdapterArgs {
  int M = 0, num_m_tiles = 0, d = 0;
  const int* tile_slot = nullptr;   // per 128-row tile: HBM slot of that request's (task, layer)
  const float* bd = nullptr;        // slot 0's down bias; slot s at + s * slot_floats
  const float* bu = nullptr;        // slot 0's up bias
  long long slot_floats = 0;
  float2* stats_out = nullptr;      // per (row, column half) partial (sum, sumsq) of y1
  int stats_ld = 0;
  const float2* r_stats = nullptr;  // partial stats of the pre-norm residual h (null: h is final)
  int r_stats_n = 0, r_stats_ld = 0;
  const float* r_gamma = nullptr;   // LN applied to h on the fly
  const float* r_beta = nullptr;
  float inv_n = 0.f;
  // fine pipeline: this layer's adapter slots are resident once *ready >= ready_seq (written
  // by the copy stream after the layer's H2D copies, cuStreamWriteValue32); null: no wait
  const uint32_t* ready = nullptr;
  uint32_t ready_seq = 0;
  int32_t* err = nullptr;           // HMI_SCHEDULING_BUG if the flag never arrives
};

struct AdapterSpec {
  const void* a = nullptr;    // [rows][d] 16-bit attention output (after Wo, bo)
  const void* h = nullptr;    // [rows][d] 16-bit layer input (pre-norm when r_stats)
  void* out = nullptr;        // [rows][d] 16-bit y1 (pre-LN1)
  const uint8_t* arena = nullptr;  // slot arena
  size_t slot_bytes = 0, off_wu = 0, off_bd = 0, off_bu = 0;
  int n_slots = 0, d = 0, r_pad = 0, rows = 0, precision = 0;
  const int* tile_slot = nullptr;
  float2* stats_out = nullptr;
  int stats_ld = 0;
  const float2* r_stats = nullptr;
  int r_stats_n = 0;
  const float* r_gamma = nullptr;
  const float* r_beta = nullptr;
};

struct AdapterPlan {
  AdapterMaps maps;
  AdapterArgs args;
  int precision = 0;
  int max_rows = 0;
};

AdapterPlan make_adapter_plan(const AdapterSpec& s);
void launch_adapter(const AdapterPlan& p, int rows, cudaStream_t stream,
                    const uint32_t* ready = nullptr, uint32_t ready_seq = 0, int32_t* err = nullptr);

}  // namespace hmi_b200
