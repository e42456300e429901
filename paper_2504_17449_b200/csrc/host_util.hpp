// SPDX-License-Identifier: Apache-2.0
//
// Host-side helpers shared by the launchers: CUDA error -> status mapping,
// thread-local error text, and TMA tensor-map encoding through the driver
// entry point (no link-time dependency on libcuda).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/hmi_gpu.h"

namespace hmi_b200 {

// Exception carrying an hmi status code; caught at the C-ABI boundary.
struct HmiError : std::runtime_error {
  int code;
  HmiError(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

void set_last_error(const std::string& msg);

#define HMI_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess) {                                                            \
      throw ::hmi_b200::HmiError(HMI_CUDA_ERROR, std::string(#call) + ": " +           \
                                                    cudaGetErrorString(_e) + " at " +   \
                                                    __FILE__ + ":" + std::to_string(__LINE__)); \
    }                                                                                   \
  } while (0)

#define HMI_CHECK(cond, code, msg)                          \
  do {                                                      \
    if (!(cond)) throw ::hmi_b200::HmiError((code), (msg)); \
  } while (0)

inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || p == nullptr) {
      throw HmiError(HMI_CUDA_ERROR, "cuTensorMapEncodeTiled entry point unavailable");
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// cuStreamWriteValue32 (stream memory operations), or null when the driver does not offer it.
using StreamWriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
inline StreamWriteValue32Fn stream_write_value32() {
  static StreamWriteValue32Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    const cudaError_t e = cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess) {
      (void)cudaGetLastError();
      return static_cast<StreamWriteValue32Fn>(nullptr);
    }
    return reinterpret_cast<StreamWriteValue32Fn>(p);
  }();
  return fn;
}

// Row-major 2-D tensor [rows][cols] with an explicit row pitch (bytes).
inline CUtensorMap make_tmap_2d(const void* base, CUtensorMapDataType dtype, uint64_t cols,
                                uint64_t rows, uint64_t row_pitch_bytes, uint32_t box_cols,
                                uint32_t box_rows, CUtensorMapSwizzle swz) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_pitch_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = tmap_encoder()(&m, dtype, 2, const_cast<void*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw HmiError(HMI_CUDA_ERROR, "cuTensorMapEncodeTiled(2d) failed: " + std::to_string(r));
  }
  return m;
}

// [groups][rows][cols] with explicit row pitch and group stride (bytes).
inline CUtensorMap make_tmap_3d(const void* base, CUtensorMapDataType dtype, uint64_t cols,
                                uint64_t rows, uint64_t groups, uint64_t row_pitch_bytes,
                                uint64_t group_stride_bytes, uint32_t box_cols,
                                uint32_t box_rows, CUtensorMapSwizzle swz) {
  CUtensorMap m;
  cuuint64_t dims[3] = {cols, rows, groups};
  cuuint64_t strides[2] = {row_pitch_bytes, group_stride_bytes};
  cuuint32_t box[3] = {box_cols, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = tmap_encoder()(&m, dtype, 3, const_cast<void*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw HmiError(HMI_CUDA_ERROR, "cuTensorMapEncodeTiled(3d) failed: " + std::to_string(r));
  }
  return m;
}

// Launch with programmatic stream serialization (the kernel may begin before its predecessor
// in the stream completes; it must griddepcontrol.wait before reading that predecessor's
// outputs). HMI_PDL=0 launches normally.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args&&... args) {
  static const bool on = std::getenv("HMI_PDL") == nullptr || std::string(std::getenv("HMI_PDL")) != "0";
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = on ? 1 : 0;
  HMI_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

inline int device_sm_count() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

}  // namespace hmi_b200
