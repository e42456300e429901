/* SPDX-License-Identifier: Apache-2.0
 *
 * hmi_gpu.h — C ABI of the B200-native batched multi-tenant hPLM forward pass.
 *
 * This is the drop-in boundary under the reference's C++ serving API. The
 * reference (proj/, C++20, CPU only) has no GPU backend; its SPEC defines a
 * scheduler `Backend` of kind {numeric, simulated} used by `stage_compute`
 * (SPEC.md:425-428, :461-469). This ABI is the third kind, `cuda`: the host
 * engine (paper_2504_17449_b200/host, or any C/C++/ctypes caller) registers
 * artefacts once and calls hmi_gpu_infer_batch() once per batch.
 *
 * Conventions
 *   - Plain pointers and sizes only; caller buffers are borrowed for the call.
 *   - Every entry point returns an int status (HMI_OK or an error class below).
 *     Status codes map 1:1 onto the reference's exception classes
 *     (proj/include/hmi/errors.hpp:10-68); hmi_gpu_last_error() returns the
 *     thread-local message. No exception crosses the ABI.
 *   - One context per GPU. hmi_gpu_infer_batch is not reentrant per context
 *     (one scheduler drains the queue); registration calls take a
 *     context mutex and apply between batches.
 *   - Float artefacts are passed exactly as stored in the reference's files:
 *     f32, row-major, declaration order (HMI1 model_io.cpp:19-36, ADP1
 *     adapter_set.cpp:38-43, PLT1 plot_io.cpp:17-33).
 */
#ifndef HMI_GPU_H_
#define HMI_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:10-68) ------------------------------------ */
#define HMI_OK 0
#define HMI_DIMENSION_ERROR 1   /* DimensionError      errors.hpp:11  */
#define HMI_VOCABULARY_ERROR 2  /* VocabularyError     errors.hpp:17  */
#define HMI_CONFLICT_ERROR 3    /* ConflictError       errors.hpp:23  */
#define HMI_CAPACITY_ERROR 4    /* CapacityError       errors.hpp:29  */
#define HMI_ROUTING_ERROR 5     /* RoutingError        errors.hpp:35  */
#define HMI_CONFIG_ERROR 6      /* ConfigError         errors.hpp:40  */
#define HMI_BUILD_ERROR 7       /* BuildError          errors.hpp:46  */
#define HMI_SCHEDULING_BUG 8    /* SchedulingBugError  errors.hpp:53  */
#define HMI_FORMAT_ERROR 9      /* FormatError         errors.hpp:59  */
#define HMI_CUDA_ERROR 100      /* CUDA runtime / driver failure        */

/* Thread-local text of the last failing call on this thread. */
const char* hmi_gpu_last_error(void);

/* ---- standalone kernel probe (K1/K2 GEMM) ------------------------------ */
/* C[M x N] = epi(A[M x K] . B[g]^T + bias[g]) for a device-side tcgen05 GEMM,
 * host buffers in/out, used by the parity tests of the GEMM kernel alone.
 *   a16      : M*K 16-bit (fp16 or bf16 bits per `precision`)
 *   b16      : groups*N*K 16-bit, B stored [g][N][K] (i.e. W^T)
 *   bias     : groups*N f32
 *   tile_slot: M/128 ints selecting the group of each 128-row tile, or NULL
 *   res0/res1: optional M*N 16-bit residuals (epi flags 2/4)
 *   epi      : bit0 ReLU, bit1 +res0, bit2 +res0+res1, bit3 f32 output
 *   bn       : N-tile width (64, 128, 192 or 256)
 *   out      : M*N, 16-bit or f32 per epi bit3
 *   elapsed_ms (nullable): device time of one launch (CUDA events)        */
int hmi_gpu_gemm_probe(int device, int M, int N, int K, int groups, const uint16_t* a16,
                       const uint16_t* b16, const float* bias, const int32_t* tile_slot,
                       const uint16_t* res0, const uint16_t* res1, int epi, int bn,
                       int precision, void* out, float* elapsed_ms);

#ifdef __cplusplus
}
#endif

#endif /* HMI_GPU_H_ */
