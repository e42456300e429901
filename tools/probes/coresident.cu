// Can a 0-smem kernel on a second stream run while a 148-CTA, ~214 KB-smem kernel spins on
// every SM waiting for it?  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cor tools/probes/coresident.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void spinner(volatile unsigned* flag, unsigned* timed_out, unsigned long long budget_ns) {
  extern __shared__ unsigned char sm[];
  sm[threadIdx.x] = 1;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (threadIdx.x == 0) {
    while (*flag == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > budget_ns) { atomicExch(timed_out, 1u); break; }
      __nanosleep(256);
    }
  }
  __syncthreads();
}

__global__ void setter(unsigned* flag) {
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) { __threadfence_system(); atomicExch(flag, 1u); }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *flag, *to;
  cudaMalloc(&flag, 4); cudaMalloc(&to, 4);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  const int smem = 214 * 1024;
  cudaFuncSetAttribute(spinner, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 2; ++mode) {
    if (mode == 1) cudaFuncSetAttribute(setter, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    for (int grid : {16, 148}) {
      cudaMemset(flag, 0, 4); cudaMemset(to, 0, 4);
      cudaDeviceSynchronize();
      spinner<<<sms, 320, smem, a>>>(flag, to, 2000000000ull);
      setter<<<grid, 128, 0, b>>>(flag);
      cudaDeviceSynchronize();
      unsigned h = 0; cudaMemcpy(&h, to, 4, cudaMemcpyDeviceToHost);
      printf("carveout_hint=%d setter_grid=%d -> %s (%s)\n", mode, grid, h ? "TIMED OUT (not co-resident)" : "co-resident",
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
