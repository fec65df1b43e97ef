// How many tcgen05.mma instructions can be in flight before issue blocks:
// one thread issues 32 MMAs (M = 128, N, K = 16, SS) back to back and stamps
// clock64 after each; a flat then linear stamp curve shows the queue depth.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_mma_queue tools/mma_queue.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2204_10319_b200/csrc/sm100_ptx.cuh"

using namespace scb::ptx;

__global__ void queue(int n, long long* out, int with_commit) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, spare;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&spare, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = slot;
  long long st[33];
  if (threadIdx.x == 0) {
    const uint64_t ad = make_sdesc(smem_u32(smem), 8u * 128, 2u);
    const uint64_t bd = make_sdesc(smem_u32(smem + 16384), 8u * 128, 2u);
    const uint32_t idesc = (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    st[0] = clock64();
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      mma_f16(tmem, ad + 2u * (k & 3), bd + 2u * (k & 3), idesc, k ? 1u : 0u);
      if (with_commit && (k % 4) == 3) mma_commit(&spare);
      st[k + 1] = clock64();
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long end = clock64();
    if (blockIdx.x == 0) {
      for (int k = 0; k <= 32; ++k) out[k] = st[k] - st[0];
      out[33] = end - st[0];
    }
  }
  tc_before();
  __syncthreads();
  if (warp == 0) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  cudaFuncSetAttribute(queue, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int n : {96, 256})
    for (int c : {0, 1}) {
      queue<<<148, 128, 100 * 1024>>>(n, d, c);
      cudaDeviceSynchronize();
      long long h[34];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("N=%d commit/4=%d issue stamps:", n, c);
      for (int k = 1; k <= 32; ++k) printf(" %lld", h[k]);
      printf(" | done %lld\n", h[33]);
    }
  return 0;
}
