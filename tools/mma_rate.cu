// tcgen05.mma throughput probe (B200): one elected thread per CTA issues
// `rounds` bursts of U back-to-back MMAs (fully unrolled, no waits inside a
// burst; one commit per burst), M = 128, K = 16, kind::f16, for several N,
// with A from shared memory (SS) or from TMEM (TS), 1 or 2 CTAs per SM.
// Prints cycles per MMA against the floor 128*N/256.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_rate tools/mma_rate.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2204_10319_b200/csrc/sm100_ptx.cuh"

using namespace scb::ptx;

template <int U, bool TS>
__global__ void rate(int n, int rounds, int commit_every, long long* out, int noise) {
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
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp > 0 && noise) {
    // smem write traffic beside the MMAs: 16-B stores into a region the MMAs
    // do not read (noise = 1), or cp.async 16-B copies from global (noise = 2)
    uint8_t* region = smem + 48 * 1024;
    const uint32_t off = (threadIdx.x - 32) * 16;
    int it = 0;
    while (!stop) {
      if (noise == 1) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
          *reinterpret_cast<uint4*>(region + ((off + r * 1536) & 16383)) = make_uint4(it, r, 0, 0);
      } else {
#pragma unroll
        for (int r = 0; r < 8; ++r)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(region + ((off + r * 1536) & 16383))),
                       "l"(out + 512 + ((threadIdx.x * 8 + r + it * 64) & 4095) * 2) : "memory");
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 4;" ::: "memory");
      }
      ++it;
    }
  }
  if (warp == 0) {
    const uint64_t ad = make_sdesc(smem_u32(smem), 8u * 128, 2u);
    const uint64_t bd = make_sdesc(smem_u32(smem + 16384), 8u * 128, 2u);
    const uint32_t idesc = (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    __syncwarp();
    const long long t0 = clock64();
    if (elect_one()) {
      for (int r = 0; r < rounds; ++r) {
#pragma unroll
        for (int k = 0; k < U; ++k) {
          if (TS)
            mma_f16_ts(tmem, tmem + 128 + 8 * (k & 3), bd + 2u * (k & 3), idesc, (r | k) ? 1u : 0u);
          else
            mma_f16(tmem, ad + 2u * (k & 3), bd + 2u * (k & 3), idesc, (r | k) ? 1u : 0u);
        }
        if (commit_every && (r % commit_every) == 0) mma_commit(&spare);
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    if (threadIdx.x == 0) stop = 1;
  }
  tc_before();
  __syncthreads();
  if (warp == 0) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

template <int U, bool TS>
void run(int n, int ctas_per_sm, int commit_every, int noise = 0) {
  static long long* d = nullptr;
  const int grid = 148 * ctas_per_sm;
  if (!d) cudaMalloc(&d, 148 * 4 * sizeof(long long) + 64 * 1024);
  const int smem = ctas_per_sm == 1 ? 200 * 1024 : 100 * 1024;
  cudaFuncSetAttribute(rate<U, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int rounds = 16384 / U;
  rate<U, TS><<<grid, noise ? 256 : 128, smem>>>(n, rounds, commit_every, d, noise);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148 * 4];
  cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < grid; ++i) s += h[i];
  const double per = s / grid / (rounds * U);
  printf("%s noise=%d U=%2d N=%3d ctas/SM=%d commit/%d: %6.1f cyc/MMA per CTA, %6.1f per SM (floor %5.1f) %s\n",
         TS ? "TS" : "SS", noise, U, n, ctas_per_sm, commit_every, per, per / ctas_per_sm, 128.0 * n / 256,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  for (int n : {64, 96, 128}) {
    for (int noise : {0, 1, 2}) {
      run<16, false>(n, 1, 1, noise);
      run<16, true>(n, 1, 1, noise);
    }
  }
  return 0;
}
