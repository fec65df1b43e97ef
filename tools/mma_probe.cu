// tcgen05.mma issue-rate probe (run on the B200): one thread per CTA issues R
// rounds of KC/16 MMAs (M = 128, N, K = 16, kind::f16, A and B from shared
// memory, fixed operands) into `nacc` rotating TMEM accumulators, then
// commits and waits.  Prints cycles per MMA for each (N, KC, nacc).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_probe tools/mma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2204_10319_b200/csrc/sm100_ptx.cuh"

using namespace scb::ptx;

__global__ void probe(int n, int kc, int nacc, int rounds, int chain, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, done, spare;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&done, 1);
    mbar_init(&spare, 1);
    mbar_arrive(&done);   // phase 0 completes
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = slot;
  if (warp == 0) {   // the whole warp runs the loop (uniform operands), one lane issues
    const uint32_t swz = kc * 2;
    const uint32_t layout = swz == 128 ? 2u : (swz == 64 ? 4u : 6u);
    const uint64_t ad = make_sdesc(smem_u32(smem), 8u * swz, layout);
    const uint64_t bd = make_sdesc(smem_u32(smem + 16384 * 2), 8u * swz, layout);
    const uint32_t idesc = (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t a_step = (uint32_t)(128 * kc * 2 >> 4), b_step = (uint32_t)(n * kc * 2 >> 4);
    __syncwarp();
    const long long t0 = clock64();
    uint32_t acc = 0, sel = 0, first = (uint32_t)nacc;
    if (mode == 1 || mode >= 3) {   // one elected lane runs the whole loop (3: + poll, commit; 4: commit; 5: poll)
      if (elect_one()) {
        for (int r = 0; r < rounds; ++r) {
          const uint64_t a = ad + (uint64_t)(sel * a_step);
          const uint64_t b = bd + (uint64_t)(sel * b_step);
          if (mode == 3 || mode == 5) mbar_wait(&done, 0);
          for (int k = 0; k < kc / 16; ++k)
            mma_f16(tmem + acc * (uint32_t)n, a + 2u * k, b + 2u * k, idesc, first ? 0u : 1u);
          if (mode == 3 || mode == 4) mma_commit(&spare);
          if (first) --first;
          if (++acc == (uint32_t)nacc) acc = 0;
          if (++sel == (uint32_t)chain) sel = 0;
        }
      }
      __syncwarp();
    } else {
      for (int r = 0; r < rounds; ++r) {
        const uint64_t a = ad + (uint64_t)(sel * a_step);
        const uint64_t b = bd + (uint64_t)(sel * b_step);
        if (mode == 2) mbar_wait(&done, 0);   // a completed barrier, like the stage-full poll
        if (elect_one()) {
          for (int k = 0; k < kc / 16; ++k) {
            mma_f16(tmem + acc * (uint32_t)n, a + 2u * k, b + 2u * k, idesc, first ? 0u : 1u);
          }
          if (mode == 2) mma_commit(&spare);
        }
        __syncwarp();
        if (first) --first;
        if (++acc == (uint32_t)nacc) acc = 0;
        if (++sel == (uint32_t)chain) sel = 0;
      }
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  tc_before();
  __syncthreads();
  if (warp == 0) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int rounds = 2000;
  for (int mode : {1, 4, 5})
    for (int kc : {64, 32})
      for (int n : {96}) {
        const int nacc = 1, chain = 2;
        probe<<<148, 128, 200 * 1024>>>(n, kc, nacc, rounds, chain, mode, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double s = 0;
        for (int i = 0; i < 148; ++i) s += h[i];
        const double per = s / 148 / (rounds * (kc / 16));
        printf("mode=%d kc=%d N=%3d: %7.1f cycles/MMA, %7.1f per iteration (nominal %5.1f/MMA) %s\n",
               mode, kc, n, per, per * (kc / 16), 128.0 * n / 256,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
