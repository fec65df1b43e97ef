// Standalone probe of the TMA forms the implicit conv uses (run on the B200):
//   tma_probe 1d            1-D tile load of 128 int32
//   tma_probe g4 <swz> <kc> gather4 of 4 fp16 rows, box {kc, 1}, swizzle swz (0/32/64/128)
// Prints PASS/FAIL per check; a fault aborts only this process.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2204_10319_b200/csrc/sm100_ptx.cuh"

using namespace scb::ptx;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

static EncodeFn enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (EncodeFn)p;
}

__global__ void k1d(const __grid_constant__ CUtensorMap m, int x, int* out) {
  __shared__ alignas(128) int buf[128];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, 512);
    tma_load_1d(buf, &m, &bar, x);
  }
  mbar_wait(&bar, 0);
  out[threadIdx.x] = buf[threadIdx.x];
}

__global__ void kg4(const __grid_constant__ CUtensorMap m, int rowbytes, int r0, int r1, int r2,
                    int r3, uint8_t* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, 4 * rowbytes);
    tma_gather4(buf, &m, &bar, 0, r0, r1, r2, r3);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 4 * rowbytes; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  EncodeFn fn = enc();
  if (!fn) { printf("no encode fn\n"); return 1; }
  if (argc > 1 && !strcmp(argv[1], "1d")) {
    const int n = 1000;
    std::vector<int> h(n);
    for (int i = 0; i < n; ++i) h[i] = i * 3;
    int *d, *o;
    cudaMalloc(&d, n * 4);
    cudaMalloc(&o, 128 * 4);
    cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    CUtensorMap m;
    cuuint64_t dims[1] = {n}, str[1] = {0};
    cuuint32_t box[1] = {128}, es[1] = {1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_INT32, 1, d, dims, str, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode 1d: %d\n", (int)r);
    for (int x : {0, 37, 900}) {
      k1d<<<1, 128>>>(m, x, o);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<int> got(128);
      cudaMemcpy(got.data(), o, 512, cudaMemcpyDeviceToHost);
      bool ok = e == cudaSuccess;
      for (int i = 0; i < 128 && ok; ++i) ok = got[i] == (x + i < n ? (x + i) * 3 : 0);
      printf("1d x=%d: %s (%s)\n", x, ok ? "PASS" : "FAIL", cudaGetErrorString(e));
      if (e != cudaSuccess) return 2;
    }
    return 0;
  }
  const int swz = argc > 2 ? atoi(argv[2]) : 128;
  const int kc = argc > 3 ? atoi(argv[3]) : 64;
  const int rows = 100, cols = 64;  // fp16 matrix [rows][cols]
  std::vector<__half> h(rows * cols);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) h[r * cols + c] = __float2half((float)(r * 100 + c));
  __half* d;
  uint8_t* o;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&o, 4 * 256);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, str[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)kc, 1}, es[2] = {1, 1};
  CUtensorMapSwizzle sw = swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swz == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d, dims, str, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode gather4 swz=%d kc=%d: %d\n", swz, kc, (int)r);
  const int rowbytes = kc * 2;
  const int idx[4] = {7, 100, 3, 42};  // 100 is out of bounds
  cudaFuncSetAttribute(kg4, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  kg4<<<1, 128, 4096>>>(m, rowbytes, idx[0], idx[1], idx[2], idx[3], o);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<uint8_t> got(4 * rowbytes);
  cudaMemcpy(got.data(), o, got.size(), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int rr = 0; rr < 4; ++rr)
    for (int c = 0; c < kc; ++c) {
      // undo the swizzle: 16-B chunk index XOR row bits, as the UMMA layout expects
      const int chunk = (c * 2) / 16, within = (c * 2) % 16;
      int phys = chunk;
      if (swz == 128) phys = chunk ^ (rr & 7);
      if (swz == 64) phys = chunk ^ ((rr >> 1) & 3);
      if (swz == 32) phys = chunk ^ ((rr >> 2) & 1);
      __half v;
      memcpy(&v, &got[rr * rowbytes + phys * 16 + within], 2);
      const float want = idx[rr] < rows ? (float)(idx[rr] * 100 + c) : 0.f;
      if (__half2float(v) != want) ++bad;
    }
  printf("gather4 swz=%d kc=%d: %s (%d bad, %s)\n", swz, kc, (bad == 0 && e == cudaSuccess) ? "PASS" : "FAIL",
         bad, cudaGetErrorString(e));
  if (bad) {  // raw dump: value at each 2-byte slot
    for (int rr = 0; rr < 4; ++rr) {
      printf(" row%d:", rr);
      for (int c = 0; c < kc && c < 64; ++c) {
        __half v;
        memcpy(&v, &got[rr * rowbytes + c * 2], 2);
        printf(" %g", __half2float(v));
      }
      printf("\n");
    }
  }
  return e == cudaSuccess ? 0 : 2;
}
