// TMEM load latency from 4 warps with / without a concurrent stream of tcgen05.mma.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2410_01359_b200/csrc/fm_ptx.cuh"
using namespace fm;
__global__ void __launch_bounds__(160, 1) k(long long* out, int with_mma, int nld) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = smem_align1024<uint8_t>(raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t tb_s;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); stop = 0; }
  if (warp == 4) tmem_alloc<512>(&tb_s);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tb_s;
  if (warp == 4) {
    if (threadIdx.x == 128 && with_mma) {
      const uint32_t id = idesc_bf16(128, 128, 0, 0);
      const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
      int r = 0;
      while (!stop) {
        mma_ss(tb + 256, sdesc_sw128(a, 16, 1024), sdesc_sw128(b, 16, 1024), id, 1);
        if (++r > 200000) break;
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
    }
  } else {
    const uint32_t lo = static_cast<uint32_t>(warp * 32) << 16;
    uint32_t r[16];
    unsigned acc = 0;
    const long long t0 = clock64();
    for (int i = 0; i < nld; ++i) {
      tmem_ld16(tb + lo + (i & 7) * 16, r);
      tmem_wait_ld();
      acc += r[0];
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) { out[blockIdx.x] = t1 - t0; out[1000 + blockIdx.x] = acc; }
    named_bar_sync(1, 128);
    if (threadIdx.x == 0) stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) { tc_fence_after(); tmem_dealloc<512>(tb); }
}
int main() {
  long long* d; cudaMalloc(&d, 2000 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  for (int m = 0; m < 2; ++m) {
    const int nld = 2000;
    k<<<148, 160, 65536 + 1024>>>(d, m, nld);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
    printf("%s: tcgen05.ld x16 + wait latency %.1f clk (%s)\n", m ? "with MMA stream" : "idle tensor core", avg / nld, cudaGetErrorString(e));
  }
  return 0;
}
