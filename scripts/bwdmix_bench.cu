// Backward MMA-mix variants (d = 128, Br = 64), issued by one converged warp:
// which GEMMs take A from TMEM (TS) vs SMEM (SS), and in which order.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -o bwdmix_bench scripts/bwdmix_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2410_01359_b200/csrc/fm_ptx.cuh"
using namespace fm;

// flags: 1 = S^T A from TMEM, 2 = dP^T A from TMEM, 4 = dQ^T A from TMEM, 8 = no S/dP interleave
template <int FLAGS>
__global__ void __launch_bounds__(128, 1) mix(long long* out, int iters) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = smem_align1024<uint8_t>(raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t tb_s;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tb_s);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tb_s;
  if (warp == 0) {
    const uint32_t kA = smem_u32(sm), vA = kA + 32768, qB = kA + 65536, dOB = kA + 81920, dsB = kA + 98304;
    const uint32_t ID_S = idesc_bf16(128, 64, 0, 0), ID_G = idesc_bf16(128, 128, 0, 1), ID_Q = idesc_bf16(128, 64, 1, 1);
    const uint32_t ID_QT = idesc_bf16(128, 64, 0, 1);
    // TMEM map (bench only, regions may alias): S 0, dP 64, dQ 128, A-operands 192/224/.. (K_A, V_A, KT_A
    // share columns — values are irrelevant), dV 256, dK 384
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      auto s_mma = [&](int kk) {
        const uint32_t ao = (kk >> 2) * 16384 + (kk & 3) * 32, bo = (kk >> 2) * 8192 + (kk & 3) * 32;
        if (FLAGS & 1) mma_ts_w(tb + 0, tb + 192 + kk * 8, sdesc_sw128(qB + bo, 16, 1024), ID_S, kk > 0);
        else mma_ss_w(tb + 0, sdesc_sw128(kA + ao, 16, 1024), sdesc_sw128(qB + bo, 16, 1024), ID_S, kk > 0);
      };
      auto dp_mma = [&](int kk) {
        const uint32_t ao = (kk >> 2) * 16384 + (kk & 3) * 32, bo = (kk >> 2) * 8192 + (kk & 3) * 32;
        if (FLAGS & 2) mma_ts_w(tb + 64, tb + 192 + kk * 8, sdesc_sw128(dOB + bo, 16, 1024), ID_S, kk > 0);
        else mma_ss_w(tb + 64, sdesc_sw128(vA + ao, 16, 1024), sdesc_sw128(dOB + bo, 16, 1024), ID_S, kk > 0);
      };
      if (FLAGS & 8) {
        for (int kk = 0; kk < 8; ++kk) s_mma(kk);
        for (int kk = 0; kk < 8; ++kk) dp_mma(kk);
      } else {
        for (int kk = 0; kk < 8; ++kk) { s_mma(kk); dp_mma(kk); }
      }
      for (int kk = 0; kk < 4; ++kk) {
        mma_ts_w(tb + 256, tb + 128 + kk * 8, sdesc_sw128(dOB + kk * 2048, 8192, 1024), ID_G, 1);
        mma_ts_w(tb + 384, tb + 160 + kk * 8, sdesc_sw128(qB + kk * 2048, 8192, 1024), ID_G, 1);
      }
      for (int kk = 0; kk < 8; ++kk) {
        if (FLAGS & 4)  // dQ^T = K^T dS^T with K^T from TMEM, dS^T (keys x rows) MN-major in smem
          mma_ts_w(tb + 128, tb + 192 + kk * 8, sdesc_sw128(dsB + kk * 2048, 16384, 1024), ID_QT, kk > 0);
        else
          mma_ss_w(tb + 128, sdesc_sw128(kA + kk * 2048, 16384, 1024), sdesc_sw128(dsB + kk * 2048, 16384, 1024), ID_Q, kk > 0);
      }
    }
    mma_commit_w(&bar);
    mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tb); }
}

template <int F>
void run(const char* name, double ideal) {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(mix<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 1024);
  const int iters = 512;
  mix<F><<<148, 128, 131072 + 1024>>>(d, iters);
  mix<F><<<148, 128, 131072 + 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%-44s %s %6.0f clk/iter (model %4.0f, ideal 1280)\n", name, cudaGetErrorString(e), avg / iters, ideal);
  cudaFree(d);
}

int main() {
  run<0>("all SS except dV/dK (current)", 384 + 384 + 512 + 384);
  run<1>("S^T TS", 256 + 384 + 512 + 384);
  run<1 | 8>("S^T TS, no interleave", 256 + 384 + 512 + 384);
  run<3>("S^T, dP^T TS", 256 + 256 + 512 + 384);
  run<3 | 8>("S^T, dP^T TS, no interleave", 256 + 256 + 512 + 384);
  run<4>("dQ^T TS", 384 + 384 + 512 + 256);
  run<5>("S^T, dQ^T TS", 256 + 384 + 512 + 256);
  run<7>("all TS", 1280);
  run<7 | 8>("all TS, no interleave", 1280);
  return 0;
}
