// Microbenchmark: cycles per tcgen05.mma (kind::f16, bf16 -> fp32, K = 16) by shape and
// operand source.  One CTA per SM; one thread issues REPS back-to-back MMAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -o umma_bench scripts/umma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2410_01359_b200/csrc/fm_ptx.cuh"

using namespace fm;

constexpr int REPS = 4096;

template <int M, int N, bool A_TMEM, int A_MN, int B_MN, int CONV = 0, int NACC = 1>
__global__ void __launch_bounds__(128, 1) bench(unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase_s;
  if (CONV && warp == 0) {
    // converged warp, elect.sync inside the MMA (fm_ptx.cuh *_w); NACC independent accumulators
    const uint32_t id = idesc_bf16(M, N, A_MN, B_MN);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    const long long t0 = clock64();
    for (int r = 0; r < REPS; r += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t off = u * 32;
        const uint32_t dcol = 256 + ((r + u) % NACC) * N;
        if constexpr (A_TMEM)
          mma_ts_w(tb + dcol, tb + u * 8, sdesc_sw128(b + off, 16384, 1024), id, 1);
        else
          mma_ss_w(tb + dcol, sdesc_sw128(a + off, 16384, 1024), sdesc_sw128(b + off, 16384, 1024), id, 1);
      }
    }
    mma_commit_w(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
  } else if (!CONV && threadIdx.x == 0) {
    const uint32_t id = idesc_bf16(M, N, A_MN, B_MN);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    const long long t0 = clock64();
    for (int r = 0; r < REPS; ++r) {
      const uint32_t off = (r & 3) * 32;
      if constexpr (A_TMEM)
        mma_ts(tb + 256, tb + (r & 3) * 8, sdesc_sw128(b + off, 16384, 1024), id, 1);
      else
        mma_ss(tb + 256, sdesc_sw128(a + off, 16384, 1024), sdesc_sw128(b + off, 16384, 1024), id, 1);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tb);
  }
}

template <int M, int N, bool AT, int AMN, int BMN, int CONV = 0, int NACC = 1>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  auto k = bench<M, N, AT, AMN, BMN, CONV, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  k<<<148, 128, 65536 + 1024>>>(d);
  k<<<148, 128, 65536 + 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double per = avg / REPS;
  const double macs = double(M) * N * 16;
  printf("%-34s %s  %7.1f clk/MMA  %7.0f MAC/clk/SM (%.0f%% of 4096)\n", name, cudaGetErrorString(e), per, macs / per,
         100.0 * macs / per / 4096);
  cudaFree(d);
}

// One backward iteration's MMA mix (d=128, Br=64): S^T TS N64 x8, dP^T SS N64 x8,
// dV / dK TS N128 x4 each, dQ^T SS N64 (A,B MN-major) x8.
template <int CONV>
__global__ void __launch_bounds__(128, 1) bwd_mix(unsigned long long* out, int iters, int use_ka) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase_s;
  if (CONV ? (warp == 0) : (threadIdx.x == 0)) {
    const uint32_t kA = smem_u32(sm), vA = kA + 32768, qB = kA + 65536, dOB = kA + 81920, dsB = kA + 98304;
if constexpr (CONV) {
    const uint32_t ID_S = idesc_bf16(128, 64, 0, 0), ID_G = idesc_bf16(128, 128, 0, 1), ID_Q = idesc_bf16(128, 64, 1, 1);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t ao = (kk >> 2) * 16384 + (kk & 3) * 32, bo = (kk >> 2) * 8192 + (kk & 3) * 32;
        if (use_ka) mma_ts_w(tb + 0, tb + 192 + kk * 8, sdesc_sw128(qB + bo, 16, 1024), ID_S, kk > 0);
        else mma_ss_w(tb + 0, sdesc_sw128(kA + ao, 16, 1024), sdesc_sw128(qB + bo, 16, 1024), ID_S, kk > 0);
        mma_ss_w(tb + 64, sdesc_sw128(vA + ao, 16, 1024), sdesc_sw128(dOB + bo, 16, 1024), ID_S, kk > 0);
      }
      for (int kk = 0; kk < 4; ++kk) {
        mma_ts_w(tb + 256, tb + 128 + kk * 8, sdesc_sw128(dOB + kk * 2048, 8192, 1024), ID_G, 1);
        mma_ts_w(tb + 384, tb + 160 + kk * 8, sdesc_sw128(qB + kk * 2048, 8192, 1024), ID_G, 1);
      }
      for (int kk = 0; kk < 8; ++kk)
        mma_ss_w(tb + 128, sdesc_sw128(kA + kk * 2048, 16384, 1024), sdesc_sw128(dsB + kk * 2048, 16384, 1024), ID_Q, kk > 0);
    }
    mma_commit_w(&bar);
    mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[blockIdx.x] = static_cast<unsigned long long>(clock64() - t0);
} else {
    const uint32_t ID_S = idesc_bf16(128, 64, 0, 0), ID_G = idesc_bf16(128, 128, 0, 1), ID_Q = idesc_bf16(128, 64, 1, 1);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t ao = (kk >> 2) * 16384 + (kk & 3) * 32, bo = (kk >> 2) * 8192 + (kk & 3) * 32;
        if (use_ka) mma_ts(tb + 0, tb + 192 + kk * 8, sdesc_sw128(qB + bo, 16, 1024), ID_S, kk > 0);
        else mma_ss(tb + 0, sdesc_sw128(kA + ao, 16, 1024), sdesc_sw128(qB + bo, 16, 1024), ID_S, kk > 0);
        mma_ss(tb + 64, sdesc_sw128(vA + ao, 16, 1024), sdesc_sw128(dOB + bo, 16, 1024), ID_S, kk > 0);
      }
      for (int kk = 0; kk < 4; ++kk) {
        mma_ts(tb + 256, tb + 128 + kk * 8, sdesc_sw128(dOB + kk * 2048, 8192, 1024), ID_G, 1);
        mma_ts(tb + 384, tb + 160 + kk * 8, sdesc_sw128(qB + kk * 2048, 8192, 1024), ID_G, 1);
      }
      for (int kk = 0; kk < 8; ++kk)
        mma_ss(tb + 128, sdesc_sw128(kA + kk * 2048, 16384, 1024), sdesc_sw128(dsB + kk * 2048, 16384, 1024), ID_Q, kk > 0);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = static_cast<unsigned long long>(clock64() - t0);
}
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tb); }
}

template <int CONV>
void run_mix(int use_ka) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(bwd_mix<CONV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 1024);
  const int iters = 512;
  bwd_mix<CONV><<<148, 128, 196608 + 1024>>>(d, iters, use_ka);
  bwd_mix<CONV><<<148, 128, 196608 + 1024>>>(d, iters, use_ka);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("bwd iteration MMA mix (K in %s, %s issue): %s %.0f clk/iteration (ideal 1280)\n", use_ka ? "TMEM" : "smem",
         CONV ? "converged" : "lane-0",
         cudaGetErrorString(e), avg / iters);
  cudaFree(d);
}

__global__ void __launch_bounds__(128, 1) qdepth(long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase_s;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const uint32_t id = idesc_bf16(128, 256, 0, 0);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 16384);
    long long t[64];
    const long long t0 = clock64();
    for (int r = 0; r < 64; ++r) {
      mma_ss(tb + 256, sdesc_sw128(a, 16, 1024), sdesc_sw128(b, 16, 1024), id, 1);
      t[r] = clock64();
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    for (int r = 0; r < 64; ++r) out[r] = t[r] - t0;
    out[64] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tb); }
}

int main() {
  {
    long long* d;
    cudaMalloc(&d, 65 * 8);
    cudaFuncSetAttribute(qdepth, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    qdepth<<<1, 128, 65536 + 1024>>>(d);
    cudaDeviceSynchronize();
    long long h[65];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("issue clock after each of 64 N=256 MMAs (128 clk each):");
    for (int r = 0; r < 64; ++r) printf(" %lld", h[r]);
    printf("\ncomplete: %lld\n", h[64]);
    cudaFree(d);
  }
  run_mix<0>(0);
  run_mix<1>(0);
  run_mix<1>(1);
  run<128, 64, false, 0, 0>("SS M128 N64  lane-0");
  run<128, 64, false, 0, 0, 1, 1>("SS M128 N64  conv 1acc");
  run<128, 64, false, 0, 0, 1, 2>("SS M128 N64  conv 2acc");
  run<128, 64, false, 0, 0, 1, 4>("SS M128 N64  conv 4acc");
  run<128, 128, false, 0, 0>("SS M128 N128 lane-0");
  run<128, 128, false, 0, 0, 1, 1>("SS M128 N128 conv 1acc");
  run<128, 128, false, 0, 0, 1, 2>("SS M128 N128 conv 2acc");
  run<128, 32, false, 0, 0, 1, 1>("SS M128 N32  conv 1acc");
  run<128, 32, false, 0, 0, 1, 4>("SS M128 N32  conv 4acc");
  run<128, 64, true, 0, 1, 1, 1>("TS M128 N64 B MN conv 1acc");
  run<128, 64, true, 0, 1, 1, 2>("TS M128 N64 B MN conv 2acc");
  run<128, 128, true, 0, 1, 1, 1>("TS M128 N128 B MN conv");
  run<128, 256, false, 0, 0, 1, 1>("SS M128 N256 conv");
  return 0;
}
