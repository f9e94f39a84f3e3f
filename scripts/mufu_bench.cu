// MUFU.EX2 and FFMA2 throughput per SM (many independent chains, 1 CTA per SM).
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include "../paper_2410_01359_b200/csrc/fm_ptx.cuh"
using namespace fm;
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(float* out, int iters, long long* cyc) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) - 1.0f;
      else if (MODE == 2) {
        uint32_t h2, r2;
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h2) : "f"(a[i]), "f"(a[i] * 0.5f));
        asm("ex2.approx.f16x2 %0, %1;" : "=r"(r2) : "r"(h2));
        __half2 hh = *reinterpret_cast<__half2*>(&r2);
        a[i] = __low2float(hh) - __high2float(hh) - 0.25f;
      } else {
        float r0, r1;
        exp2_poly2(f2pack(a[i], a[i] * 0.5f), r0, r1);
        a[i] = r0 - r1 - 0.5f;
      }
    }
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* o; long long* c;
  cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 148 * 8);
  const int iters = 4096;
  for (int mode = 0; mode < 3; ++mode) {
    for (int threads : {128, 256, 512}) {
      if (mode == 0) { k<0><<<148, threads>>>(o, iters, c); k<0><<<148, threads>>>(o, iters, c); }
      else if (mode == 1) { k<1><<<148, threads>>>(o, iters, c); k<1><<<148, threads>>>(o, iters, c); }
      else { k<2><<<148, threads>>>(o, iters, c); k<2><<<148, threads>>>(o, iters, c); }
      cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
      const double n_exp = double(threads) * iters * 8 * (mode == 0 ? 1 : 2);
      printf("%s threads=%d: %.2f exp2/clk/SM\n", mode == 0 ? "MUFU.EX2" : (mode == 1 ? "poly(FMA)" : "MUFU.EX2.F16x2"), threads, n_exp / avg);
    }
  }
  return 0;
}
