// Experiment: FFMA2 (fma.rn.f32x2, sm_100a) throughput vs FFMA, alone and mixed with
// independent integer ALU work (does FFMA2 free issue slots?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/exp_ffma2 scripts/exp_ffma2.cu && /tmp/exp_ffma2
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
template <int MODE>  // 0: FFMA x4 chains; 1: FFMA2 x4 chains (8 FMA); 2: FFMA x4 + 4 IADD; 3: FFMA2 x4 + 4 IADD
__global__ void k(float *out, long long iters) {
  float x[4]; unsigned long long y[4]; unsigned z[4];
  for (int c = 0; c < 4; ++c) { x[c] = threadIdx.x * 1e-3f + c; y[c] = ((unsigned long long)__float_as_uint(x[c]) << 32) | __float_as_uint(x[c]); z[c] = threadIdx.x + c; }
  const unsigned long long a2 = ((unsigned long long)__float_as_uint(0.999f) << 32) | __float_as_uint(0.999f);
  const unsigned long long b2 = ((unsigned long long)__float_as_uint(1e-4f) << 32) | __float_as_uint(1e-4f);
  for (long long i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 32; ++u) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (MODE == 0 || MODE == 2) x[c] = fmaf(x[c], 0.999f, 1e-4f);
        if (MODE == 1 || MODE == 3) y[c] = f2(y[c], a2, b2);
        if (MODE >= 2) asm volatile("add.u32 %0, %0, %1;" : "+r"(z[c]) : "r"(c + 1));
      }
    }
  }
  float s = 0;
  for (int c = 0; c < 4; ++c) s += x[c] + __uint_as_float((unsigned)y[c]) + (float)z[c];
  if (s == -1.f) out[threadIdx.x] = s;
}
template <int MODE>
void run(long long iters) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *o; cudaMalloc(&o, 4096);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<MODE><<<sms * 8, 256>>>(o, iters);
  cudaEventRecord(a);
  k<MODE><<<sms * 8, 256>>>(o, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float t; cudaEventElapsedTime(&t, a, b);
  double warp_iters = (double)iters * 32 * sms * 8 * 256 / 32;   // per unrolled step
  double fma = (MODE == 1 || MODE == 3 ? 8 : 4) * (MODE == 0 || MODE == 2 ? 1 : 0) + (MODE == 1 || MODE == 3 ? 8 : 0);
  double flops = warp_iters * 32 * fma * 2;
  double instr = warp_iters * 4 * (MODE >= 2 ? 2 : 1);
  printf("mode %d: %.2f TFLOP/s, %.3f warp-instr per SMSP per clock (%.3f ms)\n", MODE,
         flops / (t * 1e-3) / 1e12, instr / (sms * 4) / (t * 1e-3 * 1.965e9), t);
}
int main() { run<0>(2000); run<1>(2000); run<2>(2000); run<3>(2000); return 0; }
