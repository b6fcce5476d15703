// Experiment: throughput of legacy warp-level mma.sync m16n8k4 tf32 (HMMA.1684.F32.TF32)
// on sm_100a, independent chains per warp; and mixed with FFMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/exp_hmma scripts/exp_hmma.cu && /tmp/exp_hmma
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(float *out, long long iters) {
  unsigned a0 = __float_as_uint(1.0f + threadIdx.x), a1 = __float_as_uint(2.0f), b0 = __float_as_uint(0.5f);
  float d[CH][4];
#pragma unroll
  for (int c = 0; c < CH; ++c) for (int i = 0; i < 4; ++i) d[c][i] = 0.f;
  for (long long it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3]) : "r"(a0), "r"(a1), "r"(b0));
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == -1.f) out[threadIdx.x] = s;
}
template <int CH>
void run(int ctas, int threads, long long iters) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *o; cudaMalloc(&o, 4096);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<CH><<<sms * ctas, threads>>>(o, iters);
  cudaEventRecord(a);
  k<CH><<<sms * ctas, threads>>>(o, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float t; cudaEventElapsedTime(&t, a, b);
  double mmas = (double)CH * iters * sms * ctas * threads / 32;
  double per_smsp_clk = mmas / (sms * 4) / (t * 1e-3 * 1.965e9);
  printf("CH=%d ctas/SM=%d threads=%d: %.3f HMMA.1684 per SMSP per clock (%.3f ms)\n", CH, ctas, threads,
         per_smsp_clk, t);
}
int main() {
  run<4>(4, 256, 20000);
  run<8>(4, 256, 10000);
  run<8>(8, 256, 10000);
  run<2>(8, 256, 40000);
  return 0;
}
