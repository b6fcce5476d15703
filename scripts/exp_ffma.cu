// Experiment: FFMA throughput variants (how close to 128 FFMA/clk/SM a kernel gets).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/exp_ffma scripts/exp_ffma.cu && /tmp/exp_ffma
#include <cstdio>
#include <cuda_runtime.h>
template <int CH, int UN>
__global__ void k(float *out, long long iters, float a, float b) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = (threadIdx.x + c) * 1e-3f;
  for (long long i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < UN; ++u)
#pragma unroll
      for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == -1234.5f) out[threadIdx.x] = s;
}
template <int CH, int UN>
void run(int ctas_per_sm, int threads, long long total_per_thread) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *o; cudaMalloc(&o, 4096);
  long long iters = total_per_thread / (CH * UN);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<CH, UN><<<sms * ctas_per_sm, threads>>>(o, iters, 0.999f, 1e-4f);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k<CH, UN><<<sms * ctas_per_sm, threads>>>(o, iters, 0.999f, 1e-4f);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float t; cudaEventElapsedTime(&t, a, b); best = t < best ? t : best;
  }
  double fl = 2.0 * CH * UN * iters * (double)sms * ctas_per_sm * threads;
  printf("CH=%2d UN=%3d ctas/SM=%d threads=%d: %.2f TFLOP/s (%.3f ms)\n", CH, UN, ctas_per_sm, threads,
         fl / (best * 1e-3) / 1e12, best);
  cudaFree(o);
}
int main() {
  const long long T = 768000;
  run<8, 16>(4, 256, T);
  run<8, 64>(4, 256, T);
  run<16, 32>(4, 256, T);
  run<8, 64>(8, 256, T);
  run<8, 64>(2, 256, T);
  run<4, 64>(8, 256, T);
  run<12, 32>(4, 256, T);
  return 0;
}
