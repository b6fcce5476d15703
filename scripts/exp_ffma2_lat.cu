// Experiment: latency and low-occupancy throughput of FFMA2 (fma.rn.f32x2) vs FFMA on sm_100a:
// C dependent chains per warp, W warps per SM sub-partition; reports cycles per FMA-instruction
// per warp and FMA lanes per clock per SMSP.  MODE 0: FFMA, 1: FFMA2 (all packed operands),
// 2: FFMA2 with a broadcast scalar multiplicand (Rn.F32).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/exp_ffma2_lat scripts/exp_ffma2_lat.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ u64 f2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
template <int MODE, int C>
__global__ void k(float *out, int iters, long long *cyc, float m, float ad) {
  float x[C]; u64 y[C];
  for (int c = 0; c < C; ++c) { x[c] = threadIdx.x * 1e-3f + c; y[c] = pk(x[c], x[c] + 1.f); }
  const u64 a2 = pk(m, m * 0.9999f), b2 = pk(ad, ad * 2.f), ms = pk(m, m);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (MODE == 0) x[c] = fmaf(x[c], m, ad);
        if (MODE == 1) y[c] = f2(y[c], a2, b2);
        if (MODE == 2) y[c] = f2(y[c], ms, b2);
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int c = 0; c < C; ++c) s += x[c] + __uint_as_float((unsigned)y[c]) + __uint_as_float((unsigned)(y[c] >> 32));
  if (s == -1.f) out[threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int MODE, int C>
void run(int warps_per_smsp) {
  float *o; cudaMalloc(&o, 4096);
  long long *cyc; cudaMallocManaged(&cyc, 8);
  const int iters = 4000;
  k<MODE, C><<<148, warps_per_smsp * 128>>>(o, iters, cyc, 0.999f, 1e-4f);
  cudaDeviceSynchronize();
  k<MODE, C><<<148, warps_per_smsp * 128>>>(o, iters, cyc, 0.999f, 1e-4f);
  cudaDeviceSynchronize();
  double instr_per_warp = (double)iters * 16 * C;
  double cpi = *cyc / instr_per_warp;                        // cycles per instruction per warp
  double lanes = warps_per_smsp * 32.0 * (MODE ? 2 : 1) / cpi;    // FMA lanes per clock per SMSP
  printf("mode %d chains %d warps/SMSP %d: %.2f cycles/instr/warp, %.1f FMA lanes/clk/SMSP\n", MODE, C,
         warps_per_smsp, cpi, lanes);
}
int main() {
  for (int w : {1, 2, 4, 8}) {
    run<0, 1>(w); run<1, 1>(w); run<2, 1>(w);
    run<0, 2>(w); run<1, 2>(w); run<2, 2>(w);
    run<0, 4>(w); run<1, 4>(w); run<2, 4>(w);
    run<0, 8>(w); run<1, 8>(w); run<2, 8>(w);
  }
  return 0;
}
