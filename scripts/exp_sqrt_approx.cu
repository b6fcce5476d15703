// Exhaustive check of sqrt.approx.ftz.f32 (MUFU.SQRT) against the exact square
// root over every positive normal float32: max relative error and max error
// in ulps of the correctly rounded result.  The broadphase group radius uses
// the approximation inflated by 1.000002 (+1e-6 m), which must exceed the
// worst case found here.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/sq scripts/exp_sqrt_approx.cu && /tmp/sq
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>

__device__ unsigned long long g_max_rel;   // double bits of the max relative error
__device__ unsigned int g_max_ulp, g_below;

__global__ void check(uint32_t lo, uint32_t hi) {
  for (uint64_t b = lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < hi;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const float x = __uint_as_float((uint32_t)b);
    float a;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(x));
    const double e = sqrt((double)x);
    const double rel = fabs((double)a - e) / e;
    atomicMax(&g_max_rel, (unsigned long long)__double_as_longlong(rel));
    const float r = __fsqrt_rn(x);
    const int du = abs((int)__float_as_uint(a) - (int)__float_as_uint(r));
    atomicMax(&g_max_ulp, (unsigned)du);
    if ((double)a < e) atomicAdd(&g_below, 1u);
  }
}

int main() {
  check<<<148 * 16, 256>>>(0x00800000u, 0x7f800000u);   // all positive normal floats
  unsigned long long rel_bits;
  unsigned ulp, below;
  cudaMemcpyFromSymbol(&rel_bits, g_max_rel, 8);
  cudaMemcpyFromSymbol(&ulp, g_max_ulp, 4);
  cudaMemcpyFromSymbol(&below, g_below, 4);
  double rel;
  memcpy(&rel, &rel_bits, 8);
  printf("sqrt.approx.ftz.f32 over all positive normal floats: max rel error %.3e (2^%.2f), "
         "max %u ulp from sqrt_rn, %u results below the exact root; err=%s\n",
         rel, log2(rel), ulp, below, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
