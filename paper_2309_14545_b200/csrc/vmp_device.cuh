/* Device helpers shared by every vmp kernel (sm_100a).
 *
 * - environment staging: one cp.async.bulk (UBLKCP) global->shared copy per
 *   CTA, completed on an mbarrier, overlapped with the forward kinematics;
 * - narrowphase tests in expanded FFMA form (one test = 5 / 12 / 16 issue
 *   slots for sphere / capsule / cuboid obstacles);
 * - exact-rounding motion helpers reproducing numpy float32 semantics
 *   (reference lanes.py:91-113, motion.py:25-29,69-70).
 *
 * This file is inlined into NVRTC sources by codegen.py, so it may only use
 * builtins (no system headers).
 */
#ifndef VMP_DEVICE_CUH
#define VMP_DEVICE_CUH

#define VMP_FULL 0xffffffffu

/* -------------------------------------------------------------------- FK */

/* sin/cos for FK: Cody-Waite reduction to [-pi, pi] (2 FFMA with a split
 * 2 pi) then MUFU.SIN/COS.  Absolute error ~4e-7 for |x| < 1e5, which keeps
 * sphere centres within ~3e-6 m of float64 (north_star bar: 1e-5 m). */
__device__ __forceinline__ void vmp_sincos(float x, float *s, float *c) {
  const float k = rintf(x * 0.159154943091895336f);
  float r = fmaf(-k, 6.28318548202514648f, x);
  r = fmaf(-k, -1.74845553e-07f, r);
  __sincosf(r, s, c);
}

/* Nanosecond global timer (debug timelines only). */
__device__ __forceinline__ unsigned long long vmp_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

/* ---------------------------------------------------------------- staging */

__device__ __forceinline__ unsigned vmp_smem_addr(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void vmp_mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(vmp_smem_addr(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void vmp_bulk_g2s(void *dst, const void *src, unsigned bytes,
                                             unsigned long long *bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(vmp_smem_addr(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          vmp_smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(vmp_smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void vmp_mbar_wait(unsigned long long *bar, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(vmp_smem_addr(bar)), "r"(parity)
        : "memory");
  }
}

/* Shared -> global bulk (TMA) store of `bytes` (multiple of 16, both ends
 * 16-byte aligned), tracked in this thread's bulk-async group. */
__device__ __forceinline__ void vmp_bulk_s2g(void *dst, const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(vmp_smem_addr(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void vmp_bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
/* Wait until at most N of this thread's bulk groups still read shared memory. */
template <int N>
__device__ __forceinline__ void vmp_bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void vmp_bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
/* Make this thread's generic-proxy shared-memory writes visible to the async
 * (TMA) proxy before a bulk store reads them. */
__device__ __forceinline__ void vmp_fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

/* Stage the packed environment into shared memory (thread 0 issues one bulk
 * copy).  Returns the pointer kernels should read records from.  Callers must
 * vmp_mbar_wait(bar, 0) before the first dereference when staged. */
__device__ __forceinline__ const float4 *vmp_env_begin(const VmpEnvView &env, int stage,
                                                       float4 *smem,
                                                       unsigned long long *bar,
                                                       bool with_pairs = false) {
  const int n_f4 = with_pairs ? env.n_all_f4 : env.n_f4;
  if (!stage || n_f4 == 0) return env.rec;
  if (threadIdx.x == 0) {
    vmp_mbar_init(bar, 1);
    vmp_bulk_g2s(smem, env.rec, (unsigned)n_f4 * 16u, bar);
  }
  return smem;
}

/* ------------------------------------------------------------- narrowphase
 * Records (float4 units), built on the host by vmp_env_create (vmp.cu):
 *   sphere  k: R0 = (-2 o, -( |o|^2 - r^2 )),  R1 = (r, 0, 0, 0)
 *   capsule k: R0 = (a, -p0.a), R1 = (-2 p0, -( |p0|^2 - r^2 )), R2 = (1/|a|^2, |a|^2, r, Rb),
 *              R3 = (-2 cb, -( |cb|^2 - Rb^2 ))
 *   cuboid  k: R0..R2 = (row i of R^T, -(R^T c)_i),  R3 = (h, Rb),
 *              R4 = (-2 c, -( |c|^2 - Rb^2 ))
 * (cb, Rb) is the primitive's bounding sphere (capsule: midpoint, half length
 * + r; cuboid: centre, |h|; both + 1e-5 m), tested like a sphere obstacle for
 * the warp-level broadphase cull of the generated kernels.
 * For a robot sphere with centre c and radius rs, S = |c|^2 - rs^2 and
 *   |c - o|^2 - (r + rs)^2 = S + (-2 o).c + (|o|^2 - r^2) - 2 rs r
 * so the sphere test is 4 FFMA + 1 FSETP: S + (-2 o).c > 2 rs r - (|o|^2 - r^2).  Hit <=> value <= 0, i.e. boundary
 * contact counts as collision (reference collision.py:5-6, 206-211).
 */

__device__ __forceinline__ float vmp_sphere_S(float x, float y, float z, float rs2) {
  return fmaf(x, x, fmaf(y, y, fmaf(z, z, -rs2)));
}

/* expanded |c - o|^2 - (rs + r)^2 - r0.w of vmp_clear_sphere: clear iff > r0.w */
__device__ __forceinline__ float vmp_sphere_w(float x, float y, float z, float S, float m2rs,
                                              float4 r0, float r) {
  return fmaf(z, r0.z, fmaf(y, r0.y, fmaf(x, r0.x, fmaf(r, m2rs, S))));
}

/* true = clear (no contact) */
__device__ __forceinline__ bool vmp_clear_sphere(float x, float y, float z, float S, float m2rs,
                                                 float4 r0, float r) {
  /* the radius cross term sits on the compare side, as in the packed
   * two-sphere form (vmp_clear_sphere2), which must agree bit for bit */
  float w = fmaf(x, r0.x, S);
  w = fmaf(y, r0.y, w);
  w = fmaf(z, r0.z, w);
  return w > fmaf(r, -m2rs, r0.w);
}

__device__ __forceinline__ bool vmp_clear_capsule(float x, float y, float z, float S, float m2rs,
                                                  float4 r0, float4 r1, float4 r2) {
  float u = fmaf(x, r0.x, fmaf(y, r0.y, fmaf(z, r0.z, r0.w)));  /* (c - p0).a */
  float t = __saturatef(u * r2.x);                                /* clamp(u / |a|^2, 0, 1) */
  float w = fmaf(x, r1.x, S);
  w = fmaf(y, r1.y, w);
  w = fmaf(z, r1.z, w);                                            /* |c - p0|^2 - rs^2 - A */
  float v = fmaf(u, -2.0f, t * r2.y);                              /* t |a|^2 - 2 u */
  float e = fmaf(t, v, w);                                         /* |c - p0 - t a|^2 - rs^2 - A */
  return e > fmaf(r2.z, -m2rs, r1.w);                              /* + 2 rs r: vs (r + rs)^2 */
}

/* rs < 1: |l| - h saturated to [0, 1] is exact below 1 and >= rs^2 above, so
 * FADD.SAT replaces FADD + FMNMX without changing any verdict. */
__device__ __forceinline__ bool vmp_clear_box_small(float x, float y, float z, float rs2,
                                                    float4 r0, float4 r1, float4 r2, float4 r3) {
  float l0 = fmaf(x, r0.x, fmaf(y, r0.y, fmaf(z, r0.z, r0.w)));
  float l1 = fmaf(x, r1.x, fmaf(y, r1.y, fmaf(z, r1.z, r1.w)));
  float l2 = fmaf(x, r2.x, fmaf(y, r2.y, fmaf(z, r2.z, r2.w)));
  float e0 = __saturatef(fabsf(l0) - r3.x);
  float e1 = __saturatef(fabsf(l1) - r3.y);
  float e2 = __saturatef(fabsf(l2) - r3.z);
  float d = fmaf(e0, e0, fmaf(e1, e1, e2 * e2));
  return d > rs2;
}

__device__ __forceinline__ bool vmp_clear_box_any(float x, float y, float z, float rs2,
                                                  float4 r0, float4 r1, float4 r2, float4 r3) {
  float l0 = fmaf(x, r0.x, fmaf(y, r0.y, fmaf(z, r0.z, r0.w)));
  float l1 = fmaf(x, r1.x, fmaf(y, r1.y, fmaf(z, r1.z, r1.w)));
  float l2 = fmaf(x, r2.x, fmaf(y, r2.y, fmaf(z, r2.z, r2.w)));
  float e0 = fmaxf(fabsf(l0) - r3.x, 0.0f);
  float e1 = fmaxf(fabsf(l1) - r3.y, 0.0f);
  float e2 = fmaxf(fabsf(l2) - r3.z, 0.0f);
  float d = fmaf(e0, e0, fmaf(e1, e1, e2 * e2));
  return d > rs2;
}

__device__ __forceinline__ bool vmp_clear_box(float x, float y, float z, float rs, float rs2,
                                              float4 r0, float4 r1, float4 r2, float4 r3) {
  return rs < 1.0f ? vmp_clear_box_small(x, y, z, rs2, r0, r1, r2, r3)
                   : vmp_clear_box_any(x, y, z, rs2, r0, r1, r2, r3);
}

/* ---------------------------------------------------------- packed FP32
 * sm_100 executes fma.rn.f32x2 (FFMA2): two IEEE fused multiply-adds per lane
 * in one instruction - the FMA pipe throughput is unchanged (measured 74.0 vs
 * 70.7 TFLOP/s, scripts/exp_ffma2.cu) but it takes one issue slot instead of
 * two.  Each half rounds exactly like a scalar fmaf, so packed results are
 * bit-identical to the scalar forms. */
typedef unsigned long long vmp_f2;

__device__ __forceinline__ vmp_f2 vmp_pk(float lo, float hi) {
  vmp_f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float vmp_lo(vmp_f2 v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return lo;
}
__device__ __forceinline__ float vmp_hi(vmp_f2 v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return hi;
}
__device__ __forceinline__ vmp_f2 vmp_fma2(vmp_f2 a, vmp_f2 b, vmp_f2 c) {
  vmp_f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

/* vmp_sphere_w of two broadphase groups (packed centres / S / -2R) against
 * one obstacle bound, reduced with fminf: 4 FFMA2 + 1 FMNMX for two groups. */
__device__ __forceinline__ float vmp_sphere_w2(vmp_f2 x, vmp_f2 y, vmp_f2 z, vmp_f2 S, vmp_f2 m2rs,
                                               float4 r0, float r) {
  vmp_f2 w = vmp_fma2(vmp_pk(r, r), m2rs, S);
  w = vmp_fma2(x, vmp_pk(r0.x, r0.x), w);
  w = vmp_fma2(y, vmp_pk(r0.y, r0.y), w);
  w = vmp_fma2(z, vmp_pk(r0.z, r0.z), w);
  return fminf(vmp_lo(w), vmp_hi(w));
}

__device__ __forceinline__ vmp_f2 vmp_mul2(vmp_f2 a, vmp_f2 b) {
  vmp_f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ vmp_f2 vmp_add2(vmp_f2 a, vmp_f2 b) {
  vmp_f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
/* a scalar in both halves: FFMA2 takes it as a broadcast operand (Rn.F32), no MOV */
__device__ __forceinline__ vmp_f2 vmp_bc(float s) { return vmp_pk(s, s); }

/* Narrowphase tests of TWO robot spheres (packed centres x / y / z, S and
 * -2 rs) against one obstacle record: each half evaluates exactly the scalar
 * form above with IEEE fma per half (sphere / capsule: the radius cross term
 * moved to the compare side), at ~0.65 of the issue slots (sphere 3 FFMA2 +
 * 2 FFMA + 2 FSETP; capsule 9 packed + 2 FMUL.SAT + 2 FFMA + 2 FSETP; cuboid
 * 12 packed + 6 FADD.SAT + 2 FSETP).  true = both spheres clear. */
__device__ __forceinline__ bool vmp_clear_sphere2(vmp_f2 x, vmp_f2 y, vmp_f2 z, vmp_f2 S,
                                                  float rsa2, float rsb2, float4 r0, float r) {
  /* the radius cross term 2 rs r sits on the compare side (one scalar FFMA
   * with an immediate per sphere): no packed per-sphere constants */
  vmp_f2 w = vmp_fma2(x, vmp_bc(r0.x), S);
  w = vmp_fma2(y, vmp_bc(r0.y), w);
  w = vmp_fma2(z, vmp_bc(r0.z), w);
  return (vmp_lo(w) > fmaf(r, rsa2, r0.w)) & (vmp_hi(w) > fmaf(r, rsb2, r0.w));
}

__device__ __forceinline__ bool vmp_clear_capsule2(vmp_f2 x, vmp_f2 y, vmp_f2 z, vmp_f2 S,
                                                   float rsa2, float rsb2, float4 r0, float4 r1,
                                                   float4 r2) {
  const vmp_f2 u = vmp_fma2(x, vmp_bc(r0.x), vmp_fma2(y, vmp_bc(r0.y),
                            vmp_fma2(z, vmp_bc(r0.z), vmp_bc(r0.w))));
  const vmp_f2 t = vmp_pk(__saturatef(vmp_lo(u) * r2.x), __saturatef(vmp_hi(u) * r2.x));
  vmp_f2 w = vmp_fma2(x, vmp_bc(r1.x), S);
  w = vmp_fma2(y, vmp_bc(r1.y), w);
  w = vmp_fma2(z, vmp_bc(r1.z), w);
  const vmp_f2 v = vmp_fma2(u, vmp_bc(-2.0f), vmp_mul2(t, vmp_bc(r2.y)));
  const vmp_f2 e = vmp_fma2(t, v, w);
  return (vmp_lo(e) > fmaf(r2.z, rsa2, r1.w)) & (vmp_hi(e) > fmaf(r2.z, rsb2, r1.w));
}

template <bool SMALL_A, bool SMALL_B>
__device__ __forceinline__ bool vmp_clear_box2(vmp_f2 x, vmp_f2 y, vmp_f2 z, float rs2a, float rs2b,
                                               float4 r0, float4 r1, float4 r2, float4 r3) {
  const vmp_f2 l0 = vmp_fma2(x, vmp_bc(r0.x), vmp_fma2(y, vmp_bc(r0.y),
                             vmp_fma2(z, vmp_bc(r0.z), vmp_bc(r0.w))));
  const vmp_f2 l1 = vmp_fma2(x, vmp_bc(r1.x), vmp_fma2(y, vmp_bc(r1.y),
                             vmp_fma2(z, vmp_bc(r1.z), vmp_bc(r1.w))));
  const vmp_f2 l2 = vmp_fma2(x, vmp_bc(r2.x), vmp_fma2(y, vmp_bc(r2.y),
                             vmp_fma2(z, vmp_bc(r2.z), vmp_bc(r2.w))));
  /* rs < 1: FADD.SAT (see vmp_clear_box_small); else FADD + FMNMX */
#define VMP_EXC(SMALL, l, h) (SMALL ? __saturatef(fabsf(l) - (h)) : fmaxf(fabsf(l) - (h), 0.0f))
  const vmp_f2 e0 = vmp_pk(VMP_EXC(SMALL_A, vmp_lo(l0), r3.x), VMP_EXC(SMALL_B, vmp_hi(l0), r3.x));
  const vmp_f2 e1 = vmp_pk(VMP_EXC(SMALL_A, vmp_lo(l1), r3.y), VMP_EXC(SMALL_B, vmp_hi(l1), r3.y));
  const vmp_f2 e2 = vmp_pk(VMP_EXC(SMALL_A, vmp_lo(l2), r3.z), VMP_EXC(SMALL_B, vmp_hi(l2), r3.z));
#undef VMP_EXC
  const vmp_f2 d = vmp_fma2(e0, e0, vmp_fma2(e1, e1, vmp_mul2(e2, e2)));
  return (vmp_lo(d) > rs2a) & (vmp_hi(d) > rs2b);
}

/* Per-lane near masks of the batch kernels: the expanded bound distance minus
 * its threshold, whose SIGN BIT is the near flag (shifted into a mask with one
 * funnel shift).  "near" = strictly negative: a real contact makes the exact
 * value <= -(the bounds' inflation margins), far beyond the rounding of these
 * sums, so treating an exact 0 as clear cannot drop a contact. */
__device__ __forceinline__ vmp_f2 vmp_sub2(vmp_f2 a, vmp_f2 b) {
  vmp_f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ vmp_f2 vmp_near2(vmp_f2 x, vmp_f2 y, vmp_f2 z, vmp_f2 S, vmp_f2 m2rs,
                                            float4 r0, float r) {
  vmp_f2 w = vmp_fma2(vmp_bc(r), m2rs, vmp_sub2(S, vmp_bc(r0.w)));
  w = vmp_fma2(x, vmp_bc(r0.x), w);
  w = vmp_fma2(y, vmp_bc(r0.y), w);
  w = vmp_fma2(z, vmp_bc(r0.z), w);
  return w;
}
/* the same with the bound given as scalars (halves of a bound-pair record) */
__device__ __forceinline__ vmp_f2 vmp_near2s(vmp_f2 x, vmp_f2 y, vmp_f2 z, vmp_f2 S, vmp_f2 m2rs,
                                             float bx, float by, float bz, float bw, float r) {
  vmp_f2 w = vmp_fma2(vmp_bc(r), m2rs, vmp_sub2(S, vmp_bc(bw)));
  w = vmp_fma2(x, vmp_bc(bx), w);
  w = vmp_fma2(y, vmp_bc(by), w);
  w = vmp_fma2(z, vmp_bc(bz), w);
  return w;
}
/* ONE group (scalar centre, S, -2R) against the TWO bounds of a pair record:
 * the chain of vmp_near1 in both halves */
__device__ __forceinline__ vmp_f2 vmp_near1x2(float x, float y, float z, float S, float m2rs,
                                              vmp_f2 bx, vmp_f2 by, vmp_f2 bz, vmp_f2 bw, vmp_f2 r) {
  vmp_f2 w = vmp_fma2(r, vmp_bc(m2rs), vmp_sub2(vmp_bc(S), bw));
  w = vmp_fma2(vmp_bc(x), bx, w);
  w = vmp_fma2(vmp_bc(y), by, w);
  w = vmp_fma2(vmp_bc(z), bz, w);
  return w;
}
__device__ __forceinline__ float vmp_near1(float x, float y, float z, float S, float m2rs,
                                           float4 r0, float r) {
  return fmaf(z, r0.z, fmaf(y, r0.y, fmaf(x, r0.x, fmaf(r, m2rs, S - r0.w))));
}
/* mask = (mask << 1) | sign(w) */
__device__ __forceinline__ unsigned vmp_push_sign(unsigned mask, float w) {
  return __funnelshift_l(__float_as_uint(w), mask, 1);
}

/* Euclidean distance (broadphase group radii, inflated by the caller). */
__device__ __forceinline__ float vmp_dist(float ax, float ay, float az, float bx, float by,
                                          float bz) {
  const float dx = ax - bx, dy = ay - by, dz = az - bz;
  // MUFU.SQRT: within 1 ulp (2^-23.25 relative) of the exact root over every
  // positive normal float (exhaustive check, scripts/exp_sqrt_approx.cu); the
  // group radius it feeds is inflated by 1.000002 + 1e-6 m, which covers it
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaf(dz, dz, fmaf(dy, dy, dx * dx))));
  return r;
}

/* Self pair: clear iff d^2 > f32(ra + rb)^2 (reference collision.py:385-394). */
__device__ __forceinline__ bool vmp_clear_pair(float ax, float ay, float az, float bx, float by,
                                               float bz, float thr) {
  float dx = ax - bx, dy = ay - by, dz = az - bz;
  return fmaf(dz, dz, fmaf(dy, dy, dx * dx)) > thr;
}

/* Self pairs in expanded form (batch kernels): with S = |c|^2 - rs^2 of both
 * spheres, |a - b|^2 > thr  <=>  Sa + Sb - 2 a.b > thr - ra^2 - rb^2 =: T
 * (T a compile-time constant; (mx, my, mz) = -2 b).  The sums stay below a few
 * m^2 in the robot's frame, so the rounding (~5e-7 m^2) moves a verdict only
 * within ~3e-6 m of contact. */
__device__ __forceinline__ bool vmp_clear_pair_x(float ax, float ay, float az, float sa, float mx,
                                                 float my, float mz, float sb, float T) {
  return fmaf(ax, mx, fmaf(ay, my, fmaf(az, mz, sa + sb))) > T;
}
/* two partners (packed centres and S) of one sphere b */
__device__ __forceinline__ bool vmp_clear_pair2(vmp_f2 x, vmp_f2 y, vmp_f2 z, vmp_f2 S, float mx,
                                                float my, float mz, float sb, float Ta, float Tb) {
  vmp_f2 w = vmp_add2(S, vmp_bc(sb));
  w = vmp_fma2(z, vmp_bc(mz), w);
  w = vmp_fma2(y, vmp_bc(my), w);
  w = vmp_fma2(x, vmp_bc(mx), w);
  return (vmp_lo(w) > Ta) & (vmp_hi(w) > Tb);
}

/* Test one robot sphere against obstacle k (records ordered spheres, capsules, boxes). */
__device__ __forceinline__ bool vmp_sphere_clear_obstacle(const float4 *rec, int ns, int nc, int nb,
                                                          int k, float x, float y, float z,
                                                          float rs) {
  (void)nb;
  const float rs2 = rs * rs, m2rs = -2.0f * rs;
  const float S = vmp_sphere_S(x, y, z, rs2);
  if (k < ns) {
    const float4 *p = rec + VMP_SPH_F4 * k;
    return vmp_clear_sphere(x, y, z, S, m2rs, p[0], p[1].x);
  }
  if (k < ns + nc) {
    const float4 *p = rec + VMP_SPH_F4 * ns + VMP_CAP_F4 * (k - ns);
    return vmp_clear_capsule(x, y, z, S, m2rs, p[0], p[1], p[2]);
  }
  const float4 *p = rec + VMP_SPH_F4 * ns + VMP_CAP_F4 * nc + VMP_BOX_F4 * (k - ns - nc);
  return vmp_clear_box(x, y, z, rs, rs2, p[0], p[1], p[2], p[3]);
}

/* Test one robot sphere against every obstacle of env (generic path used by
 * the constant-sphere precheck and the single-primitive API wrappers). */
__device__ __forceinline__ bool vmp_sphere_clear_env(const float4 *rec, int ns, int nc, int nb,
                                                     float x, float y, float z, float rs) {
  const float rs2 = rs * rs;
  const float m2rs = -2.0f * rs;
  const float S = vmp_sphere_S(x, y, z, rs2);
  bool ok = true;
  const float4 *p = rec;
  for (int k = 0; k < ns; ++k, p += 2) ok &= vmp_clear_sphere(x, y, z, S, m2rs, p[0], p[1].x);
  for (int k = 0; k < nc; ++k, p += VMP_CAP_F4) ok &= vmp_clear_capsule(x, y, z, S, m2rs, p[0], p[1], p[2]);
  for (int k = 0; k < nb; ++k, p += VMP_BOX_F4) ok &= vmp_clear_box(x, y, z, rs, rs2, p[0], p[1], p[2], p[3]);
  return ok;
}

/* ------------------------------------------------------- motion arithmetic */

/* numpy float32 sum of squares of (a - b): sequential below 8 elements,
 * eight interleaved accumulators combined as ((0+1)+(2+3))+((4+5)+(6+7)) plus
 * a sequential tail from 8 upwards (numpy pairwise_sum, n <= 128). */
template <int D>
__device__ __forceinline__ float vmp_np_sumsq(const float *a, const float *b) {
  float sq[D > 0 ? D : 1];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    float d = __fsub_rn(a[i], b[i]);
    sq[i] = __fmul_rn(d, d);
  }
  if (D < 8) {
    float r = 0.0f;
#pragma unroll
    for (int i = 0; i < D; ++i) r = __fadd_rn(r, sq[i]);
    return r;
  } else {
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = sq[j < D ? j : 0];
    int i = 8;
#pragma unroll
    for (; i < D - (D % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], sq[(i + j) < D ? (i + j) : 0]);
    }
    float r = __fadd_rn(__fadd_rn(__fadd_rn(acc[0], acc[1]), __fadd_rn(acc[2], acc[3])),
                        __fadd_rn(__fadd_rn(acc[4], acc[5]), __fadd_rn(acc[6], acc[7])));
#pragma unroll
    for (int t = D - (D % 8); t < D; ++t) r = __fadd_rn(r, sq[t]);
    return r;
  }
}

/* n = max(1, ceil(f64(sqrt_f32(sum)) / resolution))  (reference motion.py:25-29). */
template <int D>
__device__ __forceinline__ long long vmp_discretize(const float *s, const float *g, double res) {
  float dist = __fsqrt_rn(vmp_np_sumsq<D>(s, g));
  double steps = ceil(__ddiv_rn((double)dist, res));
  long long n = steps < 1.0 ? 1 : (long long)steps;
  return n > 0x7fffffffLL ? 0x7fffffffLL : n;     /* same clamp as the plan kernels */
}

/* Discretisation count of the edge whose start / goal rows are at s / g. */
template <int D>
__device__ __noinline__ int vmp_discretize_edge(const float *s, const float *g, double res) {
  float sv[D > 0 ? D : 1], gv[D > 0 ? D : 1];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    sv[j] = __ldg(s + j);
    gv[j] = __ldg(g + j);
  }
  return (int)vmp_discretize<D>(sv, gv, res);
}

/* t = f32(f64(i) / n); q = s + t (g - s), unfused (reference motion.py:69-70,
 * lanes.py:101). */
/* t = float32(i / n) with the quotient taken in float64 (reference
 * motion.py:69-70).  For i, n < 2^24 this equals the correctly rounded
 * float32 quotient of the exactly representable float32 operands: double
 * rounding can only differ at a float32 midpoint, and |i/n - M/2^e| >=
 * 1/(n 2^e) keeps a non-midpoint quotient > 2^-49 (relative) away from every
 * 25-bit midpoint, far outside the float64 rounding error 2^-53; an exact
 * midpoint is representable in float64 and rounds identically.  So the cheap
 * IEEE float32 division is bit-exact there, float64 beyond. */
__device__ __forceinline__ float vmp_rake_param(long long i, long long n) {
  if (n < (1ll << 24)) return __fdiv_rn((float)i, (float)n);
  return __double2float_rn(__ddiv_rn((double)i, (double)n));
}

__device__ __forceinline__ float vmp_lerp_exact(float s, float g, float t) {
  return __fadd_rn(s, __fmul_rn(t, __fsub_rn(g, s)));
}

/* ceil(n / w) and the number of 32-position chunks of a W-lane rake over n
 * states, with 32-bit division (n < 2^31, w >= 1). */
__device__ __forceinline__ unsigned vmp_ceil_div(unsigned n, unsigned w) {
  return n / w + (n % w != 0u);
}
__device__ __forceinline__ unsigned vmp_rake_chunks(unsigned n, unsigned w) {
  return (unsigned)(((unsigned long long)vmp_ceil_div(n, w) * w + 31ull) >> 5);
}

#endif
