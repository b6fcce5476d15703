/* Kernel-argument structs shared by the host library (vmp.cu) and the
 * NVRTC-compiled per-robot modules (codegen.py inlines this file).
 * Plain C layout: both compilers must agree byte for byte. */
#ifndef VMP_ABI_H
#define VMP_ABI_H

/* Environment as seen by a kernel: packed float4 records, grouped by kind
 * (spheres: 2 float4, capsules: 4 float4, cuboids: 5 float4 each - the last
 * record of a capsule / cuboid is its bounding sphere; layout in
 * csrc/vmp_device.cuh and DESIGN.md "Data layout in HBM"). */
#define VMP_SPH_F4 2
#define VMP_CAP_F4 4
#define VMP_BOX_F4 5
#define VMP_PAIR_F4 3  /* behind the obstacle records, per kind: one record per two
                          obstacles with their bounding spheres interleaved as
                          packed operands (xa, xb, ya, yb) (za, zb, wa, wb)
                          (ra, rb, 0, 0); ceil(n / 2) records per kind */
typedef struct {
  const float4 *rec;   /* device pointer, 16-byte aligned */
  int ns, nc, nb;      /* sphere / capsule / cuboid counts */
  int n_f4;            /* per-obstacle float4 records = 2 ns + 4 nc + 5 nb */
  float ox, oy, oz;    /* origin of the environment frame: records hold obstacle
                          geometry minus it, kernels subtract it from sphere centres */
  int n_all_f4;        /* n_f4 + the bound pairs: 3 (ceil(ns / 2) + ceil(nc / 2) + ceil(nb / 2)) */
} VmpEnvView;

typedef struct {
  const float *q;      /* (dof, ld) float32 SoA batch */
  long long n;         /* configurations */
  long long ld;        /* leading dimension of q */
  VmpEnvView env;
  unsigned int *bits;  /* ceil(n / 32) packed verdicts, bit set = VALID */
  int stage;           /* 1: stage env in shared memory via cp.async.bulk; 2: with the
                          bound pairs behind the records (pair bound pass) */
  int pad_;
} VmpValidateArgs;

/* Motion workspace of the dynamic-queue rake (batches up to VMP_DQ_MAX_EDGES
 * edges per launch).  No plan: round 0 - the first chunk of every edge, discretised by
 * the item itself - is dealt out statically; an edge whose first iteration
 * passed publishes its remaining chunks as slot records, which warps then pop.
 * Only surviving edges ever enter the queue.  Workspace regions used (laid out
 * by the capacity the workspace size implies):
 *   hdr->counter[16 s]     pop counter of stripe s: its k-th pop is slot
 *                          VMP_QSTRIPES k + s (one 128 B line per stripe)
 *   dq[VMP_DQ_STATE]       (round-0 items finished) << 40 | slots reserved: one
 *                          atomicAdd per round-0 item both reserves its slots
 *                          and counts it done, so a reader gets both at once
 *   dq[VMP_DQ_CALLS]       calls on this workspace; slot tag = 1 + calls % 65535
 *                          (dq = the 64-bit words behind the header, one line each)
 *   int fail[E_dq]         per edge: INT_MAX - first failing iteration, 0 = none
 *   int n[E_dq]            per edge: discretisation count (written by round 0)
 *   u64 slots[2 * cap]     slot i = two self-validating words
 *                          w0 = tag << 48 | (chunk & 0x1ffff) << 31 | edge
 *                          w1 = tag << 48 | (chunk >> 17) << 31 | n
 *                          (each 8-byte word is written and read whole and
 *                          carries the call's tag: no fence, no zeroing)
 * vmp_k_motion_begin (one CTA) resets the counters, zeroes fail[] and bumps the
 * call count before the rake's first write (programmatic dependent launch). */
#define VMP_QSTRIPES 16           /* slot queue striped over 16 pop counters (slot % 16) */
#define VMP_DQ_STATE 0
#define VMP_DQ_CALLS 16
#define VMP_DQ_MAX_EDGES (1 << 22)
#define VMP_DQ_SLOTS_PER_EDGE 8   /* slot capacity per edge of workspace capacity (plus a
                                     fixed spare); an edge whose chunks do not fit is
                                     finished by its own warp */
#define VMP_TRACE_ITEM0 8192      /* debug timeline: per-item records start here */
#define VMP_TRACE_ITEMS 30000     /* items recorded (4 words each) */
typedef struct {
  unsigned long long counter[VMP_QSTRIPES * 16]; /* stripe s at [16 s]: one 128 B line each */
} VmpMotionHeader;

typedef struct {
  const float *starts; /* (n_edges, sld) float32 AoS */
  const float *goals;  /* (n_edges, sld) float32 AoS */
  long long n_edges;
  long long sld;       /* row stride of starts / goals in floats */
  double resolution;
  VmpEnvView env;
  VmpMotionHeader *hdr;
  unsigned long long *trace; /* debug timeline (VMP_MOTION_TRACE), normally null:
                                per CTA [entry, first wait over, warp 0-3 queue empty,
                                exit, work items taken] in globaltimer ns */
  int width;            /* rake lane width W whose block counts are reproduced */
  int backward;         /* comb strata top-down */
  int stage;
  int pad_;
  int *fail;            /* per edge failure record */
  int *n_of;            /* per edge discretisation count */
  unsigned long long *slots; /* 2 words per slot */
  unsigned long long *dq;    /* state / call-count words */
  long long slot_cap;   /* slots the workspace holds */
} VmpMotionArgs;

typedef struct {
  const float *q;      /* (dof, ld) */
  long long n;
  long long ld;
  float *out;          /* (rows, ldo) */
  long long ldo;
} VmpFkArgs;

#endif
