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
typedef struct {
  const float4 *rec;   /* device pointer, 16-byte aligned */
  int ns, nc, nb;      /* sphere / capsule / cuboid counts */
  int n_f4;            /* total float4 records = 2 ns + 4 nc + 5 nb */
  float ox, oy, oz;    /* origin of the environment frame: records hold obstacle
                          geometry minus it, kernels subtract it from sphere centres */
  int pad_;
} VmpEnvView;

typedef struct {
  const float *q;      /* (dof, ld) float32 SoA batch */
  long long n;         /* configurations */
  long long ld;        /* leading dimension of q */
  VmpEnvView env;
  unsigned int *bits;  /* ceil(n / 32) packed verdicts, bit set = VALID */
  int stage;           /* 1: stage env in shared memory via cp.async.bulk */
  int pad_;
} VmpValidateArgs;

/* Motion workspace (the per-edge arrays are laid out by the capacity the
 * workspace size implies, E_cap; every call resets the queue counters before
 * the rake starts and rewrites every per-edge record it reads):
 *   VmpMotionHeader
 *   unsigned hist[VMP_HBINS], fill[VMP_HBINS]   chunk-count histogram / scatter cursors
 *   long long off[VMP_HBINS]                    first work item of chunk round c
 *   int rank_of[E_cap]                          per edge: index of its rank record
 *   int n[E_cap], chunks[E_cap]                 per edge: discretisation count and
 *                                               chunks (multi-kernel plan only)
 *   int4 order[E_cap]                           rank records (edge, n, chunks, failure
 *                                               record) by chunk count descending; the
 *                                               failure record is INT_MAX - first failing
 *                                               iteration, 0 while none (atomicMax)
 * Work item t < E is round 0 of edge t (input order, no plan needed); item
 * E <= t < off[HBINS-1] is (round c, rank r): edge order[r], chunk c, where
 * off[c] <= t < off[c+1]; rounds >= HBINS-1 enumerate the n_big longest edges
 * (chunks >= HBINS-1) and skip absent chunks. */
#define VMP_HBINS 1024
#define VMP_QSTRIPES 16           /* item queue striped over 16 counters (t % 16) */
#define VMP_TRACE_ITEM0 8192      /* debug timeline: per-item records start here */
#define VMP_TRACE_ITEMS 30000     /* items recorded (4 words each) */
#define VMP_OFF_CACHE 64          /* round offsets a rake warp keeps in shared memory */
typedef struct {
  unsigned long long counter[VMP_QSTRIPES * 16]; /* stripe s at [16 s]: one 128 B line each */
  unsigned long long total_items; /* written by the scan kernel */
  unsigned int max_chunks;        /* max over edges of ceil(S W / 32), S = ceil(n / W) */
  unsigned int n_big;             /* edges with chunks >= VMP_HBINS - 1 */
  unsigned int done_ctas;         /* CTAs of the rake kernel that finished */
  unsigned int plan_done;         /* reserved (kept zero) */
  unsigned int pad_[2];           /* keep the arrays behind 16-byte aligned */
} VmpMotionHeader;

/* Dynamic-queue rake (batches up to VMP_DQ_MAX_EDGES edges per launch; the
 * default).  No plan: round 0 - the first chunk of every edge, discretised by
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
#define VMP_DQ_STATE 0
#define VMP_DQ_CALLS 16
#define VMP_DQ_MAX_EDGES (1 << 22)
#define VMP_DQ_SLOTS_PER_EDGE 8   /* slot capacity per edge of workspace capacity; an edge
                                     whose chunks do not fit is finished by its own warp */

typedef struct {
  const float *starts; /* (n_edges, sld) float32 AoS */
  const float *goals;  /* (n_edges, sld) float32 AoS */
  long long n_edges;
  long long sld;       /* row stride of starts / goals in floats */
  double resolution;
  VmpEnvView env;
  VmpMotionHeader *hdr;
  const long long *off; /* first work item of each chunk round */
  int4 *order;          /* rank records (edge, n, chunks, failure record), chunk count
                           descending; .w = INT_MAX - first failing iteration, 0 while none */
  const int *rank_of;   /* per edge: index of its rank record (read by failing round-0
                           items after the plan, and by finalize) */
  int *pad_ptr_;        /* reserved */
  unsigned long long *trace; /* debug timeline (VMP_MOTION_TRACE), normally null:
                                per CTA [entry, plan ready, warp 0-3 queue empty,
                                exit, work items taken] in globaltimer ns */
  int width;            /* rake lane width W whose block counts are reproduced */
  int backward;         /* comb strata top-down */
  int stage;
  int guard_waves;      /* stop prefetching queue items this many items per warp
                           before the end (4 for an isolated batch; 1 when batches
                           overlap, whose tails the next batch fills) */
  /* dynamic-queue rake */
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
