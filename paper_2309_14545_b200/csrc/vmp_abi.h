/* Kernel-argument structs shared by the host library (vmp.cu) and the
 * NVRTC-compiled per-robot modules (codegen.py inlines this file).
 * Plain C layout: both compilers must agree byte for byte. */
#ifndef VMP_ABI_H
#define VMP_ABI_H

/* Environment as seen by a kernel: packed float4 records, grouped by kind
 * (spheres: 2 float4, capsules: 3 float4, cuboids: 4 float4 each; layout in
 * DESIGN.md "Data layout in HBM"). */
typedef struct {
  const float4 *rec;   /* device pointer, 16-byte aligned */
  int ns, nc, nb;      /* sphere / capsule / cuboid counts */
  int n_f4;            /* total float4 records = 2 ns + 3 nc + 4 nb */
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

/* Motion workspace: this header, then int n[E], int chunks[E], int fail[E]. */
typedef struct {
  unsigned long long counter; /* work-item queue (zeroed before the plan kernel) */
  unsigned int max_chunks;    /* max over edges of ceil(S W / 32), S = ceil(n / W) */
  unsigned int pad_;
} VmpMotionHeader;

typedef struct {
  const float *starts; /* (n_edges, sld) float32 AoS */
  const float *goals;  /* (n_edges, sld) float32 AoS */
  long long n_edges;
  long long sld;       /* row stride of starts / goals in floats */
  double resolution;
  VmpEnvView env;
  VmpMotionHeader *hdr;
  const int *n_of;      /* discretisation count per edge (plan kernel) */
  const int *chunks_of; /* 32-position chunks per edge (plan kernel) */
  int *fail_of;         /* first failing rake iteration, INT_MAX while none */
  int width;            /* rake lane width W whose block counts are reproduced */
  int backward;         /* comb strata top-down */
  int stage;
  int pad_;
} VmpMotionArgs;

typedef struct {
  const float *q;      /* (dof, ld) */
  long long n;
  long long ld;
  float *out;          /* (rows, ldo) */
  long long ldo;
} VmpFkArgs;

#endif
