/* vmp.h - C ABI of the B200 FK + collision-checking + motion-validation path.
 *
 * The reference (arxiv 2309.14545 package `vecmp`, pure Python/NumPy) has no
 * FFI: its boundary is the Python API in pkg/src/vecmp/__init__.py:5-29.  This
 * header is what a binding behind those Python names calls (our own shims in
 * paper_2309_14545_b200/ use ctypes; INTEGRATION.md shows the binding a vecmp
 * maintainer would add).  Each entry point cites the reference interface it
 * replaces.  No C++ or torch types cross this boundary: plain pointers, sizes
 * and an opaque CUDA stream handle (cudaStream_t / CUstream, NULL = legacy).
 *
 * Conventions
 *   - return 0 on success, a negative VMP_E* code on failure; the thread-local
 *     message is available from vmp_last_error().  VMP_EARG maps to Python
 *     ValueError with the same text, VMP_ECUDA / VMP_ECOMPILE to RuntimeError.
 *   - all batch buffers are caller-owned DEVICE memory; calls are asynchronous
 *     on `stream`, perform no allocation, and handles are immutable after
 *     creation, so concurrent calls on distinct streams are safe.
 */
#ifndef VMP_H
#define VMP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VMP_OK 0
#define VMP_EARG (-1)     /* invalid argument            -> ValueError   */
#define VMP_ECUDA (-2)    /* CUDA runtime / launch error -> RuntimeError */
#define VMP_ECOMPILE (-3) /* NVRTC compile or load error -> RuntimeError */
#define VMP_ENOMEM (-4)

/* vmp_validate flags (reference collision.py:411-430 keyword arguments) */
#define VMP_PRUNE 1u         /* coarse per-link sphere prune (prune=True)            */
#define VMP_NO_EARLY_EXIT 4u /* dense mode: every test, no early exit, no broadphase  */
#define VMP_NO_SPLIT 8u      /* never use the small-batch split kernel               */
#define VMP_FORCE_SPLIT 32u  /* always use it (tests)                                */
#define VMP_TWO_PASS 64u     /* two-pass broadphase (bound mask per 32 obstacles)     */
#define VMP_PDL 1024u        /* programmatic dependent launch: this batch may start
                                while the previous kernel on the stream drains - only
                                for inputs that kernel does not write (consecutive
                                batches of resident configurations, ConfigStream)  */
/* vmp_validate_motions flags (reference motion.py:38-90) */
#define VMP_BACKWARD 16u     /* comb each stratum top-down (backward=True)            */
#define VMP_OVERLAPPED 512u  /* batches overlap on several streams (a pipeline); a
                                hint, accepted and currently without effect         */

typedef struct vmp_robot vmp_robot; /* compiled module for one KinematicProgram (+pairs) */
typedef struct vmp_env vmp_env;     /* device-resident packed obstacles                   */

typedef struct {
  int32_t dof;       /* KinematicProgram.dof           (reference program.py:40-50) */
  int32_t n_ops;     /* len(KinematicProgram)                                     */
  int32_t n_markers; /* len(KinematicProgram.checks)                              */
  int32_t has_cc;    /* module contains collision + motion kernels (pairs given)  */
} vmp_robot_desc;

/* Library version (major * 10000 + minor * 100 + patch). */
int vmp_version(void);

/* Thread-local text of the last error ("" if none). */
const char *vmp_last_error(void);

/* Compile CUDA source produced by codegen.py (the lowering of
 * schedule_program's KinematicProgram, reference program.py:82-139) with
 * NVRTC for sm_100a and write the cubin to `cubin_path`.  Needs no GPU. */
int vmp_compile(const char *cuda_source, const char *name, const char *cubin_path);

/* Load a cubin written by vmp_compile on the current device.  Replaces the
 * reference's per-program interpreter state (program.py:56-74 dispatch_ops,
 * Scratch program.py:142-154). */
int vmp_robot_load(const char *cubin_path, const vmp_robot_desc *desc, vmp_robot **out);
void vmp_robot_destroy(vmp_robot *robot);

/* Pack obstacles into device records (reference collision.py:57-119
 * _PackedEnvironment / Environment.packed(); cylinders arrive as capsules,
 * collision.py:147-153).  Inputs are host float64, row-major:
 *   spheres  n_spheres  x 4 : cx cy cz r
 *   capsules n_capsules x 7 : p0(3) p1(3) r
 *   boxes    n_boxes    x 15: centre(3) half_extents(3) rotation(9, row-major, world-from-box)
 */
int vmp_env_create(const double *spheres, int32_t n_spheres, const double *capsules,
                   int32_t n_capsules, const double *boxes, int32_t n_boxes, vmp_env **out);
/* Same, with the records expressed in a frame centred at `origin` (3 doubles,
 * rounded to float32; NULL = world origin).  vmp_validate and
 * vmp_validate_motions need the frame of the robot they run with,
 * vmp_robot_home(): its generated kernels test sphere centres minus that point
 * (folded into the forward kinematics at codegen time), so the expanded test
 * forms never cancel |c|^2-sized terms - a robot 30 m from the world origin
 * keeps the accuracy of one at the origin.  vmp_sphere_hits subtracts the
 * origin itself and accepts any frame.  Verdict semantics are unchanged
 * (reference collision.py:206-254). */
int vmp_env_create_at(const double *spheres, int32_t n_spheres, const double *capsules,
                      int32_t n_capsules, const double *boxes, int32_t n_boxes,
                      const double *origin, vmp_env **out);
void vmp_env_destroy(vmp_env *env);
/* The environment frame origin the robot's collision kernels assume: the mean
 * sphere centre at the zero configuration, rounded to 1/64 m (3 doubles). */
int vmp_robot_home(const vmp_robot *robot, double *home);
/* Bytes of the packed device records (shared-memory staging size). */
int64_t vmp_env_bytes(const vmp_env *env);

/* Every op row of the program for n configurations q (dof x ld, float32):
 * rows (n_ops x ldo).  Replaces evaluate_program's lane loop
 * (reference program.py:157-214) - the sink replay happens in the caller. */
int vmp_fk_rows(const vmp_robot *robot, const float *q, int64_t n, int64_t ld, float *rows,
                int64_t ldo, void *stream);

/* Sphere centres only: rows 3m+{0,1,2} for marker m (n_markers*3 x ldo). */
int vmp_fk_spheres(const vmp_robot *robot, const float *q, int64_t n, int64_t ld,
                   float *centres, int64_t ldo, void *stream);

/* Fused FK + self-collision + environment check of n configurations.
 * valid_bits: ceil(n/32) words, bit (i % 32) of word i/32 set = VALID.
 * Replaces validate_block / ValidationContext.validate_block
 * (reference collision.py:411-430, 433-459) for any block width. */
int vmp_validate(const vmp_robot *robot, const vmp_env *env, const float *q, int64_t n,
                 int64_t ld, uint32_t flags, uint32_t *valid_bits, void *stream);

/* Raked motion validation of n_edges straight-line motions (starts/goals:
 * n_edges x sld float32, row-major).  Replaces raked_motion_check /
 * validate_motion_rake (reference motion.py:38-90) batched over edges.
 *   width      : rake width W whose block counts are reproduced (ctx.width);
 *                32 is the native warp width
 *   valid_bits : ceil(n_edges/32) words, bit set = every state valid
 *   n_states   : optional, discretization_count per edge (motion.py:25-29)
 *   blocks     : optional, block evaluations the W-wide rake performs
 *   workspace  : >= vmp_motion_workspace_bytes(n_edges) bytes of device
 *                scratch (work queue, per-edge failure records and counts);
 *                16-byte aligned and ZERO-FILLED before its first use.  Its
 *                layout depends only on workspace_bytes, so one workspace
 *                serves batches of any size it holds; each call resets the
 *                queue and the failure records itself before it uses them
 *                (whatever an earlier call left behind)
 * Launches begin (reset) -> fused FK+CC rake -> finalize on `stream`, chained
 * by programmatic dependent launch; above 2^22 edges in sub-batches. */
int vmp_validate_motions(const vmp_robot *robot, const vmp_env *env, const float *starts,
                         const float *goals, int64_t n_edges, int64_t sld, double resolution,
                         int32_t width, uint32_t flags, uint32_t *valid_bits, int32_t *n_states,
                         int32_t *blocks, void *workspace, int64_t workspace_bytes, void *stream);

/* Device scratch bytes vmp_validate_motions needs for n_edges edges. */
int64_t vmp_motion_workspace_bytes(int64_t n_edges);

/* n = max(1, ceil(||g - s|| / resolution)) per edge with numpy float32
 * reduction order (reference motion.py:25-29, lanes.py:106-113); dim <= 128
 * (numpy sums longer rows recursively). */
int vmp_discretize(const float *starts, const float *goals, int64_t n_edges, int32_t dim,
                   int64_t sld, double resolution, int32_t *n_out, void *stream);

/* Host-buffer variants of vmp_validate / vmp_validate_motions for callers
 * with host data (the reference's per-call API: state_valid, a W = 8
 * validate_block, one raked_motion_check): copy the inputs (host, row stride
 * ld / sld floats; pinned memory makes the copies asynchronous DMA) into
 * `scratch` (device, >= the *_scratch_bytes size), run the kernels, copy the
 * verdict words (and optional per-edge n / W-lane block counts) back to host
 * memory, and synchronise `stream` - one C call per request. */
int64_t vmp_validate_host_scratch_bytes(const vmp_robot *robot, int64_t n);
int vmp_validate_host(const vmp_robot *robot, const vmp_env *env, const float *q_host, int64_t n,
                      int64_t ld, uint32_t flags, uint32_t *bits_host, void *scratch,
                      int64_t scratch_bytes, void *stream);
int64_t vmp_motions_host_scratch_bytes(const vmp_robot *robot, int64_t n_edges);
int vmp_validate_motions_host(const vmp_robot *robot, const vmp_env *env, const float *starts_host,
                              const float *goals_host, int64_t n_edges, int64_t sld,
                              double resolution, int32_t width, uint32_t flags,
                              uint32_t *bits_host, int32_t *n_states_host, int32_t *blocks_host,
                              void *scratch, int64_t scratch_bytes, void *workspace,
                              int64_t workspace_bytes, void *stream);

/* Zero-filled device memory on the current device (scratch / workspace for
 * bindings without their own allocator, e.g. a ctypes module); 0 bytes gives
 * NULL.  vmp_device_free(NULL) is a no-op. */
int vmp_device_alloc(int64_t bytes, void **out);
void vmp_device_free(void *ptr);

/* FP32 FMA-pipe microbenchmark: `launches` back-to-back launches of a kernel
 * of 4 independent FFMA chains per thread (8 x 256-thread CTAs per SM,
 * 2 * 256 * iters flop per thread per launch), timed with CUDA events on a
 * private stream; returns the achieved TFLOP/s (and ms).  bench.py uses it
 * as the measured roofline denominator of this FP32-bound path (burst: one
 * launch of a few ms; sustained: seconds of launches). */
int vmp_bench_ffma(int64_t iters, int32_t launches, double *tflops, double *ms);

/* The states the rake visits (reference motion.py:32-78 strata,
 * lanes.py:91-103 interpolate_lanes), written in the rake kernels' position
 * order with the same device arithmetic, for parity checks and callers that
 * want the sample points: edge e occupies positions [offsets[e],
 * offsets[e] + S_e W), S_e = ceil(n_e / W) (offsets: n_edges + 1 device int64,
 * exclusive prefix sum the caller computes from vmp_discretize).  Position
 * p holds index_out = k S + j (k = p mod W, j = p / W + 1; S - j + 1 with
 * VMP_BACKWARD), or 0 past n, and the state (dim floats, row p) at
 * t = f32(index / n) (index 1 past n). */
int vmp_motion_states(const float *starts, const float *goals, int64_t n_edges, int32_t dim,
                      int64_t sld, double resolution, int32_t width, uint32_t flags,
                      const int64_t *offsets, int32_t *index_out, float *states, void *stream);

/* Per-obstacle, per-lane contact of spheres of one radius against env
 * (hits: n_obstacles x n bytes, 1 = contact, obstacle order spheres,
 * capsules, boxes).  Backs sphere_vs_{sphere,capsule,cuboid}_lanes
 * (reference collision.py:263-287) and BlockValidator. */
int vmp_sphere_hits(const vmp_env *env, const float *xyz, int64_t n, int64_t ld, float radius,
                    uint8_t *hits, void *stream);

/* Lane-wise self-pair test of two sphere-centre streams a, b (3 x ld each):
 * clear[i] = |a_i - b_i|^2 > thr, thr = f32(ra + rb)^2 (reference
 * collision.py:385-394).  Backs the BlockValidator sink. */
int vmp_pair_clear(const float *a, const float *b, int64_t n, int64_t ld, float thr,
                   uint8_t *clear, void *stream);

/* Exact k-nearest neighbours (reference NNIndex.k_nearest / nearest,
 * nn.py:45-69).  points: dim x ld float32 SoA (device), n_points columns;
 * queries: n_queries x qld float32 rows (device).  Distance = sqrtf of the
 * float32 squares summed in joint order (unfused); results ascending by
 * (distance, point index) - ties go to the earlier-inserted point.
 *   visible   : optional device int64 per query - only points [0, visible[q])
 *               are candidates (a growing index queried mid-insertion)
 *   out_index : n_queries x k int32, -1 past the candidate count
 *   out_dist  : n_queries x k float32, +inf past the candidate count
 * 1 <= k <= VMP_KNN_MAX_K, 1 <= dim <= VMP_KNN_MAX_DIM. */
#define VMP_KNN_MAX_K 32
#define VMP_KNN_MAX_DIM 64
int vmp_knn(const float *points, int64_t n_points, int64_t ld, int32_t dim, const float *queries,
            int64_t n_queries, int64_t qld, const int64_t *visible, int32_t k, int32_t *out_index,
            float *out_dist, void *stream);

/* Every query-to-point distance (same arithmetic as vmp_knn) into out
 * (n_queries x ldo), any dim in [1, 12288]; the k > VMP_KNN_MAX_K and
 * dim > VMP_KNN_MAX_DIM paths sort these stably. */
int vmp_nn_distances(const float *points, int64_t n_points, int64_t ld, int32_t dim,
                     const float *queries, int64_t n_queries, int64_t qld, float *out, int64_t ldo,
                     void *stream);

/* Debug: copy up to n words of the rake kernel's timeline (recorded only when
 * the process starts with VMP_MOTION_TRACE set; 8 words per CTA of the last
 * launch: entry, plan ready, warp 0-3 queue empty, exit - globaltimer ns -
 * and work items taken).  Returns the words copied, 0 when tracing is off. */
int64_t vmp_debug_motion_trace(uint64_t *host, int64_t n);

/* Select the CUDA device used by subsequent vmp calls on this thread (robots
 * and environments remember the device they were created on). */
int vmp_set_device(int32_t device);

/* SM count of the current device and its ordinal (diagnostics). */
int vmp_device_info(int32_t *sm_count, int32_t *device);

#ifdef __cplusplus
}
#endif
#endif
