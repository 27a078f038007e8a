/*
 * capt_b200 -- B200-native CAPT batched sphere-vs-point-cloud collision query.
 *
 * C-ABI boundary of libcapt_b200.so.  Plain pointers and sizes only; every
 * entry point is stream-ordered on the caller's cudaStream_t (passed as
 * void*, NULL = legacy default stream) unless CAPT_HOST_IO is set, in which
 * case the call copies host buffers in/out and returns after the results are
 * on the host.
 *
 * The reference (arXiv 2406.02807 companion package `captree`, pure
 * Python/numpy) has no FFI; its boundary is the Python API.  Each entry point
 * below names the reference function it replaces (file:line relative to
 * /root/reference/pkg/src/captree).  INTEGRATION.md shows the ctypes binding
 * the reference would add; paper_2406_02807_b200/ is that binding.
 *
 * Status codes (capt_last_error() returns the thread-local message):
 *   CAPT_OK       0
 *   CAPT_EINVAL   1  invalid argument            -> ValueError
 *   CAPT_ERANGE   2  radius outside [r_min,r_max] -> ValueError (query.py:30-34)
 *   CAPT_ECUDA    3  CUDA runtime/launch failure  -> RuntimeError
 *   CAPT_ENOMEM   4  device allocation failed     -> MemoryError
 */
#ifndef CAPT_B200_H
#define CAPT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CAPT_OK 0
#define CAPT_EINVAL 1
#define CAPT_ERANGE 2
#define CAPT_ECUDA 3
#define CAPT_ENOMEM 4

/* capt_query / capt_leaf_indices flags */
#define CAPT_PREFILTER 0x1u   /* use_aabb_prefilter (query.py:184-186)          */
#define CAPT_CHECK_RADII 0x2u /* check_radii: report first out-of-band radius  */
#define CAPT_STATS 0x4u       /* fill counters[0..3] (see capt_query)           */
#define CAPT_INPUT_F64 0x8u   /* centers/radii are double (else float)          */
#define CAPT_HOST_IO 0x10u    /* all array arguments are host memory; blocking  */
#define CAPT_MODE_DIRECT 0x100u /* force the unbinned path (the hybrid kernel
                                   for fp32 k=3 input, else warp-per-sphere) */
#define CAPT_MODE_BINNED 0x200u /* force the leaf-binned kernels               */
#define CAPT_MODE_THREAD 0x400u /* force the one-thread-per-sphere kernel
                                   (always used with CAPT_STATS)               */
#define CAPT_K5_FFMA 0x800u     /* binned scan on the CUDA cores (FFMA2) instead
                                   of the tensor cores (tcgen05 tf32)          */
#define CAPT_MODE_WARP 0x1000u  /* unbinned: the warp-per-sphere kernel instead
                                   of the hybrid (thread classify + warp scan) */
#define CAPT_MODE_FIELD 0x2000u /* force the clearance-field pipeline (the
                                   default for fp32 k=3 queries without
                                   CAPT_STATS); EINVAL if the tree has none.
                                   With CAPT_MODE_BINNED / CAPT_MODE_DIRECT:
                                   the undecided spheres go through the
                                   binned pipeline / the warp list kernel  */

typedef struct capt_tree capt_tree;

typedef struct {
  int32_t k;              /* dimension (1..3)                                 */
  int32_t depth;          /* log2(n_leaves) descent steps (tree.py:93)        */
  int64_t n_leaves;       /* power of two (tree.py:150)                       */
  int64_t n_points;       /* points in the source cloud                       */
  int64_t total_stored;   /* sum of affordance-set sizes (BuildStats)         */
  int64_t max_affordance; /* largest set                                      */
  double r_min, r_max;    /* exactness band (BuildParams, tree.py:41-52)      */
  int64_t device_bytes;   /* size of the device slab                          */
  int32_t device;         /* CUDA ordinal holding the slab                    */
  int32_t reserved;
  int64_t n_ties;         /* split nodes with equal rank-(m/2-1)/(m/2) coords */
} capt_tree_info;

/* Thread-local message for the last non-OK status. */
const char* capt_last_error(void);
int capt_version(void);

/* Capt.__init__ (tree.py:74-97) / load_capt (tree.py:291-320): upload a tree
 * given in the reference layout (host arrays): tests (n-1) fp32 Eytzinger,
 * aff_lo/aff_hi (n*k) fp32, offsets (n+1) int64 CSR, aff_values
 * (offsets[n]*k) fp32, SoA within each set, representative first. */
int capt_tree_create(int device, int k, int64_t n_leaves, int64_t n_points,
                     double r_min, double r_max, const float* tests,
                     const float* aff_lo, const float* aff_hi,
                     const int64_t* offsets, const float* aff_values,
                     capt_tree** out);

/* construct(cloud, BuildParams(r_min, r_max), use_rmin_shortcut)
 * (tree.py:139-241), on device.  points: (n_points, k) fp32, device memory
 * unless flags has CAPT_HOST_IO.  Ties at a split go left by original index. */
int capt_tree_build(int device, int k, const float* points, int64_t n_points,
                    double r_min, double r_max, int use_rmin_shortcut,
                    uint32_t flags, void* stream, capt_tree** out);

int capt_tree_info_get(const capt_tree* tree, capt_tree_info* info);

/* Copy the tree back in the reference layout (host buffers sized from
 * capt_tree_info).  Rows 1.. of each set are in ascending original-index
 * order for device-built trees, in upload order for uploaded trees. */
int capt_tree_export(const capt_tree* tree, float* tests, float* aff_lo,
                     float* aff_hi, int64_t* offsets, float* aff_values);

void capt_tree_destroy(capt_tree* tree);

/* Position-independent device slab (for replication across GPUs: NCCL
 * broadcast the slab bytes, then capt_tree_from_slab on each rank).  With
 * CAPT_SLAB_BORROW the new tree adopts dev_slab instead of copying it (the
 * caller keeps the buffer alive and unchanged until capt_tree_destroy). */
#define CAPT_SLAB_BORROW 0x1u
int capt_tree_slab(const capt_tree* tree, const void** dev_ptr, int64_t* bytes);
int capt_tree_from_slab(int device, const void* dev_slab, int64_t bytes, uint32_t flags,
                        void* stream, capt_tree** out);

/* collides_many (query.py:184-219) when lane_width == 1; otherwise
 * collides_batch(tree, SphereBatch(...)).any_collision (query.py:126-167)
 * for every consecutive group of lane_width (power of two <= 32) spheres.
 *   centers: (n, k) float (or double with CAPT_INPUT_F64); radii: (n,)
 *   lane_mask: optional (n,) bytes, 0 = masked lane (SphereBatch.mask)
 *   out_bits: ceil((n/lane_width)/32) words; verdict g is bit g%32 of word g/32
 *   counters (optional, 6 x uint64, written with CAPT_STATS):
 *     [0] collisions (spheres, or groups when lane_width > 1)
 *     [1] boundary spheres: some scanned point has |d^2 - r^2| < 1e-6 (fp64)
 *     [2] points scanned, reference semantics (query.py:153-155): full set
 *         sizes of AABB-passing spheres; for groups, lanes in order up to and
 *         including the first colliding lane
 *     [3] spheres resolved by the float64 fix-up path
 *     [4] valid spheres rejected by the AABB prefilter (aabb_rejections)
 *     [5] reserved (0)
 *   first_bad (optional): index of the first out-of-band radius among valid
 *     lanes, -1 if none (CAPT_CHECK_RADII).  With CAPT_HOST_IO a bad radius
 *     makes the call return CAPT_ERANGE. */
int capt_query(const capt_tree* tree, const void* centers, const void* radii,
               int64_t n, int lane_width, const uint8_t* lane_mask,
               uint32_t flags, uint32_t* out_bits, uint64_t* counters,
               int64_t* first_bad, void* stream);

/* leaf_indices (tree.py:266-273): out (n,) int64 leaf of every center. */
int capt_leaf_indices(const capt_tree* tree, const void* centers, int64_t n,
                      uint32_t flags, int64_t* out, void* stream);

/* filter_cloud (morton.py:185-236), optional reach_filter pre-pass
 * (morton.py:173-182).  points (n, k) fp32; out_points must hold n rows;
 * *n_out receives the output count.  Host memory with CAPT_HOST_IO, else
 * device memory (then *n_out is written by the call before it returns). */
int capt_filter_cloud(int device, int k, const float* points, int64_t n,
                      double r_filter, int has_reach, const double* base,
                      double max_reach, uint32_t flags, float* out_points,
                      int64_t* n_out, void* stream);

/* dispersion_stats (oracle.py:141-158): out (n,) float64 distance from every
 * point to its nearest OTHER point (duplicates: 0), the value a float64
 * k-d tree query with k=2 returns.  points (n, k) fp32; host buffers with
 * CAPT_HOST_IO, else device memory.  n >= 2. */
int capt_nn_distances(int device, int k, const float* points, int64_t n,
                      uint32_t flags, double* out, void* stream);

/* Clearance field of a k = 3 tree (derived data, built on the device with
 * the tree): a uniform grid of nx*ny*nz cells of edge h from lo; cell
 * (ix,iy,iz) is number (iz*ny + iy)*nx + ix, with centre x0 =
 * fmaf((float)ix, h, c0[0]) (likewise y, z).  Per cell:
 *   witness = the cloud point nearest x0 (+inf if none within rcap);
 *   nn <= the distance from x0 to every cloud point (nn <= rcap);
 *   n_cand candidate points: the cloud points nearest x0 (fewer when fewer
 *     lie within rcap), stored as int16 offsets q = rint((p - x0) / q_step)
 *     per axis; a decoded difference fl(fl(c - x0) - q q_step) is within
 *     q_err of c - p (Euclidean) for a centre c of the cell;
 *   kd <= the distance from x0 to every cloud point that is not a candidate
 *     (kd <= rcap, a multiple of q_step).
 * box_lo/box_hi: the cloud's box.  cells: NULL, or a host buffer of
 * 8 * n_cells floats {witness x, y, z, nn, kd, candidate count, kd2, k2}:
 * kd2 = the ring drain's second-record bound (<= the distance from x0 to
 * every cloud point after the witness and the next k2 nearest).
 * cand: NULL, or a host buffer of 3 * n_cand * n_cells floats (each
 * candidate's offsets q, +inf for unused slots).  Returns CAPT_EINVAL for
 * trees without a field. */
typedef struct {
  int32_t nx, ny, nz, n_cand;
  int64_t n_cells;
  float lo[3], h;
  float box_lo[3], box_hi[3];
  float rcap, q_step;
  float c0[3], q_err;
} capt_field_info;
int capt_tree_field(const capt_tree* tree, capt_field_info* info, float* cells, float* cand);

/* The clearance field's block table (K0 keeps it in shared memory): blocks
 * of 2^shift cells per axis, dims[0..2] = blocks along x, y, z, block
 * (bx,by,bz) is entry (bz*dims[1] + by)*dims[0] + bx.  Entry q certifies
 * q * step <= the distance from the cloud to every centre whose computed
 * cell lies in the block.  dims: 4 ints {bx, by, bz, shift}; step: 1 float;
 * table: NULL or a host buffer of bx*by*bz bytes.  CAPT_EINVAL for trees
 * without a field. */
int capt_tree_field_blocks(const capt_tree* tree, int32_t* dims, float* step, uint8_t* table);

/* Stage timing of the clearance-field pipeline (measurement helper for
 * bench.py's roofline): while enabled, every field-pipeline capt_query
 * records CUDA events on its stream around the resolve kernel (K0) and the
 * list stage.  capt_stage_times waits for them and returns the summed
 * milliseconds ms[0] = K0, ms[1] = list stage, ms[2] = both, with the number
 * of calls, then clears the record.  Enabling also clears it. */
int capt_stage_timing(int enable);
int capt_stage_times(double* ms, int64_t* calls);

/* List lengths of the last field-pipeline capt_query issued on `stream` on
 * the current device (measurement helper for the list stage's roofline):
 * out[0] = spheres K0 left undecided (the candidate-record list), out[1] =
 * open in-band entries resolved by the exact bucket scan, out[2] = entries
 * taking the tree path (out-of-band radii with check_radii off, non-finite
 * or out-of-grid centres).  out holds 3 values.  Waits for the stream.
 * CAPT_EINVAL if no field query ran on that stream. */
int capt_field_list_counts(void* stream, uint32_t* out);

/* Number of kernels this library has launched in the process so far
 * (all devices/threads); used by bench.py to report gpu_launches. */
int64_t capt_kernel_launches(void);

/* Measurement helper for the roofline denominator: FFMA throughput of this
 * device in TFLOP/s (CUDA-event timed dependent-chain FMA kernel). */
int capt_measure_fp32_peak(int device, double* tflops);

/* Diagnostic: one 128x256x16 tf32 tcgen05 product through the library's
 * tensor-core operand layout; *max_rel_err = worst |D - ref| / sum|a_k b_k|. */
int capt_tc_selftest(int device, double* max_rel_err);

#ifdef __cplusplus
}
#endif
#endif /* CAPT_B200_H */
