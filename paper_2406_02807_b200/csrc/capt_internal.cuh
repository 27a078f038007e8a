// Internal definitions shared by the libcapt_b200 translation units.
//
// Device tree layout (one position-independent slab per tree; DESIGN.md
// "Data layout in HBM"):
//   SlabHeader                      (copy of the host header, 256 B)
//   T      float[n-1]               Eytzinger split values (tree.py:156)
//   box    float4[2n]               leaf AABB of the affordance set: lo.xyz,_ / hi.xyz,_
//   set    uint2[n]                 (start in float4 units, true set size m)
//   offs   int64[n+1]               reference CSR offsets (tree.py:226-228)
//   data   float4[...]              per set: xs[m4] ys[m4] zs[m4], m4 = roundup(m,4),
//                                   padding rows +inf; unused dims (k<3) are 0
//   org    float4[n]                binned-scan origin of each set: centre of the
//                                   finite points' box (xyz) and the largest
//                                   fp32 |p - o|^2 over the set (w)
//   rep    float4[n]                row 0 of each set (xyz), loaded beside the box
//   order  int32[n]                 leaves by descending set size (binned K5 takes
//                                   the costliest tiles first: shorter tail)
//   probe  float[8][n]              the binned classifier's per-leaf record, one
//                                   32-B load: representative xyz (fp32) and the
//                                   leaf box as outward-rounded fp16 (lo.xyz rounded
//                                   down, hi.xyz up -- a conservative box)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>

#include "../../include/capt_b200.h"

namespace capt {

constexpr uint64_t kSlabMagic = 0x3030324254504143ull;  // "CAPTB200"
constexpr int kSlabVersion = 5;
constexpr int kMaxK = 3;

struct SlabHeader {
  uint64_t magic;
  int32_t version;
  int32_t k;
  int32_t depth;
  int32_t pad0;
  int64_t n;          // leaves
  int64_t n_points;   // source cloud size
  int64_t total;      // sum of set sizes
  int64_t max_aff;
  int64_t n_ties;
  double r_min, r_max;
  int64_t off_T, off_box, off_set, off_offs, off_data;  // byte offsets in slab
  int64_t data_f4;    // float4 count of the data section
  int64_t bytes;      // slab size
  int64_t off_org;    // byte offset of the org section
  int64_t off_rep;    // byte offset of the rep section
  int64_t off_order;  // byte offset of the order section
  int64_t off_probe;  // byte offset of the probe section
  int64_t reserved[6];
};
static_assert(sizeof(SlabHeader) <= 256, "header must fit its 256-B section");

// Clearance field geometry (capt_field.cu): a uniform grid of nx*ny*nz cells
// of edge h starting at lo; cell centre x0(i) = fma(i, h, c0) per axis.
// blo/bhi = the cloud's box (finite representatives); rcap caps the stored
// lower bounds.  field == nullptr: no field (k < 3, or not built).
struct FieldGeom {
  int nx, ny, nz, m;   // cells per axis; point-bucket edge in cells
  int rr;              // candidate reach in cells (build only)
  int nbx, nby, nbz;   // point buckets per axis (the list stage's exact scan)
  float lo[3];         // grid origin: cell i spans lo + [i, i+1) h (cell_of)
  float c0[3];         // centre of cell 0: x0(i) = fma(i, h, c0) exactly, build and query
  float h, inv_h;
  float nc0[3];        // -c0 / h: a query's cell is round(fma(c, inv_h, nc0)) (qcell)
  float blo[3], bhi[3];
  float rcap;
  float q_step;        // candidate offsets from x0: int16 multiples of q_step (a power of two)
  float q_err;         // bound on the Euclidean error of a decoded candidate difference
  int64_t cells;
  // block table: blocks of 2^bshift cells per axis, bx*by*bz bytes; entry
  // q * bstep <= the distance from the cloud to any centre whose computed
  // cell lies in the block (bstep a power of two); K0 keeps it in shared
  // memory and skips the record of a sphere it certifies free
  int bshift, bx, by, bz;
  int bbytes;          // table bytes, rounded up to 16
  float bstep;
};

// Candidate record of a cell: the kCand cloud points nearest its centre x0,
// as int16 offsets (p - x0) / q_step per axis, and kd_q: kd_q * q_step <= the
// distance from x0 to every other cloud point.  48 words (192 B, six 32-B
// loads): words 0-15 hold the x offsets of slots 0..31 (two per word, slot 2w
// in the low half), words 16-31 the y offsets, words 32-47 the z offsets;
// x slot 31 is kd_q, y slot 31 the candidate count; unused slots hold
// kCandNone.
constexpr int kCand = 31;
constexpr int kCandWords = 48;
constexpr int kCandNone = -32768;

struct DevTree {
  int k, depth;
  int64_t n;
  int64_t total;  // sum of set sizes
  double r_min, r_max;
  const float* T;
  const float4* box;
  const uint2* set;
  const int64_t* offs;
  const float4* data;
  const float4* org;
  const float4* rep;  // row 0 of every set (the point owning the cell), +inf for padding
  const int* order;   // leaves by descending set size
  const float* probe; // 8 floats per leaf: rep xyz, fp16 box (conservative), 2 spare
  // clearance field (capt_field.cu; field == nullptr if absent)
  const float4* field;    // per cell: witness xyz + lower bound nn
  const uint32_t* cand;   // per cell: kCandWords words (candidate record, see kCand)
  const uint8_t* blk;     // block table (FieldGeom::bshift ...)
  const float4* cpts;     // the cloud's finite points (the field's bucket order)
  const uint32_t* bstart; // per point bucket (x fastest): first index into cpts; nb + 1
  FieldGeom fg;
};

}  // namespace capt

struct capt_tree {
  capt::SlabHeader h;
  int device;
  char* slab;  // device pointer
  bool owns_slab = true;  // false: borrowed from the caller (capt_tree_from_slab, CAPT_SLAB_BORROW)
  // clearance field: derived per device from the slab (capt_field.cu), one
  // allocation holding the K0 records and the candidate records
  void* field_mem = nullptr;
  float4* field = nullptr;
  uint32_t* cand = nullptr;
  uint8_t* blk = nullptr;
  float4* cpts = nullptr;
  uint32_t* bstart = nullptr;
  capt::FieldGeom fg{};
};

namespace capt {

// ---------------------------------------------------------------- launches
void note_launches(int64_t k);

// Keep stream-ordered scratch allocations cached in the device's default
// memory pool (no release at synchronisation points).
void ensure_pool(int device);

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define CAPT_CUDA(call)                                  \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return capt::cuda_fail(_e, #call); \
  } while (0)

inline DevTree view(const capt_tree* t) {
  DevTree d;
  d.k = t->h.k;
  d.depth = t->h.depth;
  d.n = t->h.n;
  d.total = t->h.total;
  d.r_min = t->h.r_min;
  d.r_max = t->h.r_max;
  d.T = reinterpret_cast<const float*>(t->slab + t->h.off_T);
  d.box = reinterpret_cast<const float4*>(t->slab + t->h.off_box);
  d.set = reinterpret_cast<const uint2*>(t->slab + t->h.off_set);
  d.offs = reinterpret_cast<const int64_t*>(t->slab + t->h.off_offs);
  d.data = reinterpret_cast<const float4*>(t->slab + t->h.off_data);
  d.org = reinterpret_cast<const float4*>(t->slab + t->h.off_org);
  d.rep = reinterpret_cast<const float4*>(t->slab + t->h.off_rep);
  d.order = reinterpret_cast<const int*>(t->slab + t->h.off_order);
  d.probe = reinterpret_cast<const float*>(t->slab + t->h.off_probe);
  d.field = t->field;
  d.cand = t->cand;
  d.blk = t->blk;
  d.cpts = t->cpts;
  d.bstart = t->bstart;
  d.fg = t->fg;
  return d;
}

inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

// Fill the header's section offsets for a tree of n leaves and data_f4
// float4s of set data; returns the slab size.
inline int64_t layout_slab(SlabHeader& h, int64_t data_f4) {
  int64_t off = 256;
  h.off_T = off;
  off = align256(off + sizeof(float) * (h.n > 1 ? h.n - 1 : 1));
  h.off_box = off;
  off = align256(off + sizeof(float4) * 2 * h.n);
  h.off_set = off;
  off = align256(off + sizeof(uint2) * h.n);
  h.off_offs = off;
  off = align256(off + sizeof(int64_t) * (h.n + 1));
  h.off_org = off;
  off = align256(off + sizeof(float4) * h.n);
  h.off_rep = off;
  off = align256(off + sizeof(float4) * h.n);
  h.off_order = off;
  off = align256(off + sizeof(int) * h.n);
  h.off_probe = off;
  off = align256(off + 32 * h.n);
  h.off_data = off;
  off = align256(off + sizeof(float4) * (data_f4 > 0 ? data_f4 : 1));
  h.data_f4 = data_f4;
  h.bytes = off;
  return off;
}

inline int depth_of(int64_t n) {
  int d = 0;
  while ((int64_t(1) << d) < n) ++d;
  return d;
}

// Fill the org, rep, order and probe sections of a slab whose data is final.
// Per-leaf derived sections (org, rep, probe, order) of a slab whose sets
// and boxes are final; with_origins = false when the build already wrote
// org, rep and probe (k_fill_b) and only the order remains.
int compute_origins(const DevTree& t, cudaStream_t s, bool with_origins = true);

int alloc_slab(capt_tree** out, int device, SlabHeader h);

// Build the clearance field of a tree whose rep section is final (k = 3 only;
// other trees keep field == nullptr).  Synchronises stream s.
int build_field(capt_tree* t, cudaStream_t s);

// The clearance-field query pipeline (fp32, k = 3, no CAPT_STATS / mode flags).
bool field_eligible(const DevTree& t, int64_t n, uint32_t flags);
int launch_field(const DevTree& t, const void* centers, const void* radii, int64_t n, int L,
                 const uint8_t* mask, uint32_t flags, uint32_t* bits, int64_t n_words,
                 unsigned long long* first_bad, cudaStream_t s);

// scratch allocation helpers (stream-ordered allocator)
template <class T>
inline cudaError_t dmalloc(T** p, size_t count, cudaStream_t s) {
  return cudaMallocAsync(reinterpret_cast<void**>(p), sizeof(T) * (count ? count : 1), s);
}

// One-time per-device set-up (function attributes apply to the current
// device only): f(device) runs once per device, its status is kept.
constexpr int kMaxDevices = 64;
struct DeviceOnce {
  std::once_flag flag[kMaxDevices];
  int rc[kMaxDevices] = {};
};
template <class F>
inline int per_device_once(DeviceOnce& o, F&& f) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
    return fail(CAPT_ECUDA, "no current CUDA device");
  std::call_once(o.flag[dev], [&] { o.rc[dev] = f(dev); });
  return o.rc[dev];
}

inline int grid_for(int64_t work, int block, int max_blocks_per_sm = 8) {
  static const int sms = [] {  // (every device of the box is the same part)
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  int64_t need = (work + block - 1) / block;
  int64_t cap = int64_t(sms) * max_blocks_per_sm;
  if (need < 1) need = 1;
  return int(need < cap ? need : cap);
}

}  // namespace capt
