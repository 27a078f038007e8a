// Clearance field: resolve most spheres of a query before any tree descent.
//
// The reference answers a sphere by descending to its leaf and scanning the
// leaf's affordance set (query.py:184-219).  Because the affordance sets are
// complete for radii inside [r_min, r_max] (Alg. 1; pinned
// by the reference's brute-force equality tests, test_acceptance.py:54-91),
// the verdict of an in-band sphere is exactly "some cloud point p has float64
// ((dx^2 + dy^2) + dz^2) <= r*r" -- the brute-force verdict (oracle.py:34-49;
// DESIGN.md section 3b).  A uniform grid over the cloud decides that verdict
// for almost every sphere without the tree, in two stages:
//
//   K0 (every sphere): one 16-B record per cell {witness w, nn}, w = the
//     cloud point nearest the cell centre x0 and nn <= dist(x0, cloud):
//       hit:  fp32 |c - w|^2 <= r^2 (1 - TAU);
//       free: nn - |c - x0| > r with a relative margin (dist is 1-Lipschitz);
//     decides ~96% (config 3) to ~99.7% (config 1) of the spheres.
//   list (the rest): the cell's candidate record -- its kCand nearest cloud
//     points (int16 offsets from x0) and kd <= the distance from x0 to every
//     other cloud point: a candidate hit decides; no candidate hit and
//     kd - |c - x0| > r (with a margin) decides free.  Simulated on configs
//     1 and 3, this leaves ~1e-6 / 1e-4 of the spheres (within a hair of
//     tangency to their (kCand+1)-th point).
//
// Spheres no certificate decides, spheres outside the band (check_radii =
// False), non-finite centres and extreme radii take the tree path (descent,
// AABB, representative probe, cooperative affordance-set scans with the
// float64 fix-up) with the reference's own semantics.
//
// Kernels:
//   build:  k_rep_box (cloud box), k_bucket_keys + radix sort (points into
//           buckets of 2 cells), k_field_cand (one CTA per 8x8x4-cell tile:
//           the kCand + 1 nearest points of every cell centre among the
//           points of the buckets the tile grown by rcap overlaps, staged
//           through shared memory), k_block_table (per 8^3-cell block, a
//           lower bound on the distance to the cloud)
//   query:  k_resolve1 / k_resolve (K0: band check, block table, grid
//                           certificates, lane groups, bit words, the list
//                           with its spheres)
//           k_list_knn     (candidate certificates; open in-band entries ->
//                           list 2, the others -> list 3)
//           k_bucket_list  (list 2: exact brute force over the points of the
//                           buckets the sphere's box overlaps)
//           k_tree_list    (list 3: the tree path, the reference's semantics)
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <limits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "capt_internal.cuh"
#include "capt_query_common.cuh"

namespace capt {

#ifndef CAPT_FIELD_CELLS
#define CAPT_FIELD_CELLS (1 << 21)  // 32 MB of K0 records: L2-resident
#endif
#ifndef CAPT_BLK_BYTES
#define CAPT_BLK_BYTES 49152  // block table bound (K0's dynamic shared memory, one CTA per SM)
#endif

namespace {

constexpr float kNNShrink = 1.0f - 0x1p-19f;    // fp32 sqrt(d^2) -> certified lower bound
constexpr int kFieldChunk = 1024;               // staged points per k_field_knn round
constexpr int kKP = kCand + 1;                  // nearest points kept per cell (+ the bound)
// The second record (ring drain): the kSecond nearest points after the
// witness as int16 offsets and the bound of the next one -- 2 candidates in
// 16 B or 5 in 32 B (config 3 lists 346 K spheres with 2, 121 K with 5: list
// stage 53 -> 39 us for 1% more K0).
#ifndef CAPT_SECOND
#define CAPT_SECOND 5
#endif
constexpr int kSecond = CAPT_SECOND;
constexpr int kSecondWords = kSecond == 2 ? 4 : 8;  // (3 kSecond + 1 slots of 16 bits)
static_assert(kSecond == 2 || kSecond == 5, "second record: 16 or 32 bytes");
// the second records follow the K0 records at an even cell count (32-B loads)
__host__ __device__ __forceinline__ size_t second_base(int64_t cells) {
  return size_t((cells + 1) & ~int64_t(1));
}

__device__ __forceinline__ int f2o(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}

// cell index along one axis; any value is safe for the certificates (they
// hold for every x0), the clamp keeps it inside the grid
__device__ __forceinline__ int cell_of(float c, float lo, float inv, int n) {
  const int i = __float2int_rd(__fmul_rn(__fsub_rn(c, lo), inv));
  return min(max(i, 0), n - 1);
}
// cell centre; the build and the query evaluate the same expression
__device__ __forceinline__ float centre_of(int i, float h, float c0) {
  return __fmaf_rn(__int2float_rn(i), h, c0);
}
// A query's cell along one axis: round(fma(c, inv_h, -c0 / h)), by the
// 1.5 * 2^23 magic-number rounding (two full-rate adds instead of two
// conversions); fi = the index as a float, for the centre fma(fi, h, c0).
// Any cell serves the certificates (they hold for every x0 with e = c - x0
// computed from it); the index lies in [0, n) iff c is in [lo, lo + n h) up
// to the rounding of t -- NaN and infinite coordinates give indices outside
// (the float bits of a non-finite or huge m are never magic + [0, n)).  K0,
// the ring drain and the list kernels all use this one function.
__device__ __forceinline__ int qcell(float c, float inv_h, float nc0, float& fi) {
  const float m = fmaf(c, inv_h, nc0) + 12582912.0f;
  fi = m - 12582912.0f;
  return __float_as_int(m) - 0x4B400000;
}
// The block table's certificate for a centre in the grid (computed cell
// ix, iy, iz): every cloud point is farther than bound >= rk = fl(r (1 +
// 2^-20)) > r (1 + 15u), so every float64 d^2 exceeds r*r (the K0 free
// argument with the block's bound in place of nn - |c - x0|).
#ifndef CAPT_K0_BLOCKS
#define CAPT_K0_BLOCKS 1
#endif
#ifndef CAPT_K0_GROUP_BLOCKS  // the table in the lane-group K0 (k_resolve) too
#define CAPT_K0_GROUP_BLOCKS 0
#endif
__device__ __forceinline__ bool block_free(const FieldGeom& g, const uint8_t* sblk, int ix, int iy,
                                           int iz, bool in, float rk) {
  if (!CAPT_K0_BLOCKS) return false;
  const unsigned bs = unsigned(g.bshift);
  const unsigned bi = ((unsigned(iz) >> bs) * unsigned(g.by) + (unsigned(iy) >> bs)) *
                          unsigned(g.bx) + (unsigned(ix) >> bs);
  const float q = float(sblk[in ? bi : 0u]);
  return in && q * g.bstep > rk;
}
// The single-sphere K0's one CTA per SM copies the block table into (dynamic)
// shared memory: tree data, so before the programmatic-dependency wait.
__device__ __forceinline__ const uint8_t* stage_block_table(const FieldGeom& g,
                                                            const uint8_t* blk) {
  extern __shared__ uint4 s_blk4[];
  const uint4* src = reinterpret_cast<const uint4*>(blk);
  for (int i = threadIdx.x; i < (g.bbytes >> 4); i += blockDim.x) s_blk4[i] = __ldg(src + i);
  __syncthreads();
  return reinterpret_cast<const uint8_t*>(s_blk4);
}

// field records stay in L2 while the sphere stream passes through it
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ float4 ldg_keep(const float4* p, uint64_t pol) {
  float4 v;
  asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float d2_fma(float dx, float dy, float dz) {
  return fmaf(dz, dz, fmaf(dy, dy, dx * dx));
}
// one 256-bit load (candidate and second records)
__device__ __forceinline__ void ld_v8u(const uint32_t* p, uint32_t (&v)[8]) {
  asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "l"(p));
}
// signed int16 slots of a word (candidate offsets)
__device__ __forceinline__ int slot_lo(uint32_t w) { return int(w << 16) >> 16; }
__device__ __forceinline__ int slot_hi(uint32_t w) { return int(w) >> 16; }
// the reference's float64 point test (query.py:96-99): ((dx^2 + dy^2) + dz^2) <= r*r
__device__ __forceinline__ bool hit_f64(float cx, float cy, float cz, float r, float4 p) {
  const double dx = __dsub_rn(double(cx), double(p.x)), dy = __dsub_rn(double(cy), double(p.y)),
               dz = __dsub_rn(double(cz), double(p.z));
  const double s = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return s <= __dmul_rn(double(r), double(r));
}

// ---------------------------------------------------------------- build

__global__ void k_rep_box(const float4* __restrict__ rep, int64_t n, int* __restrict__ box) {
  int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    const float4 p = rep[j];
    if (!isfinite(p.x) || !isfinite(p.y) || !isfinite(p.z)) continue;
    const float v[3] = {p.x, p.y, p.z};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      lo[d] = min(lo[d], f2o(v[d]));
      hi[d] = max(hi[d], f2o(v[d]));
    }
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    lo[d] = __reduce_min_sync(0xffffffffu, lo[d]);
    hi[d] = __reduce_max_sync(0xffffffffu, hi[d]);
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (lo[d] != INT_MAX) atomicMin(box + d, lo[d]);
      if (hi[d] != INT_MIN) atomicMax(box + 3 + d, hi[d]);
    }
  }
}

struct BucketGrid {
  int nbx, nby, nbz;
  int64_t nb;
};

__device__ __forceinline__ int bucket_of(const FieldGeom& g, const BucketGrid& b, float x, float y,
                                         float z) {
  const int ix = cell_of(x, g.lo[0], g.inv_h, g.nx) / g.m;
  const int iy = cell_of(y, g.lo[1], g.inv_h, g.ny) / g.m;
  const int iz = cell_of(z, g.lo[2], g.inv_h, g.nz) / g.m;
  return (iz * b.nby + iy) * b.nbx + ix;
}

__global__ void k_bucket_keys(const float4* __restrict__ rep, int64_t n, FieldGeom g,
                              BucketGrid b, uint32_t* __restrict__ keys, int* __restrict__ ids,
                              uint32_t* __restrict__ counts) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    const float4 p = rep[j];
    uint32_t key = uint32_t(b.nb);  // non-finite (padding) rows sort last
    if (isfinite(p.x) && isfinite(p.y) && isfinite(p.z)) key = bucket_of(g, b, p.x, p.y, p.z);
    keys[j] = key;
    ids[j] = int(j);
    atomicAdd(counts + key, 1u);
  }
}

__global__ void k_bucket_points(const float4* __restrict__ rep, const int* __restrict__ ids,
                                int64_t n_fin, float4* __restrict__ pts) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_fin;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float4 p = rep[ids[i]];
    pts[i] = make_float4(p.x, p.y, p.z, 0.f);
  }
}

// Insert (d2, id) into the ascending list bd[0..kKP) (the caller knows
// d2 < bd[kKP-1]); equal distances keep the earlier candidate first.
__device__ __forceinline__ void knn_insert(float (&bd)[kKP], int (&bi)[kKP], float d2, int id) {
#pragma unroll
  for (int j = kKP - 1; j > 0; --j) {
    const bool shift = d2 < bd[j - 1];
    const bool place = !shift && d2 < bd[j];
    bd[j] = shift ? bd[j - 1] : (place ? d2 : bd[j]);
    bi[j] = shift ? bi[j - 1] : (place ? id : bi[j]);
  }
  if (d2 < bd[0]) {
    bd[0] = d2;
    bi[0] = id;
  }
}

// int16 slot j of the axis block at w[0..15] (two slots per word), as raw bits
__device__ __forceinline__ uint32_t get_slot(const uint32_t* w, int j) {
  return (j & 1) ? (w[j >> 1] >> 16) : (w[j >> 1] & 0xffffu);
}
// Set int16 slot j of the axis block at w[0..15] (two slots per word).
__device__ __forceinline__ void put_slot(uint32_t* w, int j, int v) {
  const uint32_t u = uint32_t(v) & 0xffffu;
  w[j >> 1] = (j & 1) ? ((w[j >> 1] & 0xffffu) | (u << 16)) : ((w[j >> 1] & 0xffff0000u) | u);
}

// One CTA per tile of 8 x 8 x 4 cells (one cell per thread).  A point within
// rcap of a cell centre lies within R = ceil(rcap / h) + 1 cells of the cell
// on every axis (cell_of is monotone; the +1 covers its rounding), so the
// tile's candidates are the points of the buckets (edge m cells) overlapping
// the tile grown by R cells: for every (y, z) bucket row one contiguous range
// of the bucket-sorted points, staged through shared memory in chunks.  Tiles
// far from the cloud have no candidates.  Per cell: the kCand + 1 nearest
// points by fp32 distance (candidates in a fixed order: deterministic on
// every replica) -> the K0 record {nearest point, nn} and the candidate
// record (the kCand nearest as int16 offsets from x0, the bound kd_q).
constexpr int kTileX = 8, kTileY = 8, kTileZ = 4;
__global__ void __launch_bounds__(256, 1) k_field_cand(FieldGeom g, BucketGrid b,
                                                    const uint32_t* __restrict__ bstart,
                                                    const float4* __restrict__ pts,
                                                    float4* __restrict__ field,
                                                    uint32_t* __restrict__ cand) {
  __shared__ float4 sp[kFieldChunk];
  const int tx = (g.nx + kTileX - 1) / kTileX, ty = (g.ny + kTileY - 1) / kTileY;
  const int bid = blockIdx.x;
  const int x0 = (bid % tx) * kTileX, y0 = ((bid / tx) % ty) * kTileY, z0 = (bid / (tx * ty)) * kTileZ;
  const int lx = threadIdx.x % kTileX, ly = (threadIdx.x / kTileX) % kTileY,
            lz = threadIdx.x / (kTileX * kTileY);
  const bool live = x0 + lx < g.nx && y0 + ly < g.ny && z0 + lz < g.nz;
  const float INF = __int_as_float(0x7f800000);
  const float px = centre_of(x0 + lx, g.h, g.c0[0]);
  const float py = centre_of(y0 + ly, g.h, g.c0[1]);
  const float pz = centre_of(z0 + lz, g.h, g.c0[2]);
  float bd[kKP];
  int bi[kKP];
#pragma unroll
  for (int i = 0; i < kKP; ++i) {
    bd[i] = INF;
    bi[i] = -1;
  }
  const int R = g.rr;
  const int bx0 = max(x0 - R, 0) / g.m, bx1 = min(x0 + kTileX - 1 + R, g.nx - 1) / g.m;
  const int by0 = max(y0 - R, 0) / g.m, by1 = min(y0 + kTileY - 1 + R, g.ny - 1) / g.m;
  const int bz0 = max(z0 - R, 0) / g.m, bz1 = min(z0 + kTileZ - 1 + R, g.nz - 1) / g.m;
  // bucket rows nearest the tile first (rings of Chebyshev distance around
  // the tile's own row): the 32-nearest lists are close to final after the
  // first rings, so the later points mostly fail the one compare instead of
  // walking the insertion (same lists up to ties)
  const int cy = (y0 + kTileY / 2) / g.m, cz = (z0 + kTileZ / 2) / g.m;
  const int ring_max = max(max(cy - by0, by1 - cy), max(cz - bz0, bz1 - cz));
  for (int ring = 0; ring <= ring_max; ++ring) {
  for (int bz = max(bz0, cz - ring); bz <= min(bz1, cz + ring); ++bz)
    for (int by = max(by0, cy - ring); by <= min(by1, cy + ring); ++by) {
      if (max(abs(by - cy), abs(bz - cz)) != ring) continue;
      const int row = (bz * b.nby + by) * b.nbx;
      const uint32_t s0 = bstart[row + bx0], s1 = bstart[row + bx1 + 1];
      for (uint32_t c0 = s0; c0 < s1; c0 += kFieldChunk) {
        const int cnt = int(min(uint32_t(kFieldChunk), s1 - c0));
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += 256) sp[i] = pts[c0 + i];
        __syncthreads();
        for (int i = 0; i < cnt; ++i) {
          const float4 p = sp[i];
          const float d2 = d2_fma(p.x - px, p.y - py, p.z - pz);
          if (d2 < bd[kKP - 1]) knn_insert(bd, bi, d2, int(c0) + i);
        }
      }
    }
    // every point of a later ring lies at least `gap` from every cell centre
    // of the tile along y or z (its bucket row is ring + 1 rows from the
    // tile's; two cells of slack for the cell rounding and the half cell):
    // once no list of the tile reaches that far, the lists are final
    if (ring < ring_max) {
      const int gy = min((cy + ring + 1) * g.m - (y0 + kTileY - 1),
                         y0 - ((cy - ring - 1) * g.m + g.m - 1)) - 2;
      const int gz = min((cz + ring + 1) * g.m - (z0 + kTileZ - 1),
                         z0 - ((cz - ring - 1) * g.m + g.m - 1)) - 2;
      const float gap = float(min(gy, gz)) * g.h;
      const float t2 = gap > 0.f ? gap * gap * (1.0f - 0x1p-10f) : 0.f;
      if (!__syncthreads_or(bd[kKP - 1] >= t2)) break;
    }
  }
  {
    if (!live) return;
    const int64_t cell = (int64_t(z0 + lz) * g.ny + (y0 + ly)) * g.nx + (x0 + lx);
    // fp32 |x0 - p|^2 has relative error < 5u, sqrtf one more u:
    // sqrtf(d2) (1 - 2^-19) (rounded) < the real distance.  Points outside
    // the candidate buckets are farther than rcap: the bounds are capped there.
    auto lb = [&](int k) { return fminf(g.rcap, __fmul_rn(sqrtf(bd[k]), kNNShrink)); };
    // candidates: offsets (p - x0) / q_step rounded (exact in double: the
    // difference of two floats, a power-of-two scale), |offset| <= 32767;
    // the first point that does not fit (or lies beyond rcap) ends the list
    // and bounds kd
    uint32_t wd[kCandWords];
#pragma unroll
    for (int i = 0; i < kCandWords; ++i) wd[i] = 0x80008000u;  // kCandNone pairs
    int count = 0, drop = kKP - 1;  // (the first candidate not stored)
    bool open = true;
    const double inv = 1.0 / double(g.q_step);
#pragma unroll
    for (int k = 0; k < kCand; ++k) {
      if (!open || bi[k] < 0) {
        open = false;
        continue;
      }
      const float4 p = pts[bi[k]];
      const double qx = rint((double(p.x) - double(px)) * inv);
      const double qy = rint((double(p.y) - double(py)) * inv);
      const double qz = rint((double(p.z) - double(pz)) * inv);
      if (fabs(qx) > 32767.0 || fabs(qy) > 32767.0 || fabs(qz) > 32767.0 || !(lb(k) < g.rcap)) {
        drop = k;  // (every later candidate is at least as far)
        open = false;
        continue;
      }
      put_slot(wd, k, int(qx));
      put_slot(wd + 16, k, int(qy));
      put_slot(wd + 32, k, int(qz));
      ++count;
    }
    // kd: below the distance of the first point not stored (capped at rcap)
    put_slot(wd, 31, int(floor(double(lb(drop)) * inv)));  // kd_q q_step <= kd
    put_slot(wd + 16, 31, count);
    // K0's records: {nearest point w (exact), lb of the 2nd nearest} (read
    // for every sphere) and {the next kSecond nearest as offsets, kd_q: lb
    // of the point after them} (read for the spheres the first leaves open)
    const float4 w = bi[0] >= 0 ? pts[bi[0]] : make_float4(INF, INF, INF, 0.f);
    field[cell] = make_float4(w.x, w.y, w.z, lb(1));
    // second record: candidates 1 .. kSecond (the 2nd .. nearest) as int16
    // slots 3 (c - 1) + axis, then kd: lb of the first point after them
    {
      uint32_t w2[kSecondWords];
#pragma unroll
      for (int i = 0; i < kSecondWords; ++i) w2[i] = 0x80008000u;
#pragma unroll
      for (int c = 1; c <= kSecond; ++c) {
        put_slot(w2, 3 * (c - 1), get_slot(wd, c));
        put_slot(w2, 3 * (c - 1) + 1, get_slot(wd + 16, c));
        put_slot(w2, 3 * (c - 1) + 2, get_slot(wd + 32, c));
      }
      put_slot(w2, 2 * kSecondWords - 1, int(floor(double(lb(min(drop, kSecond + 1))) * inv)));
      uint4* d2 = reinterpret_cast<uint4*>(field + second_base(g.cells)) +
                  size_t(cell) * (kSecondWords / 4);
#pragma unroll
      for (int i = 0; i < kSecondWords / 4; ++i)
        d2[i] = make_uint4(w2[4 * i], w2[4 * i + 1], w2[4 * i + 2], w2[4 * i + 3]);
    }
    uint4* dst = reinterpret_cast<uint4*>(cand + cell * kCandWords);
#pragma unroll
    for (int i = 0; i < kCandWords / 4; ++i)
      dst[i] = make_uint4(wd[4 * i], wd[4 * i + 1], wd[4 * i + 2], wd[4 * i + 3]);
  }
}

// Block table (FieldGeom::bshift ...): one warp per block of 2^bshift cells
// per axis.  For every centre c whose computed cell (qcell) lies in the
// block, dist(c, cloud) >= lb0(x0) - |c - x0| >= min over the block's cells
// of lb0 - rcell, where lb0 = the certified lower bound of the distance from
// the cell centre x0 to its nearest cloud point (the witness, the same fp32
// expression k_field_cand ranks with; rcap when no point lies within rcap)
// and rcell >= |c - x0| (the host bounds the cell computation's rounding).
// Stored as floor(bound / bstep), bstep a power of two, saturated at 255;
// rounded down at every step.
__global__ void __launch_bounds__(256) k_block_table(FieldGeom g, const float4* __restrict__ field,
                                                     float rcell, uint8_t* __restrict__ blk) {
  const int lane = threadIdx.x & 31;
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nb = g.bx * g.by * g.bz;
  if (b >= nb) return;
  const int B = 1 << g.bshift;
  const int bxi = b % g.bx, byi = (b / g.bx) % g.by, bzi = b / (g.bx * g.by);
  const int x0 = bxi * B, y0 = byi * B, z0 = bzi * B;
  const int cx = min(B, g.nx - x0), cy = min(B, g.ny - y0), cz = min(B, g.nz - z0);
  float mn = g.rcap;
  for (int j = lane; j < cx * cy * cz; j += 32) {
    const int ix = x0 + j % cx, iy = y0 + (j / cx) % cy, iz = z0 + j / (cx * cy);
    const float4 w = field[(int64_t(iz) * g.ny + iy) * g.nx + ix];
    if (!isfinite(w.x)) continue;  // no point within rcap: lb0 = rcap
    const float px = centre_of(ix, g.h, g.c0[0]), py = centre_of(iy, g.h, g.c0[1]),
                pz = centre_of(iz, g.h, g.c0[2]);
    const float d2 = d2_fma(w.x - px, w.y - py, w.z - pz);
    mn = fminf(mn, fminf(g.rcap, __fmul_rn(sqrtf(d2), kNNShrink)));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if (lane == 0) {
    const float d = __fsub_rd(mn, rcell);
    const float q = d > 0.f ? floorf(__fdiv_rd(d, g.bstep)) : 0.f;
    blk[b] = uint8_t(fminf(q, 255.f));
  }
}

// ---------------------------------------------------------------- query

struct FieldArgs {
  DevTree t;
  const float* c;
  const float* r;
  int n;
  int L;
  const uint8_t* mask;
  uint32_t flags;
  uint32_t* bits;
  unsigned long long* first_bad;
  uint32_t* list;    // undecided sphere ids
  float4* list_s;    //   ... and their spheres {x, y, z, r} (K0's list; nullptr for the tree path's)
  uint32_t* list_n;
  float rlo_f, rhi_f;  // fp32 images of the double band edges
};

// K0.  A warp takes chunks of 128 consecutive spheres; lane l owns spheres
// 4l .. 4l+3 of the chunk, so a chunk is three 128-bit centre loads and one
// 128-bit radius load per lane.  For an in-band sphere (r in [r_min, r_max] in double; NaN is
// not) the verdict is certified without the tree (see the file comment):
//   * outside the grid: the raw cell index leaves [0, n) on some axis, so the
//     centre is more than r_max + h from the cloud's box -> free (this also
//     takes +-inf centres: the float64 distances are infinite, no collision);
//   * hit: fp32 |c - w|^2 <= r^2 (1 - TAU) for the cell's witness w;
//   * free: with e2 = fp32 |c - x0|^2 and A = fma(-r, 1 + 2^-20, nn):
//     A > 0 and A*A > e2 (1 + 2^-20).  fp32 e2 >= |c - x0|^2 (1 - 5u) and the
//     products lose <= 3u, so nn - r (1 + 16u) > |c - x0| (1 + 3u) and
//     dist(c, cloud) >= nn - |c - x0| > r (1 + 16u): every float64 d^2 of the
//     reference exceeds r*r.
// Everything else (NaN centres, out-of-band radii with check_radii=False,
// spheres near |dist - r| ~ h) is undecided.  Lane groups (L | 32) resolve on
// any definite hit (query.py:152-160); verdict bits are written directly
// (L <= 4: whole words; L >= 8: OR into cleared words); the undecided
// spheres of unresolved groups are appended to the list (single spheres via
// a per-CTA shared-memory buffer: list order is not sphere order).
constexpr float kK1 = 1.0f + 0x1p-20f;

struct Chunk {
  float4 p0, p1, p2, pr;  // xyz of 4 consecutive spheres in 3 float4, their radii
};

// kFull: the chunk is known to be whole (no bounds test)
template <bool kVec, bool kFull = false>
__device__ __forceinline__ Chunk load_chunk(const float* __restrict__ cf,
                                            const float* __restrict__ rf, int c, int lane, int n) {
  Chunk k;
  const int q0 = (c << 7) + 4 * lane;
  if (kVec && (kFull || (c << 7) + 128 <= n)) {
    const float4* c4 = reinterpret_cast<const float4*>(cf + 3 * size_t(q0));
    k.p0 = __ldcs(c4);
    k.p1 = __ldcs(c4 + 1);
    k.p2 = __ldcs(c4 + 2);
    k.pr = __ldcs(reinterpret_cast<const float4*>(rf + q0));
  } else {
    float t[12], u[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int q = q0 + v < n ? q0 + v : 0;
      t[3 * v] = __ldcs(cf + 3 * size_t(q));
      t[3 * v + 1] = __ldcs(cf + 3 * size_t(q) + 1);
      t[3 * v + 2] = __ldcs(cf + 3 * size_t(q) + 2);
      u[v] = __ldcs(rf + q);
    }
    k.p0 = make_float4(t[0], t[1], t[2], t[3]);
    k.p1 = make_float4(t[4], t[5], t[6], t[7]);
    k.p2 = make_float4(t[8], t[9], t[10], t[11]);
    k.pr = make_float4(u[0], u[1], u[2], u[3]);
  }
  return k;
}

// The common tail of a decided chunk: first_bad, lane-group resolution, the
// verdict bits, the list of undecided spheres.
// List entries carry the sphere ({x, y, z, r} and its index), so the list
// stage reads them coalesced instead of gathering four words per entry.  A
// warp collects its entries in a private 64-entry ring in shared memory and
// writes them out 32 at a time (one returning global atomic per 32 entries,
// coalesced stores), the rest at the end of the kernel; a chunk with more
// than 32 entries appends directly.
constexpr int kRing = 64;
struct Ring {
  float4* s;      // this warp's ring: spheres
  uint32_t* q;    //   ... and their indices
  unsigned head;  // (warp-uniform) oldest entry
  unsigned cnt;   // (warp-uniform) entries held
};

// Drain the k (<= 32) oldest ring entries, one per lane.  An entry flagged
// (bit 31 of its index: the witness was a definite miss) first meets the
// cell's second record -- the 2nd .. 6th nearest points of x0 as int16
// offsets and kd <= the distance to every other point, read only here so
// the hot records stay 16 B per cell -- the candidate certificate of
// k_list_knn with kSecond candidates: a hit sets its bit (the same warp wrote
// the chunk's words; __syncwarp orders the two), free drops it.  The rest
// are written to the list (coalesced, one atomic).
__device__ __forceinline__ void ring_drain(const FieldArgs& a, Ring& rg, unsigned k, int lane) {
  __syncwarp();
  const FieldGeom& g = a.t.fg;
  const unsigned slot = (rg.head + lane) & (kRing - 1);
  const bool mine = unsigned(lane) < k;
  uint32_t q = 0u;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (mine) {
    q = rg.q[slot];
    s = rg.s[slot];
  }
  __syncwarp();
  bool open = mine;
  if (q >> 31) {
    q &= 0x7fffffffu;
    float fx, fy, fz;
    const int ix = qcell(s.x, g.inv_h, g.nc0[0], fx);
    const int iy = qcell(s.y, g.inv_h, g.nc0[1], fy);
    const int iz = qcell(s.z, g.inv_h, g.nc0[2], fz);
    const unsigned cell =
        (unsigned(iz) * unsigned(g.ny) + unsigned(iy)) * unsigned(g.nx) + unsigned(ix);
    uint32_t w2[8];
    {
      const uint32_t* rec2 = reinterpret_cast<const uint32_t*>(a.t.field + second_base(g.cells)) +
                             size_t(cell) * kSecondWords;
      if (kSecondWords == 8) {
        ld_v8u(rec2, w2);
      } else {
        const uint4 h2 = __ldg(reinterpret_cast<const uint4*>(rec2));
        w2[0] = h2.x, w2[1] = h2.y, w2[2] = h2.z, w2[3] = h2.w;
      }
    }
    const float qs = g.q_step, qe = g.q_err * (1.0f + 0x1p-17f);
    const float ex = s.x - __fmaf_rn(fx, g.h, g.c0[0]);
    const float ey = s.y - __fmaf_rn(fy, g.h, g.c0[1]);
    const float ez = s.z - __fmaf_rn(fz, g.h, g.c0[2]);
    const float RH = s.w * (1.0f - 0x1p-18f) - qe;
    const float RM = s.w * (1.0f + 0x1p-18f) + qe;
    const float lo = RH > 0.f ? RH * RH * (1.0f - 0x1p-20f) : -1.f;
    const float hi = RM * RM * (1.0f + 0x1p-20f);
    auto sl = [&](int i) { return (i & 1) ? slot_hi(w2[i >> 1]) : slot_lo(w2[i >> 1]); };
    bool hit = false, amb = false;
#pragma unroll
    for (int c = 0; c < kSecond; ++c) {
      const int ox = sl(3 * c), oy = sl(3 * c + 1), oz = sl(3 * c + 2);
      const float vx = fmaf(-float(ox), qs, ex), vy = fmaf(-float(oy), qs, ey),
                  vz = fmaf(-float(oz), qs, ez);
      const float S = d2_fma(vx, vy, vz);
      const bool used = ox != kCandNone;
      hit |= used && S <= lo;
      amb |= used && S < hi;
    }
    const float A = float(sl(2 * kSecondWords - 1)) * qs - s.w * kK1;
    const bool free = !hit && !amb && A > 0.f && A * A > d2_fma(ex, ey, ez) * kK1;
    if (hit) {
      const uint32_t b = a.L == 1 ? q : q / uint32_t(a.L);
      atomicOr(a.bits + (b >> 5), 1u << (b & 31));
    }
    open = !hit && !free;
  }
  const unsigned om = __ballot_sync(0xffffffffu, open);
  if (om) {
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(a.list_n, unsigned(__popc(om)));
    base = __shfl_sync(0xffffffffu, base, 0) + __popc(om & ((1u << lane) - 1u));
    if (open) {
      a.list[base] = q;
      a.list_s[base] = s;
    }
  }
  rg.head = (rg.head + k) & (kRing - 1);
  rg.cnt -= k;
}

template <int LT>
__device__ __forceinline__ void emit_chunk(const FieldArgs& a, int ch, int lane, bool check,
                                           unsigned hitb, unsigned undb, unsigned badb,
                                           unsigned elig, const float (&x)[4], const float (&y)[4],
                                           const float (&z)[4], const float (&r)[4], Ring& rg) {
  const int n = a.n;
  const int q0 = (ch << 7) + 4 * lane;
  if (check && __any_sync(0xffffffffu, badb != 0)) {
#pragma unroll
    for (int v = 0; v < 4; ++v)
      if ((badb >> v) & 1u) atomicMin(a.first_bad, static_cast<unsigned long long>(q0 + v));
  }
  const int L = LT ? LT : a.L;
  // lane groups: a group with a hit is resolved
  unsigned resb;  // spheres of this lane whose group has a hit
  if (L == 1) {
    resb = hitb;
  } else if (L == 2) {
    const unsigned p = (hitb | (hitb >> 1)) & 5u;
    resb = p | (p << 1);
  } else if (L == 4) {
    resb = hitb ? 15u : 0u;
  } else {
    bool any = hitb != 0;
    for (int o = 1; o < L / 4; o <<= 1) any |= __shfl_xor_sync(0xffffffffu, any, o);
    resb = any ? 15u : 0u;
  }
  // verdict bits
  if (L == 1) {
    unsigned w = hitb << (4 * (lane & 7));
    w |= __shfl_xor_sync(0xffffffffu, w, 1);
    w |= __shfl_xor_sync(0xffffffffu, w, 2);
    w |= __shfl_xor_sync(0xffffffffu, w, 4);
    const int word = (ch << 2) + (lane >> 3);
    if ((lane & 7) == 0 && (word << 5) < n) a.bits[word] = w;
  } else if (L == 2) {
    unsigned w = ((resb & 1u) | ((resb >> 1) & 2u)) << (2 * (lane & 15));
    w |= __shfl_xor_sync(0xffffffffu, w, 1);
    w |= __shfl_xor_sync(0xffffffffu, w, 2);
    w |= __shfl_xor_sync(0xffffffffu, w, 4);
    w |= __shfl_xor_sync(0xffffffffu, w, 8);
    const int word = (ch << 1) + (lane >> 4);
    if ((lane & 15) == 0 && (word << 6) < n) a.bits[word] = w;
  } else if (L == 4) {
    const unsigned w = __ballot_sync(0xffffffffu, resb != 0);
    if (lane == 0) a.bits[ch] = w;
  } else {
    // one bit per L/4 lanes: keep every (L/4)-th ballot bit, compress
    const int st = L >> 2;
    const unsigned w = __ballot_sync(0xffffffffu, resb != 0 && (lane & (st - 1)) == 0);
    unsigned outw = 0;
    for (int j = 0; j < 32 / st; ++j) outw |= ((w >> (j * st)) & 1u) << j;
    const int g0 = (ch << 7) / L;  // first group of the chunk
    if (lane == 0 && outw) atomicOr(a.bits + (g0 >> 5), outw << (g0 & 31));
  }
  // the list
  const unsigned lst = undb & ~resb;
  const unsigned has = __ballot_sync(0xffffffffu, lst != 0);
  if (has) {
    const int cnt = __popc(lst);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const unsigned tot = unsigned(__shfl_sync(0xffffffffu, incl, 31));
    if (tot > 32u) {  // (rare: NaN or out-of-band batches) straight to the list
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(a.list_n, tot);
      base = __shfl_sync(0xffffffffu, base, 0) + unsigned(incl - cnt);
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if ((lst >> v) & 1u) {
          const unsigned at = base + __popc(lst & ((1u << v) - 1u));
          a.list[at] = uint32_t(q0 + v);
          a.list_s[at] = make_float4(x[v], y[v], z[v], r[v]);
        }
    } else {
      const unsigned pos = rg.head + rg.cnt + unsigned(incl - cnt);
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if ((lst >> v) & 1u) {
          const unsigned slot = (pos + __popc(lst & ((1u << v) - 1u))) & (kRing - 1);
          rg.q[slot] = uint32_t(q0 + v) | (((elig >> v) & 1u) << 31);
          rg.s[slot] = make_float4(x[v], y[v], z[v], r[v]);
        }
      rg.cnt += tot;
      if (rg.cnt >= 32u) ring_drain(a, rg, 32u, lane);
    }
  }
}

// Decide one chunk (see above): writes its bits and list entries.  LT: the
// lane width when known at compile time (0: a.L at run time); kFull: a whole
// unmasked chunk (no per-sphere validity test).
template <bool kMask, int LT, bool kFull, bool kBand = false>
__device__ __forceinline__ void resolve_chunk(const FieldArgs& a, const FieldGeom& g,
                                              const uint8_t* sblk, const Chunk& k, int ch,
                                              int lane, bool check, uint64_t pol, Ring& rg) {
  const float x[4] = {k.p0.x, k.p0.w, k.p1.z, k.p2.y};
  const float y[4] = {k.p0.y, k.p1.x, k.p1.w, k.p2.z};
  const float z[4] = {k.p0.z, k.p1.y, k.p2.x, k.p2.w};
  const float r[4] = {k.pr.x, k.pr.y, k.pr.z, k.pr.w};
  const int n = a.n;
  const int q0 = (ch << 7) + 4 * lane;
  const unsigned nxu = unsigned(g.nx), nyu = unsigned(g.ny), nzu = unsigned(g.nz);
  // phase 1: validity, band, cell, record load of sphere v (skip: its lane
  // group already has a hit -- no record is fetched)
  bool valid[4], inband[4], look[4];
  int ix[4], iy[4], iz[4];
  float fx[4], fy[4], fz[4];
  float4 rec[4];
  auto cell = [&](int v, bool skip) {
    valid[v] = kFull || q0 + v < n;
    if (kMask) valid[v] = valid[v] && a.mask[valid[v] ? q0 + v : 0] != 0;
    inband[v] = kBand || (r[v] >= a.rlo_f && r[v] <= a.rhi_f);
    ix[v] = qcell(x[v], g.inv_h, g.nc0[0], fx[v]);
    iy[v] = qcell(y[v], g.inv_h, g.nc0[1], fy[v]);
    iz[v] = qcell(z[v], g.inv_h, g.nc0[2], fz[v]);
    // (the index is used only inside the grid: no clamp)
    const bool in = unsigned(ix[v]) < nxu && unsigned(iy[v]) < nyu && unsigned(iz[v]) < nzu;
    const bool bfree = CAPT_K0_GROUP_BLOCKS && block_free(g, sblk, ix[v], iy[v], iz[v], in, r[v] * kK1);
    look[v] = valid[v] && inband[v] && in && !skip && !bfree;
#ifdef CAPT_FIELD_STATS
    {
      const unsigned lk = __ballot_sync(0xffffffffu, look[v]);
      const unsigned bf = __ballot_sync(0xffffffffu, valid[v] && inband[v] && !skip && bfree);
      if ((threadIdx.x & 31) == 0) {
        atomicAdd(a.list_n + 4, unsigned(__popc(lk)));
        atomicAdd(a.list_n + 5, unsigned(__popc(bf)));
      }
    }
#endif
    rec[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (look[v])
      rec[v] = ldg_keep(a.t.field + ((unsigned(iz[v]) * nyu + unsigned(iy[v])) * nxu + unsigned(ix[v])),
                        pol);
  };
  // phase 2: the certificates of sphere v
  unsigned hitb = 0, undb = 0, badb = 0, elig = 0;
  const float band_lo = 1.0f - kTau, band_hi = 1.0f + kTau;
  auto cert = [&](int v) {
    const float ex = x[v] - __fmaf_rn(fx[v], g.h, g.c0[0]);
    const float ey = y[v] - __fmaf_rn(fy[v], g.h, g.c0[1]);
    const float ez = z[v] - __fmaf_rn(fz[v], g.h, g.c0[2]);
    const float e2 = d2_fma(ex, ey, ez);
    const float r2 = r[v] * r[v];
    const float dw = d2_fma(x[v] - rec[v].x, y[v] - rec[v].y, z[v] - rec[v].z);
    const bool hit = dw <= r2 * band_lo;
    // free: the witness a definite miss and every other point beyond
    // rec.w - |c - x0| > r (rec.w: lower bound of the 2nd-nearest distance)
    const float A = rec[v].w - r[v] * kK1;  // (fl(r k) >= r (1 + 15u))
    bool free = dw > r2 * band_hi && A > 0.f && A * A > e2 * kK1;
    // the spheres the first record leaves open with the witness a definite
    // miss meet the cell's second record when their ring is drained
    elig |= unsigned(look[v] && !hit && !free && dw > r2 * band_hi) << v;
    hitb |= unsigned(look[v] && hit) << v;
    // decided: in-band and (outside the grid / skipped, or certified); with
    // check_radii an out-of-band (non-NaN) radius only reports first_bad
    const bool bad = !kBand && check && valid[v] && (r[v] < a.rlo_f || r[v] > a.rhi_f);
    badb |= unsigned(bad) << v;
    const bool decided = inband[v] && (!look[v] || hit || free);
    undb |= unsigned(valid[v] && !decided && !bad) << v;
  };
  const int L = LT ? LT : a.L;
  if (L >= 4) {
    // groups of L >= 4 spheres span L/4 whole lanes; a group with a hit
    // fetches no more records (query.py:152-160 early exit, applied to the
    // L2 traffic -- K0 is bound by it): one sphere per lane per round, each
    // round's records fetched only for the groups still without a hit
    // (config 1 K0: 158 us vs 167 with the lane's last three spheres in one
    // round, 206 with all four at once)
    bool any = false;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      cell(v, any);
      cert(v);
      any = hitb != 0u;
      for (int o = 1; o < L / 4; o <<= 1) any |= __shfl_xor_sync(0xffffffffu, any, o);
    }
  } else if (L == 2) {
    // pairs (0, 1) and (2, 3) of the lane: the second sphere of a pair is
    // fetched only if the first did not hit
    cell(0, false);
    cell(2, false);
    cert(0);
    cert(2);
    cell(1, (hitb & 1u) != 0u);
    cell(3, (hitb & 4u) != 0u);
    cert(1);
    cert(3);
  } else {
#pragma unroll
    for (int v = 0; v < 4; ++v) cell(v, false);
#pragma unroll
    for (int v = 0; v < 4; ++v) cert(v);
  }
  emit_chunk<LT>(a, ch, lane, check && !kBand, hitb, undb, badb, elig, x, y, z, r, rg);
}

// every radius of the chunk inside the band (warp-uniform; NaN is not)
__device__ __forceinline__ bool chunk_in_band(const FieldArgs& a, float r0, float r1, float r2,
                                              float r3) {
  const float rmn = fminf(fminf(r0, r1), fminf(r2, r3));
  const float rmx = fmaxf(fmaxf(r0, r1), fmaxf(r2, r3));
  // (fminf / fmaxf drop a NaN beside a number: test each radius for it)
  const bool ok = rmn >= a.rlo_f && rmx <= a.rhi_f && r0 == r0 && r1 == r1 && r2 == r2 &&
                  r3 == r3;
  return __all_sync(0xffffffffu, ok);
}

// K0's CTA shapes.  Both kernels keep one chunk per warp in registers at 64
// registers per thread (32 warps per SM; 40 warps at 48 registers were slower
// on config 3, a ping-pong prefetch of the next chunk was best at 24 warps and
// slower overall).  Lane groups: 2 CTAs of 512 threads per SM, two waves;
// single spheres (CAPT_K1_*): one persistent CTA of 1024 threads per SM, so
// one copy of the block table (up to 48 KB: blocks of 4^3 cells on a 2 M-cell
// grid) serves the SM (config 3 K0: 0.266 -> 0.248 ms against 4 CTAs of 256
// threads with 8 KB tables of 8^3-cell blocks).
#ifndef CAPT_K0_MINB
#define CAPT_K0_MINB 2
#endif
#ifndef CAPT_K0_FASTBAND  // whole in-band chunks without the out-of-band bookkeeping
#define CAPT_K0_FASTBAND 1
#endif
#ifndef CAPT_K0_WAVES  // K0 grid: CTAs per SM (resident: CAPT_K0_MINB)
#define CAPT_K0_WAVES 4
#endif

// persistent warps over the whole 128-sphere chunks; the last, partial chunk
// (scalar loads, per-sphere validity) after the loop
#ifndef CAPT_K0_BLOCK
#define CAPT_K0_BLOCK 512
#endif
template <bool kVec, bool kMask, int LT>
__global__ void __launch_bounds__(CAPT_K0_BLOCK, CAPT_K0_MINB) k_resolve(FieldArgs a) {
  constexpr int kBlock = CAPT_K0_BLOCK;
  const FieldGeom g = a.t.fg;
  const bool check = a.flags & CAPT_CHECK_RADII;
  const int n = a.n;
  const int lane = threadIdx.x & 31;
  const int nfull = n >> 7;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t pol = l2_keep_policy();
  __shared__ float4 s_ring[kBlock / 32][kRing];
  __shared__ uint32_t s_ringq[kBlock / 32][kRing];
  Ring rg{s_ring[threadIdx.x >> 5], s_ringq[threadIdx.x >> 5], 0u, 0u};
  // (the lane-group K0 does not use the block table: DESIGN section 9)
  const uint8_t* sblk = CAPT_K0_GROUP_BLOCKS ? stage_block_table(g, a.t.blk) : nullptr;
  // (launched after k_field_zero with programmatic serialisation)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int ch = w0; ch < nfull; ch += nwarps) {
    const Chunk A = load_chunk<kVec, true>(a.c, a.r, ch, lane, n);
    // whole unmasked chunks with every radius in band (the common case) shed
    // the out-of-band bookkeeping
    if (CAPT_K0_FASTBAND && !kMask && chunk_in_band(a, A.pr.x, A.pr.y, A.pr.z, A.pr.w))
      resolve_chunk<kMask, LT, !kMask, true>(a, g, sblk, A, ch, lane, check, pol, rg);
    else
      resolve_chunk<kMask, LT, !kMask>(a, g, sblk, A, ch, lane, check, pol, rg);
  }
  if ((n & 127) && w0 == nfull % nwarps) {
    const Chunk T = load_chunk<false>(a.c, a.r, nfull, lane, n);
    resolve_chunk<kMask, LT, false>(a, g, sblk, T, nfull, lane, check, pol, rg);
  }
  if (rg.cnt) ring_drain(a, rg, rg.cnt, lane);
}


// K0 for single spheres (L = 1, unmasked: collides_many), the same
// certificates with a strided lane map: lane l of a warp owns spheres
// l, 32 + l, 64 + l, 96 + l of its 128-sphere chunk, so the verdict word of
// spheres 32 v .. 32 v + 31 is one ballot and the list positions are ballot
// prefix counts.  Built for a short instruction stream and few live
// registers: phase 1 computes each sphere's cell, |c - x0|^2 and the block
// table's certificate and issues the 4 record loads (a sphere without a
// record gets {+inf, .., +inf}: its witness and Lipschitz tests then read
// "free", and only the `skip` bit keeps out-of-grid spheres decided without
// them); phase 2 consumes the records.  The centres are scalar loads (x, y,
// z of a sphere: each instruction spans 3 lines of 128 B for 32 spheres; y
// and z hit L1 after x).
// kBand (whole chunks only): every radius of the chunk is inside the band
// (warp-uniform, voted by the caller), so no sphere is out of band, bad or
// listed for its radius -- the common case sheds that bookkeeping.
// LG = 4, 8, 16 (groups of LG consecutive spheres, query.py:152-160): under
// the strided map a group is LG adjacent lanes of one slot, so its
// any-collision bit is a field of the slot's hit ballot -- the four records
// of a lane are in flight together (no dependent rounds; config 1 K0 0.141
// -> 0.123 ms against four rounds that stop at a group's first hit) and a
// chunk's 128 / LG group bits are one 4-, 2- or 1-byte store; the spheres of
// a group with a hit are not listed.
// kMask: lane masks (bit v of vm: sphere v of the lane is a valid lane; an
// invalid lane is never tested, listed or reported) -- kBand then means
// "every valid radius of the chunk is in band".
template <bool kFull, bool kBand, int LG, bool kMask>
__device__ __forceinline__ void resolve1_body(const FieldArgs& a, const FieldGeom& g,
                                              const uint8_t* sblk, int ch, int lane, bool check,
                                              uint64_t pol, Ring& rg, const float (&x)[4],
                                              const float (&y)[4], const float (&z)[4],
                                              const float (&r)[4], unsigned vm) {
  static_assert(LG == 1 || LG == 4 || LG == 8 || LG == 16, "lane-group width");
  constexpr unsigned kGroupMask = (1u << LG) - 1u;
  const int n = a.n;
  const int q0 = (ch << 7) + lane;
  const float INF = __int_as_float(0x7f800000);
  const unsigned bs = unsigned(g.bshift);
  float4 rec[4];
  float e2[4];
  unsigned inbm = 0u, lookm = 0u;
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const bool valid = (kFull || q0 + 32 * v < n) && (!kMask || ((vm >> v) & 1u));
    const bool inb = kBand ? (!kMask || valid) : (valid && r[v] >= a.rlo_f && r[v] <= a.rhi_f);
    float fx, fy, fz;
    const int ix = qcell(x[v], g.inv_h, g.nc0[0], fx);
    const int iy = qcell(y[v], g.inv_h, g.nc0[1], fy);
    const int iz = qcell(z[v], g.inv_h, g.nc0[2], fz);
    e2[v] = d2_fma(x[v] - __fmaf_rn(fx, g.h, g.c0[0]), y[v] - __fmaf_rn(fy, g.h, g.c0[1]),
                   z[v] - __fmaf_rn(fz, g.h, g.c0[2]));
    const bool in = unsigned(ix) < unsigned(g.nx) && unsigned(iy) < unsigned(g.ny) &&
                    unsigned(iz) < unsigned(g.nz);
    // the block table's certificate (block_free), branch-free: every lane
    // reads an entry (entry 0 outside the grid)
    const unsigned bi = ((unsigned(iz) >> bs) * unsigned(g.by) + (unsigned(iy) >> bs)) *
                            unsigned(g.bx) + (unsigned(ix) >> bs);
    const float bq = float(sblk[in ? bi : 0u]) * g.bstep;
    const bool look = inb && in && !(CAPT_K0_BLOCKS && bq > r[v] * kK1);
    const unsigned cell = (unsigned(iz) * unsigned(g.ny) + unsigned(iy)) * unsigned(g.nx) +
                          unsigned(ix);
    // no record: +inf (a witness miss); the sphere is decided by `look`
    rec[v] = make_float4(INF, INF, INF, INF);
    if (look) rec[v] = ldg_keep(a.t.field + cell, pol);
    inbm |= unsigned(inb) << v;
    lookm |= unsigned(look) << v;
#ifdef CAPT_FIELD_STATS
    {
      const unsigned lk = __ballot_sync(0xffffffffu, look);
      if (lane == 0) atomicAdd(a.list_n + 4, unsigned(__popc(lk)));
    }
#endif
  }
  unsigned ub[4], wd[4], elgm = 0u, badm = 0u;
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const float r2 = r[v] * r[v];
    const float dw = d2_fma(x[v] - rec[v].x, y[v] - rec[v].y, z[v] - rec[v].z);
    const float A = __fmaf_rn(-r[v], kK1, rec[v].w);  // (<= rec.w - fl(r k))
    const bool wmiss = dw > r2 * (1.0f + kTau);
    const bool hit = dw <= r2 * (1.0f - kTau);
    const bool free = wmiss && A > 0.f && A * A > e2[v] * kK1;
    const bool inb = (kBand && !kMask) || ((inbm >> v) & 1u);
    const bool valid = (kFull || q0 + 32 * v < n) && (!kMask || ((vm >> v) & 1u));
    // out of band: undecided (NaN radius, check_radii off), or only reported
    // (first_bad) with check_radii
    const bool bad = !kBand && check && valid && !inb && !(r[v] != r[v]);
    // in band: decided without a record (outside the grid, the block's
    // certificate), by the witness, or by the Lipschitz bound
    const bool open = ((lookm >> v) & 1u) && !hit && !free;
    const bool und = inb ? open : (valid && !bad);
    elgm |= unsigned(open && wmiss) << v;
    badm |= unsigned(bad) << v;
    // verdict word 4 ch + v = the ballot of sphere v
    wd[v] = __ballot_sync(0xffffffffu, ((lookm >> v) & 1u) && hit);
    if (LG > 1) {  // (this lane's group already has its hit: nothing to list)
      const bool res = (wd[v] & (kGroupMask << (lane & ~(LG - 1)))) != 0u;
      ub[v] = __ballot_sync(0xffffffffu, und && !res);
    } else {
      ub[v] = __ballot_sync(0xffffffffu, und);
    }
  }
  if (LG > 1) {
    // lane i < 128 / LG holds group (128 / LG) ch + i: field i % (32 / LG) of
    // slot i / (32 / LG)
    constexpr int kPerSlot = 32 / LG, kBits = 128 / LG;
    const int gv = (lane / kPerSlot) & 3;
    const unsigned h = gv == 0 ? wd[0] : gv == 1 ? wd[1] : gv == 2 ? wd[2] : wd[3];
    const unsigned gb =
        __ballot_sync(0xffffffffu, (h & (kGroupMask << (LG * (lane % kPerSlot)))) != 0u);
    if (lane == 0 && (kFull || (ch << 7) < n)) {
      if (kBits == 32) a.bits[ch] = gb;
      else if (kBits == 16) reinterpret_cast<uint16_t*>(a.bits)[ch] = uint16_t(gb & 0xffffu);
      else reinterpret_cast<uint8_t*>(a.bits)[ch] = uint8_t(gb & 0xffu);
    }
  } else if (kFull) {  // (the words of whole chunks: one 16-B store)
    if (lane == 0)
      *reinterpret_cast<uint4*>(a.bits + (ch << 2)) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
  } else {
#pragma unroll
    for (int v = 0; v < 4; ++v)
      if (lane == v && (ch << 7) + 32 * v < n) a.bits[(ch << 2) + v] = wd[v];
  }
  if (badm) {
#pragma unroll
    for (int v = 0; v < 4; ++v)
      if ((badm >> v) & 1u) atomicMin(a.first_bad, static_cast<unsigned long long>(q0 + 32 * v));
  }
  // the list: ballot prefix counts
  const unsigned tot = __popc(ub[0]) + __popc(ub[1]) + __popc(ub[2]) + __popc(ub[3]);
  if (tot == 0u) return;
  const unsigned lt = (1u << lane) - 1u;
  if (tot > 32u) {  // (rare: NaN or out-of-band batches) straight to the list
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(a.list_n, tot);
    base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      if ((ub[v] >> lane) & 1u) {
        const unsigned at = base + __popc(ub[v] & lt);
        a.list[at] = uint32_t(q0 + 32 * v);
        a.list_s[at] = make_float4(x[v], y[v], z[v], r[v]);
      }
      base += __popc(ub[v]);
    }
    return;
  }
  unsigned pos = rg.head + rg.cnt;
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    if ((ub[v] >> lane) & 1u) {
      const unsigned slot = (pos + __popc(ub[v] & lt)) & (kRing - 1);
      rg.q[slot] = uint32_t(q0 + 32 * v) | (((elgm >> v) & 1u) << 31);
      rg.s[slot] = make_float4(x[v], y[v], z[v], r[v]);
    }
    pos += __popc(ub[v]);
  }
  rg.cnt += tot;
  if (rg.cnt >= 32u) ring_drain(a, rg, 32u, lane);
}

template <bool kFull, int LG, bool kMask>
__device__ __forceinline__ void resolve1(const FieldArgs& a, const FieldGeom& g,
                                         const uint8_t* sblk, int ch, int lane, bool check,
                                         uint64_t pol, Ring& rg) {
  const int n = a.n;
  const int q0 = (ch << 7) + lane;
  float x[4], y[4], z[4], r[4];
  unsigned vm = 15u;
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const int q = kFull || q0 + 32 * v < n ? q0 + 32 * v : 0;
    x[v] = __ldcs(a.c + 3 * size_t(q));
    y[v] = __ldcs(a.c + 3 * size_t(q) + 1);
    z[v] = __ldcs(a.c + 3 * size_t(q) + 2);
    r[v] = __ldcs(a.r + q);
    if (kMask && a.mask[q] == 0) vm &= ~(1u << v);
  }
  // (an invalid lane's radius does not count in the vote)
  const float rin = a.rlo_f;
  if (CAPT_K0_FASTBAND && kFull &&
      chunk_in_band(a, kMask && !(vm & 1u) ? rin : r[0], kMask && !(vm & 2u) ? rin : r[1],
                    kMask && !(vm & 4u) ? rin : r[2], kMask && !(vm & 8u) ? rin : r[3])) {
    resolve1_body<true, true, LG, kMask>(a, g, sblk, ch, lane, check, pol, rg, x, y, z, r, vm);
    return;
  }
  resolve1_body<kFull, false, LG, kMask>(a, g, sblk, ch, lane, check, pol, rg, x, y, z, r, vm);
}

// (the single-sphere K0 has its own CTA shape: CAPT_K1_*)
#ifndef CAPT_K1_BLOCK
#define CAPT_K1_BLOCK 1024
#endif
#ifndef CAPT_K1_MINB
#define CAPT_K1_MINB 1
#endif
#ifndef CAPT_K1_WAVES
#define CAPT_K1_WAVES 1
#endif
template <int LG, bool kMask>
__global__ void __launch_bounds__(CAPT_K1_BLOCK, CAPT_K1_MINB) k_resolve1(FieldArgs a) {
  const FieldGeom g = a.t.fg;
  const bool check = a.flags & CAPT_CHECK_RADII;
  const int n = a.n;
  const int lane = threadIdx.x & 31;
  const int nfull = n >> 7;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t pol = l2_keep_policy();
  __shared__ float4 s_ring[CAPT_K1_BLOCK / 32][kRing];
  __shared__ uint32_t s_ringq[CAPT_K1_BLOCK / 32][kRing];
  Ring rg{s_ring[threadIdx.x >> 5], s_ringq[threadIdx.x >> 5], 0u, 0u};
  const uint8_t* sblk = stage_block_table(g, a.t.blk);
  // (launched after k_field_zero with programmatic serialisation)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int ch = w0; ch < nfull; ch += nwarps)
    resolve1<true, LG, kMask>(a, g, sblk, ch, lane, check, pol, rg);
  if ((n & 127) && w0 == nfull % nwarps)
    resolve1<false, LG, kMask>(a, g, sblk, nfull, lane, check, pol, rg);
  if (rg.cnt) ring_drain(a, rg, rg.cnt, lane);
}

// The list stage, part 1 (k_list_knn): every listed sphere meets its cell's
// candidate record -- the kCand cloud points nearest x0, stored as int16
// offsets (p - x0) / q_step, and kd_q q_step <= the distance from x0 to every
// other cloud point.  A decoded difference v = fl(fl(c - x0) - q q_step) is
// within q_err (Euclidean; q_step / 2 per axis from the offset rounding plus
// the fp32 roundings) of c - p, so with S = fp32 |v|^2 (relative error < 5u):
//   * hit:  RH = fl(r (1 - 2^-18)) - q_err (1 + 2^-17) > 0 and
//           S <= fl(RH^2)(1 - 2^-20): then |c - p| <= |v| + q_err < r(1 - 2^-19)
//           and the reference's float64 d^2 is <= r*r;
//   * miss: S >= fl(RM^2)(1 + 2^-20), RM = fl(r (1 + 2^-18)) + q_err (1 + 2^-17):
//           |c - p| >= |v| - q_err > r(1 + 2^-19): float64 d^2 > r*r;
//   * free: every candidate a miss and A = fl(kd - fl(r (1 + 2^-20))) > 0 with
//           A*A > fl(|c - x0|^2)(1 + 2^-20): every other cloud point p has
//           |p - c| >= kd - |c - x0| > r (1 + 16u) (the K0 free argument
//           with kd in place of nn).
// A candidate hit is a brute-force hit; "free" proves no point within r
// (DESIGN 3b; both need an in-band radius and a centre inside the grid).
// Candidates within about q_err of the sphere's surface are neither: the
// entry goes to the tree path.  One thread per entry: the entry itself
// (coalesced), then the record's six 32-byte loads; the list stage is bound
// by the L1 wavefronts of its gathers, so the record is one contiguous line
// and a half instead of a gather per candidate.  Hits set their bit; the
// open entries (about 1e-5 of a batch, plus every sphere the grid cannot
// take) go to a second list for part 2.


__global__ void __launch_bounds__(256) k_list_knn(FieldArgs a, uint32_t* __restrict__ list2,
                                                  uint32_t* __restrict__ list2_n,
                                                  uint32_t* __restrict__ list3,
                                                  uint32_t* __restrict__ list3_n) {
  const DevTree& t = a.t;
  const FieldGeom& g = a.t.fg;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // K0's list is complete
  const uint32_t n_list = *a.list_n;
  const int lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * blockDim.x;
  const int L = a.L;
  const float qs = g.q_step, qe = g.q_err * (1.0f + 0x1p-17f);
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j - lane < n_list; j += stride) {
    const bool act = j < n_list;
    uint32_t q = 0u;
    float4 sph = make_float4(0.f, 0.f, 0.f, 0.f);
    if (act) {
      q = __ldcs(a.list + j);
      sph = __ldcs(a.list_s + j);
    }
    const float x = sph.x, y = sph.y, z = sph.z, r = sph.w;
    float fx, fy, fz;
    const int ix = qcell(x, g.inv_h, g.nc0[0], fx);
    const int iy = qcell(y, g.inv_h, g.nc0[1], fy);
    const int iz = qcell(z, g.inv_h, g.nc0[2], fz);
    const bool cert = act && r >= a.rlo_f && r <= a.rhi_f && unsigned(ix) < unsigned(g.nx) &&
                      unsigned(iy) < unsigned(g.ny) && unsigned(iz) < unsigned(g.nz);
    bool hit = false, open = act;
    if (cert) {
      const unsigned cell =
          (unsigned(iz) * unsigned(g.ny) + unsigned(iy)) * unsigned(g.nx) + unsigned(ix);
      const uint32_t* rec = t.cand + size_t(cell) * kCandWords;
      uint32_t w[kCandWords];
#pragma unroll
      for (int i = 0; i < kCandWords / 8; ++i) {
        uint32_t v[8];
        ld_v8u(rec + 8 * i, v);
#pragma unroll
        for (int k = 0; k < 8; ++k) w[8 * i + k] = v[k];
      }
      const float ex = x - __fmaf_rn(fx, g.h, g.c0[0]);
      const float ey = y - __fmaf_rn(fy, g.h, g.c0[1]);
      const float ez = z - __fmaf_rn(fz, g.h, g.c0[2]);
      const float RH = r * (1.0f - 0x1p-18f) - qe;
      const float RM = r * (1.0f + 0x1p-18f) + qe;
      const float lo = RH > 0.f ? RH * RH * (1.0f - 0x1p-20f) : -1.f;
      const float hi = RM * RM * (1.0f + 0x1p-20f);
      bool amb = false;  // a candidate neither a definite hit nor a definite miss
#pragma unroll
      for (int k = 0; k < kCand; ++k) {
        const uint32_t wx = w[k >> 1], wy = w[16 + (k >> 1)], wz = w[32 + (k >> 1)];
        const int ox = (k & 1) ? slot_hi(wx) : slot_lo(wx);
        const int oy = (k & 1) ? slot_hi(wy) : slot_lo(wy);
        const int oz = (k & 1) ? slot_hi(wz) : slot_lo(wz);
        const float vx = fmaf(-float(ox), qs, ex), vy = fmaf(-float(oy), qs, ey),
                    vz = fmaf(-float(oz), qs, ez);
        const float S = d2_fma(vx, vy, vz);
        const bool used = ox != kCandNone;
        hit |= used && S <= lo;
        amb |= used && S < hi;
      }
      const float kd = float(slot_hi(w[15])) * qs;  // (x slot 31: kd_q, exact)
      const float A = kd - r * kK1;
      const bool free = !amb && A > 0.f && A * A > d2_fma(ex, ey, ez) * kK1;
      open = !hit && !free;
    }
    if (hit) {
      const uint32_t b = L == 1 ? q : q / uint32_t(L);
      atomicOr(a.bits + (b >> 5), 1u << (b & 31));
    }
    // open entries: in band inside the grid -> the exact bucket scan
    // (list 2); the rest (out-of-band radii with check_radii off, NaN,
    // centres outside the grid) -> the tree path (list 3)
    const unsigned lt = (1u << lane) - 1u;
    const unsigned om2 = __ballot_sync(0xffffffffu, open && cert);
    if (om2) {
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(list2_n, unsigned(__popc(om2)));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (open && cert) list2[base + __popc(om2 & lt)] = j;  // (its position in list 1)
    }
    const unsigned om3 = __ballot_sync(0xffffffffu, open && !cert);
    if (om3) {
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(list3_n, unsigned(__popc(om3)));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (open && !cert) list3[base + __popc(om3 & lt)] = j;
    }
  }
}

// The list stage, part 2a (k_bucket_list): an open entry of list 2 has an
// in-band radius and a centre inside the grid, so its verdict is the
// brute-force one (DESIGN 3b): some cloud point with the reference's float64
// ((dx^2 + dy^2) + dz^2) <= r*r.  Such a point lies within r (1 + 2^-20) of
// c on every axis, so in the point buckets (edge m cells; cell_of monotone,
// clamped) the box [c - r', c + r'] overlaps; one warp per entry scans those
// buckets row by row (one contiguous range of the bucket-sorted points per
// (y, z) bucket row), 32 points at a time, fp32 with the rows in the error
// band re-tested in float64, and stops at the first hit.
#ifndef CAPT_BUCKET_WARPS
#define CAPT_BUCKET_WARPS 2
#endif
constexpr int kBucketWarps = CAPT_BUCKET_WARPS;  // warps per entry (one CTA)
#ifndef CAPT_KNN_WAVES  // k_list_knn grid: CTAs per SM
#define CAPT_KNN_WAVES 8
#endif
#ifndef CAPT_BUCKET_UNROLL
#define CAPT_BUCKET_UNROLL 8
#endif
constexpr int kBucketUnroll = CAPT_BUCKET_UNROLL;
__global__ void __launch_bounds__(32 * kBucketWarps) k_bucket_list(
    FieldArgs a, const uint32_t* __restrict__ list2, const uint32_t* __restrict__ list2_n) {
  const DevTree& t = a.t;
  const FieldGeom& g = a.t.fg;
  __shared__ volatile int s_hit;
  __shared__ int s_skip;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t n_list = *list2_n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int L = a.L;
  for (uint32_t e = blockIdx.x; e < n_list; e += gridDim.x) {
    // (list 2 holds positions in list 1: the sphere and its index come from
    // K0's entry, one coalesced read instead of four gathers of the batch)
    const uint32_t j = list2[e];
    const uint32_t q = a.list[j];
    const uint32_t b = L == 1 ? q : q / uint32_t(L);
    if (threadIdx.x == 0) {
      s_hit = 0;
      // (a lane group already resolved by another entry: nothing to add)
      s_skip = L > 1 && ((__ldcg(a.bits + (b >> 5)) >> (b & 31)) & 1u);
    }
    __syncthreads();
    if (s_skip) {
      __syncthreads();
      continue;
    }
    const float4 s = a.list_s[j];
    const float r2 = s.w * s.w;
    const float loB = r2 * (1.0f - kTau), hiB = r2 * (1.0f + kTau);
    const float rp = s.w * (1.0f + 0x1p-20f);
    const int bx0 = cell_of(s.x - rp, g.lo[0], g.inv_h, g.nx) / g.m;
    const int bx1 = cell_of(s.x + rp, g.lo[0], g.inv_h, g.nx) / g.m;
    const int by0 = cell_of(s.y - rp, g.lo[1], g.inv_h, g.ny) / g.m;
    const int by1 = cell_of(s.y + rp, g.lo[1], g.inv_h, g.ny) / g.m;
    const int bz0 = cell_of(s.z - rp, g.lo[2], g.inv_h, g.nz) / g.m;
    const int bz1 = cell_of(s.z + rp, g.lo[2], g.inv_h, g.nz) / g.m;
    // the (y, z) bucket rows, 32 at a time: lane l reads row l's point
    // range, a warp scan flattens the ranges, and the CTA's warps then test
    // 32 points per step each, interleaved, wherever they lie (a point's row
    // by a binary search over the lanes' inclusive offsets), until one warp
    // finds a hit
    const int ny_rows = by1 - by0 + 1, rows = ny_rows * (bz1 - bz0 + 1);
    // (every exit test is warp-uniform: lane 0's read of the flag)
    auto stop = [&]() { return __shfl_sync(0xffffffffu, int(s_hit), 0) != 0; };
    for (int r0 = 0; r0 < rows && !stop(); r0 += 32) {
      uint32_t i0 = 0, len = 0;
      if (r0 + lane < rows) {
        const int by = by0 + (r0 + lane) % ny_rows, bz = bz0 + (r0 + lane) / ny_rows;
        const int row = (bz * g.nby + by) * g.nbx;
        i0 = __ldg(t.bstart + row + bx0);
        len = __ldg(t.bstart + row + bx1 + 1) - i0;
      }
      uint32_t incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      // (kBucketUnroll point loads of a lane in flight per step)
      for (uint32_t k0 = 32u * wid; k0 < total && !stop();
           k0 += 32u * kBucketWarps * kBucketUnroll) {
        float4 p[kBucketUnroll];
        bool in[kBucketUnroll];
#pragma unroll
        for (int u = 0; u < kBucketUnroll; ++u) {
          const uint32_t k = k0 + 32u * kBucketWarps * u + lane;
          int lo = 0;
#pragma unroll
          for (int step = 16; step; step >>= 1) {
            const uint32_t v = __shfl_sync(0xffffffffu, incl, lo + step - 1);
            if (v <= k) lo += step;
          }
          const uint32_t base = __shfl_sync(0xffffffffu, i0, lo);
          const uint32_t excl = __shfl_sync(0xffffffffu, incl - len, lo);
          in[u] = k < total;
          p[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (in[u]) p[u] = __ldg(t.cpts + base + (k - excl));
        }
        bool hit = false;
#pragma unroll
        for (int u = 0; u < kBucketUnroll; ++u) {
          const float d2 = d2_fma(s.x - p[u].x, s.y - p[u].y, s.z - p[u].z);
          hit |= in[u] && (d2 <= loB || (d2 < hiB && hit_f64(s.x, s.y, s.z, s.w, p[u])));
        }
        if (__any_sync(0xffffffffu, hit) && lane == 0) s_hit = 1;
        __syncwarp();
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_hit) atomicOr(a.bits + (b >> 5), 1u << (b & 31));
  }
}

// The list stage, part 2 (k_tree_list): the tree path over the entries part
// 1 left open, with the reference's semantics (query.py:184-219): descent,
// AABB prefilter, set scan.  The entries are few (about 1e-5 of a batch) and
// their sets long (config 3: up to 6,851 rows), so the kernel is built for
// short dependent chains: one warp per entry, the descent 5 levels per round
// trip (warp_descend), the leaf's probe record (conservative fp16 AABB
// reject, representative probe), then the set in steps of 512 rows (twelve
// 128-bit loads in flight per lane), fp32 with the rows in the error band
// re-tested in float64 on the spot; spheres outside the fast path
// (non-finite, extreme radii) take the exact float64 scan.
// The tree path for one sphere (warp-cooperative; the reference's semantics,
// query.py:184-219): descent, probe record (conservative fp16 AABB,
// representative), set scan 512 rows per step with band rows re-tested in
// float64 inline; spheres outside the fast path (non-finite, extreme radii)
// take the exact float64 scan.
__device__ __forceinline__ bool tree_verdict(const FieldArgs& a, const float (&c)[3], float r,
                                          int lane) {
  const DevTree& t = a.t;
  const bool prefilter = a.flags & CAPT_PREFILTER;
  const float band_lo = 1.0f - kTau, band_hi = 1.0f + kTau;
    const int leaf = int(warp_descend<float>(t, c, lane));
    const float r2 = r * r;
    const bool cfin = isfinite(c[0]) && isfinite(c[1]) && isfinite(c[2]);
    const bool fast = cfin && r2 >= kR2Min && r2 <= kR2Max;
    // non-finite centre with a finite radius never collides (float64 r^2 is finite)
    int st = fast ? 2 : ((!cfin && isfinite(r)) ? 0 : 3);
    float pr[8];
    ld_v8(t.probe + 8 * leaf, pr);
    if (prefilter && fast) {
      const float2 l01 = h2f2(pr[3]), l2h0 = h2f2(pr[4]), h12 = h2f2(pr[5]);
      const float rx = fmaxf(fmaxf(l01.x - c[0], 0.f), c[0] - l2h0.y);
      const float ry = fmaxf(fmaxf(l01.y - c[1], 0.f), c[1] - h12.x);
      const float rz = fmaxf(fmaxf(l2h0.x - c[2], 0.f), c[2] - h12.y);
      if (d2_fma(rx, ry, rz) > r2 * band_hi) st = 0;
    }
    if (st == 0) return false;
    const float loB = r2 * band_lo, hiB = r2 * band_hi;
    bool verdict = st == 2 && d2_fma(c[0] - pr[0], c[1] - pr[1], c[2] - pr[2]) <= loB;
    const uint2 set = __ldg(t.set + leaf);
    if (!verdict && st == 2) {
      const float* xs = reinterpret_cast<const float*>(t.data + set.x);
      const uint32_t m4 = (set.y + 3u) & ~3u;
      for (uint32_t p0 = 0; p0 < m4 && !verdict; p0 += 512) {
        float4 px[4], py[4], pz[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t p = p0 + 128 * u + 4 * lane;
          const uint32_t pc = p < m4 ? p : 0u;
          px[u] = __ldg(reinterpret_cast<const float4*>(xs + pc));
          py[u] = __ldg(reinterpret_cast<const float4*>(xs + m4 + pc));
          pz[u] = __ldg(reinterpret_cast<const float4*>(xs + 2 * m4 + pc));
        }
        bool hit = false;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (p0 + 128 * u + 4 * lane >= m4) continue;  // (padding rows are +inf: misses)
          const float X[4] = {px[u].x, px[u].y, px[u].z, px[u].w},
                      Y[4] = {py[u].x, py[u].y, py[u].z, py[u].w},
                      Z[4] = {pz[u].x, pz[u].y, pz[u].z, pz[u].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float d2 = d2_fma(c[0] - X[k], c[1] - Y[k], c[2] - Z[k]);
            // (a row in the error band: the reference's float64 test, inline)
            hit |= d2 <= loB ||
                   (d2 < hiB && hit_f64(c[0], c[1], c[2], r, make_float4(X[k], Y[k], Z[k], 0.f)));
          }
        }
        verdict = __any_sync(0xffffffffu, hit);
      }
    }
    if (st == 3 && !verdict) {
      const double c64[3] = {double(c[0]), double(c[1]), double(c[2])};
      verdict = warp_scan_f64(t, set, c64, double(r), lane);
    }
  return verdict;
}

__global__ void __launch_bounds__(256) k_tree_list(FieldArgs a, const uint32_t* __restrict__ list3,
                                                   const uint32_t* __restrict__ list3_n) {
  // launched with programmatic stream serialisation: scheduled while part 1
  // drains, reads its list only after it has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t n_list = *list3_n;
  const int lane = threadIdx.x & 31;
  const int L = a.L;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t e = warp; e < n_list; e += nwarps) {
    const uint32_t j = list3[e];  // (a position in list 1)
    const uint32_t q = a.list[j];
    const uint32_t b = L == 1 ? q : q / uint32_t(L);
    // (a lane group already resolved by another entry: nothing to add)
    // (warp-uniform: lane 0's read decides for the warp)
    if (L > 1 && __shfl_sync(0xffffffffu, (__ldcg(a.bits + (b >> 5)) >> (b & 31)) & 1u, 0)) continue;
    const float4 sph = a.list_s[j];
    const float c[3] = {sph.x, sph.y, sph.z};
    const bool verdict = tree_verdict(a, c, sph.w, lane);
    if (verdict && lane == 0) atomicOr(a.bits + (b >> 5), 1u << (b & 31));
  }
}

// ---------------------------------------------------------------- small batches
//
// One kernel for batches below kSmallBatch spheres: the fixed cost of the
// pipeline above (zero kernel, K0, three list kernels) is most of a small
// call.  A warp takes 32 lane groups (32 L spheres, one verdict word) at a
// time, 32 spheres per sub-step, one per lane: K0's certificates (band,
// block table, witness, Lipschitz); each sphere they leave open -- in a
// group without a hit -- is then resolved by the whole warp, one at a time:
// its cell's candidate record (lane k decodes candidate k), then the exact
// bucket scan (in band, inside the grid) or the tree path (the rest).  The
// verdict word is written whole (no zeroing, no atomics).

// Candidate record of the sphere's cell, one candidate per lane: 1 = a
// certified hit, 0 = certified free, 2 = open (the k_list_knn tests).
__device__ __forceinline__ int cand_verdict_warp(const DevTree& t, float x, float y, float z,
                                                 float r, int lane) {
  const FieldGeom& g = t.fg;
  float fx, fy, fz;
  const int ix = qcell(x, g.inv_h, g.nc0[0], fx);
  const int iy = qcell(y, g.inv_h, g.nc0[1], fy);
  const int iz = qcell(z, g.inv_h, g.nc0[2], fz);
  const unsigned cell =
      (unsigned(iz) * unsigned(g.ny) + unsigned(iy)) * unsigned(g.nx) + unsigned(ix);
  const uint32_t* rec = t.cand + size_t(cell) * kCandWords;
  const float qs = g.q_step, qe = g.q_err * (1.0f + 0x1p-17f);
  const float ex = x - __fmaf_rn(fx, g.h, g.c0[0]);
  const float ey = y - __fmaf_rn(fy, g.h, g.c0[1]);
  const float ez = z - __fmaf_rn(fz, g.h, g.c0[2]);
  const float RH = r * (1.0f - 0x1p-18f) - qe;
  const float RM = r * (1.0f + 0x1p-18f) + qe;
  const float lo = RH > 0.f ? RH * RH * (1.0f - 0x1p-20f) : -1.f;
  const float hi = RM * RM * (1.0f + 0x1p-20f);
  bool hit = false, amb = false;
  if (lane < kCand) {
    const int k = lane;
    const uint32_t wx = __ldg(rec + (k >> 1)), wy = __ldg(rec + 16 + (k >> 1)),
                   wz = __ldg(rec + 32 + (k >> 1));
    const int ox = (k & 1) ? slot_hi(wx) : slot_lo(wx);
    const int oy = (k & 1) ? slot_hi(wy) : slot_lo(wy);
    const int oz = (k & 1) ? slot_hi(wz) : slot_lo(wz);
    const float vx = fmaf(-float(ox), qs, ex), vy = fmaf(-float(oy), qs, ey),
                vz = fmaf(-float(oz), qs, ez);
    const float S = d2_fma(vx, vy, vz);
    const bool used = ox != kCandNone;
    hit = used && S <= lo;
    amb = used && S < hi;
  }
  if (__any_sync(0xffffffffu, hit)) return 1;
  const float kd = float(slot_hi(__ldg(rec + 15))) * qs;  // (x slot 31: kd_q, exact)
  const float A = kd - r * kK1;
  const bool free = !__any_sync(0xffffffffu, amb) && A > 0.f && A * A > d2_fma(ex, ey, ez) * kK1;
  return free ? 0 : 2;
}

// The exact bucket scan of k_bucket_list with one warp.
__device__ __forceinline__ bool bucket_verdict_warp(const DevTree& t, float4 s, int lane) {
  const FieldGeom& g = t.fg;
  const float r2 = s.w * s.w;
  const float loB = r2 * (1.0f - kTau), hiB = r2 * (1.0f + kTau);
  const float rp = s.w * (1.0f + 0x1p-20f);
  const int bx0 = cell_of(s.x - rp, g.lo[0], g.inv_h, g.nx) / g.m;
  const int bx1 = cell_of(s.x + rp, g.lo[0], g.inv_h, g.nx) / g.m;
  const int by0 = cell_of(s.y - rp, g.lo[1], g.inv_h, g.ny) / g.m;
  const int by1 = cell_of(s.y + rp, g.lo[1], g.inv_h, g.ny) / g.m;
  const int bz0 = cell_of(s.z - rp, g.lo[2], g.inv_h, g.nz) / g.m;
  const int bz1 = cell_of(s.z + rp, g.lo[2], g.inv_h, g.nz) / g.m;
  const int ny_rows = by1 - by0 + 1, rows = ny_rows * (bz1 - bz0 + 1);
  bool verdict = false;
  for (int r0 = 0; r0 < rows && !verdict; r0 += 32) {
    uint32_t i0 = 0, len = 0;
    if (r0 + lane < rows) {
      const int by = by0 + (r0 + lane) % ny_rows, bz = bz0 + (r0 + lane) / ny_rows;
      const int row = (bz * g.nby + by) * g.nbx;
      i0 = __ldg(t.bstart + row + bx0);
      len = __ldg(t.bstart + row + bx1 + 1) - i0;
    }
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    for (uint32_t k0 = 0; k0 < total && !verdict; k0 += 32) {
      const uint32_t k = k0 + lane;
      int lo = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, incl, lo + step - 1);
        if (v <= k) lo += step;
      }
      const uint32_t base = __shfl_sync(0xffffffffu, i0, lo);
      const uint32_t excl = __shfl_sync(0xffffffffu, incl - len, lo);
      bool hit = false;
      if (k < total) {
        const float4 p = __ldg(t.cpts + base + (k - excl));
        const float d2 = d2_fma(s.x - p.x, s.y - p.y, s.z - p.z);
        hit = d2 <= loB || (d2 < hiB && hit_f64(s.x, s.y, s.z, s.w, p));
      }
      verdict = __any_sync(0xffffffffu, hit);
    }
  }
  return verdict;
}

__global__ void __launch_bounds__(256) k_resolve_small(FieldArgs a) {
  const DevTree& t = a.t;
  const FieldGeom g = t.fg;
  // (small batches read the block table through L1 instead of staging it)
  const uint8_t* sblk = t.blk;
  const bool check = a.flags & CAPT_CHECK_RADII;
  const int lane = threadIdx.x & 31;
  const int L = a.L;
  const int64_t n = a.n, n_groups = n / L, n_words = (n_groups + 31) / 32;
  const uint64_t pol = l2_keep_policy();
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t wi = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; wi < n_words;
       wi += nw) {
    unsigned word = 0u;
    for (int sub = 0; sub < L; ++sub) {
      const int64_t q = wi * 32 * L + sub * 32 + lane;
      const int gb = (sub * 32 + lane) / L;  // this lane's group bit in the word
      const bool valid = q < n && (!a.mask || a.mask[q]);
      float x = 0.f, y = 0.f, z = 0.f, r = 0.f;
      if (q < n) {
        x = __ldg(a.c + 3 * q);
        y = __ldg(a.c + 3 * q + 1);
        z = __ldg(a.c + 3 * q + 2);
        r = __ldg(a.r + q);
      }
      const bool inb = valid && r >= a.rlo_f && r <= a.rhi_f;
      const bool bad = check && valid && !inb && r == r;
      if (bad) atomicMin(a.first_bad, static_cast<unsigned long long>(q));
      float fx, fy, fz;
      const int ix = qcell(x, g.inv_h, g.nc0[0], fx);
      const int iy = qcell(y, g.inv_h, g.nc0[1], fy);
      const int iz = qcell(z, g.inv_h, g.nc0[2], fz);
      const bool in = unsigned(ix) < unsigned(g.nx) && unsigned(iy) < unsigned(g.ny) &&
                      unsigned(iz) < unsigned(g.nz);
      const bool look = inb && in && !block_free(g, sblk, ix, iy, iz, in, r * kK1);
      float4 rec = make_float4(0.f, 0.f, 0.f, 0.f);
      if (look)
        rec = ldg_keep(t.field + ((unsigned(iz) * unsigned(g.ny) + unsigned(iy)) *
                                      unsigned(g.nx) + unsigned(ix)), pol);
      const float r2 = r * r;
      const float dw = d2_fma(x - rec.x, y - rec.y, z - rec.z);
      const bool hit = look && dw <= r2 * (1.0f - kTau);
      const float A = rec.w - r * kK1;
      const float e2 = d2_fma(x - __fmaf_rn(fx, g.h, g.c0[0]), y - __fmaf_rn(fy, g.h, g.c0[1]),
                              z - __fmaf_rn(fz, g.h, g.c0[2]));
      const bool free = dw > r2 * (1.0f + kTau) && A > 0.f && A * A > e2 * kK1;
      // decided: in band and (no record needed, witness hit, Lipschitz free);
      // an out-of-band radius with check_radii only reports first_bad
      const bool open = valid && !bad && !(inb && (!look || hit || free));
      // this sub-step's group bits with a hit
      const unsigned hb = __ballot_sync(0xffffffffu, hit);
      if (L == 1) {
        word |= hb;
      } else {
        const int per = 32 / L;  // (L <= 32) groups of this sub-step
        const unsigned lm = L == 32 ? 0xffffffffu : ((1u << L) - 1u);
        for (int j = 0; j < per; ++j)
          if ((hb >> (j * L)) & lm) word |= 1u << (sub * per + j);
      }
      // the open spheres of groups without a hit, one at a time by the warp
      unsigned um = __ballot_sync(0xffffffffu, open && !((word >> gb) & 1u));
      while (um) {
        const int u = __ffs(int(um)) - 1;
        um &= um - 1u;
        const int ub = __shfl_sync(0xffffffffu, gb, u);
        if ((word >> ub) & 1u) continue;  // (its group got a hit meanwhile)
        const float ux = __shfl_sync(0xffffffffu, x, u), uy = __shfl_sync(0xffffffffu, y, u),
                    uz = __shfl_sync(0xffffffffu, z, u), ur = __shfl_sync(0xffffffffu, r, u);
        const bool ucert = __shfl_sync(0xffffffffu, int(inb && in), u) != 0;
        bool v;
        if (ucert) {
          const int cv = cand_verdict_warp(t, ux, uy, uz, ur, lane);
          v = cv == 1 || (cv == 2 && bucket_verdict_warp(t, make_float4(ux, uy, uz, ur), lane));
        } else {
          const float cu[3] = {ux, uy, uz};
          v = tree_verdict(a, cu, ur, lane);
        }
        if (v) word |= 1u << ub;
      }
    }
    if (lane == 0) a.bits[wi] = word;
  }
}

}  // namespace

// ---------------------------------------------------------------- host

int build_field(capt_tree* tree, cudaStream_t s) {
  if (tree->field_mem) {
    cudaFree(tree->field_mem);
    tree->field_mem = nullptr;
    tree->field = nullptr;
    tree->cand = nullptr;
    tree->blk = nullptr;
    tree->cpts = nullptr;
    tree->bstart = nullptr;
  }
  if (tree->h.k != 3) return CAPT_OK;
  const DevTree t = view(tree);
  const int64_t n = t.n;
  int* d_box = nullptr;
  CAPT_CUDA(cudaMallocAsync(&d_box, 6 * sizeof(int), s));
  const int init[6] = {INT_MAX, INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MIN};
  CAPT_CUDA(cudaMemcpyAsync(d_box, init, sizeof(init), cudaMemcpyHostToDevice, s));
  k_rep_box<<<grid_for(n, 256, 4), 256, 0, s>>>(t.rep, n, d_box);
  CAPT_CUDA(cudaGetLastError());
  int hb[6];
  CAPT_CUDA(cudaMemcpyAsync(hb, d_box, sizeof(hb), cudaMemcpyDeviceToHost, s));
  CAPT_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(d_box, s);
  if (hb[0] == INT_MAX) return CAPT_OK;  // no finite point
  auto of = [](int o) {
    const int i = o >= 0 ? o : o ^ 0x7fffffff;
    float f;
    memcpy(&f, &i, 4);
    return f;
  };
  FieldGeom g;
  memset(&g, 0, sizeof(g));
  double ext[3];
  for (int d = 0; d < 3; ++d) {
    g.blo[d] = of(hb[d]);
    g.bhi[d] = of(hb[3 + d]);
    ext[d] = double(g.bhi[d]) - double(g.blo[d]);
  }
  const double rmax = tree->h.r_max;
  if (!(rmax > 0.0) || !std::isfinite(rmax)) return CAPT_OK;
  // cell edge: about CAPT_FIELD_CELLS cells over the box grown by r_max + h;
  // not below r_max / 16 (bounds the buckets at ~20^3 cells)
  const double budget = double(CAPT_FIELD_CELLS);
  double h = std::cbrt((ext[0] + 2 * rmax) * (ext[1] + 2 * rmax) * (ext[2] + 2 * rmax) / budget);
  h = std::max(h, rmax / 16.0);
  int64_t dims[3];
  for (int it = 0; it < 200; ++it) {
    int64_t tot = 1;
    for (int d = 0; d < 3; ++d) {
      dims[d] = std::max<int64_t>(1, int64_t(std::ceil((ext[d] + 2 * (rmax + h)) / h)));
      tot *= dims[d];
    }
    if (tot <= int64_t(budget * 1.05)) break;
    h *= 1.02;
  }
  g.h = float(h);
  h = double(g.h);
  g.inv_h = float(1.0 / h);
  for (int d = 0; d < 3; ++d) {
    g.lo[d] = float(double(g.blo[d]) - (rmax + h));
    g.c0[d] = float(double(g.lo[d]) + 0.5 * h);
    g.nc0[d] = float(-double(g.c0[d]) / h);
  }
  g.nx = int(dims[0]);
  g.ny = int(dims[1]);
  g.nz = int(dims[2]);
  g.cells = dims[0] * dims[1] * dims[2];
  // stored bounds are capped at rcap >= r_max + h (> r_max + |c - x0| for a
  // centre inside its cell); a point within rcap of a cell centre has its
  // computed cell within ceil(rcap / h) + 1 cells of it per axis, + 1 more
  // for the rounding of cell_of: rr; point buckets of m = 2 cells
  g.rcap = float(rmax + h);
  g.m = 2;
  g.rr = int(std::ceil(double(g.rcap) / h)) + 2;
  // candidate offsets: int16 multiples of a power-of-two step covering rcap;
  // the decoded difference fl(fl(c - x0) - q step) is within, per axis,
  // step / 2 (offset rounding) + u |c - x0| + u |fl(c - x0) - q step| of
  // c - p (u = 2^-24, |c - x0| <= h, |q step| <= 2 rcap): q_err bounds the
  // Euclidean sum, rounded up
  {
    const double u = std::ldexp(1.0, -24);
    const double step = std::ldexp(1.0, int(std::ceil(std::log2(double(g.rcap) / 32767.0))));
    g.q_step = float(step);
    const double ax = 0.5 * step + 4.0 * u * (h + 2.0 * double(g.rcap) + step);
    g.q_err = std::nextafter(float(std::sqrt(3.0) * ax * (1.0 + 1e-6)), INFINITY);
  }
  BucketGrid b;
  b.nbx = (g.nx + g.m - 1) / g.m;
  b.nby = (g.ny + g.m - 1) / g.m;
  b.nbz = (g.nz + g.m - 1) / g.m;
  b.nb = int64_t(b.nbx) * b.nby * b.nbz;

  uint32_t *keys = nullptr, *keys_out = nullptr, *counts = nullptr, *bstart = nullptr;
  int *ids = nullptr, *ids_out = nullptr;
  void* tmp = nullptr;
  size_t tb_sort = 0, tb_scan = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb_sort, keys, keys_out, ids, ids_out, int(n), 0, 32, s);
  cub::DeviceScan::ExclusiveSum(nullptr, tb_scan, counts, bstart, int(b.nb + 2), s);
  struct Scratch {
    cudaStream_t s;
    std::vector<void*> p;
    ~Scratch() {
      for (void* q : p) cudaFreeAsync(q, s);
    }
  } scratch{s, {}};
  auto get = [&](auto** ptr, size_t count) {
    const cudaError_t e = dmalloc(ptr, count, s);
    if (e == cudaSuccess) scratch.p.push_back(*ptr);
    return e;
  };
  CAPT_CUDA(get(&keys, n));
  CAPT_CUDA(get(&keys_out, n));
  CAPT_CUDA(get(&ids, n));
  CAPT_CUDA(get(&ids_out, n));
  CAPT_CUDA(get(&counts, b.nb + 2));
  CAPT_CUDA(get(&bstart, b.nb + 2));
  CAPT_CUDA(get(reinterpret_cast<char**>(&tmp), std::max(tb_sort, tb_scan) + 16));
  CAPT_CUDA(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * (b.nb + 2), s));
  k_bucket_keys<<<grid_for(n, 256, 8), 256, 0, s>>>(t.rep, n, g, b, keys, ids, counts);
  CAPT_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb_sort, keys, keys_out, ids, ids_out, int(n), 0,
                                            32, s));
  CAPT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb_scan, counts, bstart, int(b.nb + 2), s));
  uint32_t n_fin = 0;
  CAPT_CUDA(cudaMemcpyAsync(&n_fin, bstart + b.nb, 4, cudaMemcpyDeviceToHost, s));
  CAPT_CUDA(cudaStreamSynchronize(s));
  // block table: the smallest blocks whose table fits CAPT_BLK_BYTES; bstep
  // the power of two covering rcap in 255 steps; rcell bounds |c - x0| for a
  // centre c whose computed cell is x0's: per axis t = fma(c, inv_h, nc0)
  // is within 2^-24 (|c| / h + |c0| / h + |t|) of (c - c0) / h (inv_h and
  // nc0 rounded, one fma rounding), the cell is round(t), and fma(i, h, c0)
  // is within 2^-24 |x0| of i h + c0
  {
    int bs = 1;
    auto nbk = [&](int sh) {
      return int64_t((g.nx + (1 << sh) - 1) >> sh) * ((g.ny + (1 << sh) - 1) >> sh) *
             ((g.nz + (1 << sh) - 1) >> sh);
    };
    while (nbk(bs) > int64_t(CAPT_BLK_BYTES)) ++bs;
    g.bshift = bs;
    g.bx = (g.nx + (1 << bs) - 1) >> bs;
    g.by = (g.ny + (1 << bs) - 1) >> bs;
    g.bz = (g.nz + (1 << bs) - 1) >> bs;
    g.bbytes = int((nbk(bs) + 15) & ~int64_t(15));
    g.bstep = float(std::ldexp(1.0, int(std::ceil(std::log2(double(g.rcap) / 255.0)))));
  }
  double mu = 0.0;
  {
    const double u = std::ldexp(1.0, -24), hh = double(g.h);
    const int nd[3] = {g.nx, g.ny, g.nz};
    for (int d = 0; d < 3; ++d) {
      const double lo_h = std::fabs(double(g.lo[d])) / hh, c0_h = std::fabs(double(g.c0[d])) / hh;
      const double t_err = u * (lo_h + nd[d] + 2.0 + c0_h + nd[d] + 1.0);
      const double x0_err = u * (std::fabs(double(g.c0[d])) + (nd[d] + 1.0) * hh);
      mu = std::max(mu, hh * t_err + x0_err);
    }
  }
  const float rcell = std::nextafter(
      float(std::sqrt(3.0) * (0.5 * double(g.h) + mu) * (1.0 + std::ldexp(1.0, -20))), INFINITY);
  // one allocation: K0 records | candidate records | block table | the
  // points in bucket order | the bucket starts (the list stage's exact scan)
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t off_cand =  // (K0 records | second records; 32-B loads)
      al(sizeof(float4) * second_base(g.cells) + 4 * size_t(kSecondWords) * size_t(g.cells));
  const size_t off_blk = off_cand + al(sizeof(uint32_t) * kCandWords * size_t(g.cells));
  const size_t off_cpts = off_blk + al(size_t(g.bbytes));
  const size_t off_bst = off_cpts + al(sizeof(float4) * std::max<size_t>(n_fin, 1));
  const size_t bytes = off_bst + sizeof(uint32_t) * size_t(b.nb + 2);
  char* mem = nullptr;
  cudaError_t e = cudaMalloc(&mem, bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(clearance field)");
  float4* field = reinterpret_cast<float4*>(mem);
  uint32_t* cand = reinterpret_cast<uint32_t*>(mem + off_cand);
  float4* cpts = reinterpret_cast<float4*>(mem + off_cpts);
  uint32_t* bst = reinterpret_cast<uint32_t*>(mem + off_bst);
  g.nbx = b.nbx;
  g.nby = b.nby;
  g.nbz = b.nbz;
  e = cudaMemcpyAsync(bst, bstart, sizeof(uint32_t) * size_t(b.nb + 2), cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) {
    cudaFree(mem);
    return cuda_fail(e, "clearance field build");
  }
  k_bucket_points<<<grid_for(n_fin, 256, 8), 256, 0, s>>>(t.rep, ids_out, n_fin, cpts);
  {
    const int64_t tiles = int64_t((g.nx + kTileX - 1) / kTileX) * ((g.ny + kTileY - 1) / kTileY) *
                          ((g.nz + kTileZ - 1) / kTileZ);
    k_field_cand<<<int(tiles), 256, 0, s>>>(g, b, bstart, cpts, field, cand);
  }
  uint8_t* blk = reinterpret_cast<uint8_t*>(mem + off_blk);
  e = cudaMemsetAsync(blk, 0, size_t(g.bbytes), s);
  if (e == cudaSuccess) {
    const int nbk = g.bx * g.by * g.bz;
    k_block_table<<<(nbk + 7) / 8, 256, 0, s>>>(g, field, rcell, blk);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaFree(mem);
    return cuda_fail(e, "clearance field build");
  }
  note_launches(7);
  tree->field_mem = mem;
  tree->field = field;
  tree->cand = cand;
  tree->blk = blk;
  tree->cpts = cpts;
  tree->bstart = bst;
  tree->fg = g;
  return CAPT_OK;
}

// below this many spheres (auto mode) one fused kernel (k_resolve_small)
// beats the pipeline's fixed cost: on the tabletop cloud up to ~768 K spheres,
// on the dense config-3 cloud (more spheres left to the in-warp paths) not
// beyond ~256 K (profiles/small_crossover.py); 512 K is the compromise
#ifndef CAPT_SMALL_BATCH
#define CAPT_SMALL_BATCH (int64_t(1) << 19)
#endif

bool field_eligible(const DevTree& t, int64_t n, uint32_t flags) {
  if (!t.field || t.k != 3 || (flags & (CAPT_INPUT_F64 | CAPT_STATS))) return false;
  if (n >= (int64_t(1) << 31) - (int64_t(1) << 24)) return false;
  // fp32 r^2 of every in-band radius must stay normal and finite
  if (!(t.r_min >= 0x1p-50) || !(t.r_max <= 0x1p50)) return false;
  if (flags & CAPT_MODE_FIELD) return true;
  return !(flags & (CAPT_MODE_DIRECT | CAPT_MODE_BINNED | CAPT_MODE_THREAD | CAPT_MODE_WARP));
}

// The pipeline's zeroing (list counter; the verdict words when lane groups
// OR into them) as a kernel, so K0 can follow it with programmatic launch.
__global__ void k_field_zero(uint32_t* __restrict__ ctr, uint32_t* __restrict__ bits,
                             int64_t n_words) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t i0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i0 < 8) ctr[i0] = 0u;
  for (int64_t i = i0; i < n_words; i += int64_t(gridDim.x) * blockDim.x) bits[i] = 0u;
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl_f(void (*kernel)(KArgs...), int grid, int block, size_t smem,
                                cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Per-(device, stream) scratch for the list: reused across calls instead of
// a cudaMallocAsync / cudaFreeAsync pair per call.  A call holds the entry's
// lock while it enqueues its kernels, so two host threads issuing queries on
// the same stream cannot interleave their uses of the buffer (the stream
// orders the kernels of each call after the previous call's).
struct ListScratch {
  std::mutex mu;
  uint32_t* buf = nullptr;  // counters (8 words: list_n, list2_n) | list | list2 | list_s
  int64_t cap = 0;          // capacity of each list (entries, a multiple of 4)
};
static std::mutex g_scratch_mu;
static std::map<std::pair<int, cudaStream_t>, ListScratch*>* g_scratch = nullptr;

static ListScratch* scratch_for(int dev, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  if (!g_scratch) g_scratch = new std::map<std::pair<int, cudaStream_t>, ListScratch*>();
  ListScratch*& e = (*g_scratch)[{dev, s}];
  if (!e) e = new ListScratch();  // (kept for the process: streams are reused)
  return e;
}

// Stage timing (capt_stage_timing / capt_stage_times): CUDA events on the
// launching stream around K0 and the list stage of every field-pipeline call,
// read back and summed on request (no synchronisation inside the calls).
struct StageEvents {
  static constexpr int kMax = 2048;
  std::mutex mu;
  bool on = false;
  int n = 0;
  cudaEvent_t ev[kMax][3] = {};
};
static StageEvents g_stage[kMaxDevices];

static int stage_record(int dev, int call, int k, cudaStream_t s) {
  StageEvents& st = g_stage[dev];
  std::lock_guard<std::mutex> lk(st.mu);
  if (!st.ev[call][k]) CAPT_CUDA(cudaEventCreate(&st.ev[call][k]));
  CAPT_CUDA(cudaEventRecord(st.ev[call][k], s));
  return CAPT_OK;
}

int launch_field(const DevTree& t, const void* centers, const void* radii, int64_t n, int L,
                 const uint8_t* mask, uint32_t flags, uint32_t* bits, int64_t n_words,
                 unsigned long long* first_bad, cudaStream_t s) {
  FieldArgs a;
  a.t = t;
  a.c = static_cast<const float*>(centers);
  a.r = static_cast<const float*>(radii);
  a.n = int(n);
  a.L = L;
  a.mask = mask;
  a.flags = flags & ~uint32_t(CAPT_MODE_BINNED | CAPT_MODE_DIRECT | CAPT_MODE_FIELD);
  a.bits = bits;
  a.first_bad = first_bad;
  float lo = float(t.r_min), hi = float(t.r_max);
  if (double(lo) < t.r_min) lo = nextafterf(lo, INFINITY);
  if (double(hi) > t.r_max) hi = nextafterf(hi, -INFINITY);
  a.rlo_f = lo;
  a.rhi_f = hi;
  if (n < CAPT_SMALL_BATCH && !(flags & CAPT_MODE_FIELD)) {
    const int64_t nwd = (n / L + 31) / 32;
    k_resolve_small<<<grid_for(nwd * 32, 256, 8), 256, 0, s>>>(a);
    CAPT_CUDA(cudaGetLastError());
    note_launches(1);
    return CAPT_OK;
  }
  int dev = 0;
  CAPT_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(CAPT_ECUDA, "device index out of range");
  ListScratch* sc = scratch_for(dev, s);
  std::lock_guard<std::mutex> lk(sc->mu);
  if (sc->cap < n) {
    if (sc->buf) CAPT_CUDA(cudaFreeAsync(sc->buf, s));
    sc->buf = nullptr;
    sc->cap = 0;
    const int64_t cap = (n + 3) & ~int64_t(3);
    CAPT_CUDA(dmalloc(&sc->buf, 7 * size_t(cap) + 8, s));
    sc->cap = cap;
  }
  // counters: list_n (K0's list), list2_n (the bucket scan), list3_n (the
  // tree path); lists: list | list2 | list_s (4 words) | list3
  a.list_n = sc->buf;
  a.list = sc->buf + 8;
  uint32_t* const list2_n = sc->buf + 1;
  uint32_t* const list3_n = sc->buf + 2;
  uint32_t* const list2 = sc->buf + 8 + sc->cap;
  a.list_s = reinterpret_cast<float4*>(sc->buf + 8 + 2 * sc->cap);
  uint32_t* const list3 = sc->buf + 8 + 6 * sc->cap;
  {
    const int64_t zw = L >= 8 ? n_words : 0;
    k_field_zero<<<grid_for(zw + 8, 256, 4), 256, 0, s>>>(a.list_n, bits, zw);
    CAPT_CUDA(cudaGetLastError());
    note_launches(1);
  }
  int tcall = -1;
  {
    StageEvents& st = g_stage[dev];
    std::lock_guard<std::mutex> lk2(st.mu);
    if (st.on && st.n < StageEvents::kMax) tcall = st.n++;
  }
  if (tcall >= 0) {
    const int rc = stage_record(dev, tcall, 0, s);
    if (rc) return rc;
  }
  // (the lane-group K0 for other widths and lane masks: 128-bit loads when
  // the inputs are 16-byte aligned)
  const bool vec = (reinterpret_cast<uintptr_t>(centers) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(radii) & 15) == 0;
  const int grid = grid_for(((n + 127) / 128) * 32, CAPT_K0_BLOCK, CAPT_K0_WAVES);
  // the single-sphere K0 stages the block table in dynamic shared memory
  // (above the 48 KB default with its rings: opted in once per device)
  const size_t sm1 = size_t(t.fg.bbytes);
  {
    static std::mutex mu;
    static bool opted[kMaxDevices] = {};
    std::lock_guard<std::mutex> lk1(mu);
    if (!opted[dev]) {
      const auto opt_in = [](auto kernel) {
        return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    CAPT_BLK_BYTES);
      };
      CAPT_CUDA(opt_in(k_resolve1<1, false>));
      CAPT_CUDA(opt_in(k_resolve1<4, false>));
      CAPT_CUDA(opt_in(k_resolve1<8, false>));
      CAPT_CUDA(opt_in(k_resolve1<16, false>));
      CAPT_CUDA(opt_in(k_resolve1<1, true>));
      CAPT_CUDA(opt_in(k_resolve1<4, true>));
      CAPT_CUDA(opt_in(k_resolve1<8, true>));
      CAPT_CUDA(opt_in(k_resolve1<16, true>));
      opted[dev] = true;
    }
  }
  const size_t sm = CAPT_K0_GROUP_BLOCKS ? sm1 : 0;
  const bool bits16 = (reinterpret_cast<uintptr_t>(bits) & 15) == 0;
  const int grid1 = grid_for(((n + 127) / 128) * 32, CAPT_K1_BLOCK, CAPT_K1_WAVES);
  const auto k1 = [&](auto kernel) {
    return launch_pdl_f(kernel, grid1, CAPT_K1_BLOCK, sm1, s, a);
  };
  if (L == 1 && bits16) CAPT_CUDA(mask ? k1(k_resolve1<1, true>) : k1(k_resolve1<1, false>));
  else if (L == 4) CAPT_CUDA(mask ? k1(k_resolve1<4, true>) : k1(k_resolve1<4, false>));
  else if (L == 8) CAPT_CUDA(mask ? k1(k_resolve1<8, true>) : k1(k_resolve1<8, false>));
  else if (L == 16) CAPT_CUDA(mask ? k1(k_resolve1<16, true>) : k1(k_resolve1<16, false>));
  else if (mask && vec)
    CAPT_CUDA(launch_pdl_f(k_resolve<true, true, 0>, grid, CAPT_K0_BLOCK, sm, s, a));
  else if (mask)
    CAPT_CUDA(launch_pdl_f(k_resolve<false, true, 0>, grid, CAPT_K0_BLOCK, sm, s, a));
  else if (vec)
    CAPT_CUDA(launch_pdl_f(k_resolve<true, false, 0>, grid, CAPT_K0_BLOCK, sm, s, a));
  else
    CAPT_CUDA(launch_pdl_f(k_resolve<false, false, 0>, grid, CAPT_K0_BLOCK, sm, s, a));
  CAPT_CUDA(cudaGetLastError());
  note_launches(1);
  if (tcall >= 0) {
    const int rc = stage_record(dev, tcall, 1, s);
    if (rc) return rc;
  }
  // the list stage: persistent grids (the list lengths are known on the device only)
  CAPT_CUDA(launch_pdl_f(k_list_knn, grid_for(n, 256, CAPT_KNN_WAVES), 256, 0, s, a, list2, list2_n, list3,
                         list3_n));
  CAPT_CUDA(launch_pdl_f(k_bucket_list, grid_for(int64_t(n) * 32 * kBucketWarps, 32 * kBucketWarps, 64 / kBucketWarps),
                         32 * kBucketWarps, 0, s, a, static_cast<const uint32_t*>(list2),
                         static_cast<const uint32_t*>(list2_n)));
  CAPT_CUDA(launch_pdl_f(k_tree_list, grid_for(int64_t(n) * 32, 256, 8), 256, 0, s, a,
                         static_cast<const uint32_t*>(list3), static_cast<const uint32_t*>(list3_n)));
  CAPT_CUDA(cudaGetLastError());
  note_launches(3);
  if (tcall >= 0) {
    const int rc = stage_record(dev, tcall, 2, s);
    if (rc) return rc;
  }
#ifdef CAPT_FIELD_STATS  // diagnostics build (build_ext -D CAPT_FIELD_STATS --out ...)
  uint32_t nl[6] = {0, 0, 0, 0, 0, 0};
  CAPT_CUDA(cudaMemcpyAsync(nl, a.list_n, 24, cudaMemcpyDeviceToHost, s));
  CAPT_CUDA(cudaStreamSynchronize(s));
  fprintf(stderr,
          "[capt field] n=%lld L=%d list=%u (%.4f%%) bucket scan=%u tree path=%u records=%u "
          "(%.3f) block-free=%u (%.3f)\n",
          (long long)n, L, nl[0], 100.0 * nl[0] / double(n), nl[1], nl[2], nl[4],
          nl[4] / double(n), nl[5], nl[5] / double(n));
#endif
  return CAPT_OK;
}

}  // namespace capt

using namespace capt;

extern "C" int capt_tree_field(const capt_tree* tree, capt_field_info* info, float* cells,
                               float* cand) {
  if (!tree || !info) return fail(CAPT_EINVAL, "NULL argument");
  if (!tree->field) return fail(CAPT_EINVAL, "tree has no clearance field (k < 3)");
  const FieldGeom& g = tree->fg;
  memset(info, 0, sizeof(*info));
  info->nx = g.nx;
  info->ny = g.ny;
  info->nz = g.nz;
  info->n_cand = kCand;
  info->n_cells = g.cells;
  info->h = g.h;
  info->rcap = g.rcap;
  info->q_step = g.q_step;
  info->q_err = g.q_err;
  for (int d = 0; d < 3; ++d) {
    info->lo[d] = g.lo[d];
    info->c0[d] = g.c0[d];
    info->box_lo[d] = g.blo[d];
    info->box_hi[d] = g.bhi[d];
  }
  if (!cells && !cand) return CAPT_OK;
  CAPT_CUDA(cudaSetDevice(tree->device));
  const size_t nc = size_t(g.cells);
  const size_t nrec = second_base(g.cells) + size_t(kSecondWords / 4) * nc;
  std::vector<float4> rec(nrec);
  std::vector<uint32_t> w(nc * kCandWords);
  CAPT_CUDA(cudaMemcpy(rec.data(), tree->field, sizeof(float4) * nrec, cudaMemcpyDeviceToHost));
  CAPT_CUDA(cudaMemcpy(w.data(), tree->cand, sizeof(uint32_t) * w.size(), cudaMemcpyDeviceToHost));
  auto slot = [&](size_t cell, int axis, int j) {
    const uint32_t v = w[cell * kCandWords + 16 * axis + (j >> 1)];
    return int(int16_t(uint16_t((j & 1) ? (v >> 16) : (v & 0xffffu))));
  };
  const float INF = std::numeric_limits<float>::infinity();
  for (size_t i = 0; i < nc; ++i) {
    if (cells) {
      float* o = cells + 8 * i;
      o[0] = rec[i].x;
      o[1] = rec[i].y;
      o[2] = rec[i].z;
      o[3] = rec[i].w;
      o[4] = float(slot(i, 0, 31)) * g.q_step;  // kd
      o[5] = float(slot(i, 1, 31));            // candidates
      uint32_t kd2;  // the second record's bound: its last 16-bit slot
      memcpy(&kd2, &rec[second_base(g.cells) + size_t(kSecondWords / 4) * (i + 1) - 1].w, 4);
      o[6] = float(int16_t(uint16_t(kd2 >> 16))) * g.q_step;
      o[7] = float(kSecond);  // (o[6] bounds the (kSecond + 2)-th nearest)
    }
    if (cand) {  // offsets (p - x0) / q_step, kCandNone for unused slots
      for (int k = 0; k < kCand; ++k)
        for (int d = 0; d < 3; ++d) {
          const int q = slot(i, d, k);
          cand[(i * kCand + k) * 3 + d] = q == kCandNone ? INF : float(q);
        }
    }
  }
  return CAPT_OK;
}

extern "C" int capt_tree_field_blocks(const capt_tree* tree, int32_t* dims, float* step,
                                      uint8_t* table) {
  if (!tree || !dims || !step) return fail(CAPT_EINVAL, "NULL argument");
  if (!tree->field || !tree->blk) return fail(CAPT_EINVAL, "tree has no clearance field (k < 3)");
  const FieldGeom& g = tree->fg;
  dims[0] = g.bx;
  dims[1] = g.by;
  dims[2] = g.bz;
  dims[3] = g.bshift;
  *step = g.bstep;
  if (table) {
    CAPT_CUDA(cudaSetDevice(tree->device));
    CAPT_CUDA(cudaMemcpy(table, tree->blk, size_t(g.bx) * g.by * g.bz, cudaMemcpyDeviceToHost));
  }
  return CAPT_OK;
}

extern "C" int capt_field_list_counts(void* stream, uint32_t* out) {
  if (!out) return fail(CAPT_EINVAL, "NULL argument");
  int dev = 0;
  CAPT_CUDA(cudaGetDevice(&dev));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ListScratch* sc = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    if (g_scratch) {
      auto it = g_scratch->find({dev, s});
      if (it != g_scratch->end()) sc = it->second;
    }
  }
  if (!sc) return fail(CAPT_EINVAL, "no field query on this stream");
  std::lock_guard<std::mutex> lk(sc->mu);
  if (!sc->buf) return fail(CAPT_EINVAL, "no field query on this stream");
  uint32_t h[3] = {0, 0, 0};
  CAPT_CUDA(cudaMemcpyAsync(h, sc->buf, sizeof(h), cudaMemcpyDeviceToHost, s));
  CAPT_CUDA(cudaStreamSynchronize(s));
  out[0] = h[0];
  out[1] = h[1];
  out[2] = h[2];
  return CAPT_OK;
}

extern "C" int capt_stage_timing(int enable) {
  int dev = 0;
  CAPT_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(CAPT_ECUDA, "device index out of range");
  StageEvents& st = g_stage[dev];
  std::lock_guard<std::mutex> lk(st.mu);
  st.on = enable != 0;
  st.n = 0;
  return CAPT_OK;
}

extern "C" int capt_stage_times(double* ms, int64_t* calls) {
  if (!ms || !calls) return fail(CAPT_EINVAL, "NULL argument");
  int dev = 0;
  CAPT_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(CAPT_ECUDA, "device index out of range");
  StageEvents& st = g_stage[dev];
  std::lock_guard<std::mutex> lk(st.mu);
  ms[0] = ms[1] = ms[2] = 0.0;
  for (int i = 0; i < st.n; ++i) {
    CAPT_CUDA(cudaEventSynchronize(st.ev[i][2]));
    float a = 0.f, b = 0.f;
    CAPT_CUDA(cudaEventElapsedTime(&a, st.ev[i][0], st.ev[i][1]));
    CAPT_CUDA(cudaEventElapsedTime(&b, st.ev[i][1], st.ev[i][2]));
    ms[0] += a;
    ms[1] += b;
    ms[2] += a + b;
  }
  *calls = st.n;
  st.n = 0;
  return CAPT_OK;
}
