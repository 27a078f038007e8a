// Clearance field: resolve most spheres of a query before any tree descent.
//
// The reference answers a sphere by descending to its leaf and scanning the
// leaf's affordance set (query.py:184-219).  Because the affordance sets are
// complete for radii inside [r_min, r_max] (Alg. 1; pinned
// by the reference's brute-force equality tests, test_acceptance.py:54-91),
// the verdict of an in-band sphere is exactly "some cloud point lies within
// r of the centre" -- the brute-force verdict (oracle.py:34-49).  Two
// certificates decide that verdict for most spheres without the tree:
//
//   * hit:  some cloud point w has fp32 |c - w|^2 <= r^2 (1 - TAU)  (the
//           same definite-hit band as the representative probe);
//   * free: a lower bound of the distance from c to every cloud point
//           exceeds r with a relative margin.  The bound comes from a
//           uniform grid whose cells store nn <= dist(x0, cloud) for the
//           cell centre x0: dist(c, cloud) >= nn - |c - x0| (the distance
//           function is 1-Lipschitz), or from the cloud's box.
//
// Each cell is one 16-B record {witness xyz, nn}, witness = the cloud point
// nearest x0: one L2-resident 128-bit load per sphere.  Spheres that neither
// certificate decides (a few percent; near |dist - r| ~ cell size), spheres
// outside the band (check_radii=False), non-finite centres and extreme radii
// go to a compact list that the tree path (descent, AABB, representative
// probe, cooperative affordance-set scans with the float64 fix-up) resolves
// with the reference's own semantics.
//
// Kernels:
//   build:  k_rep_box (cloud box), k_bucket_keys + radix sort (points into
//           buckets of >= rcap), k_field_nn (one CTA per bucket: exact
//           nearest point of every cell centre among the 27 neighbouring
//           buckets, staged through shared memory)
//   query:  k_resolve  (per sphere: band check, box / field certificates,
//                       lane-group resolution, bit words, compact list)
//           k_resolve_list (the tree path over the list)
#include <cub/cub.cuh>
#include <cuda_fp16.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "capt_binned.cuh"
#include "capt_tc.cuh"
#include "capt_internal.cuh"
#include "capt_query_common.cuh"

namespace capt {

#ifndef CAPT_FIELD_CELLS
#define CAPT_FIELD_CELLS (1 << 21)  // 32 MB of records: L2-resident
#endif

namespace {

constexpr float kFreeMargin = 1.0f + 0x1p-20f;  // (r + e)(1 + 16u): see k_resolve
constexpr float kNNShrink = 1.0f - 0x1p-19f;    // fp32 sqrt(d^2) -> certified lower bound
constexpr int kFieldChunk = 1024;               // staged points per k_field_nn round
constexpr int kCellsPerThread = 4;

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
// fp16 octant bound o of a cell (octant array: 8 halves per cell)
__device__ __forceinline__ float oct_bound(const float4* oct, unsigned cell, unsigned o) {
  const unsigned short hb =
      __ldg(reinterpret_cast<const unsigned short*>(oct) + 8 * size_t(cell) + o);
  return __half2float(__ushort_as_half(hb));
}
__device__ __forceinline__ float d2_fma(float dx, float dy, float dz) {
  return fmaf(dz, dz, fmaf(dy, dy, dx * dx));
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
       i += int64_t(gridDim.x) * blockDim.x)
    pts[i] = rep[ids[i]];
}

// One CTA per bucket: every cell of the bucket against every point of the
// 27 neighbouring buckets (points farther than rcap from a cell centre lie
// outside them: bucket edge m*h >= rcap + 2h, see build_field), the
// candidates staged through shared memory in chunks.
__global__ void __launch_bounds__(256, 1) k_field_nn(FieldGeom g, BucketGrid b,
                                                  const uint32_t* __restrict__ bstart,
                                                  const float4* __restrict__ pts,
                                                  float4* __restrict__ field) {
  __shared__ float4 sp[kFieldChunk];
  const int bid = blockIdx.x;
  const int bx = bid % b.nbx, by = (bid / b.nbx) % b.nby, bz = bid / (b.nbx * b.nby);
  const int x0 = bx * g.m, y0 = by * g.m, z0 = bz * g.m;
  const int cx = min(g.m, g.nx - x0), cy = min(g.m, g.ny - y0), cz = min(g.m, g.nz - z0);
  const int ncells = cx * cy * cz;
  const float INF = __int_as_float(0x7f800000);
  const float hh = g.oct_half;
  for (int pass = 0; pass < ncells; pass += 256 * kCellsPerThread) {
    float px[kCellsPerThread], py[kCellsPerThread], pz[kCellsPerThread], best[kCellsPerThread];
    float ob[kCellsPerThread][8];  // squared distance from each octant box
    int bi[kCellsPerThread];
#pragma unroll
    for (int k = 0; k < kCellsPerThread; ++k) {
      const int j = pass + k * 256 + threadIdx.x;
      const int lx = j % cx, ly = (j / cx) % cy, lz = j / (cx * cy);
      px[k] = centre_of(x0 + lx, g.h, g.c0[0]);
      py[k] = centre_of(y0 + ly, g.h, g.c0[1]);
      pz[k] = centre_of(z0 + lz, g.h, g.c0[2]);
      best[k] = INF;
      bi[k] = -1;
#pragma unroll
      for (int o = 0; o < 8; ++o) ob[k][o] = INF;
    }
    for (int nz = max(bz - 1, 0); nz <= min(bz + 1, b.nbz - 1); ++nz)
      for (int ny = max(by - 1, 0); ny <= min(by + 1, b.nby - 1); ++ny)
        for (int nx = max(bx - 1, 0); nx <= min(bx + 1, b.nbx - 1); ++nx) {
          const int nbid = (nz * b.nby + ny) * b.nbx + nx;
          const uint32_t s0 = bstart[nbid], s1 = bstart[nbid + 1];
          for (uint32_t c0 = s0; c0 < s1; c0 += kFieldChunk) {
            const int cnt = int(min(uint32_t(kFieldChunk), s1 - c0));
            __syncthreads();
            for (int i = threadIdx.x; i < cnt; i += 256) sp[i] = pts[c0 + i];
            __syncthreads();
            for (int i = 0; i < cnt; ++i) {
              const float4 p = sp[i];
#pragma unroll
              for (int k = 0; k < kCellsPerThread; ++k) {
                const float ax = p.x - px[k], ay = p.y - py[k], az = p.z - pz[k];
                const float d2 = d2_fma(ax, ay, az);
                if (d2 < best[k]) {
                  best[k] = d2;
                  bi[k] = int(c0) + i;
                }
                // gap from the octant box [x0, x0 + hh] (bit 1) / [x0 - hh, x0] (bit 0)
                const float gx1 = fmaxf(fmaxf(-ax, ax - hh), 0.f), gx0 = fmaxf(fmaxf(ax, -ax - hh), 0.f);
                const float gy1 = fmaxf(fmaxf(-ay, ay - hh), 0.f), gy0 = fmaxf(fmaxf(ay, -ay - hh), 0.f);
                const float gz1 = fmaxf(fmaxf(-az, az - hh), 0.f), gz0 = fmaxf(fmaxf(az, -az - hh), 0.f);
                const float xy[4] = {fmaf(gy0, gy0, gx0 * gx0), fmaf(gy0, gy0, gx1 * gx1),
                                     fmaf(gy1, gy1, gx0 * gx0), fmaf(gy1, gy1, gx1 * gx1)};
                const float zz0 = gz0 * gz0, zz1 = gz1 * gz1;
#pragma unroll
                for (int o = 0; o < 4; ++o) {
                  ob[k][o] = fminf(ob[k][o], xy[o] + zz0);
                  ob[k][o + 4] = fminf(ob[k][o + 4], xy[o] + zz1);
                }
              }
            }
          }
        }
#pragma unroll
    for (int k = 0; k < kCellsPerThread; ++k) {
      const int j = pass + k * 256 + threadIdx.x;
      // fp32 |x0 - p|^2 has relative error < 5u, sqrtf one more u:
      // sqrtf(d2) (1 - 2^-19) (rounded) < the real distance
      const int bsel = bi[k] >= 0 ? bi[k] : 0;
      const float nn = fminf(g.rcap, __fmul_rn(sqrtf(best[k]), kNNShrink));
      // octant bounds: the same relative margin and an absolute one for the
      // rounded gaps, capped where the candidate search ends, fp16 rounded down
      unsigned short hb[8];
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        float lb = fmaf(sqrtf(ob[k][o]), kNNShrink, -g.oct_abs);
        lb = fminf(fmaxf(lb, 0.f), g.oct_cap);
        hb[o] = __half_as_ushort(__float2half_rd(lb));
      }
      if (j < ncells) {
        const int lx = j % cx, ly = (j / cx) % cy, lz = j / (cx * cy);
        const int64_t cell = (int64_t(z0 + lz) * g.ny + (y0 + ly)) * g.nx + (x0 + lx);
        const float4 w = bi[k] >= 0 ? pts[bsel] : make_float4(INF, INF, INF, 0.f);
        field[cell] = make_float4(w.x, w.y, w.z, nn);
        field[g.cells + cell] = make_float4(
            __uint_as_float(unsigned(hb[0]) | (unsigned(hb[1]) << 16)),
            __uint_as_float(unsigned(hb[2]) | (unsigned(hb[3]) << 16)),
            __uint_as_float(unsigned(hb[4]) | (unsigned(hb[5]) << 16)),
            __uint_as_float(unsigned(hb[6]) | (unsigned(hb[7]) << 16)));
      }
    }
  }
}

// Distance-sorted set copy.  Keys: fp32 |p - o| (o = the set's origin) of
// every stored row (padding rows +inf), sorted within each set; the scan of a
// sphere (c, r) can stop at the first row with |p - o| > r + |c - o| (a row
// beyond it is farther than r from c).  Stored distances are rounded down.
__global__ void k_sort_keys(DevTree t, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                            int* __restrict__ seg_begin, int* __restrict__ seg_end) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = warp; j < t.n; j += nwarps) {
    const uint2 st = t.set[j];
    const uint32_t m4 = (st.y + 3u) & ~3u;
    const float* base = reinterpret_cast<const float*>(t.data + st.x);
    const int64_t b = int64_t(st.x) * 4 / 3;
    const float4 o = t.org[j];
    if (lane == 0) {
      seg_begin[j] = int(b);
      seg_end[j] = int(b + m4);
    }
    for (uint32_t i = lane; i < m4; i += 32) {
      float d = __int_as_float(0x7f800000);
      if (i < st.y) {
        const float dx = base[i] - o.x, dy = base[m4 + i] - o.y, dz = base[2 * m4 + i] - o.z;
        d = sqrtf(d2_fma(dx, dy, dz));
        if (!(d <= 3.0e38f)) d = __int_as_float(0x7f800000);  // (+inf rows of padding leaves)
      }
      keys[b + i] = __float_as_uint(d);
      vals[b + i] = i;
    }
  }
}

__global__ void k_sort_gather(DevTree t, const uint32_t* __restrict__ keys,
                              const uint32_t* __restrict__ vals, float* __restrict__ sdata,
                              float* __restrict__ sdist) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = warp; j < t.n; j += nwarps) {
    const uint2 st = t.set[j];
    const uint32_t m4 = (st.y + 3u) & ~3u;
    const float* src = reinterpret_cast<const float*>(t.data + st.x);
    float* dst = sdata + int64_t(st.x) * 4;
    const int64_t b = int64_t(st.x) * 4 / 3;
    for (uint32_t i = lane; i < m4; i += 32) {
      const uint32_t k = vals[b + i];
      dst[i] = src[k];
      dst[m4 + i] = src[m4 + k];
      dst[2 * m4 + i] = src[2 * m4 + k];
      // fp32 |p - o| has relative error < 4u: (1 - 2^-19) rounds it below the real distance
      sdist[b + i] = __fmul_rn(__uint_as_float(keys[b + i]), 1.0f - 0x1p-19f);
    }
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
  uint32_t* list;    // sphere ids the tree path resolves
  uint32_t* list_n;
  float rlo_f, rhi_f;  // fp32 images of the double band edges
};

// K0.  A warp takes chunks of 128 consecutive spheres; lane l owns spheres
// 4l .. 4l+3 of the chunk, so a chunk is three 128-bit centre loads and one
// 128-bit radius load per lane (the next chunk is loaded while this one is
// decided).  For an in-band sphere (r in [r_min, r_max] in double; NaN is
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
// spheres of unresolved groups are appended to the list in sphere order (a
// group's spheres stay contiguous) with one atomic per warp and chunk.
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
// verdict bits, the list of undecided spheres (in sphere order).
// A CTA's list entries collect in shared memory (one shared atomic per warp
// and chunk instead of a returning global atomic on every chunk's critical
// path) and are copied out once at the end of the kernel; a full buffer
// falls back to direct appends.
#ifndef CAPT_K0_LISTBUF
#define CAPT_K0_LISTBUF 4096
#endif
constexpr int kListBuf = CAPT_K0_LISTBUF;
struct ListBuf {
  uint32_t* buf;  // shared memory (nullptr: append to the global list directly)
  uint32_t* n;    // entries reserved in buf (may run past kListBuf)
  uint32_t* end;  // the first reservation that did not fit (its range is a hole)
};

template <int LT>
__device__ __forceinline__ void emit_chunk(const FieldArgs& a, int ch, int lane, bool check,
                                           unsigned hitb, unsigned undb, unsigned badb,
                                           ListBuf lb = {nullptr, nullptr, nullptr}) {
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
  // the list, in sphere order
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
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    unsigned base = 0;
    bool local = false;
    if (lane == 0) {
      if (lb.buf) {
        base = atomicAdd(lb.n, unsigned(tot));
        local = base + unsigned(tot) <= unsigned(kListBuf);
        if (!local && base < unsigned(kListBuf)) atomicMin(lb.end, base);
      }
      if (!local) base = atomicAdd(a.list_n, unsigned(tot));
    }
    base = __shfl_sync(0xffffffffu, base, 0) + unsigned(incl - cnt);
    local = __shfl_sync(0xffffffffu, local, 0);
    uint32_t* dst = local ? lb.buf : a.list;
#pragma unroll
    for (int v = 0; v < 4; ++v)
      if ((lst >> v) & 1u) dst[base + __popc(lst & ((1u << v) - 1u))] = uint32_t(q0 + v);
  }
}

// Decide one chunk (see above): writes its bits and list entries.  LT: the
// lane width when known at compile time (0: a.L at run time); kFull: a whole
// unmasked chunk (no per-sphere validity test).
template <bool kMask, int LT, bool kFull>
__device__ __forceinline__ void resolve_chunk(const FieldArgs& a, const FieldGeom& g,
                                              const Chunk& k, int ch, int lane, bool check,
                                              uint64_t pol, ListBuf lb = {nullptr, nullptr, nullptr}) {
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
  float4 rec[4];
  auto cell = [&](int v, bool skip) {
    valid[v] = kFull || q0 + v < n;
    if (kMask) valid[v] = valid[v] && a.mask[valid[v] ? q0 + v : 0] != 0;
    inband[v] = r[v] >= a.rlo_f && r[v] <= a.rhi_f;
    ix[v] = __float2int_rd(__fmul_rn(__fsub_rn(x[v], g.lo[0]), g.inv_h));
    iy[v] = __float2int_rd(__fmul_rn(__fsub_rn(y[v], g.lo[1]), g.inv_h));
    iz[v] = __float2int_rd(__fmul_rn(__fsub_rn(z[v], g.lo[2]), g.inv_h));
    // (the index is used only inside the grid: no clamp)
    const bool in = unsigned(ix[v]) < nxu && unsigned(iy[v]) < nyu && unsigned(iz[v]) < nzu;
    look[v] = valid[v] && inband[v] && in && !skip;
    rec[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (look[v])
      rec[v] = ldg_keep(a.t.field + ((unsigned(iz[v]) * nyu + unsigned(iy[v])) * nxu + unsigned(ix[v])),
                        pol);
  };
  // phase 2: the certificates of sphere v
  unsigned hitb = 0, undb = 0, badb = 0;
  const float band_lo = 1.0f - kTau;
  auto cert = [&](int v) {
    const float ex = x[v] - centre_of(ix[v], g.h, g.c0[0]);
    const float ey = y[v] - centre_of(iy[v], g.h, g.c0[1]);
    const float ez = z[v] - centre_of(iz[v], g.h, g.c0[2]);
    const float e2 = d2_fma(ex, ey, ez);
    const float r2 = r[v] * r[v];
    const bool hit = d2_fma(x[v] - rec[v].x, y[v] - rec[v].y, z[v] - rec[v].z) <= r2 * band_lo;
    const float A = rec[v].w - r[v] * kK1;  // (fl(r k) >= r (1 + 15u))
    const bool free = A > 0.f && A * A > e2 * kK1;
    hitb |= unsigned(look[v] && hit) << v;
    // decided: in-band and (outside the grid / skipped, or certified); with
    // check_radii an out-of-band (non-NaN) radius only reports first_bad
    const bool bad = check && valid[v] && (r[v] < a.rlo_f || r[v] > a.rhi_f);
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
  emit_chunk<LT>(a, ch, lane, check, hitb, undb, badb, lb);
}

// K0 CTAs per SM the register allocation must allow: one chunk per warp in
// registers, 4 (54 registers; 5: 48 registers, slower on config 3); with the
// ping-pong prefetch (CAPT_K0_PREFETCH) 3 was best (78 registers)
#ifndef CAPT_K0_MINB
#define CAPT_K0_MINB 4
#endif

// persistent warps over the whole 128-sphere chunks, two per round (ping-pong
// registers: the next chunk's loads are in flight while one is decided); the
// last, partial chunk (scalar loads, per-sphere validity) after the loop
template <bool kVec, bool kMask, int LT>
#ifndef CAPT_K0_BLOCK
#define CAPT_K0_BLOCK 256
#endif
__global__ void __launch_bounds__(CAPT_K0_BLOCK, CAPT_K0_MINB) k_resolve(FieldArgs a) {
  const FieldGeom g = a.t.fg;
  const bool check = a.flags & CAPT_CHECK_RADII;
  const int n = a.n;
  const int lane = threadIdx.x & 31;
  const int nfull = n >> 7;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t pol = l2_keep_policy();
  __shared__ uint32_t s_list[LT == 8 ? 1 : kListBuf];
  __shared__ uint32_t s_ln, s_end, s_gbase;
  if (threadIdx.x == 0) {
    s_ln = 0u;
    s_end = uint32_t(kListBuf);
  }
  __syncthreads();
  // (8-sphere groups: most groups resolve on a hit, lists are short -- the
  // buffer's shared memory would cost the record loads L1 capacity instead:
  // config 1 K0 170 vs 166 us)
  const ListBuf lb = LT == 8 ? ListBuf{nullptr, nullptr, nullptr} : ListBuf{s_list, &s_ln, &s_end};
  // (launched after k_field_zero with programmatic serialisation)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  int ch = w0;
#ifndef CAPT_K0_PREFETCH  // one chunk in registers: 166 us at 4 CTAs/SM vs 175 (ping-pong, 3 CTAs)
  for (; ch < nfull; ch += nwarps) {
    const Chunk A = load_chunk<kVec, true>(a.c, a.r, ch, lane, n);
    resolve_chunk<kMask, LT, !kMask>(a, g, A, ch, lane, check, pol, lb);
  }
  if (false) {
#else
  if (ch < nfull) {
#endif
    Chunk A = load_chunk<kVec, true>(a.c, a.r, ch, lane, n), B;
    while (true) {
      const int c1 = ch + nwarps;
      if (c1 < nfull) B = load_chunk<kVec, true>(a.c, a.r, c1, lane, n);
      resolve_chunk<kMask, LT, !kMask>(a, g, A, ch, lane, check, pol);
      if (c1 >= nfull) break;
      const int c2 = c1 + nwarps;
      if (c2 < nfull) A = load_chunk<kVec, true>(a.c, a.r, c2, lane, n);
      resolve_chunk<kMask, LT, !kMask>(a, g, B, c1, lane, check, pol);
      if (c2 >= nfull) break;
      ch = c2;
    }
  }
  if ((n & 127) && w0 == nfull % nwarps) {
    const Chunk T = load_chunk<false>(a.c, a.r, nfull, lane, n);
    resolve_chunk<kMask, LT, false>(a, g, T, nfull, lane, check, pol, lb);
  }
  // the CTA's buffered list entries, in one reservation
  __syncthreads();
  const uint32_t cnt = min(s_ln, s_end);  // (entries past a non-fitting reservation went global)
  if (threadIdx.x == 0 && cnt) s_gbase = atomicAdd(a.list_n, cnt);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) a.list[s_gbase + i] = s_list[i];
}

// K0 with TMA bulk copies (the default for unmasked, 16-B aligned batches).
// Persistent CTAs of 8 warps take tiles of 1024 spheres; one thread streams
// each tile's centres (12 KB) and radii (4 KB) into a ring of kStages
// shared-memory stages with cp.async.bulk (completion on the stage's
// mbarrier, L2 evict-first), so the sphere stream stays in flight without
// holding registers; warp w decides chunk w of the tile from shared memory
// (resolve_chunk), the stage is refilled once every warp is past it.  The
// spheres after the last whole tile take the register path.
constexpr int kTileSpheres = 1024;
constexpr int kStages = 3;
constexpr uint32_t kTileC = kTileSpheres * 12, kTileR = kTileSpheres * 4;
constexpr size_t kTmaSmem = size_t(kStages) * (kTileC + kTileR) + 64;

__device__ __forceinline__ uint64_t l2_stream_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(mbar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(tc::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(mbar)), "l"(pol)
      : "memory");
}

template <int LT>
__global__ void __launch_bounds__(256, 4) k_resolve_tma(FieldArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* const sc = reinterpret_cast<float*>(smem);
  float* const sr = reinterpret_cast<float*>(smem + kStages * kTileC);
  uint64_t* const full = reinterpret_cast<uint64_t*>(smem + kStages * (kTileC + kTileR));
  const FieldGeom g = a.t.fg;
  const bool check = a.flags & CAPT_CHECK_RADII;
  const int n = a.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ntiles = n / kTileSpheres;
  const uint64_t keep = l2_keep_policy();
  if (threadIdx.x == 0) {
    for (int st = 0; st < kStages; ++st) tc::mbar_init(&full[st], 1);
    tc::fence_async_smem();
  }
  __syncthreads();
  auto issue = [&](int tile, int st) {
    const uint64_t pol = l2_stream_policy();
    mbar_expect_tx(&full[st], kTileC + kTileR);
    bulk_g2s(sc + st * (kTileC / 4), a.c + size_t(tile) * kTileSpheres * 3, kTileC, &full[st], pol);
    bulk_g2s(sr + st * (kTileR / 4), a.r + size_t(tile) * kTileSpheres, kTileR, &full[st], pol);
  };
  if (threadIdx.x == 0)
    for (int st = 0; st < kStages; ++st) {
      const int tile = blockIdx.x + st * gridDim.x;
      if (tile < ntiles) issue(tile, st);
    }
  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it % kStages;
    tc::mbar_wait(&full[st], uint32_t((it / kStages) & 1));
    const float4* c4 = reinterpret_cast<const float4*>(sc + st * (kTileC / 4) + warp * 384) + 3 * lane;
    Chunk k;
    k.p0 = c4[0];
    k.p1 = c4[1];
    k.p2 = c4[2];
    k.pr = reinterpret_cast<const float4*>(sr + st * (kTileR / 4) + warp * 128)[lane];
    resolve_chunk<false, LT, true>(a, g, k, tile * (kTileSpheres / 128) + warp, lane, check, keep);
    __syncthreads();  // every warp is past stage st
    if (threadIdx.x == 0) {
      const int next = tile + kStages * gridDim.x;
      if (next < ntiles) issue(next, st);
    }
  }
  // the spheres after the last whole tile: register path, one chunk per warp
  const int nchunks = (n + 127) >> 7;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int ch = ntiles * (kTileSpheres / 128) + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
       ch < nchunks; ch += nwarps) {
    const Chunk k = load_chunk<true>(a.c, a.r, ch, lane, n);
    if ((ch << 7) + 128 <= n) resolve_chunk<false, LT, true>(a, g, k, ch, lane, check, keep);
    else resolve_chunk<false, LT, false>(a, g, k, ch, lane, check, keep);
  }
}

// List filter: the octant certificate.  Each cell also stores, per octant
// (bit d set: the centre is at or above x0 on axis d -- an exact sign test),
// an fp16 lower bound of the distance from the octant's box to the cloud
// (rounded down at build, the box grown by the cell-index rounding); an
// undecided in-band sphere whose bound exceeds fl(r (1 + 2^-20)) is free.
// Survivors are compacted in order within each warp (one atomic per warp).
// One 2-byte load per listed sphere instead of an octant record for every
// sphere in K0 (32-byte records there cost more than the shorter list saves).
__device__ __forceinline__ bool octant_free(const FieldArgs& a, const FieldGeom& g, float x,
                                            float y, float z, float r) {
  const int ix = __float2int_rd(__fmul_rn(__fsub_rn(x, g.lo[0]), g.inv_h));
  const int iy = __float2int_rd(__fmul_rn(__fsub_rn(y, g.lo[1]), g.inv_h));
  const int iz = __float2int_rd(__fmul_rn(__fsub_rn(z, g.lo[2]), g.inv_h));
  const bool in = unsigned(ix) < unsigned(g.nx) && unsigned(iy) < unsigned(g.ny) &&
                  unsigned(iz) < unsigned(g.nz);
  if (!in || !(r >= a.rlo_f && r <= a.rhi_f)) return false;
  const unsigned o = (x - centre_of(ix, g.h, g.c0[0]) >= 0.f ? 1u : 0u) |
                     (y - centre_of(iy, g.h, g.c0[1]) >= 0.f ? 2u : 0u) |
                     (z - centre_of(iz, g.h, g.c0[2]) >= 0.f ? 4u : 0u);
  const unsigned cell =
      (unsigned(iz) * unsigned(g.ny) + unsigned(iy)) * unsigned(g.nx) + unsigned(ix);
  return oct_bound(a.t.field + g.cells, cell, o) > r * kK1;
}

__global__ void __launch_bounds__(256) k_list_octant(FieldArgs a, uint32_t* __restrict__ out,
                                                     uint32_t* __restrict__ out_n) {
  const FieldGeom g = a.t.fg;
  const uint32_t n_list = *a.list_n;
  const int lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t j0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; j0 < n_list; j0 += stride) {
    const uint32_t j = j0 + lane;
    const bool act = j < n_list;
    const uint32_t q = act ? a.list[j] : 0u;
    bool keep = act;
    if (act) {
      const float x = __ldg(a.c + 3 * size_t(q)), y = __ldg(a.c + 3 * size_t(q) + 1),
                  z = __ldg(a.c + 3 * size_t(q) + 2), r = __ldg(a.r + q);
      keep = !octant_free(a, g, x, y, z, r);
    }
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    unsigned base = 0;
    if (lane == 0 && km) base = atomicAdd(out_n, unsigned(__popc(km)));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (keep) out[base + __popc(km & ((1u << lane) - 1u))] = q;
  }
}

// The tree path over the list (the reference's semantics for every sphere it
// holds).  The list is short but its spheres are the hard ones, so the kernel
// is built for short dependent-load chains: a warp takes 8 entries; lanes 0-7
// descend (T through L1), load the leaf's probe record
// (conservative AABB reject, representative probe); then 4 lanes per entry
// scan its set, 64 points per step (12 128-bit loads in flight per lane),
// fp32 with the float64 re-scan of the band.  (One entry per lane with a
// serial warp scan, or a per-thread scan, measured ~73 us for config 1's 85 K
// entries: the warp waits on its longest chain.)
constexpr int kLE = 8;  // list entries per warp

template <bool kOct>
__global__ void __launch_bounds__(256) k_resolve_list(FieldArgs a) {
  const DevTree& t = a.t;
  // launched with programmatic stream serialisation: scheduled while K0
  // drains, reads K0's list only after K0 has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t n_list = *a.list_n;
  const int lane = threadIdx.x & 31;
  const int slot = lane >> 2, sl = lane & 3;
  const int L = a.L;
  const bool prefilter = a.flags & CAPT_PREFILTER;
  const float band_lo = 1.0f - kTau, band_hi = 1.0f + kTau;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t j0 = warp * kLE; j0 < n_list; j0 += nwarps * kLE) {
    const uint32_t j = j0 + lane;
    const bool active = lane < kLE && j < n_list;
    const uint32_t q = active ? a.list[j] : 0u;
    float cx = 0.f, cy = 0.f, cz = 0.f, r = 0.f;
    if (active) {
      cx = __ldg(a.c + 3 * size_t(q));
      cy = __ldg(a.c + 3 * size_t(q) + 1);
      cz = __ldg(a.c + 3 * size_t(q) + 2);
      r = __ldg(a.r + q);
    }
    const uint32_t gid = active ? q / uint32_t(L) : 0xffffffffu - lane;
    const unsigned gm = L > 1 ? __match_any_sync(0xffffffffu, gid) : (1u << lane);
    int st = 0, leaf = 0;
    bool verdict = false;
    float r2 = 0.f;
    // the octant certificate first (k_list_octant when the list is filtered)
    const bool sure_free = kOct && active && octant_free(a, a.t.fg, cx, cy, cz, r);
    if (active && !sure_free) {
      // descent (tree.py:266-273)
      int i = 0;
      for (int s = 0; s < t.depth; ++s) {  // (the top levels stay in L1)
        const int ax = s % 3;
        const float cv = ax == 0 ? cx : (ax == 1 ? cy : cz);
        i = 2 * i + 1 + (cv > __ldg(t.T + i) ? 1 : 0);
      }
      leaf = i - int(t.n - 1);
      // classification (as k_bin_count3 / k_query_hybrid)
      r2 = r * r;
      const bool cfin = isfinite(cx) && isfinite(cy) && isfinite(cz);
      const bool fast = cfin && r2 >= kR2Min && r2 <= kR2Max;
      st = fast ? 2 : ((!cfin && isfinite(r)) ? 0 : 3);
      float pr[8];
      ld_v8(t.probe + 8 * leaf, pr);
      if (prefilter) {
        const float2 l01 = h2f2(pr[3]), l2h0 = h2f2(pr[4]), h12 = h2f2(pr[5]);
        const float rx = fmaxf(fmaxf(l01.x - cx, 0.f), cx - l2h0.y);
        const float ry = fmaxf(fmaxf(l01.y - cy, 0.f), cy - h12.x);
        const float rz = fmaxf(fmaxf(l2h0.x - cz, 0.f), cz - h12.y);
        st = (fast && d2_fma(rx, ry, rz) > r2 * band_hi) ? 0 : st;
      }
      verdict = st == 2 && d2_fma(cx - pr[0], cy - pr[1], cz - pr[2]) <= r2 * band_lo;
    }
    const unsigned hitm = __ballot_sync(0xffffffffu, verdict);
    const bool scan = (st == 2 || st == 3) && !verdict && (hitm & gm) == 0;
    uint2 set = make_uint2(0u, 0u);
    if (scan) set = __ldg(t.set + leaf);
    // the scan, load-balanced over the warp: entry e's set is split into
    // items of 64 points; in each step slot k (lanes 4k .. 4k+3, 16 points
    // per lane) takes item 8 step + k of the concatenated item list, so the
    // warp takes ceil(sum items / 8) steps instead of the longest set's
    const bool scan32 = scan && st == 2;
    const uint32_t m4e = scan32 ? ((set.y + 3u) & ~3u) : 0u;   // lanes 0-7: entry lane
    // rows to scan: with the distance-sorted copy, only those within
    // r + |c - o| of the set's origin (fl, rounded up: see sorted_limit)
    uint32_t lime = m4e;
    if (scan32 && t.sdata && m4e > 256u) {  // (short sets: scanning beats the search)
      const float4 o = __ldg(t.org + leaf);
      const float e = sqrtf(d2_fma(cx - o.x, cy - o.y, cz - o.z));
      // (|r|: a negative radius collides like its magnitude, d^2 <= r*r)
      const float cut = __fmul_ru(__fadd_ru(fabsf(r), e), 1.0f + 0x1p-18f);
      lime = sorted_limit(t.sdist + int64_t(set.x) * 4 / 3, m4e, cut);
    }
    const uint32_t items = (lime + 63u) >> 6;
    uint32_t incl = items;  // inclusive prefix over lanes 0-7
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t tv = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += tv;
    }
    uint32_t pre[kLE];  // inclusive prefix of every entry (uniform)
#pragma unroll
    for (int e = 0; e < kLE; ++e) pre[e] = __shfl_sync(0xffffffffu, incl, e);
    const uint32_t total = pre[kLE - 1];
    const float loB0 = r2 * band_lo, hiB0 = r2 * band_hi;
    bool hit_e = false, amb_e = false;  // lanes 0-7: their entry's result
    for (uint32_t s0 = 0; s0 < total; s0 += kLE) {
      const uint32_t item = s0 + slot;
      int e = 0;
#pragma unroll
      for (int k = 0; k < kLE - 1; ++k) e += item >= pre[k] ? 1 : 0;
      const uint32_t first = e ? pre[e - 1] : 0u;
      // entry e's data (shuffles are warp-wide; lanes past the end read entry 7)
      const float sx = __shfl_sync(0xffffffffu, cx, e);
      const float sy = __shfl_sync(0xffffffffu, cy, e);
      const float sz = __shfl_sync(0xffffffffu, cz, e);
      const float loB = __shfl_sync(0xffffffffu, loB0, e);
      const float hiB = __shfl_sync(0xffffffffu, hiB0, e);
      const uint32_t sset = __shfl_sync(0xffffffffu, set.x, e);
      const uint32_t m4 = __shfl_sync(0xffffffffu, m4e, e);    // SoA stride
      const uint32_t lim = __shfl_sync(0xffffffffu, lime, e);  // rows to scan
      const bool done = __shfl_sync(0xffffffffu, hit_e, e);  // entry already hit: skip
      const bool live = item < total && !done;
      const float* base = t.sdata ? t.sdata + int64_t(sset) * 4
                                  : reinterpret_cast<const float*>(t.data + sset);
      const uint32_t p0 = (item - first) * 64u;
      bool hit = false, amb = false;
      if (live) {
        // all 12 loads in flight: rows past the set are clamped to row 0 and
        // masked out of the result
        float4 px[4], py[4], pz[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t p = p0 + 16 * u + 4 * sl;
          const uint32_t pc = p < lim ? p : 0u;
          px[u] = __ldg(reinterpret_cast<const float4*>(base + pc));
          py[u] = __ldg(reinterpret_cast<const float4*>(base + m4 + pc));
          pz[u] = __ldg(reinterpret_cast<const float4*>(base + 2 * m4 + pc));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool in = p0 + 16 * u + 4 * sl < lim;
          const float xs[4] = {px[u].x, px[u].y, px[u].z, px[u].w},
                      ys[4] = {py[u].x, py[u].y, py[u].z, py[u].w},
                      zs[4] = {pz[u].x, pz[u].y, pz[u].z, pz[u].w};
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const float d2 = d2_fma(sx - xs[w], sy - ys[w], sz - zs[w]);
            hit |= in && d2 <= loB;
            amb |= in && d2 < hiB;
          }
        }
      }
      // fold the step's results into the owning entries (lanes 0-7)
      const unsigned hb = __ballot_sync(0xffffffffu, hit);
      const unsigned ab = __ballot_sync(0xffffffffu, amb);
#pragma unroll
      for (int k = 0; k < kLE; ++k) {
        const uint32_t ik = s0 + k;
        int ek = 0;
#pragma unroll
        for (int j = 0; j < kLE - 1; ++j) ek += ik >= pre[j] ? 1 : 0;
        if (ek == lane && ik < total) {
          hit_e |= ((hb >> (4 * k)) & 15u) != 0;
          amb_e |= ((ab >> (4 * k)) & 15u) != 0;
        }
      }
    }
    if (scan && st == 2) verdict = hit_e;
    // float64 re-scans (fp32 band hits; st == 3: the exact path only), one
    // entry at a time by the whole warp (a per-thread scan of a 600-point set
    // is a chain of dependent loads that outlasts the rest of the kernel)
    unsigned exact = __ballot_sync(0xffffffffu, scan && !verdict && (st == 3 || amb_e));
    while (exact) {
      const int src = __ffs(exact) - 1;
      exact &= exact - 1;
      const double c64[3] = {__shfl_sync(0xffffffffu, double(cx), src),
                             __shfl_sync(0xffffffffu, double(cy), src),
                             __shfl_sync(0xffffffffu, double(cz), src)};
      const double r64 = __shfl_sync(0xffffffffu, double(r), src);
      const uint2 sset = make_uint2(__shfl_sync(0xffffffffu, set.x, src),
                                    __shfl_sync(0xffffffffu, set.y, src));
      const uint32_t slim = __shfl_sync(0xffffffffu, lime, src);
      const bool sfast = __shfl_sync(0xffffffffu, st == 2, src);
      const uint32_t sm4 = (sset.y + 3u) & ~3u;
      // a fast sphere's rows beyond its cutoff are float64 misses: the sorted
      // copy's first slim rows hold every possible hit
      const bool h64 =
          (sfast && t.sdata)
              ? warp_scan_f64_rows(t.sdata + int64_t(sset.x) * 4, sm4, min(slim, sset.y),
                                   t.k, c64, __dmul_rn(r64, r64), lane)
              : warp_scan_f64(t, sset, c64, r64, lane);
      if (lane == src) verdict = h64;
    }
    // one OR per hit sphere (L = 1) or per group (first hitting lane)
    const unsigned vm = __ballot_sync(0xffffffffu, verdict);
    if (verdict && lane == __ffs(vm & gm) - 1) {
      const uint32_t b = L == 1 ? q : q / uint32_t(L);
      atomicOr(a.bits + (b >> 5), 1u << (b & 31));
    }
  }
}

}  // namespace

// ---------------------------------------------------------------- host

static int build_sorted(capt_tree* tree, cudaStream_t s) {
  if (tree->sdata) cudaFree(tree->sdata);
  if (tree->sdist) cudaFree(tree->sdist);
  tree->sdata = tree->sdist = nullptr;
  const DevTree t = view(tree);
  const int64_t nf = tree->h.data_f4 * 4;  // floats of the data section
  const int64_t items = nf / 3;
  if (items <= 0 || items >= (int64_t(1) << 31)) return CAPT_OK;  // (no sorted copy)
  uint32_t *keys = nullptr, *keys_o = nullptr, *vals = nullptr, *vals_o = nullptr;
  int *sb = nullptr, *se = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  CAPT_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, tb, keys, keys_o, vals, vals_o, int(items),
                                                int(t.n), sb, se, s));
  cudaError_t e = cudaSuccess;
  float *sdata = nullptr, *sdist = nullptr;
  e = cudaMalloc(&sdata, sizeof(float) * size_t(nf));
  if (e == cudaSuccess) e = cudaMalloc(&sdist, sizeof(float) * size_t(items));
  if (e == cudaSuccess) e = dmalloc(&keys, items, s);
  if (e == cudaSuccess) e = dmalloc(&keys_o, items, s);
  if (e == cudaSuccess) e = dmalloc(&vals, items, s);
  if (e == cudaSuccess) e = dmalloc(&vals_o, items, s);
  if (e == cudaSuccess) e = dmalloc(&sb, t.n, s);
  if (e == cudaSuccess) e = dmalloc(&se, t.n, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&tmp, tb + 16, s);
  if (e == cudaSuccess) {
    k_sort_keys<<<grid_for(t.n * 32, 256, 8), 256, 0, s>>>(t, keys, vals, sb, se);
    e = cub::DeviceSegmentedSort::SortPairs(tmp, tb, keys, keys_o, vals, vals_o, int(items),
                                            int(t.n), sb, se, s);
  }
  if (e == cudaSuccess) {
    k_sort_gather<<<grid_for(t.n * 32, 256, 8), 256, 0, s>>>(t, keys_o, vals_o, sdata, sdist);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(keys, s);
  cudaFreeAsync(keys_o, s);
  cudaFreeAsync(vals, s);
  cudaFreeAsync(vals_o, s);
  cudaFreeAsync(sb, s);
  cudaFreeAsync(se, s);
  cudaFreeAsync(tmp, s);
  if (e != cudaSuccess) {
    cudaFree(sdata);
    cudaFree(sdist);
    if (e == cudaErrorMemoryAllocation) {  // optional acceleration: run without it
      cudaGetLastError();
      return CAPT_OK;
    }
    return cuda_fail(e, "sorted set copy");
  }
  note_launches(3);
  tree->sdata = sdata;
  tree->sdist = sdist;
  return CAPT_OK;
}

int build_field(capt_tree* tree, cudaStream_t s) {
  if (tree->field) {
    cudaFree(tree->field);
    tree->field = nullptr;
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
  }
  g.nx = int(dims[0]);
  g.ny = int(dims[1]);
  g.nz = int(dims[2]);
  g.cells = dims[0] * dims[1] * dims[2];
  // stored bounds are capped at rcap >= r_max + h (> r_max + |c - x0| for a
  // centre inside its cell); buckets of m cells with m h >= rcap + 2h: a
  // point outside a centre's 27 neighbouring buckets is more than rcap away
  // even when its computed cell index is off by one
  g.rcap = float(rmax + h);
  g.m = int(std::ceil(double(g.rcap) / h)) + 2;
  // octant boxes: a centre assigned to a cell lies within h/2 + delta of its
  // x0 per axis (delta covers the rounding of the cell index and of x0);
  // half-edge hh = h/2 + delta rounded up; absolute slack for the rounded
  // gaps; bounds capped at rcap - sqrt(3) hh (points beyond the candidate
  // search are farther than that from every octant point)
  {
    double maxabs = 0.0;
    int64_t maxdim = std::max<int64_t>(dims[0], std::max<int64_t>(dims[1], dims[2]));
    for (int d = 0; d < 3; ++d)
      maxabs = std::max(maxabs, std::max(std::fabs(double(g.lo[d])),
                                         std::fabs(double(g.lo[d]) + dims[d] * h)));
    const double u = std::ldexp(1.0, -24);
    const double delta = h * std::ldexp(1.0, -12) + 8 * u * (double(maxdim) * h + maxabs);
    g.oct_half = std::nextafter(float(0.5 * h + delta), INFINITY);
    g.oct_abs = float(16 * u * (maxabs + double(g.rcap) + h));
    g.oct_cap = std::max(0.0f, float(double(g.rcap) - std::sqrt(3.0) * double(g.oct_half)) *
                                   (1.0f - 0x1p-20f));
  }
  BucketGrid b;
  b.nbx = (g.nx + g.m - 1) / g.m;
  b.nby = (g.ny + g.m - 1) / g.m;
  b.nbz = (g.nz + g.m - 1) / g.m;
  b.nb = int64_t(b.nbx) * b.nby * b.nbz;

  uint32_t *keys = nullptr, *keys_out = nullptr, *counts = nullptr, *bstart = nullptr;
  int *ids = nullptr, *ids_out = nullptr;
  float4* pts = nullptr;
  void* tmp = nullptr;
  size_t tb_sort = 0, tb_scan = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb_sort, keys, keys_out, ids, ids_out, int(n), 0, 32, s);
  cub::DeviceScan::ExclusiveSum(nullptr, tb_scan, counts, bstart, int(b.nb + 2), s);
  CAPT_CUDA(dmalloc(&keys, n, s));
  CAPT_CUDA(dmalloc(&keys_out, n, s));
  CAPT_CUDA(dmalloc(&ids, n, s));
  CAPT_CUDA(dmalloc(&ids_out, n, s));
  CAPT_CUDA(dmalloc(&counts, b.nb + 2, s));
  CAPT_CUDA(dmalloc(&bstart, b.nb + 2, s));
  CAPT_CUDA(dmalloc(&pts, n, s));
  CAPT_CUDA(cudaMallocAsync(&tmp, std::max(tb_sort, tb_scan) + 16, s));
  CAPT_CUDA(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * (b.nb + 2), s));
  k_bucket_keys<<<grid_for(n, 256, 8), 256, 0, s>>>(t.rep, n, g, b, keys, ids, counts);
  CAPT_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb_sort, keys, keys_out, ids, ids_out, int(n), 0,
                                            32, s));
  CAPT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb_scan, counts, bstart, int(b.nb + 2), s));
  uint32_t n_fin = 0;
  CAPT_CUDA(cudaMemcpyAsync(&n_fin, bstart + b.nb, 4, cudaMemcpyDeviceToHost, s));
  CAPT_CUDA(cudaStreamSynchronize(s));
  k_bucket_points<<<grid_for(n_fin, 256, 8), 256, 0, s>>>(t.rep, ids_out, n_fin, pts);
  float4* field = nullptr;
  cudaError_t e = cudaMalloc(&field, 2 * sizeof(float4) * size_t(g.cells));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(clearance field)");
  k_field_nn<<<int(b.nb), 256, 0, s>>>(g, b, bstart, pts, field);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(keys, s);
  cudaFreeAsync(keys_out, s);
  cudaFreeAsync(ids, s);
  cudaFreeAsync(ids_out, s);
  cudaFreeAsync(counts, s);
  cudaFreeAsync(bstart, s);
  cudaFreeAsync(pts, s);
  cudaFreeAsync(tmp, s);
  if (e != cudaSuccess) {
    cudaFree(field);
    return cuda_fail(e, "clearance field build");
  }
  note_launches(6);
  tree->field = field;
  tree->fg = g;
  return build_sorted(tree, s);
}

constexpr int64_t kFieldMinBatch = 8192;

bool field_eligible(const DevTree& t, int64_t n, uint32_t flags) {
  if (!t.field || t.k != 3 || (flags & (CAPT_INPUT_F64 | CAPT_STATS))) return false;
  if (n >= (int64_t(1) << 31) - (int64_t(1) << 24)) return false;
  // fp32 r^2 of every in-band radius must stay normal and finite
  if (!(t.r_min >= 0x1p-50) || !(t.r_max <= 0x1p50)) return false;
  if (flags & CAPT_MODE_FIELD) return true;  // (+ MODE_BINNED / MODE_DIRECT: the list path)
  // below a few thousand spheres the one-kernel warp path has less fixed cost
  // (two kernels, two memsets here: ~13 us at 1 K spheres vs ~8)
  if (n < kFieldMinBatch) return false;
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
static cudaError_t launch_pdl_f(void (*kernel)(KArgs...), int grid, int block, cudaStream_t s,
                                Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Stage timing (capt_stage_timing / capt_stage_times): CUDA events on the
// launching stream around K0 and the list stage of every field-pipeline call,
// read back and summed on request (no synchronisation inside the calls).
struct StageEvents {
  static constexpr int kMax = 2048;
  bool on = false;
  int n = 0;
  cudaEvent_t ev[kMax][3] = {};
  void record(int call, int k, cudaStream_t s) {
    if (!ev[call][k]) cudaEventCreate(&ev[call][k]);
    cudaEventRecord(ev[call][k], s);
  }
};
static StageEvents g_stage;

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
  a.flags = flags;
  a.bits = bits;
  a.first_bad = first_bad;
  float lo = float(t.r_min), hi = float(t.r_max);
  if (double(lo) < t.r_min) lo = nextafterf(lo, INFINITY);
  if (double(hi) > t.r_max) hi = nextafterf(hi, -INFINITY);
  a.rlo_f = lo;
  a.rhi_f = hi;
  CAPT_CUDA(dmalloc(&a.list_n, 8, s));
  CAPT_CUDA(dmalloc(&a.list, n, s));
  {
    const int64_t zw = L >= 8 ? n_words : 0;
    k_field_zero<<<grid_for(zw + 8, 256, 4), 256, 0, s>>>(a.list_n, bits, zw);
    CAPT_CUDA(cudaGetLastError());
    note_launches(1);
  }
  const int tcall = (g_stage.on && g_stage.n < StageEvents::kMax) ? g_stage.n++ : -1;
  if (tcall >= 0) g_stage.record(tcall, 0, s);
  const bool vec = (reinterpret_cast<uintptr_t>(centers) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(radii) & 15) == 0;
  const int grid = grid_for(((n + 127) / 128) * 32, CAPT_K0_BLOCK, 8 * 256 / CAPT_K0_BLOCK);
  // unmasked 16-B aligned batches: the TMA-fed kernel (specialised for single
  // spheres and 8-sphere groups, configs 0-4); everything else the register path
  static const bool use_tma = getenv("CAPT_K0_TMA") != nullptr;
  if (vec && !mask && use_tma && n >= kTileSpheres) {
    static bool attr = false;
    if (!attr) {
      for (auto f : {k_resolve_tma<1>, k_resolve_tma<8>, k_resolve_tma<0>})
        CAPT_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTmaSmem)));
      attr = true;
    }
    const int gt = grid_for(((n + kTileSpheres - 1) / kTileSpheres) * 256, 256, 4);
    if (L == 1) k_resolve_tma<1><<<gt, 256, kTmaSmem, s>>>(a);
    else if (L == 8) k_resolve_tma<8><<<gt, 256, kTmaSmem, s>>>(a);
    else k_resolve_tma<0><<<gt, 256, kTmaSmem, s>>>(a);
  }
  else if (vec && !mask && L == 1) CAPT_CUDA(launch_pdl_f(k_resolve<true, false, 1>, grid, CAPT_K0_BLOCK, s, a));
  else if (vec && !mask && L == 8) CAPT_CUDA(launch_pdl_f(k_resolve<true, false, 8>, grid, CAPT_K0_BLOCK, s, a));
  else if (mask) CAPT_CUDA(launch_pdl_f(k_resolve<false, true, 0>, grid, CAPT_K0_BLOCK, s, a));
  else CAPT_CUDA(launch_pdl_f(k_resolve<false, false, 0>, grid, CAPT_K0_BLOCK, s, a));
  CAPT_CUDA(cudaGetLastError());
  note_launches(1);
  if (tcall >= 0) g_stage.record(tcall, 1, s);
  // the list: one warp-cooperative kernel, or -- for large batches over large
  // affordance sets, where the tensor-core binned scan amortises each set
  // over up to 128 spheres -- the leaf-binned pipeline in list mode
  static const int force = [] {
    const char* e = getenv("CAPT_FIELD_LIST");
    return !e ? 0 : (e[0] == 'b' ? 2 : 1);
  }();
  bool binned = force ? force == 2 : (n >= (int64_t(1) << 22) && t.total >= 512 * t.n);
  if (flags & CAPT_MODE_FIELD) {
    if (flags & CAPT_MODE_BINNED) binned = true;
    if (flags & CAPT_MODE_DIRECT) binned = false;
  }
  flags &= ~uint32_t(CAPT_MODE_BINNED | CAPT_MODE_DIRECT | CAPT_MODE_FIELD);
  int rc = CAPT_OK;
  FieldArgs a2 = a;  // the filtered list (binned path)
  if (binned) {
    // (K1 in list mode applies the octant certificate itself)
    static const bool filt = getenv("CAPT_OCT_FILTER") != nullptr;
    if (filt) {
      CAPT_CUDA(dmalloc(&a2.list_n, 1, s));
      CAPT_CUDA(dmalloc(&a2.list, n, s));
      CAPT_CUDA(cudaMemsetAsync(a2.list_n, 0, 4, s));
      k_list_octant<<<grid_for(int64_t(n) / 64 + 1, 256, 2), 256, 0, s>>>(a, a2.list, a2.list_n);
      CAPT_CUDA(cudaGetLastError());
      note_launches(1);
    }
    rc = launch_binned(t, centers, radii, n, L, nullptr, flags, bits, n_words, first_bad, s,
                       a2.list, a2.list_n);
  } else {
    // grid for the worst case (every sphere listed): 8 entries per warp
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid_for(int64_t(n) * 4 + 32, 256, 8));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CAPT_CUDA(cudaLaunchKernelEx(&cfg, k_resolve_list<true>, a));
    CAPT_CUDA(cudaGetLastError());
    note_launches(1);
  }
  if (tcall >= 0) g_stage.record(tcall, 2, s);
  static const bool debug = getenv("CAPT_DEBUG") != nullptr;
  if (debug) {
    uint32_t nl = 0, nl2 = 0;
    CAPT_CUDA(cudaMemcpyAsync(&nl, a.list_n, 4, cudaMemcpyDeviceToHost, s));
    if (a2.list != a.list) CAPT_CUDA(cudaMemcpyAsync(&nl2, a2.list_n, 4, cudaMemcpyDeviceToHost, s));
    CAPT_CUDA(cudaStreamSynchronize(s));
    fprintf(stderr, "[capt field] n=%lld L=%d undecided=%u (%.3f%%) after octants=%u (%.3f%%) list=%s\n",
            (long long)n, L, nl, 100.0 * nl / double(n ? n : 1), nl2, 100.0 * nl2 / double(n ? n : 1),
            binned ? "binned" : "thread");
  }
  cudaFreeAsync(a.list, s);
  cudaFreeAsync(a.list_n, s);
  if (a2.list != a.list) {
    cudaFreeAsync(a2.list, s);
    cudaFreeAsync(a2.list_n, s);
  }
  return rc;
}

}  // namespace capt

using namespace capt;

extern "C" int capt_tree_field(const capt_tree* tree, capt_field_info* info, float* cells) {
  if (!tree || !info) return fail(CAPT_EINVAL, "NULL argument");
  if (!tree->field) return fail(CAPT_EINVAL, "tree has no clearance field (k < 3)");
  const FieldGeom& g = tree->fg;
  memset(info, 0, sizeof(*info));
  info->nx = g.nx;
  info->ny = g.ny;
  info->nz = g.nz;
  info->n_cells = g.cells;
  info->h = g.h;
  info->rcap = g.rcap;
  info->oct_half = g.oct_half;
  for (int d = 0; d < 3; ++d) {
    info->lo[d] = g.lo[d];
    info->c0[d] = g.c0[d];
    info->box_lo[d] = g.blo[d];
    info->box_hi[d] = g.bhi[d];
  }
  if (cells) {  // device: all witness records, then all octant records; out: interleaved
    CAPT_CUDA(cudaSetDevice(tree->device));
    std::vector<float4> tmp(2 * size_t(g.cells));
    CAPT_CUDA(cudaMemcpy(tmp.data(), tree->field, 2 * sizeof(float4) * size_t(g.cells),
                         cudaMemcpyDeviceToHost));
    float4* out = reinterpret_cast<float4*>(cells);
    for (int64_t i = 0; i < g.cells; ++i) {
      out[2 * i] = tmp[i];
      out[2 * i + 1] = tmp[g.cells + i];
    }
  }
  return CAPT_OK;
}

extern "C" int capt_stage_timing(int enable) {
  g_stage.on = enable != 0;
  g_stage.n = 0;
  return CAPT_OK;
}

extern "C" int capt_stage_times(double* ms, int64_t* calls) {
  if (!ms || !calls) return fail(CAPT_EINVAL, "NULL argument");
  ms[0] = ms[1] = ms[2] = 0.0;
  for (int i = 0; i < g_stage.n; ++i) {
    CAPT_CUDA(cudaEventSynchronize(g_stage.ev[i][2]));
    float a = 0.f, b = 0.f;
    CAPT_CUDA(cudaEventElapsedTime(&a, g_stage.ev[i][0], g_stage.ev[i][1]));
    CAPT_CUDA(cudaEventElapsedTime(&b, g_stage.ev[i][1], g_stage.ev[i][2]));
    ms[0] += a;
    ms[1] += b;
    ms[2] += a + b;
  }
  *calls = g_stage.n;
  g_stage.n = 0;
  return CAPT_OK;
}
