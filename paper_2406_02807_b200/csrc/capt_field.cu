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

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "capt_binned.cuh"
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
__device__ __forceinline__ float centre_of(int i, float h, float lo) {
  return __fmaf_rn(__fadd_rn(__int2float_rn(i), 0.5f), h, lo);
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
  for (int pass = 0; pass < ncells; pass += 256 * kCellsPerThread) {
    float px[kCellsPerThread], py[kCellsPerThread], pz[kCellsPerThread], best[kCellsPerThread];
    int bi[kCellsPerThread];
#pragma unroll
    for (int k = 0; k < kCellsPerThread; ++k) {
      const int j = pass + k * 256 + threadIdx.x;
      const int lx = j % cx, ly = (j / cx) % cy, lz = j / (cx * cy);
      px[k] = centre_of(x0 + lx, g.h, g.lo[0]);
      py[k] = centre_of(y0 + ly, g.h, g.lo[1]);
      pz[k] = centre_of(z0 + lz, g.h, g.lo[2]);
      best[k] = INF;
      bi[k] = -1;
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
                const float d2 = d2_fma(px[k] - p.x, py[k] - p.y, pz[k] - p.z);
                if (d2 < best[k]) {
                  best[k] = d2;
                  bi[k] = int(c0) + i;
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
      const int b = bi[k] >= 0 ? bi[k] : 0;
      const float nn = fminf(g.rcap, __fmul_rn(sqrtf(best[k]), kNNShrink));
      if (j < ncells) {
        const int lx = j % cx, ly = (j / cx) % cy, lz = j / (cx * cy);
        const int64_t cell = (int64_t(z0 + lz) * g.ny + (y0 + ly)) * g.nx + (x0 + lx);
        const float4 w = bi[k] >= 0 ? pts[b] : make_float4(INF, INF, INF, 0.f);
        field[cell] = make_float4(w.x, w.y, w.z, nn);
      }
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

// K0: per sphere (V in flight per thread, inputs prefetched one iteration
// ahead with evict-first loads):
//   status 1 = hit, 0 = free / masked, 2 = the tree path decides.
// In-band fp32 spheres with a finite centre are tested against
//   (a) the cloud box: fp32 gap^2 > r^2 (1 + TAU) -> free (every point lies
//       in the box; fp32 gap^2 has relative error < 5u);
//   (b) the cell's witness: fp32 |c - w|^2 <= r^2 (1 - TAU) -> hit;
//   (c) the cell's bound: nn > fl(fl(r + e) (1 + 2^-20)), e = sqrtf(fp32
//       |c - x0|^2) -> free.  e overestimates nothing by more than 3.6u
//       relative, the sum and product lose <= 2u, so nn > (r + |c - x0|)
//       (1 + 10u) and dist(c, cloud) >= nn - |c - x0| > r (1 + 10u): every
//       float64 d^2 of the reference is > r*r.
// Lane groups (L | 32) resolve on any definite hit (query.py:152-160); the
// verdict bits are written directly (L = 1: one word per warp; L > 1: OR
// into cleared words); unresolved spheres of unresolved groups are appended
// to the list with one atomic per warp.
template <int V>
__global__ void __launch_bounds__(256) k_resolve(FieldArgs a) {
  const FieldGeom g = a.t.fg;
  const float4* __restrict__ field = a.t.field;
  const float* __restrict__ cf = a.c;
  const float* __restrict__ rf = a.r;
  const bool check = a.flags & CAPT_CHECK_RADII;
  const int n = a.n;
  const int n_pad = (n + 31) & ~31;
  const int lane = threadIdx.x & 31;
  const int L = a.L;
  const unsigned seg = L >= 32 ? 0xffffffffu : ((1u << L) - 1u) << ((lane / L) * L);
  const float band_lo = 1.0f - kTau, band_hi = 1.0f + kTau;
  const int stride = gridDim.x * blockDim.x * V;
  float nx[V], ny[V], nz[V], nr[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int q = blockIdx.x * blockDim.x * V + v * blockDim.x + threadIdx.x;
    const int qq = q < n ? q : 0;
    nx[v] = __ldcs(cf + 3 * qq);
    ny[v] = __ldcs(cf + 3 * qq + 1);
    nz[v] = __ldcs(cf + 3 * qq + 2);
    nr[v] = __ldcs(rf + qq);
  }
  for (int base = blockIdx.x * blockDim.x * V; base < n_pad; base += stride) {
    float cx[V], cy[V], cz[V], r[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      cx[v] = nx[v];
      cy[v] = ny[v];
      cz[v] = nz[v];
      r[v] = nr[v];
      const int qn = base + stride + v * blockDim.x + threadIdx.x;
      const int qq = qn < n ? qn : 0;
      nx[v] = __ldcs(cf + 3 * qq);
      ny[v] = __ldcs(cf + 3 * qq + 1);
      nz[v] = __ldcs(cf + 3 * qq + 2);
      nr[v] = __ldcs(rf + qq);
    }
    int st[V];
    bool bad_any = false;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int q = base + v * blockDim.x + threadIdx.x;
      bool valid = q < n;
      if (a.mask && valid) valid = a.mask[q] != 0;
      const bool inband = r[v] >= a.rlo_f && r[v] <= a.rhi_f;  // false for NaN
      // the reference's band check (query.py:194-197) does not flag NaN
      const bool bad = check && valid && (r[v] < a.rlo_f || r[v] > a.rhi_f);
      bad_any |= bad;
      const float r2 = r[v] * r[v];
      const bool cfin = isfinite(cx[v]) && isfinite(cy[v]) && isfinite(cz[v]);
      const bool elig = valid && inband && cfin && r2 >= kR2Min && r2 <= kR2Max;
      // (a) the cloud box
      const float gx = fmaxf(fmaxf(g.blo[0] - cx[v], 0.f), cx[v] - g.bhi[0]);
      const float gy = fmaxf(fmaxf(g.blo[1] - cy[v], 0.f), cy[v] - g.bhi[1]);
      const float gz = fmaxf(fmaxf(g.blo[2] - cz[v], 0.f), cz[v] - g.bhi[2]);
      const bool boxfree = d2_fma(gx, gy, gz) > r2 * band_hi;
      int s = (!valid || bad) ? 0 : 2;
      if (elig && !boxfree) {
        const int ix = cell_of(cx[v], g.lo[0], g.inv_h, g.nx);
        const int iy = cell_of(cy[v], g.lo[1], g.inv_h, g.ny);
        const int iz = cell_of(cz[v], g.lo[2], g.inv_h, g.nz);
        const float4 rec = __ldg(field + (iz * g.ny + iy) * g.nx + ix);
        // (b) the witness
        const bool hit = d2_fma(cx[v] - rec.x, cy[v] - rec.y, cz[v] - rec.z) <= r2 * band_lo;
        // (c) the Lipschitz bound from the cell centre
        const float ex = cx[v] - centre_of(ix, g.h, g.lo[0]);
        const float ey = cy[v] - centre_of(iy, g.h, g.lo[1]);
        const float ez = cz[v] - centre_of(iz, g.h, g.lo[2]);
        const float e = sqrtf(d2_fma(ex, ey, ez));
        const bool free = rec.w > __fmul_rn(__fadd_rn(r[v], e), kFreeMargin);
        s = hit ? 1 : (free ? 0 : 2);
      } else if (elig) {
        s = 0;
      }
      st[v] = s;
    }
    if (check && __any_sync(0xffffffffu, bad_any)) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int q = base + v * blockDim.x + threadIdx.x;
        bool valid = q < n;
        if (a.mask && valid) valid = a.mask[q] != 0;
        if (valid && (r[v] < a.rlo_f || r[v] > a.rhi_f))
          atomicMin(a.first_bad, static_cast<unsigned long long>(q));
      }
    }
    // verdict bits and lane-group resolution
    unsigned act[V], tot = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const unsigned hm = __ballot_sync(0xffffffffu, st[v] == 1);
      const int qw = base + v * blockDim.x + (threadIdx.x & ~31);  // first sphere of the warp
      if (L == 1) {
        if (lane == 0 && qw < n) a.bits[qw >> 5] = hm;
      } else {
        unsigned gb = 0;
        const unsigned gmask = L >= 32 ? 0xffffffffu : (1u << L) - 1u;
        for (int j = 0; j < 32 / L; ++j)
          if ((hm >> (j * L)) & gmask) gb |= 1u << j;
        const int g0 = qw / L;
        if (lane == 0 && gb) atomicOr(a.bits + (g0 >> 5), gb << (g0 & 31));
      }
      const bool resolved = (hm & seg) != 0;
      act[v] = __ballot_sync(0xffffffffu, st[v] == 2 && !resolved);
      tot += __popc(act[v]);
    }
    if (tot) {
      unsigned j = 0;
      if (lane == 0) j = atomicAdd(a.list_n, tot);
      j = __shfl_sync(0xffffffffu, j, 0);
      const unsigned lt = (1u << lane) - 1u;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if ((act[v] >> lane) & 1u)
          a.list[j + __popc(act[v] & lt)] = uint32_t(base + v * blockDim.x + threadIdx.x);
        j += __popc(act[v]);
      }
    }
  }
}

// The tree path over the list (the reference's semantics for every sphere it
// holds): per thread descent (top levels from shared memory), the leaf's
// probe record (conservative AABB reject, representative probe), then each
// warp scans the sets of its unresolved spheres one after the other,
// cooperatively (fp32 with the float64 re-scan of the band).  A list entry's
// lane group is recovered with __match_any_sync on q / L (K0 appends a
// group's spheres contiguously); a hit resolves the group's other entries.
constexpr int kListSmemLevels = 11;
constexpr int kListSmem = (1 << kListSmemLevels) - 1;

__global__ void __launch_bounds__(256) k_resolve_list(FieldArgs a) {
  __shared__ float sT[kListSmem];
  const DevTree& t = a.t;
  const int n_smem = int(t.n - 1 < kListSmem ? t.n - 1 : kListSmem);
  for (int i = threadIdx.x; i < n_smem; i += blockDim.x) sT[i] = t.T[i];
  __syncthreads();
  const uint32_t n_list = *a.list_n;
  const int lane = threadIdx.x & 31;
  const int L = a.L;
  const bool prefilter = a.flags & CAPT_PREFILTER;
  const float band_lo = 1.0f - kTau, band_hi = 1.0f + kTau;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t j0 = warp * 32; j0 < n_list; j0 += nwarps * 32) {
    const uint32_t j = j0 + lane;
    const bool active = j < n_list;
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
    // descent (tree.py:266-273)
    int i = 0, s = 0;
    for (; s < t.depth; ++s) {
      const int ax = s % 3;
      const float cv = ax == 0 ? cx : (ax == 1 ? cy : cz);
      const float tv = i < n_smem ? sT[i] : __ldg(t.T + i);
      i = 2 * i + 1 + (cv > tv ? 1 : 0);
    }
    const int leaf = i - int(t.n - 1);
    // classification (as k_bin_count3 / k_query_hybrid)
    const float r2 = r * r;
    const bool cfin = isfinite(cx) && isfinite(cy) && isfinite(cz);
    const bool fast = cfin && r2 >= kR2Min && r2 <= kR2Max;
    int st = fast ? 2 : ((!cfin && isfinite(r)) ? 0 : 3);
    st = active ? st : 0;
    float pr[8];
    ld_v8(t.probe + 8 * leaf, pr);
    if (prefilter) {
      const float2 l01 = h2f2(pr[3]), l2h0 = h2f2(pr[4]), h12 = h2f2(pr[5]);
      const float rx = fmaxf(fmaxf(l01.x - cx, 0.f), cx - l2h0.y);
      const float ry = fmaxf(fmaxf(l01.y - cy, 0.f), cy - h12.x);
      const float rz = fmaxf(fmaxf(l2h0.x - cz, 0.f), cz - h12.y);
      st = (fast && d2_fma(rx, ry, rz) > r2 * band_hi) ? 0 : st;
    }
    bool verdict = st == 2 && d2_fma(cx - pr[0], cy - pr[1], cz - pr[2]) <= r2 * band_lo;
    const unsigned hitm = __ballot_sync(0xffffffffu, verdict);
    unsigned todo = __ballot_sync(0xffffffffu, (st == 2 || st == 3) && !verdict);
    todo &= ~__ballot_sync(0xffffffffu, (hitm & gm) != 0);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const float sx = __shfl_sync(0xffffffffu, cx, src);
      const float sy = __shfl_sync(0xffffffffu, cy, src);
      const float sz = __shfl_sync(0xffffffffu, cz, src);
      const float sr = __shfl_sync(0xffffffffu, r, src);
      const int sst = __shfl_sync(0xffffffffu, st, src);
      const int sleaf = __shfl_sync(0xffffffffu, leaf, src);
      const unsigned sgm = __shfl_sync(0xffffffffu, gm, src);
      const uint2 set = __ldg(t.set + sleaf);
      int v = 2;
      if (sst == 2) {
        const float sr2 = sr * sr;
        v = warp_scan_f32(t, set, sx, sy, sz, sr2 * band_lo, sr2 * band_hi, lane);
      }
      bool hit = v == 1;
      if (v == 2) {
        const double c64[3] = {sx, sy, sz};
        hit = warp_scan_f64(t, set, c64, double(sr), lane);
      }
      if (hit) {
        if (lane == src) verdict = true;
        todo &= ~sgm;
      }
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
  for (int d = 0; d < 3; ++d) g.lo[d] = float(double(g.blo[d]) - (rmax + h));
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
  cudaError_t e = cudaMalloc(&field, sizeof(float4) * size_t(g.cells));
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
  return CAPT_OK;
}

bool field_eligible(const DevTree& t, int64_t n, uint32_t flags) {
  if (!t.field || t.k != 3 || (flags & (CAPT_INPUT_F64 | CAPT_STATS))) return false;
  if (n >= (int64_t(1) << 31) - (int64_t(1) << 24)) return false;
  if (flags & CAPT_MODE_FIELD) return true;  // (+ MODE_BINNED / MODE_DIRECT: the list path)
  return !(flags & (CAPT_MODE_DIRECT | CAPT_MODE_BINNED | CAPT_MODE_THREAD | CAPT_MODE_WARP));
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
  a.flags = flags;
  a.bits = bits;
  a.first_bad = first_bad;
  float lo = float(t.r_min), hi = float(t.r_max);
  if (double(lo) < t.r_min) lo = nextafterf(lo, INFINITY);
  if (double(hi) > t.r_max) hi = nextafterf(hi, -INFINITY);
  a.rlo_f = lo;
  a.rhi_f = hi;
  CAPT_CUDA(dmalloc(&a.list_n, 1, s));
  CAPT_CUDA(dmalloc(&a.list, n, s));
  CAPT_CUDA(cudaMemsetAsync(a.list_n, 0, 4, s));
  if (L > 1) CAPT_CUDA(cudaMemsetAsync(bits, 0, 4 * (n_words ? n_words : 1), s));
  constexpr int V = 4;
  k_resolve<V><<<grid_for((n + V - 1) / V, 256, 8), 256, 0, s>>>(a);
  CAPT_CUDA(cudaGetLastError());
  note_launches(1);
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
  if (binned) {
    rc = launch_binned(t, centers, radii, n, L, nullptr, flags, bits, n_words, first_bad, s,
                       a.list, a.list_n);
  } else {
    k_resolve_list<<<grid_for(int64_t(1) << 30, 256, 4), 256, 0, s>>>(a);
    CAPT_CUDA(cudaGetLastError());
    note_launches(1);
  }
  cudaFreeAsync(a.list, s);
  cudaFreeAsync(a.list_n, s);
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
  for (int d = 0; d < 3; ++d) {
    info->lo[d] = g.lo[d];
    info->box_lo[d] = g.blo[d];
    info->box_hi[d] = g.bhi[d];
  }
  if (cells) {
    CAPT_CUDA(cudaSetDevice(tree->device));
    CAPT_CUDA(cudaMemcpy(cells, tree->field, sizeof(float4) * size_t(g.cells),
                         cudaMemcpyDeviceToHost));
  }
  return CAPT_OK;
}
