// Device CAPT construction: construct(cloud, BuildParams) (tree.py:139-241).
//
// The reference recursion (Alg. 1) is restated as
//   1. pad to n = 2^depth leaves with +inf points (tree.py:150-154);
//   2. presort the point indices once per axis by (coordinate, index) with a
//      stable radix sort, then per level: the split value of every node is
//      the rank-(m/2-1) element of its axis list (np.argpartition,
//      tree.py:199-202; ties broken by original index) and every other axis
//      list is stably partitioned (flag scan + scatter) so each node's range
//      stays sorted -- no re-sorting;
//   3. every leaf's cell is replayed from T (conftest.py:11-31 pattern);
//   4. every leaf's affordance set is computed independently as
//        {rep} U {finite p != rep : dist^2_fp64(p, cell) <= r_max^2}
//      (padding leaf: {inf-row} U {...}; r_min shortcut: {rep} alone,
//      tree.py:164-188).  This equals the recursive definition because the
//      float64 point-box distance is monotone under cell inclusion, so a point
//      afforded by the leaf cell survives every ancestor's filter
//      (tree.py:209-218).  Candidates come from a uniform grid of point
//      buckets (edge >= r_max / 2): one warp per leaf scans the buckets its
//      cell grown by r_max overlaps, then the exact float64 test of
//      tree.py:209-213 decides membership;
//   5. count pass -> exclusive scan -> fill pass into the padded slab layout.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>

#include <cuda_fp16.h>

#include "capt_internal.cuh"

#ifndef CAPT_BUCKET_SCALE
#define CAPT_BUCKET_SCALE 0.5  // point-bucket edge / r_max (build; 1.0: 15% slower on configs 1 and 3)
#endif

namespace capt {

__device__ __forceinline__ uint32_t f32_key(float f) {
  if (f == 0.0f) f = 0.0f;  // -0.0 and +0.0 compare equal: same key
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void k_init(const float* __restrict__ pts, int64_t n0, int64_t n, int k,
                       float* __restrict__ X, uint32_t* __restrict__ keys, int32_t* __restrict__ idx) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    for (int d = 0; d < k; ++d) {
      const float v = i < n0 ? pts[i * k + d] : __int_as_float(0x7f800000);
      X[d * n + i] = v;
      keys[d * n + i] = f32_key(v);
    }
    idx[i] = int32_t(i);
  }
}

// One thread per node of the level: split value + tie detection.
__global__ void k_split(int64_t n_seg, int64_t m, int a, int64_t n, const float* __restrict__ X,
                        const int32_t* __restrict__ Pa, float* __restrict__ T,
                        unsigned long long* __restrict__ ties) {
  for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < n_seg;
       s += int64_t(gridDim.x) * blockDim.x) {
    const int64_t half = m / 2;
    const float t = X[a * n + Pa[s * m + half - 1]];
    const float t2 = X[a * n + Pa[s * m + half]];
    T[n_seg - 1 + s] = t;
    if (t == t2 && isfinite(t)) atomicAdd(ties, 1ull);
  }
}

__global__ void k_flags(int64_t n, int64_t m, const int32_t* __restrict__ Pa,
                        uint8_t* __restrict__ left) {
  for (int64_t pos = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; pos < n;
       pos += int64_t(gridDim.x) * blockDim.x)
    left[Pa[pos]] = (pos % m) < (m / 2);
}

__global__ void k_gather_flags(int64_t n, const int32_t* __restrict__ Pd,
                               const uint8_t* __restrict__ left, int32_t* __restrict__ f) {
  for (int64_t pos = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; pos < n;
       pos += int64_t(gridDim.x) * blockDim.x)
    f[pos] = left[Pd[pos]];
}

__global__ void k_partition(int64_t n, int64_t m, const int32_t* __restrict__ Pd,
                            const int32_t* __restrict__ f, const int32_t* __restrict__ sc,
                            int32_t* __restrict__ out) {
  for (int64_t pos = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; pos < n;
       pos += int64_t(gridDim.x) * blockDim.x) {
    const int64_t base = pos - pos % m;
    const int64_t lb = int64_t(sc[pos]) - int64_t(sc[base]);
    const int64_t dst = f[pos] ? base + lb : base + m / 2 + (pos - base - lb);
    out[dst] = Pd[pos];
  }
}

struct Cell {
  float lo[3], hi[3];
};

// Replay the split walls from the root to leaf j (conftest.py:11-31).
__device__ __forceinline__ Cell leaf_cell(const float* __restrict__ T, int64_t n, int depth, int k,
                                          int64_t j) {
  Cell c;
  for (int d = 0; d < 3; ++d) {
    c.lo[d] = -INFINITY;
    c.hi[d] = INFINITY;
  }
  int64_t node = 0;
  for (int L = 0; L < depth; ++L) {
    const int a = L % k;
    const bool right = (j >> (depth - 1 - L)) & 1;
    const float t = T[node];
    if (right) c.lo[a] = t;
    else c.hi[a] = t;
    node = 2 * node + 1 + (right ? 1 : 0);
  }
  return c;
}

// float64 squared distance of finite p to the cell, numpy order (geom.py:130-134)
__device__ __forceinline__ double dist_cell64(int k, const double* p, const Cell& c) {
  double s = 0.0;
  for (int d = 0; d < k; ++d) {
    double r = fmax(__dsub_rn(double(c.lo[d]), p[d]), 0.0);
    r = fmax(r, __dsub_rn(p[d], double(c.hi[d])));
    const double sq = __dmul_rn(r, r);
    s = (d == 0) ? sq : __dadd_rn(s, sq);
  }
  return s;
}

struct BuildView {
  int k, depth;
  int64_t n, n0;
  const float* X;      // k * n, SoA
  const int32_t* rep;  // n (leaf -> point index)
  const float* T;
  double r_min_sq, r_max_sq;
  float r2_hi;         // fp32 r_max^2 with an upward margin (clear-miss prefilter)
  float r2_in;         // fp32 r_max^2 with a downward margin (clear members)
  int shortcut;
};

// shortcut test (tree.py:176-181): sum max(|rep-lo|, |rep-hi|)^2 <= r_min^2
__device__ __forceinline__ bool shortcut_fires(const BuildView& v, const Cell& c, int32_t p) {
  double s = 0.0;
  for (int d = 0; d < v.k; ++d) {
    const double x = double(v.X[d * v.n + p]);
    const double a = fabs(__dsub_rn(x, double(c.lo[d])));
    const double b = fabs(__dsub_rn(x, double(c.hi[d])));
    const double m = a >= b ? a : b;
    const double sq = __dmul_rn(m, m);
    s = (d == 0) ? sq : __dadd_rn(s, sq);
  }
  return s <= v.r_min_sq;
}

// ---------------------------------------------------------------------------
// Bucketed affordance sets.  The finite points are sorted into a uniform grid
// of buckets of edge b (x fastest); a leaf's candidates are the points of the
// buckets its cell grown by r' = r_max (1 + 2^-20) overlaps, clamped to the
// grid.  bucket(x) = floor((x - lo) / b) is monotone in x, and a point with
// float64 dist^2(p, cell) <= r_max^2 lies within r' of the cell on every
// axis, so it is among the candidates; the exact test (tree.py:209-213)
// decides.  One warp per leaf: the x-buckets of one (y, z) row are one
// contiguous range of the sorted points, scanned 32 points at a time (an fp32
// box distance with a relative margin rejects the clear misses first).
// ---------------------------------------------------------------------------
struct Buckets {
  double lo[3], inv_b;
  int dims[3];
  const uint32_t* start;  // nb + 1
  const float4* pts;      // sorted points {x, y, z, index bits}
};

__device__ __forceinline__ int bucket_of(const Buckets& B, int d, double x) {
  double t = floor(__dmul_rn(__dsub_rn(x, B.lo[d]), B.inv_b));
  if (!(t >= 0.0)) t = 0.0;  // (also -inf)
  return t >= double(B.dims[d] - 1) ? B.dims[d] - 1 : int(t);
}

__global__ void k_bucket_key(int k, int64_t n0, Buckets B, const float* __restrict__ X, int64_t n,
                             uint32_t* __restrict__ key, int32_t* __restrict__ id,
                             uint32_t* __restrict__ count) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n0;
       i += int64_t(gridDim.x) * blockDim.x) {
    int c[3] = {0, 0, 0};
    for (int d = 0; d < k; ++d) c[d] = bucket_of(B, d, double(X[d * n + i]));
    const uint32_t kk = (uint32_t(c[2]) * uint32_t(B.dims[1]) + uint32_t(c[1])) * uint32_t(B.dims[0]) +
                        uint32_t(c[0]);
    key[i] = kk;
    id[i] = int32_t(i);
    atomicAdd(count + kk, 1u);
  }
}

__global__ void k_bucket_gather(int k, int64_t n0, const float* __restrict__ X, int64_t n,
                                const int32_t* __restrict__ id, float4* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n0;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t p = id[i];
    float v[3] = {0.f, 0.f, 0.f};
    for (int d = 0; d < k; ++d) v[d] = X[d * n + p];
    out[i] = make_float4(v[0], v[1], v[2], __int_as_float(p));
  }
}

// fp32 lower bound s of the squared box distance: a relative margin of 2^-20
// on every gap covers the roundings, so s <= d^2 <= s (1 + 2^-18) for the
// float64 d^2 of dist_cell64.  s > r2_hi: a clear miss; s <= r2_in = fl(r_max^2)
// (1 - 2^-16): a clear member (d^2 <= s (1 + 2^-18) < r_max^2); only the
// band between them needs the exact float64 expression.
__device__ __forceinline__ float cell_lb32(int k, const float4 q, const Cell& c) {
  const float v[3] = {q.x, q.y, q.z};
  float s = 0.f;
  for (int d = 0; d < k; ++d) {
    float g = fmaxf(fmaxf(c.lo[d] - v[d], 0.f), v[d] - c.hi[d]);
    g *= (1.0f - 0x1p-20f);
    s = fmaf(g, g, s);
  }
  return s;
}

// Candidates of leaf j's set (excluding its representative), in a fixed
// order (bucket rows, then sorted point order): visit(lane_hit, point).
template <class F>
__device__ __forceinline__ void warp_afforded(const BuildView& v, const Buckets& B, const Cell& c,
                                              int32_t self, int lane, F&& visit) {
  const double rp = v.r_max_sq > 0.0 ? sqrt(v.r_max_sq) * (1.0 + 0x1p-20) : 0.0;
  int b0[3] = {0, 0, 0}, b1[3] = {0, 0, 0};
  for (int d = 0; d < v.k; ++d) {
    b0[d] = bucket_of(B, d, __dsub_rn(double(c.lo[d]), rp));
    b1[d] = bucket_of(B, d, __dadd_rn(double(c.hi[d]), rp));
  }
  // the (y, z) bucket rows, 32 at a time: lane l reads row l's point range,
  // a warp scan flattens the ranges, and the warp tests 32 candidates per
  // step wherever they lie (a candidate's row by a binary search over the
  // lanes' inclusive offsets) -- rows of a few points keep the lanes busy;
  // the order (rows, then sorted points) is fixed
  const int ny_rows = b1[1] - b0[1] + 1, rows = ny_rows * (b1[2] - b0[2] + 1);
  for (int r0 = 0; r0 < rows; r0 += 32) {
    uint32_t i0 = 0, len = 0;
    if (r0 + lane < rows) {
      const int by = b0[1] + (r0 + lane) % ny_rows, bz = b0[2] + (r0 + lane) / ny_rows;
      const uint32_t row = (uint32_t(bz) * uint32_t(B.dims[1]) + uint32_t(by)) * uint32_t(B.dims[0]);
      i0 = __ldg(B.start + row + b0[0]);
      len = __ldg(B.start + row + b1[0] + 1) - i0;
    }
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    for (uint32_t k0 = 0; k0 < total; k0 += 32) {
      const uint32_t k = k0 + lane;
      int lo = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const uint32_t w = __shfl_sync(0xffffffffu, incl, lo + step - 1);
        if (w <= k) lo += step;
      }
      const uint32_t base = __shfl_sync(0xffffffffu, i0, lo);
      const uint32_t excl = __shfl_sync(0xffffffffu, incl - len, lo);
      bool hit = false;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k < total) {
        q = __ldg(B.pts + base + (k - excl));
        const float s32 = cell_lb32(v.k, q, c);
        if (__float_as_int(q.w) != self && s32 <= v.r2_hi) {
          if (s32 <= v.r2_in) {
            hit = true;
          } else {
            const double pq[3] = {double(q.x), double(q.y), double(q.z)};
            hit = dist_cell64(v.k, pq, c) <= v.r_max_sq;
          }
        }
      }
      visit(hit, q);
    }
  }
}

__global__ void __launch_bounds__(256) k_count_b(BuildView v, Buckets B,
                                                 uint32_t* __restrict__ sizes) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < v.n; j += nw) {
    const Cell c = leaf_cell(v.T, v.n, v.depth, v.k, j);
    const int32_t p = v.rep[j];
    uint32_t m = 0;
    if (!(p < v.n0 && v.shortcut && shortcut_fires(v, c, p)))
      warp_afforded(v, B, c, p, lane, [&](bool hit, float4) {
        m += __popc(__ballot_sync(0xffffffffu, hit));
      });
    if (lane == 0) sizes[j] = 1 + m;
  }
}

__global__ void __launch_bounds__(256) k_fill_b(BuildView v, Buckets B,
                                                const uint2* __restrict__ set,
                                                float4* __restrict__ data,
                                                float4* __restrict__ box,
                                                float4* __restrict__ org,
                                                float4* __restrict__ rep,
                                                float* __restrict__ probe) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const float INF = __int_as_float(0x7f800000);
  for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < v.n; j += nw) {
    const Cell c = leaf_cell(v.T, v.n, v.depth, v.k, j);
    const int32_t p = v.rep[j];
    const uint2 st = set[j];
    const uint32_t m4 = (st.y + 3u) & ~3u;
    float* dst = reinterpret_cast<float*>(data + st.x);
    // row 0: the representative (+inf for a padding leaf)
    float rx[3] = {0.f, 0.f, 0.f};
    for (int d = 0; d < v.k; ++d) rx[d] = p < v.n0 ? v.X[d * v.n + p] : INF;
    float blo[3] = {rx[0], rx[1], rx[2]}, bhi[3] = {rx[0], rx[1], rx[2]};
    // the finite rows' box (the origin of the binned scan; a padding leaf's
    // +inf row is left out, as in k_origins)
    const bool rfin = p < v.n0;
    float flo[3], fhi[3];
    for (int d = 0; d < 3; ++d) {
      flo[d] = rfin ? rx[d] : INF;
      fhi[d] = rfin ? rx[d] : -INF;
    }
    if (lane < 3) dst[lane * m4] = rx[lane];
    uint32_t w = 1;
    if (st.y > 1)
      warp_afforded(v, B, c, p, lane, [&](bool hit, float4 q) {
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const uint32_t at = w + __popc(b & ((1u << lane) - 1u));
          const float qv[3] = {q.x, q.y, q.z};
          for (int d = 0; d < 3; ++d) {
            dst[d * m4 + at] = d < v.k ? qv[d] : 0.f;
            blo[d] = fminf(blo[d], qv[d]);
            bhi[d] = fmaxf(bhi[d], qv[d]);
            flo[d] = fminf(flo[d], qv[d]);
            fhi[d] = fmaxf(fhi[d], qv[d]);
          }
        }
        w += __popc(b);
      });
    // padding rows (+inf), unused axes 0
    for (uint32_t i = st.y + lane; i < m4; i += 32)
      for (int d = 0; d < 3; ++d) dst[d * m4 + i] = d < v.k ? INF : 0.f;
    float o[3], bb = 0.f;
    for (int d = 0; d < 3; ++d) {
      for (int s = 16; s; s >>= 1) {
        blo[d] = fminf(blo[d], __shfl_xor_sync(0xffffffffu, blo[d], s));
        bhi[d] = fmaxf(bhi[d], __shfl_xor_sync(0xffffffffu, bhi[d], s));
        flo[d] = fminf(flo[d], __shfl_xor_sync(0xffffffffu, flo[d], s));
        fhi[d] = fmaxf(fhi[d], __shfl_xor_sync(0xffffffffu, fhi[d], s));
      }
      if (d >= v.k) blo[d] = bhi[d] = 0.f;
      // origin = the finite box's centre; org.w >= max |p - o|^2 (the
      // farthest corner of the finite box, rounded up): the binned scan's
      // error band only needs an upper bound
      o[d] = flo[d] <= fhi[d] ? 0.5f * flo[d] + 0.5f * fhi[d] : 0.f;
      const float e =
          flo[d] <= fhi[d] ? fmaxf(__fsub_ru(fhi[d], o[d]), __fsub_ru(o[d], flo[d])) : 0.f;
      bb = __fmaf_ru(e, e, bb);
    }
    if (lane == 0) {
      box[2 * j] = make_float4(blo[0], blo[1], blo[2], 0.f);
      box[2 * j + 1] = make_float4(bhi[0], bhi[1], bhi[2], 0.f);
      org[j] = make_float4(o[0], o[1], o[2], __fmul_ru(bb, 1.0f + 0x1p-20f));
      const float4 rp = make_float4(rx[0], rx[1], rx[2], 0.f);
      rep[j] = rp;
      const __half2 h0 = __halves2half2(__float2half_rd(blo[0]), __float2half_rd(blo[1]));
      const __half2 h1 = __halves2half2(__float2half_rd(blo[2]), __float2half_ru(bhi[0]));
      const __half2 h2 = __halves2half2(__float2half_ru(bhi[1]), __float2half_ru(bhi[2]));
      float4* pr = reinterpret_cast<float4*>(probe + 8 * j);
      pr[0] = make_float4(rp.x, rp.y, rp.z, __uint_as_float(*reinterpret_cast<const unsigned*>(&h0)));
      pr[1] = make_float4(__uint_as_float(*reinterpret_cast<const unsigned*>(&h1)),
                          __uint_as_float(*reinterpret_cast<const unsigned*>(&h2)), 0.f, 0.f);
    }
  }
}

__global__ void k_set_layout(int64_t n, const uint32_t* __restrict__ sizes,
                             const int64_t* __restrict__ f4_excl, const int64_t* __restrict__ off_excl,
                             uint2* __restrict__ set, int64_t* __restrict__ offs) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    set[j] = make_uint2(uint32_t(f4_excl[j]), sizes[j]);
    offs[j] = off_excl[j];
    if (j == n - 1) offs[n] = off_excl[j] + sizes[j];
  }
}

__host__ __device__ inline int64_t f4_count(uint32_t m) { return 3 * int64_t((m + 3u) & ~3u) / 4; }

__global__ void k_widen(int64_t n, const uint32_t* __restrict__ sizes, int64_t* __restrict__ c4,
                        int64_t* __restrict__ cm) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    c4[j] = f4_count(sizes[j]);
    cm[j] = sizes[j];
  }
}

// Scratch arena for one build (freed at the end).
struct Scratch {
  cudaStream_t s;
  void* ptrs[64];
  int np = 0;
  template <class T>
  T* get(size_t count) {
    void* p = nullptr;
    if (np == 64) return nullptr;
    if (cudaMallocAsync(&p, (count ? count : 1) * sizeof(T), s) != cudaSuccess) return nullptr;
    ptrs[np++] = p;
    return static_cast<T*>(p);
  }
  ~Scratch() {
    for (int i = 0; i < np; ++i) cudaFreeAsync(ptrs[i], s);
  }
};

}  // namespace capt

using namespace capt;

extern "C" int capt_tree_build(int device, int k, const float* points, int64_t n0, double r_min,
                               double r_max, int use_rmin_shortcut, uint32_t flags, void* stream,
                               capt_tree** out) {
  if (!out) return fail(CAPT_EINVAL, "out is NULL");
  *out = nullptr;
  if (n0 <= 0) return fail(CAPT_EINVAL, "cannot build a tree over an empty cloud");
  if (k < 1 || k > kMaxK) return fail(CAPT_EINVAL, "k must be 1..3 on the device path");
  if (!(r_min > 0 && r_min <= r_max) || !std::isfinite(r_min) || !std::isfinite(r_max))
    return fail(CAPT_EINVAL, "need 0 < r_min <= r_max, finite");
  if (n0 > (int64_t(1) << 30)) return fail(CAPT_EINVAL, "cloud too large");
  CAPT_CUDA(cudaSetDevice(device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int depth = depth_of(n0);
  const int64_t n = int64_t(1) << depth;
  Scratch S;
  S.s = s;

  const float* d_pts = points;
  if (flags & CAPT_HOST_IO) {
    float* p = S.get<float>(size_t(n0) * k);
    if (!p) return fail(CAPT_ENOMEM, "scratch allocation");
    CAPT_CUDA(cudaMemcpyAsync(p, points, sizeof(float) * n0 * k, cudaMemcpyHostToDevice, s));
    d_pts = p;
  }
  float* X = S.get<float>(size_t(n) * k);
  uint32_t* keys = S.get<uint32_t>(size_t(n) * k);
  uint32_t* keys_out = S.get<uint32_t>(size_t(n));
  int32_t* idx = S.get<int32_t>(size_t(n));
  int32_t* P[3] = {nullptr, nullptr, nullptr};
  for (int d = 0; d < k; ++d) P[d] = S.get<int32_t>(size_t(n));
  int32_t* Ptmp = S.get<int32_t>(size_t(n));
  uint8_t* left = S.get<uint8_t>(size_t(n));
  int32_t* f = S.get<int32_t>(size_t(n));
  int32_t* sc = S.get<int32_t>(size_t(n));
  float* T = S.get<float>(size_t(n > 1 ? n - 1 : 1));
  unsigned long long* ties = S.get<unsigned long long>(1);
  uint32_t* sizes = S.get<uint32_t>(size_t(n));
  int64_t* f4x = S.get<int64_t>(size_t(n));
  int64_t* offx = S.get<int64_t>(size_t(n));
  if (!X || !keys || !keys_out || !idx || !Ptmp || !left || !f || !sc || !T || !ties || !sizes ||
      !f4x || !offx)
    return fail(CAPT_ENOMEM, "scratch allocation");
  for (int d = 0; d < k; ++d)
    if (!P[d]) return fail(CAPT_ENOMEM, "scratch allocation");
  CAPT_CUDA(cudaMemsetAsync(ties, 0, 8, s));
  const int G = grid_for(n, 256, 8);
  k_init<<<G, 256, 0, s>>>(d_pts, n0, n, k, X, keys, idx);
  CAPT_CUDA(cudaGetLastError());

  // 1. presort every axis by (coordinate key, index): stable LSD radix sort
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys_out, idx, P[0], int(n), 0, 32, s);
  size_t tb2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, f, sc, int(n), s);
  void* tmp = S.get<char>(tb > tb2 ? tb : tb2);
  if (!tmp) return fail(CAPT_ENOMEM, "scratch allocation");
  const size_t tbytes = tb > tb2 ? tb : tb2;
  for (int d = 0; d < k; ++d) {
    size_t t = tbytes;
    CAPT_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t, keys + size_t(d) * n, keys_out, idx, P[d],
                                              int(n), 0, 32, s));
  }

  // the cloud's extremes per axis (bucket grid): first / last finite entry
  // of each presorted list, kept before the partitions reorder them
  int32_t* P0sorted[3] = {nullptr, nullptr, nullptr};
  for (int d = 0; d < k; ++d) {
    P0sorted[d] = S.get<int32_t>(size_t(n0));
    if (!P0sorted[d]) return fail(CAPT_ENOMEM, "scratch allocation");
    CAPT_CUDA(cudaMemcpyAsync(P0sorted[d], P[d], sizeof(int32_t) * n0, cudaMemcpyDeviceToDevice, s));
  }

  // 2. level-by-level median split with stable partitions
  for (int L = 0; L < depth; ++L) {
    const int64_t n_seg = int64_t(1) << L;
    const int64_t m = n >> L;
    const int a = L % k;
    k_split<<<grid_for(n_seg, 256, 8), 256, 0, s>>>(n_seg, m, a, n, X, P[a], T, ties);
    k_flags<<<G, 256, 0, s>>>(n, m, P[a], left);
    for (int d = 0; d < k; ++d) {
      if (d == a) continue;
      k_gather_flags<<<G, 256, 0, s>>>(n, P[d], left, f);
      size_t t = tbytes;
      CAPT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, t, f, sc, int(n), s));
      k_partition<<<G, 256, 0, s>>>(n, m, P[d], f, sc, Ptmp);
      int32_t* sw = P[d];
      P[d] = Ptmp;
      Ptmp = sw;
    }
    CAPT_CUDA(cudaGetLastError());
  }

  // 3-4. per-leaf affordance counts
  BuildView v;
  v.k = k;
  v.depth = depth;
  v.n = n;
  v.n0 = n0;
  v.X = X;
  v.rep = P[0];
  v.T = T;
  v.r_min_sq = r_min * r_min;
  v.r_max_sq = r_max * r_max;
  v.r2_hi = float(r_max * r_max) * (1.0f + 0x1p-16f);
  // (the relative-error argument needs r_max^2 well inside the normal floats)
  v.r2_in = (r_max * r_max > 0x1p-100 && r_max * r_max < 0x1p100)
                ? float(r_max * r_max) * (1.0f - 0x1p-16f)
                : -1.0f;
  v.shortcut = use_rmin_shortcut;
  // the point buckets (edge >= r_max, at most ~2^21 buckets)
  Buckets B;
  {
    float hb[6];
    {
      // the cloud's box: the first / last entries of the presorted axis lists
      // hold the extremes (finite points sort before the +inf padding)
      for (int d = 0; d < 3; ++d) {
        hb[d] = 0.f;
        hb[3 + d] = 0.f;
      }
      int32_t ends[6] = {0, 0, 0, 0, 0, 0};
      for (int d = 0; d < k; ++d) {
        CAPT_CUDA(cudaMemcpyAsync(ends + d, P0sorted[d], 4, cudaMemcpyDeviceToHost, s));
        CAPT_CUDA(cudaMemcpyAsync(ends + 3 + d, P0sorted[d] + (n0 - 1), 4, cudaMemcpyDeviceToHost, s));
      }
      CAPT_CUDA(cudaStreamSynchronize(s));
      for (int d = 0; d < k; ++d) {
        CAPT_CUDA(cudaMemcpyAsync(hb + d, X + size_t(d) * n + ends[d], 4, cudaMemcpyDeviceToHost, s));
        CAPT_CUDA(cudaMemcpyAsync(hb + 3 + d, X + size_t(d) * n + ends[3 + d], 4, cudaMemcpyDeviceToHost, s));
      }
      CAPT_CUDA(cudaStreamSynchronize(s));
    }
    double ext[3] = {0.0, 0.0, 0.0}, vol = 1.0;
    for (int d = 0; d < 3; ++d) {
      B.lo[d] = 0.0;
      B.dims[d] = 1;
    }
    for (int d = 0; d < k; ++d) {
      B.lo[d] = double(hb[d]);
      ext[d] = double(hb[3 + d]) - double(hb[d]);
    }
    double b = r_max * CAPT_BUCKET_SCALE;
    for (int it = 0; it < 400; ++it) {
      vol = 1.0;
      for (int d = 0; d < k; ++d) vol *= std::floor(ext[d] / b) + 1.0;
      if (vol <= double(1 << 21)) break;
      b *= 1.1;
    }
    B.inv_b = 1.0 / b;
    int64_t nb = 1;
    for (int d = 0; d < k; ++d) {
      B.dims[d] = int(std::floor(ext[d] / b) + 1.0);
      nb *= B.dims[d];
    }
    uint32_t* bkey = S.get<uint32_t>(size_t(n0));
    uint32_t* bkeyS = S.get<uint32_t>(size_t(n0));
    int32_t* bid = S.get<int32_t>(size_t(n0));
    int32_t* bidS = S.get<int32_t>(size_t(n0));
    uint32_t* cnt = S.get<uint32_t>(size_t(nb + 1));
    uint32_t* start = S.get<uint32_t>(size_t(nb + 1));
    float4* bp = S.get<float4>(size_t(n0));
    if (!bkey || !bkeyS || !bid || !bidS || !cnt || !start || !bp)
      return fail(CAPT_ENOMEM, "scratch allocation");
    CAPT_CUDA(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (nb + 1), s));
    k_bucket_key<<<grid_for(n0, 256, 8), 256, 0, s>>>(k, n0, B, X, n, bkey, bid, cnt);
    size_t t1 = 0, t2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, bkey, bkeyS, bid, bidS, int(n0), 0, 32, s);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, cnt, start, int(nb + 1), s);
    void* tmpb = S.get<char>(std::max(t1, t2));
    if (!tmpb) return fail(CAPT_ENOMEM, "scratch allocation");
    CAPT_CUDA(cub::DeviceRadixSort::SortPairs(tmpb, t1, bkey, bkeyS, bid, bidS, int(n0), 0, 32, s));
    CAPT_CUDA(cub::DeviceScan::ExclusiveSum(tmpb, t2, cnt, start, int(nb + 1), s));
    k_bucket_gather<<<grid_for(n0, 256, 8), 256, 0, s>>>(k, n0, X, n, bidS, bp);
    B.start = start;
    B.pts = bp;
  }
  k_count_b<<<grid_for(n * 32, 256, 8), 256, 0, s>>>(v, B, sizes);
  CAPT_CUDA(cudaGetLastError());

  // 5. layout: exclusive scans of padded float4 counts and of set sizes
  {
    int64_t* c4 = S.get<int64_t>(size_t(n));
    int64_t* cm = S.get<int64_t>(size_t(n));
    if (!c4 || !cm) return fail(CAPT_ENOMEM, "scratch allocation");
    k_widen<<<G, 256, 0, s>>>(n, sizes, c4, cm);
    size_t t1 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t1, c4, f4x, int(n), s);
    void* tmp2 = S.get<char>(t1);
    if (!tmp2) return fail(CAPT_ENOMEM, "scratch allocation");
    CAPT_CUDA(cub::DeviceScan::ExclusiveSum(tmp2, t1, c4, f4x, int(n), s));
    CAPT_CUDA(cub::DeviceScan::ExclusiveSum(tmp2, t1, cm, offx, int(n), s));
  }
  int64_t last_f4 = 0, last_off = 0;
  uint32_t last_size = 0;
  unsigned long long n_ties = 0;
  CAPT_CUDA(cudaMemcpyAsync(&last_f4, f4x + n - 1, 8, cudaMemcpyDeviceToHost, s));
  CAPT_CUDA(cudaMemcpyAsync(&last_off, offx + n - 1, 8, cudaMemcpyDeviceToHost, s));
  CAPT_CUDA(cudaMemcpyAsync(&last_size, sizes + n - 1, 4, cudaMemcpyDeviceToHost, s));
  CAPT_CUDA(cudaMemcpyAsync(&n_ties, ties, 8, cudaMemcpyDeviceToHost, s));
  uint32_t max_size = 0;
  {
    uint32_t* d_max = S.get<uint32_t>(1);
    size_t t = 0;
    cub::DeviceReduce::Max(nullptr, t, sizes, d_max, int(n), s);
    void* tmp3 = S.get<char>(t);
    if (!d_max || !tmp3) return fail(CAPT_ENOMEM, "scratch allocation");
    CAPT_CUDA(cub::DeviceReduce::Max(tmp3, t, sizes, d_max, int(n), s));
    CAPT_CUDA(cudaMemcpyAsync(&max_size, d_max, 4, cudaMemcpyDeviceToHost, s));
  }
  CAPT_CUDA(cudaStreamSynchronize(s));
  const int64_t data_f4 = last_f4 + f4_count(last_size);
  if (data_f4 > 0xffffffffll) return fail(CAPT_EINVAL, "tree too large for 32-bit float4 offsets");

  SlabHeader h;
  memset(&h, 0, sizeof(h));
  h.magic = kSlabMagic;
  h.version = kSlabVersion;
  h.k = k;
  h.n = n;
  h.depth = depth;
  h.n_points = n0;
  h.total = last_off + last_size;
  h.max_aff = max_size;
  h.n_ties = int64_t(n_ties);
  h.r_min = r_min;
  h.r_max = r_max;
  layout_slab(h, data_f4);
  int rc = alloc_slab(out, device, h);
  if (rc) return rc;
  capt_tree* t = *out;
  DevTree dv = view(t);
  cudaError_t e = cudaMemcpyAsync(t->slab, &h, sizeof(h), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && n > 1)
    e = cudaMemcpyAsync(const_cast<float*>(dv.T), T, sizeof(float) * (n - 1), cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) {
    k_set_layout<<<G, 256, 0, s>>>(n, sizes, f4x, offx, const_cast<uint2*>(dv.set),
                                   const_cast<int64_t*>(dv.offs));
    k_fill_b<<<grid_for(n * 32, 256, 8), 256, 0, s>>>(
        v, B, dv.set, const_cast<float4*>(dv.data), const_cast<float4*>(dv.box),
        const_cast<float4*>(dv.org), const_cast<float4*>(dv.rep), const_cast<float*>(dv.probe));
    e = cudaGetLastError();
    if (e == cudaSuccess && compute_origins(dv, s, false)) e = cudaErrorLaunchFailure;
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    capt_tree_destroy(t);
    *out = nullptr;
    return cuda_fail(e, "tree build");
  }
  rc = build_field(t, s);
  if (rc) {
    capt_tree_destroy(t);
    *out = nullptr;
  }
  return rc;
}
