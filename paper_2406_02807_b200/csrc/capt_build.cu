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
//      (tree.py:209-218).  Candidates come from a stackless traversal of the
//      implicit tree pruned by a conservative fp32 box-box distance, then
//      the exact float64 test of tree.py:209-213 decides membership;
//   5. count pass -> exclusive scan -> fill pass into the padded slab layout.
#include <cub/cub.cuh>

#include <cmath>
#include <cstring>

#include "capt_internal.cuh"

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

// Conservative lower bound test: may the node cell hold a point within r of
// the leaf cell?  (fp32 with a relative margin; exact test happens per point)
__device__ __forceinline__ bool cells_near(int k, const float* nlo, const float* nhi,
                                           const Cell& c, float r2_hi) {
  float s = 0.f;
  for (int d = 0; d < k; ++d) {
    if (nlo[d] == INFINITY) return false;  // all-padding subtree
    float g = 0.f;
    if (nlo[d] > c.hi[d]) g = nlo[d] - c.hi[d];
    else if (c.lo[d] > nhi[d]) g = c.lo[d] - nhi[d];
    g *= (1.0f - 0x1p-20f);
    s = fmaf(g, g, s);
  }
  return s <= r2_hi;
}

struct BuildView {
  int k, depth;
  int64_t n, n0;
  const float* X;      // k * n, SoA
  const int32_t* rep;  // n (leaf -> point index)
  const float* T;
  double r_min_sq, r_max_sq;
  float r2_hi;         // fp32 r_max^2 upper margin for pruning
  int shortcut;
};

// Stackless DFS over the implicit tree; visit(point index) for every finite
// leaf representative (other than `self`) whose cell may be within r_max of
// cell `c`, applying the exact membership test.
template <class F>
__device__ __forceinline__ void for_each_afforded(const BuildView& v, const Cell& c, int64_t self,
                                                  F&& visit) {
  float lo[3] = {-INFINITY, -INFINITY, -INFINITY}, hi[3] = {INFINITY, INFINITY, INFINITY};
  float savedHi[48], savedLo[48];
  int64_t i = 0;
  int level = 0;
  const int64_t inner = v.n - 1;
  while (true) {
    bool descend = false;
    if (cells_near(v.k, lo, hi, c, v.r2_hi)) {
      if (i >= inner) {
        const int64_t leaf = i - inner;
        const int32_t p = v.rep[leaf];
        if (leaf != self && p < v.n0) {
          double q[3];
          for (int d = 0; d < v.k; ++d) q[d] = double(v.X[d * v.n + p]);
          if (dist_cell64(v.k, q, c) <= v.r_max_sq) visit(p);
        }
      } else {
        descend = true;
      }
    }
    if (descend) {
      const int a = level % v.k;
      savedHi[level] = hi[a];
      hi[a] = v.T[i];
      i = 2 * i + 1;
      ++level;
      continue;
    }
    // advance to the next node in DFS order
    bool done = false;
    while (true) {
      if (i == 0) {
        done = true;
        break;
      }
      const int64_t parent = (i - 1) / 2;
      const int a = (level - 1) % v.k;
      if (i & 1) {  // left child -> right sibling
        hi[a] = savedHi[level - 1];
        savedLo[level - 1] = lo[a];
        lo[a] = v.T[parent];
        i = i + 1;
        break;
      }
      lo[a] = savedLo[level - 1];  // right child -> up
      i = parent;
      --level;
    }
    if (done) break;
  }
}

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

__global__ void k_count(BuildView v, uint32_t* __restrict__ sizes) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < v.n;
       j += int64_t(gridDim.x) * blockDim.x) {
    const Cell c = leaf_cell(v.T, v.n, v.depth, v.k, j);
    const int32_t p = v.rep[j];
    uint32_t m = 1;
    if (!(p < v.n0 && v.shortcut && shortcut_fires(v, c, p)))
      for_each_afforded(v, c, j, [&](int32_t) { ++m; });
    sizes[j] = m;
  }
}

__global__ void k_fill(BuildView v, const uint2* __restrict__ set, float4* __restrict__ data,
                       float4* __restrict__ box) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < v.n;
       j += int64_t(gridDim.x) * blockDim.x) {
    const Cell c = leaf_cell(v.T, v.n, v.depth, v.k, j);
    const int32_t p = v.rep[j];
    const uint2 st = set[j];
    const uint32_t m4 = (st.y + 3u) & ~3u;
    float* dst = reinterpret_cast<float*>(data + st.x);
    float blo[3], bhi[3];
    for (int d = 0; d < 3; ++d) {
      const float x = d < v.k ? (p < v.n0 ? v.X[d * v.n + p] : INFINITY) : 0.f;
      dst[d * m4] = x;
      blo[d] = x;
      bhi[d] = x;
    }
    uint32_t w = 1;
    if (st.y > 1) {
      for_each_afforded(v, c, j, [&](int32_t q) {
        for (int d = 0; d < v.k; ++d) {
          const float x = v.X[d * v.n + q];
          dst[d * m4 + w] = x;
          blo[d] = fminf(blo[d], x);
          bhi[d] = fmaxf(bhi[d], x);
        }
        ++w;
      });
    }
    for (uint32_t i = st.y; i < m4; ++i)
      for (int d = 0; d < 3; ++d) dst[d * m4 + i] = d < v.k ? INFINITY : 0.f;
    for (int d = v.k; d < 3; ++d)
      for (uint32_t i = 1; i < st.y; ++i) dst[d * m4 + i] = 0.f;
    box[2 * j] = make_float4(blo[0], blo[1], blo[2], 0.f);
    box[2 * j + 1] = make_float4(bhi[0], bhi[1], bhi[2], 0.f);
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
  void* ptrs[48];
  int np = 0;
  template <class T>
  T* get(size_t count) {
    void* p = nullptr;
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
  v.shortcut = use_rmin_shortcut;
  k_count<<<grid_for(n, 128, 16), 128, 0, s>>>(v, sizes);
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
    k_fill<<<grid_for(n, 128, 16), 128, 0, s>>>(v, dv.set, const_cast<float4*>(dv.data),
                                                const_cast<float4*>(dv.box));
    e = cudaGetLastError();
    if (e == cudaSuccess && compute_origins(dv, s)) e = cudaErrorLaunchFailure;
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
