// Device Z-order point filter: filter_cloud (morton.py:185-236) with the
// optional reach_filter pre-pass (morton.py:173-182).
//
// Per axis permutation (itertools.permutations order), on the survivors:
//   1. bounds: fp32 min/max per axis (orderable-key atomics);
//   2. keys:   float64 quantisation q = floor((p - lo) / span * (2^b - 1)),
//              clamped, degenerate axes -> 0, bits interleaved with perm[0]
//              most significant (morton.py:95-126), all with __d*_rn ops;
//   3. order:  survivors are listed in ascending original index, then a
//              stable LSD radix sort by key gives the (key, index) order of
//              np.lexsort((idx, keys)) (morton.py:209);
//   4. gap scan (morton.py:141-170): keep j iff dist64(p_j, last kept) > r^2.
//              Parallel form: nxt[j] = first i > j with dist64(p_i, p_j) > r^2
//              (one warp per j, ballot over 32 candidates at a time); the kept
//              set is the chain 0 -> nxt[0] -> ..., marked by pointer jumping
//              (log2 m doubling tables, then log2 m marking rounds); anchors
//              are a max-scan of kept positions.
// Orphan repair (morton.py:212-235): every dropped point whose anchor was
// dropped later is re-added, in ascending original index, iff no final
// survivor lies within r_filter (float64 test against the survivors of the
// neighbouring cells of a uniform grid, k_orphans).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "capt_internal.cuh"

namespace capt {

namespace {

__device__ __forceinline__ uint32_t okey(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float okey_inv(uint32_t u) {
  u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
  return __uint_as_float(u);
}

// reach pre-pass keep flags: ((p - base)^2 summed in numpy order) <= reach^2
__global__ void k_reach(int k, int64_t n, const float* __restrict__ p, double b0, double b1,
                        double b2, double reach_sq, uint8_t* __restrict__ keep) {
  const double b[3] = {b0, b1, b2};
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int d = 0; d < k; ++d) {
      const double t = __dsub_rn(double(p[i * k + d]), b[d]);
      const double sq = __dmul_rn(t, t);
      s = d == 0 ? sq : __dadd_rn(s, sq);
    }
    keep[i] = s <= reach_sq;
  }
}

__global__ void k_bounds(int k, int64_t m, const int32_t* __restrict__ idx,
                         const float* __restrict__ p, uint32_t* __restrict__ mn,
                         uint32_t* __restrict__ mx) {
  uint32_t lmn[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, lmx[3] = {0, 0, 0};
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int32_t i = idx[j];
    for (int d = 0; d < k; ++d) {
      const uint32_t u = okey(p[int64_t(i) * k + d]);
      lmn[d] = min(lmn[d], u);
      lmx[d] = max(lmx[d], u);
    }
  }
  for (int d = 0; d < k; ++d) {
    uint32_t a = lmn[d], b = lmx[d];
    for (int o = 16; o > 0; o >>= 1) {
      a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(mn + d, a);
      atomicMax(mx + d, b);
    }
  }
}

__device__ __forceinline__ uint64_t spread(uint64_t v, int k, int bits) {
  uint64_t out = 0;
  for (int b = 0; b < bits; ++b) out |= ((v >> b) & 1ull) << (b * k);
  return out;
}

// quantize + morton_keys (morton.py:95-126)
__global__ void k_keys(int k, int bits, int64_t m, const int32_t* __restrict__ idx,
                       const float* __restrict__ p, const uint32_t* __restrict__ mn,
                       const uint32_t* __restrict__ mx, int perm0, int perm1, int perm2,
                       uint64_t* __restrict__ keys) {
  const int perm[3] = {perm0, perm1, perm2};
  const uint64_t amax = (1ull << bits) - 1;
  double lo[3], span[3];
  bool degen[3];
  for (int d = 0; d < k; ++d) {
    lo[d] = double(okey_inv(mn[d]));
    const double hi = double(okey_inv(mx[d]));
    span[d] = __dsub_rn(hi, lo[d]);
    degen[d] = span[d] == 0.0;
    if (degen[d]) span[d] = 1.0;
  }
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += int64_t(gridDim.x) * blockDim.x) {
    const int32_t i = idx[j];
    uint64_t q[3] = {0, 0, 0};
    for (int d = 0; d < k; ++d) {
      const double frac = __ddiv_rn(__dsub_rn(double(p[int64_t(i) * k + d]), lo[d]), span[d]);
      const double f = floor(__dmul_rn(frac, double(amax)));
      uint64_t v = uint64_t(f);
      if (v > amax) v = amax;
      q[d] = degen[d] ? 0 : v;
    }
    uint64_t key = 0;
    for (int a = 0; a < k; ++a) key |= spread(q[perm[a]], k, bits) << (k - 1 - a);
    keys[j] = key;
  }
}

__global__ void k_gather(int k, int64_t m, const int32_t* __restrict__ idx,
                         const float* __restrict__ p, float* __restrict__ q) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += int64_t(gridDim.x) * blockDim.x)
    for (int d = 0; d < k; ++d) q[j * k + d] = p[int64_t(idx[j]) * k + d];
}

__device__ __forceinline__ double dist64(int k, const float* a, const float* b) {
  double s = 0.0;
  for (int d = 0; d < k; ++d) {
    const double t = __dsub_rn(double(a[d]), double(b[d]));
    const double sq = __dmul_rn(t, t);
    s = d == 0 ? sq : __dadd_rn(s, sq);
  }
  return s;
}

// nxt[j] = first i > j with dist64(q_i, q_j) > r2 (m if none); one warp per j
__global__ void k_next(int k, int64_t m, const float* __restrict__ q, double r2,
                       int32_t* __restrict__ nxt) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = warp; j < m; j += nwarps) {
    float pj[3];
    for (int d = 0; d < k; ++d) pj[d] = q[j * k + d];
    int64_t res = m;
    for (int64_t base = j + 1; base < m; base += 32) {
      const int64_t i = base + lane;
      const bool far = i < m && dist64(k, q + i * k, pj) > r2;
      const uint32_t b = __ballot_sync(0xffffffffu, far);
      if (b) {
        res = base + __ffs(b) - 1;
        break;
      }
    }
    if (lane == 0) nxt[j] = int32_t(res);
  }
}

__global__ void k_jump(int64_t m, const int32_t* __restrict__ J, int32_t* __restrict__ J2) {
  for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x <= m;
       x += int64_t(gridDim.x) * blockDim.x)
    J2[x] = J[J[x]];
}

__global__ void k_mark(int64_t m, const int32_t* __restrict__ J, uint8_t* __restrict__ mk) {
  for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < m;
       x += int64_t(gridDim.x) * blockDim.x)
    if (mk[x]) {
      const int32_t y = J[x];
      if (y < m) mk[y] = 1;
    }
}

__global__ void k_kept_pos(int64_t m, const uint8_t* __restrict__ mk, int32_t* __restrict__ a) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += int64_t(gridDim.x) * blockDim.x)
    a[j] = mk[j] ? int32_t(j) : -1;
}

// removed positions: anchor_of[idx[j]] = idx[anchor(j)], survivor flag cleared
__global__ void k_drop(int64_t m, const uint8_t* __restrict__ mk, const int32_t* __restrict__ anc,
                       const int32_t* __restrict__ idx, int32_t* __restrict__ anchor_of,
                       uint8_t* __restrict__ surv) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += int64_t(gridDim.x) * blockDim.x)
    if (!mk[j]) {
      anchor_of[idx[j]] = idx[anc[j]];
      surv[idx[j]] = 0;
    }
}

__global__ void k_candidates(int64_t n0, const uint8_t* __restrict__ surv,
                             const int32_t* __restrict__ anchor_of, uint8_t* __restrict__ cand) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n0;
       i += int64_t(gridDim.x) * blockDim.x)
    cand[i] = !surv[i] && !surv[anchor_of[i]];
}

// Orphan check (morton.py:212-235): candidate c is an orphan iff no final
// survivor lies within r (the float64 test of the brute-force reference).
// Survivors are bucketed on a uniform grid of edge cs >= r (1 + 2^-20):
// bucket(x) = floor((x - lo) / cs) per axis in float64, clamped to the grid
// (monotone in x), so a survivor within r of c differs from c by at most one
// bucket per axis; keys are x-fastest, so the three x-buckets of one (y, z)
// row are one key range of the sorted survivors, found by binary search.
struct OrphanGrid {
  double lo[3], inv_cs;
  int dims[3];
};

__device__ __forceinline__ int og_cell(const OrphanGrid& G, int d, float x) {
  const double t = floor(__dmul_rn(__dsub_rn(double(x), G.lo[d]), G.inv_cs));
  return t < 0.0 ? 0 : (t >= double(G.dims[d] - 1) ? G.dims[d] - 1 : int(t));
}

__global__ void k_orphan_keys(int k, OrphanGrid G, int64_t m, const int32_t* __restrict__ sidx,
                              const float* __restrict__ p, uint32_t* __restrict__ key,
                              int32_t* __restrict__ val) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += int64_t(gridDim.x) * blockDim.x) {
    const float* q = p + int64_t(sidx[j]) * k;
    int c[3] = {0, 0, 0};
    for (int d = 0; d < k; ++d) c[d] = og_cell(G, d, q[d]);
    key[j] = (uint32_t(c[2]) * uint32_t(G.dims[1]) + uint32_t(c[1])) * uint32_t(G.dims[0]) +
             uint32_t(c[0]);
    val[j] = sidx[j];
  }
}

__device__ __forceinline__ int64_t lower_bound_u32(const uint32_t* a, int64_t n, uint32_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_orphans(int k, OrphanGrid G, int64_t nc, const int32_t* __restrict__ cidx,
                          int64_t ns, const uint32_t* __restrict__ skey,
                          const int32_t* __restrict__ sval, const float* __restrict__ p,
                          double r2, uint8_t* __restrict__ orphan) {
  for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < nc;
       c += int64_t(gridDim.x) * blockDim.x) {
    float pc[3] = {0.f, 0.f, 0.f};
    int cc[3] = {0, 0, 0};
    for (int d = 0; d < k; ++d) {
      pc[d] = p[int64_t(cidx[c]) * k + d];
      cc[d] = og_cell(G, d, pc[d]);
    }
    bool found = false;
    const int z0 = k > 2 ? max(cc[2] - 1, 0) : 0, z1 = k > 2 ? min(cc[2] + 1, G.dims[2] - 1) : 0;
    const int y0 = k > 1 ? max(cc[1] - 1, 0) : 0, y1 = k > 1 ? min(cc[1] + 1, G.dims[1] - 1) : 0;
    const int x0 = max(cc[0] - 1, 0), x1 = min(cc[0] + 1, G.dims[0] - 1);
    for (int z = z0; z <= z1 && !found; ++z)
      for (int y = y0; y <= y1 && !found; ++y) {
        const uint32_t row = (uint32_t(z) * uint32_t(G.dims[1]) + uint32_t(y)) * uint32_t(G.dims[0]);
        const int64_t b = lower_bound_u32(skey, ns, row + uint32_t(x0));
        const int64_t e = lower_bound_u32(skey, ns, row + uint32_t(x1) + 1u);
        for (int64_t i = b; i < e; ++i)
          if (dist64(k, pc, p + int64_t(sval[i]) * k) <= r2) {
            found = true;
            break;
          }
      }
    orphan[c] = !found;
  }
}

__global__ void k_emit(int k, int64_t m, const int32_t* __restrict__ idx,
                       const float* __restrict__ p, float* __restrict__ out) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += int64_t(gridDim.x) * blockDim.x)
    for (int d = 0; d < k; ++d) out[j * k + d] = p[int64_t(idx[j]) * k + d];
}

struct Arena {
  cudaStream_t s;
  std::vector<void*> ptrs;
  template <class T>
  T* get(size_t count) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, (count ? count : 1) * sizeof(T), s) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~Arena() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
};

// stable compaction of [0, n) by flags -> out (ascending), returns count
int select_flagged(Arena& A, const uint8_t* flags, int64_t n, int32_t* out, int64_t* count) {
  cub::CountingInputIterator<int32_t> it(0);
  int64_t* d_cnt = A.get<int64_t>(1);
  size_t tb = 0;
  cub::DeviceSelect::Flagged(nullptr, tb, it, flags, out, d_cnt, n, A.s);
  void* tmp = A.get<char>(tb);
  if (!d_cnt || !tmp) return fail(CAPT_ENOMEM, "scratch allocation");
  CAPT_CUDA(cub::DeviceSelect::Flagged(tmp, tb, it, flags, out, d_cnt, n, A.s));
  CAPT_CUDA(cudaMemcpyAsync(count, d_cnt, 8, cudaMemcpyDeviceToHost, A.s));
  CAPT_CUDA(cudaStreamSynchronize(A.s));
  return CAPT_OK;
}

// stable compaction of idx[] by flags (order preserved)
int select_values(Arena& A, const int32_t* in, const uint8_t* flags, int64_t n, int32_t* out,
                  int64_t* count) {
  int64_t* d_cnt = A.get<int64_t>(1);
  size_t tb = 0;
  cub::DeviceSelect::Flagged(nullptr, tb, in, flags, out, d_cnt, n, A.s);
  void* tmp = A.get<char>(tb);
  if (!d_cnt || !tmp) return fail(CAPT_ENOMEM, "scratch allocation");
  CAPT_CUDA(cub::DeviceSelect::Flagged(tmp, tb, in, flags, out, d_cnt, n, A.s));
  CAPT_CUDA(cudaMemcpyAsync(count, d_cnt, 8, cudaMemcpyDeviceToHost, A.s));
  CAPT_CUDA(cudaStreamSynchronize(A.s));
  return CAPT_OK;
}

struct MaxOp {
  __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

bool next_perm(int* p, int k) {
  int i = k - 2;
  while (i >= 0 && p[i] > p[i + 1]) --i;
  if (i < 0) return false;
  int j = k - 1;
  while (p[j] < p[i]) --j;
  std::swap(p[i], p[j]);
  for (int a = i + 1, b = k - 1; a < b; ++a, --b) std::swap(p[a], p[b]);
  return true;
}

}  // namespace

}  // namespace capt

using namespace capt;

#define TRY(x)              \
  do {                      \
    int _rc = (x);          \
    if (_rc) return _rc;    \
  } while (0)

extern "C" int capt_filter_cloud(int device, int k, const float* points, int64_t n,
                                 double r_filter, int has_reach, const double* base,
                                 double max_reach, uint32_t flags, float* out_points,
                                 int64_t* n_out, void* stream) {
  if (!n_out) return fail(CAPT_EINVAL, "n_out is NULL");
  if (k < 1 || k > kMaxK) return fail(CAPT_EINVAL, "k must be 1..3 on the device path");
  if (n < 0) return fail(CAPT_EINVAL, "negative point count");
  if (std::isnan(r_filter) || std::isinf(r_filter))
    return fail(CAPT_EINVAL, "r_filter must be finite");
  if (has_reach && !(max_reach > 0)) return fail(CAPT_EINVAL, "max_reach must be > 0");
  if (n > (int64_t(1) << 30)) return fail(CAPT_EINVAL, "cloud too large");
  const bool host = flags & CAPT_HOST_IO;
  if (n == 0) {
    *n_out = 0;
    return CAPT_OK;
  }
  if (!points || !out_points) return fail(CAPT_EINVAL, "NULL array argument");
  CAPT_CUDA(cudaSetDevice(device));
  Arena A;
  A.s = static_cast<cudaStream_t>(stream);
  cudaStream_t s = A.s;
  const int G = grid_for(n, 256, 8);

  const float* d_in = points;
  if (host) {
    float* p = A.get<float>(size_t(n) * k);
    if (!p) return fail(CAPT_ENOMEM, "scratch allocation");
    CAPT_CUDA(cudaMemcpyAsync(p, points, sizeof(float) * n * k, cudaMemcpyHostToDevice, s));
    d_in = p;
  }
  // reach pre-pass (order preserving) -> pts0
  const float* pts0 = d_in;
  int64_t n0 = n;
  if (has_reach) {
    double b[3] = {0, 0, 0};
    for (int d = 0; d < k; ++d) b[d] = base[d];
    uint8_t* keep = A.get<uint8_t>(n);
    int32_t* sel = A.get<int32_t>(n);
    float* p0 = A.get<float>(size_t(n) * k);
    if (!keep || !sel || !p0) return fail(CAPT_ENOMEM, "scratch allocation");
    k_reach<<<G, 256, 0, s>>>(k, n, d_in, b[0], b[1], b[2], max_reach * max_reach, keep);
    TRY(select_flagged(A, keep, n, sel, &n0));
    if (n0) k_emit<<<grid_for(n0, 256, 8), 256, 0, s>>>(k, n0, sel, d_in, p0);
    pts0 = p0;
  }
  if (n0 == 0 || r_filter < 0) {  // empty after reach, or reach-only call
    if (n0) {
      if (host) CAPT_CUDA(cudaMemcpyAsync(out_points, pts0, sizeof(float) * n0 * k, cudaMemcpyDeviceToHost, s));
      else CAPT_CUDA(cudaMemcpyAsync(out_points, pts0, sizeof(float) * n0 * k, cudaMemcpyDeviceToDevice, s));
    }
    CAPT_CUDA(cudaStreamSynchronize(s));
    *n_out = n0;
    return CAPT_OK;
  }

  const double r2 = r_filter * r_filter;
  const int bits = (63 / k) < 21 ? 63 / k : 21;
  uint8_t* surv = A.get<uint8_t>(n0);
  int32_t* anchor_of = A.get<int32_t>(n0);
  int32_t* idx = A.get<int32_t>(n0);       // survivors, ascending index
  int32_t* idxS = A.get<int32_t>(n0);      // survivors, sorted (key, index)
  int32_t* final_idx = A.get<int32_t>(n0); // last pass's kept list (sorted order)
  uint64_t* keys = A.get<uint64_t>(n0);
  uint64_t* keysS = A.get<uint64_t>(n0);
  float* q = A.get<float>(size_t(n0) * k);
  uint32_t* mnmx = A.get<uint32_t>(6);
  int32_t* anc = A.get<int32_t>(n0);
  int32_t* kp = A.get<int32_t>(n0);
  uint8_t* mk = A.get<uint8_t>(n0 + 1);
  int levels = 1;
  while ((int64_t(1) << levels) < n0 + 1) ++levels;
  std::vector<int32_t*> J(levels + 1);
  for (auto& x : J) x = A.get<int32_t>(n0 + 1);
  if (!surv || !anchor_of || !idx || !idxS || !final_idx || !keys || !keysS || !q || !mnmx ||
      !anc || !kp || !mk)
    return fail(CAPT_ENOMEM, "scratch allocation");
  for (auto x : J)
    if (!x) return fail(CAPT_ENOMEM, "scratch allocation");
  CAPT_CUDA(cudaMemsetAsync(surv, 1, n0, s));
  CAPT_CUDA(cudaMemsetAsync(anchor_of, 0xff, sizeof(int32_t) * n0, s));

  // sort / scan temp storage (sized for n0)
  size_t tb_sort = 0, tb_scan = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb_sort, keys, keysS, idx, idxS, n0, 0, 64, s);
  cub::DeviceScan::InclusiveScan(nullptr, tb_scan, kp, anc, MaxOp(), n0, s);
  void* tmp = A.get<char>(tb_sort > tb_scan ? tb_sort : tb_scan);
  if (!tmp) return fail(CAPT_ENOMEM, "scratch allocation");

  int64_t m = n0;
  bool any_pass = false;
  int perm[3] = {0, 1, 2};
  do {
    if (m <= 1) break;
    // survivors in ascending original index
    TRY(select_flagged(A, surv, n0, idx, &m));
    const int Gm = grid_for(m, 256, 8);
    const uint32_t init[6] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0, 0, 0};
    CAPT_CUDA(cudaMemcpyAsync(mnmx, init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_bounds<<<Gm, 256, 0, s>>>(k, m, idx, pts0, mnmx, mnmx + 3);
    k_keys<<<Gm, 256, 0, s>>>(k, bits, m, idx, pts0, mnmx, mnmx + 3, perm[0], perm[1], perm[2],
                              keys);
    size_t t = tb_sort;
    const int end_bit = bits * k;
    CAPT_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t, keys, keysS, idx, idxS, m, 0, end_bit, s));
    k_gather<<<Gm, 256, 0, s>>>(k, m, idxS, pts0, q);
    // gap scan: next pointers, doubling tables, chain marking
    k_next<<<grid_for(m * 32, 256, 8), 256, 0, s>>>(k, m, q, r2, J[0]);
    CAPT_CUDA(cudaMemcpyAsync(J[0] + m, &m, 4, cudaMemcpyHostToDevice, s));  // sentinel J[m] = m
    int T = 1;
    while ((int64_t(1) << T) < m + 1) ++T;
    for (int lv = 0; lv + 1 < T; ++lv)
      k_jump<<<grid_for(m + 1, 256, 8), 256, 0, s>>>(m, J[lv], J[lv + 1]);
    CAPT_CUDA(cudaMemsetAsync(mk, 0, m + 1, s));
    CAPT_CUDA(cudaMemsetAsync(mk, 1, 1, s));
    for (int lv = T - 1; lv >= 0; --lv) k_mark<<<Gm, 256, 0, s>>>(m, J[lv], mk);
    // anchors: last kept position before each removed one
    k_kept_pos<<<Gm, 256, 0, s>>>(m, mk, kp);
    t = tb_scan;
    CAPT_CUDA(cub::DeviceScan::InclusiveScan(tmp, t, kp, anc, MaxOp(), m, s));
    k_drop<<<Gm, 256, 0, s>>>(m, mk, anc, idxS, anchor_of, surv);
    CAPT_CUDA(cudaGetLastError());
    int64_t nk = 0;
    TRY(select_values(A, idxS, mk, m, final_idx, &nk));
    m = nk;
    any_pass = true;
  } while (next_perm(perm, k));

  // final survivors in output order
  const int32_t* fin = final_idx;
  if (!any_pass) {  // n0 == 1: no pass ran
    TRY(select_flagged(A, surv, n0, idx, &m));
    fin = idx;
  }
  // orphan repair
  uint8_t* cand = A.get<uint8_t>(n0);
  int32_t* cidx = A.get<int32_t>(n0);
  uint8_t* orph = A.get<uint8_t>(n0);
  int32_t* oidx = A.get<int32_t>(n0);
  if (!cand || !cidx || !orph || !oidx) return fail(CAPT_ENOMEM, "scratch allocation");
  int64_t nc = 0, no = 0;
  if (any_pass) {
    k_candidates<<<grid_for(n0, 256, 8), 256, 0, s>>>(n0, surv, anchor_of, cand);
    TRY(select_flagged(A, cand, n0, cidx, &nc));
    if (nc) {
      // the grid over the survivors' box (the last pass's bounds cover them)
      uint32_t hb[6];
      CAPT_CUDA(cudaMemcpyAsync(hb, mnmx, sizeof(hb), cudaMemcpyDeviceToHost, s));
      CAPT_CUDA(cudaStreamSynchronize(s));
      OrphanGrid G;
      double ext = 0.0;
      for (int d = 0; d < 3; ++d) {
        G.lo[d] = 0.0;
        G.dims[d] = 1;
      }
      auto inv = [](uint32_t u) {
        u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
        float f;
        std::memcpy(&f, &u, 4);
        return double(f);
      };
      for (int d = 0; d < k; ++d) {
        G.lo[d] = inv(hb[d]);
        ext = std::max(ext, inv(hb[3 + d]) - G.lo[d]);
      }
      // cells of edge >= r (1 + 2^-20), at most ~2^8 per axis (keys fit in 32 bits)
      const double cs = std::max(r_filter * (1.0 + std::ldexp(1.0, -20)), ext / 256.0);
      G.inv_cs = cs > 0.0 ? 1.0 / cs : 0.0;
      if (!(cs > 0.0) || !std::isfinite(G.inv_cs)) G.inv_cs = 0.0;  // (one bucket)
      else
        for (int d = 0; d < k; ++d)
          G.dims[d] = int(std::min(258.0, std::floor((inv(hb[3 + d]) - G.lo[d]) / cs) + 2.0));
      // 1/cs rounded: the bucket map stays monotone; cs' = 1/inv_cs >= r still
      // holds up to a relative 2^-52, far inside the 2^-20 margin
      uint32_t* skey = A.get<uint32_t>(m);
      uint32_t* skeyS = A.get<uint32_t>(m);
      int32_t* sval = A.get<int32_t>(m);
      int32_t* svalS = A.get<int32_t>(m);
      if (!skey || !skeyS || !sval || !svalS) return fail(CAPT_ENOMEM, "scratch allocation");
      k_orphan_keys<<<grid_for(m, 256, 8), 256, 0, s>>>(k, G, m, fin, pts0, skey, sval);
      size_t t = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, t, skey, skeyS, sval, svalS, m, 0, 32, s);
      void* tmp2 = t <= tb_sort ? tmp : A.get<char>(t);
      if (!tmp2) return fail(CAPT_ENOMEM, "scratch allocation");
      CAPT_CUDA(cub::DeviceRadixSort::SortPairs(tmp2, t, skey, skeyS, sval, svalS, m, 0, 32, s));
      k_orphans<<<grid_for(nc, 128, 8), 128, 0, s>>>(k, G, nc, cidx, m, skeyS, svalS, pts0, r2,
                                                     orph);
      TRY(select_values(A, cidx, orph, nc, oidx, &no));
    }
  }
  float* d_out = out_points;
  if (host) {
    d_out = A.get<float>(size_t(m + no) * k);
    if (!d_out) return fail(CAPT_ENOMEM, "scratch allocation");
  }
  k_emit<<<grid_for(m, 256, 8), 256, 0, s>>>(k, m, fin, pts0, d_out);
  if (no) k_emit<<<grid_for(no, 256, 8), 256, 0, s>>>(k, no, oidx, pts0, d_out + m * k);
  CAPT_CUDA(cudaGetLastError());
  if (host)
    CAPT_CUDA(cudaMemcpyAsync(out_points, d_out, sizeof(float) * (m + no) * k,
                              cudaMemcpyDeviceToHost, s));
  CAPT_CUDA(cudaStreamSynchronize(s));
  *n_out = m + no;
  return CAPT_OK;
}
