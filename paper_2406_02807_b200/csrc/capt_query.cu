// Batched sphere-vs-point-cloud collision query (the hot path).
//
// Replaces collides_many (query.py:184-219) and collides_batch(...).
// any_collision (query.py:126-167).  Three kernels:
//   * warp    (this file, k_query_warp): one warp per sphere / lane group,
//     the latency path for batches too small to bin (see below).
//   * thread  (this file, k_query_direct, also the CAPT_STATS counter
//     kernel): one thread per sphere -- branchless Eytzinger
//     descent with the top 12 levels in shared memory (tree.py:266-273),
//     fp32 leaf-AABB reject (query.py:202-208), float4 SoA scan of the
//     affordance set (query.py:96-99), warp-ballot bit packing, and for
//     lane_width > 1 a per-group __ballot_sync vote after every 4-point chunk
//     (edge-validation early exit, query.py:152-160).
//   * binned  (capt_binned.cu): for large batches, spheres are bucketed by
//     leaf and every leaf's set is staged once in shared memory.
//
// Exactness.  The reference evaluates in float64 on fp32 data.  The descent
// compares fp32 values, so an fp32 compare is identical.  Squared distances
// are computed in fp32 with a proven relative error < 5u (u = 2^-24); any
// comparison within a relative band TAU = 2^-19 of r^2 is re-evaluated with
// the reference's exact float64 expression ((dx^2 + dy^2) + dz^2, no FMA,
// __dadd_rn/__dmul_rn), so verdicts are bit-identical to the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <type_traits>
#include <vector>

#include "capt_binned.cuh"
#include "capt_internal.cuh"
#include "capt_query_common.cuh"

namespace capt {

constexpr int kBlock = 256;

template <typename InT>
struct SphereIn;

template <>
struct SphereIn<float> {
  __device__ static void load(const void* c, const void* r, int64_t q, int k, double c64[3],
                              double& r64) {
    const float* cf = static_cast<const float*>(c);
    c64[0] = c64[1] = c64[2] = 0.0;
#pragma unroll
    for (int d = 0; d < kMaxK; ++d)
      if (d < k) c64[d] = double(__ldg(cf + q * k + d));
    r64 = double(__ldg(static_cast<const float*>(r) + q));
  }
};
template <>
struct SphereIn<double> {
  __device__ static void load(const void* c, const void* r, int64_t q, int k, double c64[3],
                              double& r64) {
    const double* cd = static_cast<const double*>(c);
    c64[0] = c64[1] = c64[2] = 0.0;
#pragma unroll
    for (int d = 0; d < kMaxK; ++d)
      if (d < k) c64[d] = __ldg(cd + q * k + d);
    r64 = __ldg(static_cast<const double*>(r) + q);
  }
};

// Sphere status in the direct kernel
enum : int { ST_FALSE = 0, ST_TRUE = 1, ST_SCAN = 2, ST_SLOW = 3, ST_SKIP = 4 };

template <typename InT, bool kStats>
__global__ void __launch_bounds__(kBlock)
    k_query_direct(DevTree t, const void* __restrict__ centers, const void* __restrict__ radii,
                   int64_t n, int L, const uint8_t* __restrict__ lane_mask, uint32_t flags,
                   uint32_t* __restrict__ out_bits, int64_t n_words,
                   unsigned long long* __restrict__ counters,
                   unsigned long long* __restrict__ first_bad) {
  __shared__ float sT[kSmemNodes];
  __shared__ uint32_t sWords[kBlock / 32];
  const int n_smem = int(t.n - 1 < kSmemNodes ? t.n - 1 : kSmemNodes);
  for (int i = threadIdx.x; i < n_smem; i += blockDim.x) sT[i] = t.T[i];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const bool prefilter = flags & CAPT_PREFILTER;
  const bool check = flags & CAPT_CHECK_RADII;
  const uint32_t seg = (L >= 32) ? 0xffffffffu : ((1u << L) - 1u);
  const uint32_t my_seg = seg << ((lane / L) * L);
  const int64_t n_tiles = (n + kBlock - 1) / kBlock;

  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t q = tile * kBlock + threadIdx.x;
    bool valid = q < n;
    if (valid && lane_mask) valid = lane_mask[q] != 0;
    double c64[3] = {0.0, 0.0, 0.0}, r64 = 0.0;
    if (valid) SphereIn<InT>::load(centers, radii, q, t.k, c64, r64);
    if (valid && check && (r64 < t.r_min || r64 > t.r_max))
      atomicMin(first_bad, static_cast<unsigned long long>(q));

    int status = ST_FALSE;
    int64_t leaf = 0;
    uint2 set = make_uint2(0, 0);
    float cx = 0.f, cy = 0.f, cz = 0.f, r2 = 0.f, loB = 0.f, hiB = 0.f;
    bool passed = false;  // AABB passed (scanned)
    bool leaf_ok = false; // reached the AABB test (finite centre)
    if (valid) {
      if constexpr (std::is_same<InT, float>::value) {
        const float cf[3] = {float(c64[0]), float(c64[1]), float(c64[2])};
        leaf = descend_t<float>(t, sT, n_smem, cf);
      } else {
        leaf = descend(t, sT, n_smem, c64);
      }
      status = classify(t, leaf, c64, r64, prefilter, cx, cy, cz, r2, loB, hiB);
      passed = status == ST_SCAN || status == ST_SLOW;
      leaf_ok = passed || prefilter;
      if (passed) set = __ldg(t.set + leaf);
    }

    // ---- scan: warp-uniform loop over 4-point chunks ----
    bool hit = false, amb = false, bnd_cand = false;
    uint32_t pos = 0;
    const float* base = reinterpret_cast<const float*>(t.data + set.x);
    const uint32_t m4 = (set.y + 3u) & ~3u;
    while (__any_sync(0xffffffffu, status == ST_SCAN)) {
      if (status == ST_SCAN) {
        const float4 px = __ldg(reinterpret_cast<const float4*>(base + pos));
        const float4 py = __ldg(reinterpret_cast<const float4*>(base + m4 + pos));
        const float4 pz = __ldg(reinterpret_cast<const float4*>(base + 2 * m4 + pos));
        test4(px, py, pz, cx, cy, cz, r2, loB, hiB, hit, amb, bnd_cand, kStats);
        pos += 4;
        if (hit && !kStats) status = ST_TRUE;
        else if (pos >= m4) status = hit ? ST_TRUE : (amb ? ST_SLOW : ST_FALSE);
      }
      if (!kStats && L > 1) {
        const uint32_t done = __ballot_sync(0xffffffffu, status == ST_TRUE);
        if ((done & my_seg) && status == ST_SCAN) status = ST_SKIP;
      }
    }
    // ---- float64 fix-up (exact reference arithmetic) ----
    if (!kStats && L > 1) {
      const uint32_t done = __ballot_sync(0xffffffffu, status == ST_TRUE);
      if ((done & my_seg) && status == ST_SLOW) status = ST_SKIP;
    }
    bool slow = false, boundary = false;
    if (status == ST_SLOW || (kStats && bnd_cand)) {
      slow = status == ST_SLOW;
      bool b = false;
      const bool h64 = scan_f64(t, set, c64, r64, kStats ? &b : nullptr);
      status = h64 ? ST_TRUE : ST_FALSE;
      boundary = b;
    }
    const bool verdict = status == ST_TRUE;

    // ---- bit packing ----
    const uint32_t bits = __ballot_sync(0xffffffffu, verdict);
    uint32_t gbits = bits;
    if (L > 1) {
      gbits = 0;
      for (int j = 0; j < 32 / L; ++j)
        if ((bits >> (j * L)) & seg) gbits |= 1u << j;
    }
    if (L <= 8) {
      if (threadIdx.x < kBlock / 32) sWords[threadIdx.x] = 0;
      __syncthreads();
      if (lane == 0) {
        const int per = 32 / L;                   // group bits per warp
        const int bitpos = warp * per;            // within the tile
        atomicOr(&sWords[bitpos >> 5], gbits << (bitpos & 31));
      }
      __syncthreads();
      const int words_per_tile = (kBlock / L) / 32;
      if (threadIdx.x < words_per_tile) {
        const int64_t w = tile * words_per_tile + threadIdx.x;
        if (w < n_words) out_bits[w] = sWords[threadIdx.x];
      }
    } else if (lane == 0 && gbits) {
      const int64_t g0 = (tile * kBlock + warp * 32) / L;
      atomicOr(out_bits + (g0 >> 5), gbits << (g0 & 31));
    }

    // ---- counters (reference semantics) ----
    if (kStats) {
      unsigned long long c_hit, c_bnd = boundary, c_scan = 0, c_fix = slow;
      unsigned long long c_rej = (valid && !passed && leaf_ok) ? 1ull : 0ull;
      if (L == 1) {
        c_hit = verdict;
        c_scan = passed ? set.y : 0;
      } else {
        // lanes in order up to and including the first colliding lane
        const uint32_t segbits = bits & my_seg;
        const int first = segbits ? __ffs(segbits) - 1 : 32;
        c_scan = (passed && lane <= first) ? set.y : 0;
        c_hit = ((lane % L) == 0) && (segbits != 0);
      }
      c_hit = warp_sum(c_hit);
      c_bnd = warp_sum(c_bnd);
      c_scan = warp_sum(c_scan);
      c_fix = warp_sum(c_fix);
      c_rej = warp_sum(c_rej);
      if (lane == 0) {
        atomicAdd(counters + 4, c_rej);
        atomicAdd(counters + 0, c_hit);
        atomicAdd(counters + 1, c_bnd);
        atomicAdd(counters + 2, c_scan);
        atomicAdd(counters + 3, c_fix);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Warp-per-sphere kernel (latency path for batches too small to bin).
//
// One warp owns one lane group (L spheres, scanned in lane order with the
// reference's early exit, query.py:152-160).  For each sphere the 32 lanes
//   * descend 5 Eytzinger levels per round: lane j loads node j of the
//     31-node subtree under the current node, the path is then walked with
//     shuffles -- one L1/L2 round trip per 5 levels instead of per level;
//   * scan the affordance set cooperatively, 128 points per iteration
//     (coalesced SoA loads), with a warp vote after every iteration;
//   * re-run the exact float64 scan cooperatively for band/slow spheres.
// ---------------------------------------------------------------------------
template <typename InT>
__global__ void __launch_bounds__(kBlock)
    k_query_warp(DevTree t, const void* __restrict__ centers, const void* __restrict__ radii,
                 int64_t n, int L, const uint8_t* __restrict__ lane_mask, uint32_t flags,
                 uint32_t* __restrict__ out_bits, unsigned long long* __restrict__ first_bad) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const bool prefilter = flags & CAPT_PREFILTER;
  const bool check = flags & CAPT_CHECK_RADII;
  const int64_t n_groups = n / L;
  for (int64_t g = warp; g < n_groups; g += nwarps) {
    bool verdict = false;
    for (int l = 0; l < L; ++l) {
      const int64_t q = g * L + l;
      if (lane_mask && !lane_mask[q]) continue;
      double c64[3], r64;
      SphereIn<InT>::load(centers, radii, q, t.k, c64, r64);
      if (check && lane == 0 && (r64 < t.r_min || r64 > t.r_max))
        atomicMin(first_bad, static_cast<unsigned long long>(q));
      if (verdict) continue;  // radii of later lanes are still checked
      int64_t leaf;
      if constexpr (std::is_same<InT, float>::value) {
        const float cf[3] = {float(c64[0]), float(c64[1]), float(c64[2])};
        leaf = warp_descend<float>(t, cf, lane);
      } else {
        leaf = warp_descend<double>(t, c64, lane);
      }
      const uint2 set = __ldg(t.set + leaf);
      const float4 rp = __ldg(t.rep + leaf);
      float cx, cy, cz, r2, loB, hiB;
      const int status = classify(t, leaf, c64, r64, prefilter, cx, cy, cz, r2, loB, hiB);
      if (status == ST_FALSE) continue;
      int v = 2;
      if (status == ST_SCAN) {
        // representative probe: row 0 of the set owns the cell holding the
        // centre; a definite fp32 hit (same band as the scan) ends the sphere
        const float dx = cx - rp.x, dy = cy - rp.y, dz = cz - rp.z;
        v = fmaf(dz, dz, fmaf(dy, dy, dx * dx)) <= loB
                ? 1
                : warp_scan_f32(t, set, cx, cy, cz, loB, hiB, lane);
      }
      verdict = (v == 1) || (v == 2 && warp_scan_f64(t, set, c64, r64, lane));
    }
    if (verdict && lane == 0) atomicOr(out_bits + (g >> 5), 1u << (g & 31));
  }
}


// ---------------------------------------------------------------------------
// Hybrid unbinned kernel (fp32 inputs, k = 3): the classifier of the binned
// pipeline's K1, one sphere per thread -- 13 shared-memory levels, one
// 256-bit probe record load, conservative AABB reject, representative probe,
// group resolution by ballot -- then the warp scans the sets of its still
// unresolved spheres one after the other, cooperatively (warp_scan_f32 /
// warp_scan_f64).  Every sphere's descent runs in parallel; only the rare
// unresolved ones pay a serial scan.
// ---------------------------------------------------------------------------
constexpr int kHybSmem = 8191;  // top 13 levels
constexpr int64_t kHybridMin = int64_t(1) << 15;
__global__ void __launch_bounds__(kBlock) k_query_hybrid(
    DevTree t, const float* __restrict__ centers, const float* __restrict__ radii, int64_t n,
    int L, const uint8_t* __restrict__ lane_mask, uint32_t flags, uint32_t* __restrict__ out_bits,
    unsigned long long* __restrict__ first_bad, float rlo_f, float rhi_f) {
  __shared__ float sT[kHybSmem];
  const int n_smem = int(t.n - 1 < kHybSmem ? t.n - 1 : kHybSmem);
  for (int i = threadIdx.x; i < n_smem; i += blockDim.x) sT[i] = t.T[i];
  __syncthreads();
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(sT));
  const int dsm = t.depth < 13 ? t.depth : 13;
  const int lane = threadIdx.x & 31;
  const bool prefilter = flags & CAPT_PREFILTER;
  const bool check = flags & CAPT_CHECK_RADII;
  const unsigned seg = L >= 32 ? 0xffffffffu : ((1u << L) - 1u) << ((lane / L) * L);
  const float band_lo = 1.0f - kTau, band_hi = 1.0f + kTau;
  const float INF = __int_as_float(0x7f800000);
  const int64_t n_pad = (n + 31) & ~int64_t(31);
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q - lane < n_pad;
       q += int64_t(gridDim.x) * blockDim.x) {
    bool valid = q < n;
    if (valid && lane_mask) valid = lane_mask[q] != 0;
    float cx = 0.f, cy = 0.f, cz = 0.f, r = 0.f;
    if (valid) {
      cx = __ldg(centers + 3 * q);
      cy = __ldg(centers + 3 * q + 1);
      cz = __ldg(centers + 3 * q + 2);
      r = __ldg(radii + q);
    }
    if (check && valid && (r < rlo_f || r > rhi_f))
      atomicMin(first_bad, static_cast<unsigned long long>(q));
    // descent: 13 shared levels on absolute addresses, the rest from T
    unsigned ad = sbase;
    int s = 0;
    {
      const unsigned k0 = 4u - sbase, k1 = 8u - sbase;
      for (; s + 3 <= dsm; s += 3) {
        ad = 2 * ad + (cx > lds_f32(ad) ? k1 : k0);
        ad = 2 * ad + (cy > lds_f32(ad) ? k1 : k0);
        ad = 2 * ad + (cz > lds_f32(ad) ? k1 : k0);
      }
    }
    unsigned off = ad - sbase;
    for (; s < dsm; ++s) {
      const int ax = s % 3;
      const float c = ax == 0 ? cx : (ax == 1 ? cy : cz);
      off = 2 * off + (c > lds_f32(sbase + off) ? 8u : 4u);
    }
    for (; s < t.depth; ++s) {
      const int ax = s % 3;
      const float c = ax == 0 ? cx : (ax == 1 ? cy : cz);
      off = 2 * off + (c > __ldg(t.T + (off >> 2)) ? 8u : 4u);
    }
    const int64_t leaf = int64_t(off >> 2) - (t.n - 1);
    // classification (see k_bin_count3: conservative AABB, probe)
    const float r2 = r * r;
    const bool cfin = isfinite(cx) && isfinite(cy) && isfinite(cz);
    const bool fast = cfin && r2 >= kR2Min && r2 <= kR2Max;
    int st = fast ? 2 : ((!cfin && isfinite(r)) ? 0 : 3);
    st = valid ? st : 0;
    float pr[8];
    ld_v8(t.probe + 8 * leaf, pr);
    if (prefilter) {
      const float2 l01 = h2f2(pr[3]), l2h0 = h2f2(pr[4]), h12 = h2f2(pr[5]);
      const float rx = fmaxf(fmaxf(l01.x - cx, 0.f), cx - l2h0.y);
      const float ry = fmaxf(fmaxf(l01.y - cy, 0.f), cy - h12.x);
      const float rz = fmaxf(fmaxf(l2h0.x - cz, 0.f), cz - h12.y);
      const float ss = fmaf(rz, rz, fmaf(ry, ry, rx * rx));
      st = (fast && ss > r2 * band_hi) ? 0 : st;
    }
    const float dx = cx - pr[0], dy = cy - pr[1], dz = cz - pr[2];
    bool verdict = st == 2 && fmaf(dz, dz, fmaf(dy, dy, dx * dx)) <= r2 * band_lo;
    // unresolved spheres of unresolved groups: cooperative scans
    unsigned done_groups = __ballot_sync(0xffffffffu, verdict);
    unsigned todo = __ballot_sync(0xffffffffu, (st == 2 || st == 3) && !verdict);
    const unsigned leaf_lo = unsigned(leaf);
    while (true) {
      // drop lanes whose group already has a hit
      if (L > 1) {
        unsigned resolved = 0;
        for (int g0 = 0; g0 < 32; g0 += L) {
          const unsigned m = (L >= 32 ? 0xffffffffu : ((1u << L) - 1u)) << g0;
          if (done_groups & m) resolved |= m;
        }
        todo &= ~resolved;
      }
      if (!todo) break;
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const float sx = __shfl_sync(0xffffffffu, cx, src);
      const float sy = __shfl_sync(0xffffffffu, cy, src);
      const float sz = __shfl_sync(0xffffffffu, cz, src);
      const float sr = __shfl_sync(0xffffffffu, r, src);
      const int sst = __shfl_sync(0xffffffffu, st, src);
      const unsigned sleaf = __shfl_sync(0xffffffffu, leaf_lo, src);
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
        done_groups |= 1u << src;
      }
    }
    // bit packing: one bit per lane group (atomicOr into cleared words)
    const unsigned bits = __ballot_sync(0xffffffffu, verdict);
    if (lane == 0 && bits) {
      const int64_t wbase = q - lane;  // first sphere of this warp
      if (L == 1) {
        atomicOr(out_bits + (wbase >> 5), bits);
      } else {
        uint32_t gb = 0;
        for (int j = 0; j < 32 / L; ++j)
          if ((bits >> (j * L)) & (L >= 32 ? 0xffffffffu : ((1u << L) - 1u))) gb |= 1u << j;
        const int64_t g0 = wbase / L;
        atomicOr(out_bits + (g0 >> 5), gb << (g0 & 31));
      }
    }
    (void)seg;
  }
}

template <typename InT>
__global__ void k_leaf_indices(DevTree t, const void* __restrict__ centers, int64_t n,
                               int64_t* __restrict__ out) {
  __shared__ float sT[kSmemNodes];
  const int n_smem = int(t.n - 1 < kSmemNodes ? t.n - 1 : kSmemNodes);
  for (int i = threadIdx.x; i < n_smem; i += blockDim.x) sT[i] = t.T[i];
  __syncthreads();
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
       q += int64_t(gridDim.x) * blockDim.x) {
    double c64[3], r64;
    SphereIn<InT>::load(centers, centers, q, t.k, c64, r64);
    out[q] = descend(t, sT, n_smem, c64);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

struct HostIO {
  // device mirrors of host arguments (CAPT_HOST_IO)
  void* centers = nullptr;
  void* radii = nullptr;
  uint8_t* mask = nullptr;
  uint32_t* bits = nullptr;
  unsigned long long* counters = nullptr;
  unsigned long long* first_bad = nullptr;
  cudaStream_t s = nullptr;
  ~HostIO() {
    if (centers) cudaFreeAsync(centers, s);
    if (radii) cudaFreeAsync(radii, s);
    if (mask) cudaFreeAsync(mask, s);
    if (bits) cudaFreeAsync(bits, s);
    if (counters) cudaFreeAsync(counters, s);
    if (first_bad) cudaFreeAsync(first_bad, s);
  }
};

int launch_direct(const DevTree& t, const void* centers, const void* radii, int64_t n, int L,
                  const uint8_t* mask, uint32_t flags, uint32_t* bits, int64_t n_words,
                  unsigned long long* counters, unsigned long long* first_bad, cudaStream_t s) {
  const bool f64 = flags & CAPT_INPUT_F64;
  const bool stats = flags & CAPT_STATS;
  // hybrid for batches with enough warps to hide its serial per-warp scans
  // (measured crossover with the warp kernel between 16 K and 64 K spheres)
  const bool hybrid_ok = !f64 && t.k == 3 && !(flags & CAPT_MODE_WARP) &&
                         (n >= kHybridMin || (flags & CAPT_MODE_DIRECT));
  if (!stats && !(flags & CAPT_MODE_THREAD) && hybrid_ok) {
    if (L <= 8) CAPT_CUDA(cudaMemsetAsync(bits, 0, 4 * (n_words ? n_words : 1), s));
    float lo = float(t.r_min), hi = float(t.r_max);
    if (double(lo) < t.r_min) lo = nextafterf(lo, INFINITY);
    if (double(hi) > t.r_max) hi = nextafterf(hi, -INFINITY);
    k_query_hybrid<<<grid_for(n, kBlock, 4), kBlock, 0, s>>>(
        t, static_cast<const float*>(centers), static_cast<const float*>(radii), n, L, mask, flags,
        bits, first_bad, lo, hi);
    CAPT_CUDA(cudaGetLastError());
    note_launches(1);
    return CAPT_OK;
  }
  if (!stats && !(flags & CAPT_MODE_THREAD)) {
    if (L <= 8) CAPT_CUDA(cudaMemsetAsync(bits, 0, 4 * (n_words ? n_words : 1), s));
    const int grid = grid_for((n / L) * 32, kBlock, 8);
    if (f64)
      k_query_warp<double><<<grid, kBlock, 0, s>>>(t, centers, radii, n, L, mask, flags, bits, first_bad);
    else
      k_query_warp<float><<<grid, kBlock, 0, s>>>(t, centers, radii, n, L, mask, flags, bits, first_bad);
    CAPT_CUDA(cudaGetLastError());
    note_launches(1);
    return CAPT_OK;
  }
  const int64_t n_tiles = (n + kBlock - 1) / kBlock;
  const int grid = grid_for(n_tiles * kBlock, kBlock, 8);
#define LAUNCH(T, S) \
  k_query_direct<T, S><<<grid, kBlock, 0, s>>>(t, centers, radii, n, L, mask, flags, bits, n_words, counters, first_bad)
  if (f64) {
    if (stats) LAUNCH(double, true); else LAUNCH(double, false);
  } else {
    if (stats) LAUNCH(float, true); else LAUNCH(float, false);
  }
#undef LAUNCH
  CAPT_CUDA(cudaGetLastError());
  note_launches(1);
  return CAPT_OK;
}

// ---------------------------------------------------------------------------
// float64 inputs on the clearance-field pipeline.  Reference callers pass
// float64 arrays (query.py:192-193); when a sphere's four values are fp32
// values, the fp32 kernels see exactly the reference's inputs.  k_split_f64
// converts every sphere, marks the exact ones valid for the field pipeline
// (which then skips the others as masked lanes) and lists the inexact ones;
// k_list_f64 answers the listed spheres with the reference's float64
// arithmetic (band check, descent, AABB prefilter, set scan) and ORs their
// verdicts into the words the field pipeline wrote.  A group's bit is the OR
// of its valid lanes' verdicts either way (query.py:126-167).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_split_f64(const double* __restrict__ c,
                                                      const double* __restrict__ r, int64_t n,
                                                      const uint8_t* __restrict__ umask,
                                                      float* __restrict__ c32,
                                                      float* __restrict__ r32,
                                                      uint8_t* __restrict__ m32,
                                                      uint32_t* __restrict__ list,
                                                      uint32_t* __restrict__ list_n) {
  const int lane = threadIdx.x & 31;
  for (int64_t q0 = int64_t(blockIdx.x) * blockDim.x; q0 < n; q0 += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = q0 + threadIdx.x;
    bool inexact = false;
    if (q < n) {
      const double v[4] = {__ldcs(c + 3 * q), __ldcs(c + 3 * q + 1), __ldcs(c + 3 * q + 2),
                           __ldcs(r + q)};
      bool exact = true;
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        const float f = __double2float_rn(v[d]);
        exact &= double(f) == v[d] || (isnan(v[d]) && isnan(f));
        if (d < 3) c32[3 * q + d] = f; else r32[q] = f;
      }
      const bool valid = !umask || umask[q];
      m32[q] = uint8_t(valid && exact);
      inexact = valid && !exact;
    }
    const unsigned b = __ballot_sync(0xffffffffu, inexact);
    if (b) {
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(list_n, unsigned(__popc(b)));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (inexact) list[base + __popc(b & ((1u << lane) - 1u))] = uint32_t(q);
    }
  }
}

__global__ void __launch_bounds__(kBlock) k_list_f64(DevTree t, const double* __restrict__ c,
                                                     const double* __restrict__ r, int L,
                                                     uint32_t flags,
                                                     const uint32_t* __restrict__ list,
                                                     const uint32_t* __restrict__ list_n,
                                                     uint32_t* __restrict__ bits,
                                                     unsigned long long* __restrict__ first_bad) {
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const bool prefilter = flags & CAPT_PREFILTER;
  const bool check = flags & CAPT_CHECK_RADII;
  const uint32_t m = *list_n;
  for (uint32_t e = warp; e < m; e += nwarps) {
    const uint32_t q = list[e];
    const uint32_t g = q / uint32_t(L);
    double c64[3], r64;
    SphereIn<double>::load(c, r, q, 3, c64, r64);
    // (query.py:194-197: a NaN radius is not flagged)
    if (check && lane == 0 && (r64 < t.r_min || r64 > t.r_max))
      atomicMin(first_bad, static_cast<unsigned long long>(q));
    // (warp-uniform: lane 0's read decides for the warp)
    if (L > 1 && __shfl_sync(0xffffffffu, (__ldcg(bits + (g >> 5)) >> (g & 31)) & 1u, 0)) continue;
    const int64_t leaf = warp_descend<double>(t, c64, lane);
    const uint2 set = __ldg(t.set + leaf);
    float cx, cy, cz, r2, loB, hiB;
    const int status = classify(t, leaf, c64, r64, prefilter, cx, cy, cz, r2, loB, hiB);
    if (status == ST_FALSE) continue;
    int v = 2;
    if (status == ST_SCAN) v = warp_scan_f32(t, set, cx, cy, cz, loB, hiB, lane);
    const bool verdict = (v == 1) || (v == 2 && warp_scan_f64(t, set, c64, r64, lane));
    if (verdict && lane == 0) atomicOr(bits + (g >> 5), 1u << (g & 31));
  }
}

static int launch_field_f64(const DevTree& t, const void* d_c, const void* d_r, int64_t n, int L,
                            const uint8_t* d_m, uint32_t fl, uint32_t* d_bits, int64_t n_words,
                            unsigned long long* d_bad, cudaStream_t s) {
  struct Scratch {
    cudaStream_t s;
    char* p = nullptr;
    ~Scratch() {
      if (p) cudaFreeAsync(p, s);
    }
  } sc{s};
  const size_t nn = size_t(n);
  const size_t off_r = 12 * nn, off_m = 16 * nn, off_l = (17 * nn + 15) & ~size_t(15);
  CAPT_CUDA(dmalloc(&sc.p, off_l + 4 * nn + 16, s));
  float* c32 = reinterpret_cast<float*>(sc.p);
  float* r32 = reinterpret_cast<float*>(sc.p + off_r);
  uint8_t* m32 = reinterpret_cast<uint8_t*>(sc.p + off_m);
  uint32_t* list_n = reinterpret_cast<uint32_t*>(sc.p + off_l);
  uint32_t* list = list_n + 4;
  CAPT_CUDA(cudaMemsetAsync(list_n, 0, 4, s));
  k_split_f64<<<grid_for(n, kBlock, 8), kBlock, 0, s>>>(static_cast<const double*>(d_c),
                                                        static_cast<const double*>(d_r), n, d_m,
                                                        c32, r32, m32, list, list_n);
  CAPT_CUDA(cudaGetLastError());
  note_launches(1);
  const int rc = launch_field(t, c32, r32, n, L, m32, fl & ~uint32_t(CAPT_INPUT_F64), d_bits,
                              n_words, d_bad, s);
  if (rc) return rc;
  k_list_f64<<<grid_for(int64_t(n) * 32, kBlock, 4), kBlock, 0, s>>>(
      t, static_cast<const double*>(d_c), static_cast<const double*>(d_r), L, fl, list, list_n,
      d_bits, d_bad);
  CAPT_CUDA(cudaGetLastError());
  note_launches(1);
  return CAPT_OK;
}

// One query over device buffers on stream s (direct or binned pipeline).
int query_device(const DevTree& t, const void* d_c, const void* d_r, int64_t n, int L,
                 const uint8_t* d_m, uint32_t flags, uint32_t* d_bits,
                 unsigned long long* d_cnt, unsigned long long* d_bad, cudaStream_t s) {
  const int64_t n_words = (n / L + 31) / 32;
  if (d_bad) CAPT_CUDA(cudaMemsetAsync(d_bad, 0xff, 8, s));
  if (d_cnt && (flags & CAPT_STATS)) CAPT_CUDA(cudaMemsetAsync(d_cnt, 0, 48, s));
  if (L > 8 || n == 0) CAPT_CUDA(cudaMemsetAsync(d_bits, 0, 4 * (n_words ? n_words : 1), s));
  if (n == 0) return CAPT_OK;
  uint32_t fl = flags;
  if (!d_bad) fl &= ~CAPT_CHECK_RADII;
  if (field_eligible(t, n, fl))
    return launch_field(t, d_c, d_r, n, L, d_m, fl, d_bits, n_words, d_bad, s);
  if ((fl & CAPT_INPUT_F64) && field_eligible(t, n, fl & ~uint32_t(CAPT_INPUT_F64)))
    return launch_field_f64(t, d_c, d_r, n, L, d_m, fl, d_bits, n_words, d_bad, s);
  if (fl & CAPT_MODE_FIELD)
    return fail(CAPT_EINVAL, "clearance-field pipeline unavailable for this tree/input");
  return binned_preferred(t, n, fl)
             ? launch_binned(t, d_c, d_r, n, L, d_m, fl, d_bits, n_words, d_bad, s)
             : launch_direct(t, d_c, d_r, n, L, d_m, fl, d_bits, n_words, d_cnt, d_bad, s);
}

// Host-buffer queries larger than one chunk: a two-stream pipeline so the
// host->device copy of chunk i+1 overlaps the kernels of chunk i.  Chunks are
// multiples of 32 lane groups, so every chunk owns whole verdict words; they
// are written into one device array copied back once at the end (a
// per-chunk copy into pageable user memory would block the host thread and
// serialise the pipeline).
//
// Each call takes a PipeState (two worker streams, events, a pinned buffer
// for the per-chunk first_bad and counters) from a per-device free list, so
// concurrent calls on one tree never share them (a Capt is safe for any
// number of concurrent readers, tree.py:67-71).
struct PipeState {
  static constexpr int kMaxChunks = 1024;
  cudaStream_t w[2] = {nullptr, nullptr};
  cudaEvent_t start = nullptr, done[2] = {nullptr, nullptr};
  unsigned long long* pinned = nullptr;  // per chunk: first_bad + 6 counters
  // pageable inputs: two pinned staging buffers (centres + radii + mask of
  // one chunk each), filled by host threads while the other one's copy and
  // kernels run; staged[b] is recorded after the copy out of buffer b
  char* stage[2] = {nullptr, nullptr};
  size_t stage_bytes = 0;
  cudaEvent_t staged[2] = {nullptr, nullptr};
};

// memcpy with up to `threads` host threads (pageable -> pinned staging)
static void parallel_copy(char* dst, const char* src, size_t bytes, int threads) {
  constexpr size_t kMinPerThread = size_t(8) << 20;
  const int t = int(std::min<size_t>(threads, std::max<size_t>(1, bytes / kMinPerThread)));
  if (t <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t per = (bytes + t - 1) / t;
  for (int i = 1; i < t; ++i) {
    const size_t a = per * i, b = std::min(bytes, a + per);
    if (a < b) th.emplace_back([=] { std::memcpy(dst + a, src + a, b - a); });
  }
  std::memcpy(dst, src, std::min(per, bytes));
  for (auto& x : th) x.join();
}

static bool is_pageable(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();  // (clear the sticky-free error of a plain host pointer)
    return true;
  }
  return at.type == cudaMemoryTypeUnregistered;
}

struct PipePool {
  std::mutex mu;
  std::vector<PipeState*> free_list;
};
static PipePool g_pipes[kMaxDevices];

static PipeState* pipe_acquire(int device) {
  if (device < 0 || device >= kMaxDevices) return nullptr;
  {
    std::lock_guard<std::mutex> lk(g_pipes[device].mu);
    auto& fl = g_pipes[device].free_list;
    if (!fl.empty()) {
      PipeState* p = fl.back();
      fl.pop_back();
      return p;
    }
  }
  PipeState* p = new PipeState();
  bool ok = true;
  for (int i = 0; i < 2; ++i) {
    ok = ok && cudaStreamCreateWithFlags(&p->w[i], cudaStreamNonBlocking) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&p->done[i], cudaEventDisableTiming) == cudaSuccess;
  }
  ok = ok && cudaEventCreateWithFlags(&p->start, cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaHostAlloc(reinterpret_cast<void**>(&p->pinned),
                           sizeof(unsigned long long) * 7 * PipeState::kMaxChunks,
                           cudaHostAllocDefault) == cudaSuccess;
  if (!ok) {
    for (int i = 0; i < 2; ++i) {
      if (p->w[i]) cudaStreamDestroy(p->w[i]);
      if (p->done[i]) cudaEventDestroy(p->done[i]);
    }
    if (p->start) cudaEventDestroy(p->start);
    if (p->pinned) cudaFreeHost(p->pinned);
    delete p;
    return nullptr;
  }
  return p;
}

static void pipe_release(int device, PipeState* p) {
  std::lock_guard<std::mutex> lk(g_pipes[device].mu);
  g_pipes[device].free_list.push_back(p);
}

int query_host_pipelined(const capt_tree* tree, const DevTree& t, const void* centers,
                         const void* radii, int64_t n, int L, const uint8_t* lane_mask,
                         uint32_t flags, uint32_t* out_bits, uint64_t* counters,
                         int64_t* first_bad, cudaStream_t s, int64_t chunk) {
  const size_t in_elem = (flags & CAPT_INPUT_F64) ? sizeof(double) : sizeof(float);
  const int64_t n_chunks = (n + chunk - 1) / chunk;
  if (n_chunks > PipeState::kMaxChunks) return fail(CAPT_EINVAL, "batch too large for the pipeline");
  PipeState* p = pipe_acquire(tree->device);
  if (!p) return fail(CAPT_ECUDA, "pipeline streams unavailable");
  // every exit path: device buffers freed in stream order, the worker
  // streams joined into s, s drained, the state returned to the pool
  struct Call {
    PipeState* p;
    int device;
    cudaStream_t s;
    void* c[2] = {nullptr, nullptr};
    void* r[2] = {nullptr, nullptr};
    uint8_t* m[2] = {nullptr, nullptr};
    unsigned long long* aux[2] = {nullptr, nullptr};  // first_bad + 6 counters
    uint32_t* d_bits = nullptr;
    ~Call() {
      for (int i = 0; i < 2; ++i) {
        if (c[i]) cudaFreeAsync(c[i], p->w[i]);
        if (r[i]) cudaFreeAsync(r[i], p->w[i]);
        if (m[i]) cudaFreeAsync(m[i], p->w[i]);
        if (aux[i]) cudaFreeAsync(aux[i], p->w[i]);
        cudaEventRecord(p->done[i], p->w[i]);
        cudaStreamWaitEvent(s, p->done[i], 0);
      }
      if (d_bits) cudaFreeAsync(d_bits, s);
      cudaStreamSynchronize(s);
      cudaStreamSynchronize(p->w[0]);
      cudaStreamSynchronize(p->w[1]);
      pipe_release(device, p);
    }
  } call{p, tree->device, s};
  const int64_t words_total = (n / L + 31) / 32;
  CAPT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&call.d_bits), 4 * words_total, s));
  CAPT_CUDA(cudaEventRecord(p->start, s));
  for (int i = 0; i < 2; ++i) {
    cudaStream_t w = p->w[i];
    CAPT_CUDA(cudaStreamWaitEvent(w, p->start, 0));
    CAPT_CUDA(cudaMallocAsync(&call.c[i], in_elem * t.k * chunk, w));
    CAPT_CUDA(cudaMallocAsync(&call.r[i], in_elem * chunk, w));
    if (lane_mask) CAPT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&call.m[i]), chunk, w));
    CAPT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&call.aux[i]), 8 * 7, w));
  }
  // pageable (plain malloc'd / numpy) inputs go through pinned staging
  // buffers filled by host threads: a pageable cudaMemcpyAsync is staged by
  // the driver one thread at a time and blocks the calling thread
  const bool pageable = is_pageable(centers) || is_pageable(radii) ||
                        (lane_mask && is_pageable(lane_mask));
  const size_t cb = in_elem * t.k * size_t(chunk), rb = in_elem * size_t(chunk);
  const size_t need = cb + rb + (lane_mask ? size_t(chunk) : 0);
  const int nthreads = int(std::min(8u, std::max(1u, std::thread::hardware_concurrency() / 2)));
  if (pageable && p->stage_bytes < need) {
    for (int i = 0; i < 2; ++i) {
      if (p->stage[i]) cudaFreeHost(p->stage[i]);
      p->stage[i] = nullptr;
    }
    p->stage_bytes = 0;
    for (int i = 0; i < 2; ++i) {
      CAPT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p->stage[i]), need, cudaHostAllocDefault));
      if (!p->staged[i]) CAPT_CUDA(cudaEventCreateWithFlags(&p->staged[i], cudaEventDisableTiming));
    }
    p->stage_bytes = need;
  }
  for (int64_t ci = 0; ci < n_chunks; ++ci) {
    const int b = int(ci & 1);
    cudaStream_t w = p->w[b];
    const int64_t base = ci * chunk;
    const int64_t len = n - base < chunk ? n - base : chunk;
    const char* hc = static_cast<const char*>(centers) + in_elem * t.k * base;
    const char* hr = static_cast<const char*>(radii) + in_elem * base;
    const uint8_t* hm = lane_mask ? lane_mask + base : nullptr;
    if (pageable) {
      // (buffer b's previous copy to the device has completed)
      CAPT_CUDA(cudaEventSynchronize(p->staged[b]));
      char* st = p->stage[b];
      parallel_copy(st, hc, in_elem * t.k * len, nthreads);
      parallel_copy(st + cb, hr, in_elem * len, nthreads);
      if (hm) std::memcpy(st + cb + rb, hm, size_t(len));
      hc = st;
      hr = st + cb;
      if (hm) hm = reinterpret_cast<const uint8_t*>(st + cb + rb);
    }
    CAPT_CUDA(cudaMemcpyAsync(call.c[b], hc, in_elem * t.k * len, cudaMemcpyHostToDevice, w));
    CAPT_CUDA(cudaMemcpyAsync(call.r[b], hr, in_elem * len, cudaMemcpyHostToDevice, w));
    if (lane_mask)
      CAPT_CUDA(cudaMemcpyAsync(call.m[b], hm, len, cudaMemcpyHostToDevice, w));
    if (pageable) CAPT_CUDA(cudaEventRecord(p->staged[b], w));
    const int rc = query_device(t, call.c[b], call.r[b], len, L, lane_mask ? call.m[b] : nullptr,
                               flags, call.d_bits + base / L / 32, call.aux[b] + 1, call.aux[b], w);
    if (rc) return rc;
    CAPT_CUDA(cudaMemcpyAsync(p->pinned + 7 * ci, call.aux[b], 8 * 7, cudaMemcpyDeviceToHost, w));
  }
  for (int i = 0; i < 2; ++i) {
    CAPT_CUDA(cudaEventRecord(p->done[i], p->w[i]));
    CAPT_CUDA(cudaStreamWaitEvent(s, p->done[i], 0));
  }
  CAPT_CUDA(cudaMemcpyAsync(out_bits, call.d_bits, 4 * words_total, cudaMemcpyDeviceToHost, s));
  CAPT_CUDA(cudaStreamSynchronize(s));
  int64_t fb = -1;
  uint64_t cnt[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t ci = 0; ci < n_chunks; ++ci) {
    const unsigned long long* a = p->pinned + 7 * ci;
    if (fb < 0 && a[0] != ~0ull) fb = ci * chunk + int64_t(a[0]);
    for (int j = 0; j < 6; ++j) cnt[j] += a[1 + j];
  }
  if (first_bad) *first_bad = fb;
  if (counters && (flags & CAPT_STATS)) memcpy(counters, cnt, sizeof(cnt));
  if ((flags & CAPT_CHECK_RADII) && fb >= 0) {
    set_error("radius outside the tree's exactness band");
    return CAPT_ERANGE;
  }
  return CAPT_OK;
}

}  // namespace capt

using namespace capt;

extern "C" int capt_query(const capt_tree* tree, const void* centers, const void* radii,
                          int64_t n, int L, const uint8_t* lane_mask, uint32_t flags,
                          uint32_t* out_bits, uint64_t* counters, int64_t* first_bad,
                          void* stream) {
  if (!tree) return fail(CAPT_EINVAL, "NULL tree");
  if (n < 0) return fail(CAPT_EINVAL, "negative sphere count");
  if (L < 1 || L > 32 || (L & (L - 1))) return fail(CAPT_EINVAL, "lane width must be a power of two <= 32");
  if (n % L) return fail(CAPT_EINVAL, "sphere count must be a multiple of the lane width");
  if (n > 0 && (!centers || !radii || !out_bits)) return fail(CAPT_EINVAL, "NULL array argument");
  if ((flags & CAPT_STATS) && !counters) return fail(CAPT_EINVAL, "CAPT_STATS needs counters");
  CAPT_CUDA(cudaSetDevice(tree->device));
  ensure_pool(tree->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const DevTree t = view(tree);
  const int64_t n_groups = n / L;
  const int64_t n_words = (n_groups + 31) / 32;
  const bool host = flags & CAPT_HOST_IO;
  const size_t in_elem = (flags & CAPT_INPUT_F64) ? sizeof(double) : sizeof(float);

  // group-sequential counters (STATS with lane groups) are additive per chunk
#ifndef CAPT_PIPE_CHUNK_LOG2
#define CAPT_PIPE_CHUNK_LOG2 22
#endif
  const int64_t chunk = int64_t(1) << CAPT_PIPE_CHUNK_LOG2;  // spheres per pipeline chunk (multiple of 32 * L)
  if (host && n > chunk) {
    return query_host_pipelined(tree, t, centers, radii, n, L, lane_mask, flags, out_bits,
                                counters, first_bad, s, chunk);
  }

  HostIO io;
  io.s = s;
  const void* d_c = centers;
  const void* d_r = radii;
  const uint8_t* d_m = lane_mask;
  uint32_t* d_bits = out_bits;
  unsigned long long* d_cnt = reinterpret_cast<unsigned long long*>(counters);
  unsigned long long* d_bad = reinterpret_cast<unsigned long long*>(first_bad);
  if (host) {
    CAPT_CUDA(cudaMallocAsync(&io.centers, in_elem * t.k * (n ? n : 1), s));
    CAPT_CUDA(cudaMallocAsync(&io.radii, in_elem * (n ? n : 1), s));
    CAPT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&io.bits), 4 * (n_words ? n_words : 1), s));
    CAPT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&io.counters), 8 * 6, s));
    CAPT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&io.first_bad), 8, s));
    if (n) {
      CAPT_CUDA(cudaMemcpyAsync(io.centers, centers, in_elem * t.k * n, cudaMemcpyHostToDevice, s));
      CAPT_CUDA(cudaMemcpyAsync(io.radii, radii, in_elem * n, cudaMemcpyHostToDevice, s));
    }
    if (lane_mask) {
      CAPT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&io.mask), n ? n : 1, s));
      if (n) CAPT_CUDA(cudaMemcpyAsync(io.mask, lane_mask, n, cudaMemcpyHostToDevice, s));
    }
    d_c = io.centers;
    d_r = io.radii;
    d_m = io.mask;
    d_bits = io.bits;
    d_cnt = io.counters;
    d_bad = io.first_bad;
  }
  {
    const int rc = query_device(t, d_c, d_r, n, L, d_m, flags, d_bits, d_cnt, d_bad, s);
    if (rc) return rc;
  }
  if (host) {
    if (n_words) CAPT_CUDA(cudaMemcpyAsync(out_bits, d_bits, 4 * n_words, cudaMemcpyDeviceToHost, s));
    int64_t fb = -1;
    CAPT_CUDA(cudaMemcpyAsync(&fb, d_bad, 8, cudaMemcpyDeviceToHost, s));
    uint64_t cnt[6] = {0, 0, 0, 0, 0, 0};
    if (flags & CAPT_STATS) CAPT_CUDA(cudaMemcpyAsync(cnt, d_cnt, 48, cudaMemcpyDeviceToHost, s));
    CAPT_CUDA(cudaStreamSynchronize(s));
    if (first_bad) *first_bad = fb;
    if (counters && (flags & CAPT_STATS)) memcpy(counters, cnt, sizeof(cnt));
    if ((flags & CAPT_CHECK_RADII) && fb >= 0) {
      set_error("radius outside the tree's exactness band");
      return CAPT_ERANGE;
    }
  }
  return CAPT_OK;
}

extern "C" int capt_leaf_indices(const capt_tree* tree, const void* centers, int64_t n,
                                 uint32_t flags, int64_t* out, void* stream) {
  if (!tree) return fail(CAPT_EINVAL, "NULL tree");
  if (n < 0) return fail(CAPT_EINVAL, "negative count");
  if (n == 0) return CAPT_OK;
  if (!centers || !out) return fail(CAPT_EINVAL, "NULL array argument");
  CAPT_CUDA(cudaSetDevice(tree->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const DevTree t = view(tree);
  const bool host = flags & CAPT_HOST_IO;
  const size_t in_elem = (flags & CAPT_INPUT_F64) ? sizeof(double) : sizeof(float);
  void* d_c = const_cast<void*>(centers);
  int64_t* d_out = out;
  if (host) {
    CAPT_CUDA(cudaMallocAsync(&d_c, in_elem * t.k * n, s));
    CAPT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_out), 8 * n, s));
    CAPT_CUDA(cudaMemcpyAsync(d_c, centers, in_elem * t.k * n, cudaMemcpyHostToDevice, s));
  }
  const int grid = grid_for(n, 256, 8);
  if (flags & CAPT_INPUT_F64)
    k_leaf_indices<double><<<grid, 256, 0, s>>>(t, d_c, n, d_out);
  else
    k_leaf_indices<float><<<grid, 256, 0, s>>>(t, d_c, n, d_out);
  CAPT_CUDA(cudaGetLastError());
  if (host) {
    CAPT_CUDA(cudaMemcpyAsync(out, d_out, 8 * n, cudaMemcpyDeviceToHost, s));
    CAPT_CUDA(cudaFreeAsync(d_c, s));
    CAPT_CUDA(cudaFreeAsync(d_out, s));
    CAPT_CUDA(cudaStreamSynchronize(s));
  }
  return CAPT_OK;
}
