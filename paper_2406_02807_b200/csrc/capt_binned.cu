// Leaf-binned query pipeline (the large-batch hot path).
//
// The reference itself groups spheres by leaf and scans each affordance set
// once as a dense (spheres x points) distance matrix (query.py:209-218).  On
// B200 that becomes:
//   K1 k_bin_count3   per sphere: band check, descent (top 13 levels in smem),
//                     fp32 AABB reject (float64 fix-up in the band), the
//                     representative probe (a definite hit resolves the sphere
//                     and its whole lane group), warp-aggregated per-leaf
//                     counts; spheres needing the exact path go to a queue
//                     (k_bin_count: generic k / float64 inputs)
//   K2 k_scan_tiles   per-leaf start offsets and first-tile indices, one CTA;
//                     K3a writes the (leaf, chunk of <= 1024 spheres) tiles
//   K3 k_part_bucket, k_part_leaf: group K1's compact list of binned spheres
//                     by leaf in two shared-memory-ranked passes (bucket of
//                     leaves, then leaf) into a permutation; K5 gathers the
//                     float4 {c, r} records through it
//   K5 k_binned_scan  persistent CTAs pull tiles from an atomic counter; the
//                     leaf's set is staged once into shared memory in local
//                     coordinates b = p - o with w = |b|^2, and each thread
//                     holds 8 spheres as 4 packed fp32x2 pairs:
//                         t = w - 2 a.b    (3 FFMA2 per 2 tests)
//                         min = min3(min, t_j, t_j+1)   (FMNMX3)
//                     a sphere collides iff min_t <= r^2 - |a|^2; a proven
//                     error band (64u relative to |a|^2 + |b|^2 + r^2) sends
//                     the rare ambiguous sphere to the exact queue
//   K6 k_slow         K5's hits (by list index) -> sphere verdicts; exact
//                     float64 scan of the queue, one warp per sphere
//   K7 k_pack         verdict bytes -> bit words, OR over each lane group
#include <cub/cub.cuh>
#include <cuda_fp16.h>

#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "capt_binned.cuh"
#include "capt_query_common.cuh"
#include "capt_tc.cuh"

namespace capt {

namespace {

constexpr int kBT = 128;           // threads per binned CTA
constexpr int kS = 8;              // spheres per thread (4 packed pairs)
constexpr int kTS = kBT * kS;      // spheres per tile
// Compile-time tunables (build_ext --out ... -D NAME=VALUE builds a variant).
// Measured on config 1 (K5 us): TS 128/NC 64 265; 128/128 404 (4 CTAs/SM);
// 256/128 577; 512/64 ~1100; 128/32 371; 256/64 with 256 threads 286
// (config 3: 4384 vs 5659); a two-accumulator ping-pong over chunks was
// slower at both configs (fewer CTAs/SM).
#ifndef CAPT_TC_TS
#define CAPT_TC_TS 128
#endif
#ifndef CAPT_TC_NC
#define CAPT_TC_NC 64
#endif
constexpr int kTsTc = CAPT_TC_TS;  // spheres per tile, tensor-core K5
constexpr int kChunk = 512;        // staged points per shared-memory chunk
constexpr float kBand = 0x1p-18f;  // 64u

// Programmatic dependent launch: each stage after K1 is launched with
// programmatic stream serialisation, so its CTAs are scheduled while the
// previous stage drains; it waits (griddepcontrol.wait) before reading the
// previous stage's output.  Every stage signals its dependents once its CTAs
// are past their last write.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename InT>
__device__ __forceinline__ void load_sphere(const void* c, const void* r, int64_t q, int k,
                                            double c64[3], double& r64) {
  c64[0] = c64[1] = c64[2] = 0.0;
  if constexpr (std::is_same<InT, float>::value) {
    const float* cf = static_cast<const float*>(c);
#pragma unroll
    for (int d = 0; d < kMaxK; ++d)
      if (d < k) c64[d] = double(__ldg(cf + q * k + d));
    r64 = double(__ldg(static_cast<const float*>(r) + q));
  } else {
    const double* cd = static_cast<const double*>(c);
#pragma unroll
    for (int d = 0; d < kMaxK; ++d)
      if (d < k) c64[d] = __ldg(cd + q * k + d);
    r64 = __ldg(static_cast<const double*>(r) + q);
  }
}

struct SphereClass {
  int status;  // 0 false, 2 scan, 3 slow
  int64_t leaf;
  float cx, cy, cz, rf;
};

template <typename InT>
__device__ __forceinline__ SphereClass classify_sphere(const DevTree& t, const float* sT, int n_smem,
                                                       const BinArgs& a, int64_t q, bool check) {
  SphereClass sc;
  sc.status = 0;
  sc.leaf = 0;
  bool valid = q < a.n;
  if (valid && a.mask) valid = a.mask[q] != 0;
  if (!valid) return sc;
  double c64[3], r64;
  load_sphere<InT>(a.centers, a.radii, q, t.k, c64, r64);
  if (check && (r64 < t.r_min || r64 > t.r_max))
    atomicMin(a.first_bad, static_cast<unsigned long long>(q));
  if constexpr (std::is_same<InT, float>::value) {
    const float cf[3] = {float(c64[0]), float(c64[1]), float(c64[2])};
    sc.leaf = descend_t<float>(t, sT, n_smem, cf);
  } else {
    sc.leaf = descend(t, sT, n_smem, c64);
  }
  float r2, loB, hiB;
  sc.status = classify(t, sc.leaf, c64, r64, a.flags & CAPT_PREFILTER, sc.cx, sc.cy, sc.cz, r2,
                       loB, hiB);
  sc.rf = float(r64);
  return sc;
}

// fp32 inputs: branch-light classification without any float64 work on the
// common path.  Band check against the fp32 images of the double band edges
// (r < r_min in double <=> r < smallest float >= r_min).  Returns 0 (false),
// 2 (binned fp32 scan) or 3 (exact float64 scan; AABB already decided).
__device__ __forceinline__ int classify_f32(const DevTree& t, const float* sT, int n_smem,
                                            const BinArgs& a, int64_t q, bool check, int& leaf) {
  const float* cf = static_cast<const float*>(a.centers);
  float c[3] = {0.f, 0.f, 0.f};
  for (int d = 0; d < t.k; ++d) c[d] = __ldg(cf + q * t.k + d);
  const float r = __ldg(static_cast<const float*>(a.radii) + q);
  if (check && (r < a.rlo_f || r > a.rhi_f))
    atomicMin(a.first_bad, static_cast<unsigned long long>(q));
  int i = 0;
  if (t.k == 3) {
    // levels 0..11 (node ids < 4095) come from shared memory, 3 axes per step
    const float c0 = c[0], c1 = c[1], c2 = c[2];
    const int dsm = t.depth < 12 ? t.depth : 12;
    int s = 0;
    for (; s + 3 <= dsm; s += 3) {
      i = 2 * i + 1 + (c0 > sT[i] ? 1 : 0);
      i = 2 * i + 1 + (c1 > sT[i] ? 1 : 0);
      i = 2 * i + 1 + (c2 > sT[i] ? 1 : 0);
    }
    for (; s < t.depth; ++s) {
      const int ax = s % 3;
      const float cv = ax == 0 ? c0 : (ax == 1 ? c1 : c2);
      const float tv = s < dsm ? sT[i] : __ldg(t.T + i);
      i = 2 * i + 1 + (cv > tv ? 1 : 0);
    }
  } else {
    int ax = 0;
    for (int s = 0; s < t.depth; ++s) {
      const float tv = (i < n_smem) ? sT[i] : __ldg(t.T + i);
      const float cv = ax == 0 ? c[0] : (ax == 1 ? c[1] : c[2]);
      i = 2 * i + 1 + (cv > tv ? 1 : 0);
      ax = (ax + 1 == t.k) ? 0 : ax + 1;
    }
  }
  leaf = i - int(t.n - 1);
  const bool cfin = isfinite(c[0]) && isfinite(c[1]) && isfinite(c[2]);
  const float r2 = r * r;
  const bool fast = cfin && r2 >= kR2Min && r2 <= kR2Max;
  if (!fast && !cfin && isfinite(r)) return 0;  // finite r^2 in float64: never collides
  const bool prefilter = a.flags & CAPT_PREFILTER;
  if (!prefilter) return fast ? 2 : 3;
  const float4 lo = __ldg(t.box + 2 * leaf);
  const float4 hi = __ldg(t.box + 2 * leaf + 1);
  if (fast) {
    const float rx = fmaxf(fmaxf(lo.x - c[0], 0.f), c[0] - hi.x);
    const float ry = fmaxf(fmaxf(lo.y - c[1], 0.f), c[1] - hi.y);
    const float rz = fmaxf(fmaxf(lo.z - c[2], 0.f), c[2] - hi.z);
    const float s = fmaf(rz, rz, fmaf(ry, ry, rx * rx));
    if (s > r2 * (1.0f + kTau)) return 0;
    if (s < r2 * (1.0f - kTau)) return 2;
  }
  const double c64[3] = {c[0], c[1], c[2]};
  const double r64 = r;
  if (!aabb_keep64(t.k, lo, hi, c64, __dmul_rn(r64, r64))) return 0;
  return fast ? 2 : 3;
}

// Warp-collective: per-leaf histogram (warp-aggregated, fire-and-forget
// atomics), compact list entry for K3 (one list atomic per warp), exact-path
// list.
__device__ __forceinline__ void record_bin(const BinArgs& a, int64_t q, int status, int leaf,
                                           float4 rc) {
  const bool scan = status == 2;
  const unsigned act = __ballot_sync(0xffffffffu, scan);
  const int lane = threadIdx.x & 31;
  unsigned lbase = 0;
  if (act && lane == 0) lbase = atomicAdd(a.list_n, __popc(act));
  if (scan) {
    const unsigned peers = __match_any_sync(act, unsigned(leaf));
    if (lane == __ffs(peers) - 1) atomicAdd(a.counts + leaf, __popc(peers));
  }
  lbase = __shfl_sync(0xffffffffu, lbase, 0);
  if (scan) {
    const unsigned j = lbase + __popc(act & ((1u << lane) - 1u));
    a.lrec[j] = rc;
    a.lmeta[j] = make_int2(int(q), leaf);
    a.lhit[j] = 0;
  }
  if (status == 3) {
    const unsigned i = atomicAdd(a.slow_n, 1u);
    a.slow[i] = make_int2(int(q), leaf);
  }
}

// Warp-collective representative probe before binning.  Row 0 of a leaf's
// set is the point that owns the leaf's cell -- the cell the sphere centre
// lies in -- so it is the likeliest hit.  A definite fp32 hit (same error band
// as the scan) resolves the sphere; with lane groups (query.py:152-160 early
// exit) it resolves the whole group, whose other spheres are then never
// binned.  Returns the status to bin with.
__device__ __forceinline__ int rep_probe(const BinArgs& a, int64_t q, int status, int leaf,
                                         float cx, float cy, float cz, float r) {
  bool hit = false;
  if (status == 2) {
    const float4 rp = __ldg(a.t.rep + leaf);
    const float dx = cx - rp.x, dy = cy - rp.y, dz = cz - rp.z;
    const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    hit = d2 <= (r * r) * (1.0f - kTau);
  }
  if (q < a.n) a.verdict[q] = hit ? 1 : 0;  // every byte written: no memset
  bool resolved = hit;
  if (a.L > 1) {
    const unsigned hb = __ballot_sync(0xffffffffu, hit);
    const int lane = threadIdx.x & 31;
    const unsigned seg = a.L >= 32 ? 0xffffffffu : ((1u << a.L) - 1u) << ((lane / a.L) * a.L);
    resolved = (hb & seg) != 0;
  }
  return resolved ? 0 : status;
}

// K1: classify, per-leaf histogram (warp-aggregated), exact-path list
template <typename InT>
__global__ void __launch_bounds__(256) k_bin_count(BinArgs a) {
  __shared__ float sT[kSmemNodes];
  const DevTree& t = a.t;
  const int n_smem = int(t.n - 1 < kSmemNodes ? t.n - 1 : kSmemNodes);
  for (int i = threadIdx.x; i < n_smem; i += blockDim.x) sT[i] = t.T[i];
  __syncthreads();
  const bool check = a.flags & CAPT_CHECK_RADII;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t n_pad = (a.n + 31) & ~int64_t(31);
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n_pad; q += stride) {
    int status = 0, leaf = -1;
    bool valid = q < a.n;
    if (valid && a.mask) valid = a.mask[q] != 0;
    if (valid) {
      if constexpr (std::is_same<InT, float>::value) {
        status = classify_f32(t, sT, n_smem, a, q, check, leaf);
      } else {
        const SphereClass sc = classify_sphere<InT>(t, sT, n_smem, a, q, check);
        status = sc.status;
        leaf = int(sc.leaf);
      }
    }
    float c[3] = {0.f, 0.f, 0.f}, r = 0.f;
    if (status == 2) {  // binned spheres are exact fp32 values
      for (int d = 0; d < t.k; ++d) {
        if constexpr (std::is_same<InT, float>::value)
          c[d] = static_cast<const float*>(a.centers)[q * t.k + d];
        else
          c[d] = float(static_cast<const double*>(a.centers)[q * t.k + d]);
      }
      if constexpr (std::is_same<InT, float>::value) r = static_cast<const float*>(a.radii)[q];
      else r = float(static_cast<const double*>(a.radii)[q]);
    }
    status = rep_probe(a, q, status, leaf, c[0], c[1], c[2], r);
    record_bin(a, q, status, leaf, make_float4(c[0], c[1], c[2], r));
  }
}

// K1 specialised for k = 3, fp32 input (the hot path): V spheres per thread
// in flight (one sphere per lane: the inputs stay coalesced -- a thread-per-
// group variant sharing the descent prefix of an 8-sphere group was measured
// 2x slower), 32-bit indexing, the top 13 levels of T in shared memory walked
// on absolute shared addresses (LDS, FSETP, SEL, IADD3 per level), one
// 256-bit probe record per sphere, one list atomic per warp.
// split levels K1 keeps in shared memory: 13 (32 KB, 4 CTAs/SM; 339 us)
// beats 14 (64 KB, 3 CTAs/SM; 370-401 us) on config 1
#ifndef CAPT_K1_SMEM_LEVELS
#define CAPT_K1_SMEM_LEVELS 13
#endif
constexpr int kSmemNodes3 = (1 << CAPT_K1_SMEM_LEVELS) - 1;
// K1 min CTAs per SM (caps registers at 64): 4 beats 1 (70 regs) by ~10%
#ifndef CAPT_K1_MINB
#define CAPT_K1_MINB 4
#endif
// spheres in flight per K1 thread: 4 (339 us) beats 2 (442) and 6 (482)
constexpr int kK1V = 4;
template <int V>
__global__ void __launch_bounds__(256, CAPT_K1_MINB) k_bin_count3(BinArgs a) {
  extern __shared__ __align__(16) float sT[];  // kSmemNodes3 floats (dynamic: may exceed 48 KB)
  const DevTree& t = a.t;
  const int n_smem = int(t.n - 1 < kSmemNodes3 ? t.n - 1 : kSmemNodes3);
  for (int i = threadIdx.x; i < n_smem; i += blockDim.x) sT[i] = t.T[i];
  __syncthreads();
  pdl_wait();  // the counters are cleared by k_zero (T staging overlaps it)
  const bool check = a.flags & CAPT_CHECK_RADII;
  const bool prefilter = a.flags & CAPT_PREFILTER;
  const float* __restrict__ cf = static_cast<const float*>(a.centers);
  const float* __restrict__ rf = static_cast<const float*>(a.radii);
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(sT));
  const int dsm = t.depth < CAPT_K1_SMEM_LEVELS ? t.depth : CAPT_K1_SMEM_LEVELS;
  const int nl1 = int(t.n - 1);
  const int n = int(a.n);
  const int n_pad = (n + 31) & ~31;
  const int lane = threadIdx.x & 31;
  const unsigned seg = a.L >= 32 ? 0xffffffffu : ((1u << a.L) - 1u) << ((lane / a.L) * a.L);
  const float band_lo = 1.0f - kTau, band_hi = 1.0f + kTau;
  const int stride = gridDim.x * blockDim.x * V;
  // streaming (evict-first) input loads, software-pipelined one iteration
  // ahead: the DRAM latency of iteration i+1 hides behind iteration i
  float nx[V], ny[V], nz[V], nr[V];
  int nsid[V];  // sphere ids (the list entries in list mode)
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int q = blockIdx.x * blockDim.x * V + v * blockDim.x + threadIdx.x;
    const int qq = q < n ? q : 0;
    nsid[v] = qq;
    nx[v] = __ldcs(cf + 3 * qq);
    ny[v] = __ldcs(cf + 3 * qq + 1);
    nz[v] = __ldcs(cf + 3 * qq + 2);
    nr[v] = __ldcs(rf + qq);
  }
  for (int base = blockIdx.x * blockDim.x * V; base < n_pad; base += stride) {
    float cx[V], cy[V], cz[V], r[V];
    int sid[V];
    bool valid[V];
    unsigned off[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      cx[v] = nx[v];
      cy[v] = ny[v];
      cz[v] = nz[v];
      r[v] = nr[v];
      sid[v] = nsid[v];
      const int qn = base + stride + v * blockDim.x + threadIdx.x;
      const int qq = qn < n ? qn : 0;
      nsid[v] = qq;
      nx[v] = __ldcs(cf + 3 * qq);
      ny[v] = __ldcs(cf + 3 * qq + 1);
      nz[v] = __ldcs(cf + 3 * qq + 2);
      nr[v] = __ldcs(rf + qq);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int q = base + v * blockDim.x + threadIdx.x;
      valid[v] = q < n;
      if (a.mask && valid[v]) valid[v] = a.mask[q] != 0;
      off[v] = 0;
    }
    if (check) {  // out-of-band radii are rare: one warp vote, then the atomics
      bool bad = false;
#pragma unroll
      for (int v = 0; v < V; ++v) bad |= valid[v] && (r[v] < a.rlo_f || r[v] > a.rhi_f);
      if (__any_sync(0xffffffffu, bad)) {
#pragma unroll
        for (int v = 0; v < V; ++v)
          if (valid[v] && (r[v] < a.rlo_f || r[v] > a.rhi_f))
            atomicMin(a.first_bad,
                      static_cast<unsigned long long>(base + v * blockDim.x + threadIdx.x));
      }
    }
    // shared-memory levels on absolute shared-window addresses:
    // addr(child) = 2 addr + (4 or 8) - sbase, one LDS + compare + select + IMAD
    int s = 0;
    {
      unsigned ad[V];
#pragma unroll
      for (int v = 0; v < V; ++v) ad[v] = sbase;
      const unsigned k0 = 4u - sbase, k1 = 8u - sbase;
      for (; s + 3 <= dsm; s += 3) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          unsigned x = ad[v];
          x = 2 * x + (cx[v] > lds_f32(x) ? k1 : k0);
          x = 2 * x + (cy[v] > lds_f32(x) ? k1 : k0);
          x = 2 * x + (cz[v] > lds_f32(x) ? k1 : k0);
          ad[v] = x;
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) off[v] = ad[v] - sbase;
    }
    // the remaining (< 3) shared levels, then the global ones; the axis is
    // uniform per level, selected without branches
#pragma unroll 1
    for (; s < dsm; ++s) {
      const int ax = s % 3;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const float c = ax == 0 ? cx[v] : (ax == 1 ? cy[v] : cz[v]);
        off[v] = 2 * off[v] + (c > lds_f32(sbase + off[v]) ? 8u : 4u);
      }
    }
#pragma unroll 1
    for (; s < t.depth; ++s) {
      const int ax = s % 3;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const float c = ax == 0 ? cx[v] : (ax == 1 ? cy[v] : cz[v]);
        off[v] = 2 * off[v] + (c > __ldg(t.T + (off[v] >> 2)) ? 8u : 4u);
      }
    }
    // per-sphere classification, branch-free.  The AABB test (on the probe
    // record's outward-rounded fp16 box) only has to
    // be conservative here: every point of a set lies inside the set's box and
    // the reference's float64 box distance is a monotone function of the same
    // rounded differences, so s_box <= s_point and a sphere the reference
    // rejects by its AABB (query.py:202-208) has no colliding point -- the
    // prefilter never changes a verdict, only the work.  A sphere is rejected
    // only when the fp32 box distance is clearly above r^2 (relative band
    // TAU); the band itself is kept and left to the scan.  Exact reference
    // AABB semantics (the aabb-rejection counter) live in the counter kernel.
    int leaf[V], status[V];
    bool hit[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      leaf[v] = int(off[v] >> 2) - nl1;
      const float r2 = r[v] * r[v];
      const bool cfin = isfinite(cx[v]) && isfinite(cy[v]) && isfinite(cz[v]);
      const bool fast = cfin && r2 >= kR2Min && r2 <= kR2Max;
      // non-finite centre with a finite radius never collides (float64 r^2 is finite)
      int st = fast ? 2 : ((!cfin && isfinite(r[v])) ? 0 : 3);
      st = valid[v] ? st : 0;
      // one 32-B load: representative + outward-rounded fp16 box
      float pr[8];
      ld_v8(t.probe + 8 * leaf[v], pr);
      const float4 rp = make_float4(pr[0], pr[1], pr[2], 0.f);
      if (prefilter) {
        const float2 l01 = h2f2(pr[3]), l2h0 = h2f2(pr[4]), h12 = h2f2(pr[5]);
        const float rx = fmaxf(fmaxf(l01.x - cx[v], 0.f), cx[v] - l2h0.y);
        const float ry = fmaxf(fmaxf(l01.y - cy[v], 0.f), cy[v] - h12.x);
        const float rz = fmaxf(fmaxf(l2h0.x - cz[v], 0.f), cz[v] - h12.y);
        const float ss = fmaf(rz, rz, fmaf(ry, ry, rx * rx));
        st = (fast && ss > r2 * band_hi) ? 0 : st;
      }
      const float dx = cx[v] - rp.x, dy = cy[v] - rp.y, dz = cz[v] - rp.z;
      hit[v] = st == 2 && fmaf(dz, dz, fmaf(dy, dy, dx * dx)) <= r2 * band_lo;
      status[v] = st;
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int q = base + v * blockDim.x + threadIdx.x;
      if (q < n) a.verdict[sid[v]] = hit[v] ? 1 : 0;  // every byte written: no memset
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      bool resolved = hit[v];
      if (a.L > 1) resolved = (__ballot_sync(0xffffffffu, hit[v]) & seg) != 0;
      if (resolved) status[v] = 0;
    }
    // binned spheres go to the compact list (one returning atomic per warp,
    // issued before the per-leaf counts so its latency overlaps them); the
    // counts are fire-and-forget reductions; the rank inside the leaf is
    // drawn by K3
    unsigned act[V], tot = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      act[v] = __ballot_sync(0xffffffffu, status[v] == 2);
      tot += __popc(act[v]);
    }
    unsigned lbase = 0;
    if (tot && lane == 0) lbase = atomicAdd(a.list_n, tot);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int q = sid[v];
      if (status[v] == 2) {
        const unsigned peers = __match_any_sync(act[v], unsigned(leaf[v]));
        if (lane == __ffs(peers) - 1) atomicAdd(a.counts + leaf[v], __popc(peers));
      }
      if (status[v] == 3) {
        const unsigned j = atomicAdd(a.slow_n, 1u);
        a.slow[j] = make_int2(q, leaf[v]);
      }
    }
    if (tot) {
      unsigned j = __shfl_sync(0xffffffffu, lbase, 0);
      const unsigned lt = (1u << lane) - 1u;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (status[v] == 2) {
          const unsigned p = j + __popc(act[v] & lt);
          __stcs(a.lrec + p, make_float4(cx[v], cy[v], cz[v], r[v]));
          a.lhit[p] = 0;
          __stcs(a.lmeta + p, make_int2(sid[v], leaf[v]));
        }
        j += __popc(act[v]);
      }
    }
  }
  pdl_trigger();
}

// K3: group K1's compact list by leaf in two coalescing passes instead of
// one random scatter with a returning atomic per sphere (both of which are
// L2-transaction bound at this size).  Only 8-byte (leaf, list index) pairs
// move; K5 gathers each tile's records through the permutation.
//   K3a k_part_bucket: a CTA takes 4096 list entries, ranks them per leaf
//       bucket (<= 256 buckets of 2^bshift consecutive leaves) with shared
//       memory atomics, reserves each bucket's run with ONE global atomic and
//       writes (leaf, list index) pairs -- runs of ~16 pairs per bucket.
//       Bucket b's region starts at start[b << bshift] (the leaf scan).
//   K3b k_part_leaf: a CTA takes 4096 bucket-ordered pairs (their leaves span
//       one or a few buckets), ranks them per leaf in shared memory, reserves
//       per leaf with one global atomic, and writes perm[start[leaf] + rank]
//       (writes stay inside the buckets' regions).
constexpr int kBuckets = 256;
constexpr int kPartItems = 4096;  // entries per CTA pass
constexpr int kPartPer = kPartItems / 256;
constexpr int kLeafSpan = 2048;  // K3b shared-memory leaf counters

__global__ void __launch_bounds__(256) k_part_bucket(BinArgs a) {
  __shared__ uint32_t hist[kBuckets];
  __shared__ uint32_t gbase[kBuckets];
  pdl_wait();
  const uint32_t n = *a.list_n;
  const int tid = threadIdx.x;
  // the K5 tile list: every chunk of <= ts spheres of a leaf, leaf by leaf in
  // the tree's order (K2 gave each leaf its first tile index); one warp per
  // leaf, its lanes write the leaf's tiles
  {
    const int lane = tid & 31;
    const int64_t wg = (int64_t(blockIdx.x) * blockDim.x + tid) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t j = wg; j < a.t.n; j += nw) {
      const int leaf = a.t.order[j];
      const uint32_t total = a.counts[leaf];
      const uint32_t ts = a.ts;
      const uint32_t nt = (total + ts - 1) / ts;
      if (!nt) continue;
      const uint32_t t0 = a.tstart[j], s0 = a.start[leaf];
      const uint2 st = a.t.set[leaf];
      const float4 org = a.t.org[leaf];
      for (uint32_t k = lane; k < nt; k += 32) {
        TileMeta tm;
        tm.leaf = leaf;
        tm.setx = st.x;
        tm.m = st.y;
        tm.pad[0] = tm.pad[1] = tm.pad[2] = 0;
        tm.org = org;
        tm.s0 = s0 + k * ts;
        tm.cnt = int(min(ts, total - k * ts));
        a.tiles[t0 + k] = tm;
      }
    }
  }
  for (uint32_t c0 = blockIdx.x * kPartItems; c0 < n; c0 += gridDim.x * kPartItems) {
    hist[tid] = 0;
    __syncthreads();
    int leaf[kPartPer];
    uint32_t rank[kPartPer];
#pragma unroll
    for (int i = 0; i < kPartPer; ++i) {
      const uint32_t j = c0 + i * 256 + tid;
      leaf[i] = j < n ? __ldcs(&a.lmeta[j].y) : -1;
    }
#pragma unroll
    for (int i = 0; i < kPartPer; ++i)
      if (leaf[i] >= 0) rank[i] = atomicAdd(&hist[leaf[i] >> a.bshift], 1u);
    __syncthreads();
    const uint32_t hc = hist[tid];
    if (hc) gbase[tid] = a.start[tid << a.bshift] + atomicAdd(a.bcursor + tid, hc);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kPartPer; ++i) {
      if (leaf[i] >= 0) {
        const uint32_t j = c0 + i * 256 + tid;
        a.part[gbase[leaf[i] >> a.bshift] + rank[i]] = make_int2(leaf[i], int(j));
      }
    }
    __syncthreads();
  }
  pdl_trigger();
}

__global__ void __launch_bounds__(256) k_part_leaf(BinArgs a) {
  __shared__ uint32_t cnt[kLeafSpan];
  __shared__ int lmin_s, lmax_s;
  pdl_wait();
  const uint32_t n = *a.list_n;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  for (uint32_t c0 = blockIdx.x * kPartItems; c0 < n; c0 += gridDim.x * kPartItems) {
    int2 it[kPartPer];  // (leaf, list index)
    int lo = INT_MAX, hi = -1;
#pragma unroll
    for (int i = 0; i < kPartPer; ++i) {
      const uint32_t j = c0 + i * 256 + tid;
      it[i] = j < n ? __ldcs(a.part + j) : make_int2(-1, -1);
      if (it[i].x >= 0) {
        lo = min(lo, it[i].x);
        hi = max(hi, it[i].x);
      }
    }
    if (tid == 0) {
      lmin_s = INT_MAX;
      lmax_s = -1;
    }
    for (int i = tid; i < kLeafSpan; i += 256) cnt[i] = 0;
    __syncthreads();
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lane == 0) {
      atomicMin(&lmin_s, lo);
      atomicMax(&lmax_s, hi);
    }
    __syncthreads();
    const int lmin = lmin_s;
    const bool local = lmax_s - lmin < kLeafSpan;
    uint32_t rank[kPartPer];
    if (local) {
#pragma unroll
      for (int i = 0; i < kPartPer; ++i)
        if (it[i].x >= 0) rank[i] = atomicAdd(&cnt[it[i].x - lmin], 1u);
      __syncthreads();
      for (int i = tid; i < kLeafSpan; i += 256) {
        const uint32_t c = cnt[i];
        if (c) cnt[i] = a.start[lmin + i] + atomicAdd(a.cursor + lmin + i, c);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < kPartPer; ++i) {
      const int2 e = it[i];
      if (e.x < 0) continue;
      const uint32_t pos = local ? cnt[e.x - lmin] + rank[i]
                                 : a.start[e.x] + atomicAdd(a.cursor + e.x, 1u);
      a.perm[pos] = uint32_t(e.y);
    }
    __syncthreads();
  }
  pdl_trigger();
}

// K2: one CTA turns the per-leaf counts into per-leaf start offsets (leaf
// order; K3's buckets are leaf ranges) and per-leaf first-tile indices in
// tile order (the tile list itself is written by K3a's CTAs).  Tiles are laid
// out leaf by leaf in the tree's order section (descending set size), so the
// persistent K5 CTAs draw the costliest tiles first and the tail of the
// launch is made of small ones.  One launch instead of two device-wide scans
// (this stage is pure latency at every batch size).
// large trees (more leaves than a few single-CTA passes cover): device-wide
// scans instead
__global__ void k_tile_counts(BinArgs a, uint32_t* __restrict__ tc) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < a.t.n;
       j += int64_t(gridDim.x) * blockDim.x)
    tc[j] = (a.counts[a.t.order[j]] + a.ts - 1) / a.ts;
}
__global__ void k_tile_total(BinArgs a, const uint32_t* __restrict__ tc) {
  *a.n_tiles = a.tstart[a.t.n - 1] + tc[a.t.n - 1];
}
constexpr int64_t kScanSingleMax = 32768;  // leaves handled by the one-CTA K2

constexpr int kScanT = 512;
constexpr int kScanI = 16;  // leaves per thread per pass
__global__ void __launch_bounds__(kScanT) k_scan_tiles(BinArgs a) {
  using Scan = cub::BlockScan<uint32_t, kScanT>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint32_t carry[2];
  pdl_wait();
  const int nl = int(a.t.n);
  const int tid = threadIdx.x;
  if (tid == 0) carry[0] = carry[1] = 0;
  for (int p0 = 0; p0 < nl; p0 += kScanT * kScanI) {
    // blocked arrangement, direct 128-bit loads: leaves p0 + 16 tid + i
    const int b0 = p0 + kScanI * tid;
    const int nv = max(0, min(kScanI, nl - b0));
    uint32_t c[kScanI], ord[kScanI], tc[kScanI];
    if (nv == kScanI) {
#pragma unroll
      for (int k = 0; k < kScanI / 4; ++k) {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(a.counts + b0) + k);
        const uint4 y = __ldg(reinterpret_cast<const uint4*>(a.t.order + b0) + k);
        c[4 * k] = x.x; c[4 * k + 1] = x.y; c[4 * k + 2] = x.z; c[4 * k + 3] = x.w;
        ord[4 * k] = y.x; ord[4 * k + 1] = y.y; ord[4 * k + 2] = y.z; ord[4 * k + 3] = y.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < kScanI; ++i) {
        c[i] = i < nv ? a.counts[b0 + i] : 0u;
        ord[i] = i < nv ? uint32_t(a.t.order[b0 + i]) : 0u;
      }
    }
#pragma unroll
    for (int i = 0; i < kScanI; ++i) tc[i] = i < nv ? (a.counts[ord[i]] + a.ts - 1) / a.ts : 0u;
    uint32_t cs = 0, ts = 0;
#pragma unroll
    for (int i = 0; i < kScanI; ++i) {
      cs += c[i];
      ts += tc[i];
    }
    __syncthreads();  // carry visible; scan storage free
    const uint32_t c0 = carry[0], t0 = carry[1];
    uint32_t cpre, tpre, ctot, ttot;
    Scan(tmp).ExclusiveSum(cs, cpre, ctot);
    __syncthreads();
    Scan(tmp).ExclusiveSum(ts, tpre, ttot);
    cpre += c0;
    tpre += t0;
#pragma unroll
    for (int i = 0; i < kScanI; ++i) {  // c[] / tc[] become the exclusive prefixes
      const uint32_t cv = c[i], tv = tc[i];
      c[i] = cpre;
      tc[i] = tpre;
      cpre += cv;
      tpre += tv;
    }
    if (nv == kScanI) {
#pragma unroll
      for (int k = 0; k < kScanI / 4; ++k) {
        reinterpret_cast<uint4*>(a.start + b0)[k] =
            make_uint4(c[4 * k], c[4 * k + 1], c[4 * k + 2], c[4 * k + 3]);
        reinterpret_cast<uint4*>(a.tstart + b0)[k] =
            make_uint4(tc[4 * k], tc[4 * k + 1], tc[4 * k + 2], tc[4 * k + 3]);
      }
    } else {
      for (int i = 0; i < nv; ++i) {
        a.start[b0 + i] = c[i];
        a.tstart[b0 + i] = tc[i];
      }
    }
    __syncthreads();
    if (tid == 0) {
      carry[0] = c0 + ctot;
      carry[1] = t0 + ttot;
    }
  }
  __syncthreads();
  if (tid == 0) *a.n_tiles = carry[1];
  pdl_trigger();
}

// ---- packed fp32x2 helpers (sm_100: FFMA2 / FMNMX3) ----
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ uint32_t okey(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float okey_inv(uint32_t u) {
  u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
  return __uint_as_float(u);
}

struct __align__(16) SmemBinned {
  ulonglong2 A[kChunk];  // {bx,bx}, {by,by}
  ulonglong2 B[kChunk];  // {bz,bz}, {w,w}
  uint32_t minkey[kTS];  // per sphere: min over the phases (orderable key)
  float lim_lo[kTS];     // per sphere: thr - band (min <= it: definite hit)
  float lim_hi[kTS];     // per sphere: thr + band (min > it: definite miss)
  uint32_t hitmask[kTS / kS];
  int tile;
};

// Eight spheres of one thread in local coordinates of the set origin o:
// t = |b|^2 - 2 a.b compared with thr = r^2 - |a|^2 (a = c - o, b = p - o).
// Only the packed -2a and the running minima live in registers; the decision
// limits sit in shared memory (read every 8 point groups and at the end).
struct Spheres8 {
  unsigned long long Kx[kS / 2], Ky[kS / 2], Kz[kS / 2];
  float mn[kS];
  int base;        // tile-local index of sphere 0 of this slot
  uint32_t real;   // bit i: sphere base + i exists
};

// The tile-local spheres slot*kS .. slot*kS + kS-1 (those < count); the
// slot's owner (phase 0) writes their decision limits.
__device__ __forceinline__ void load_spheres(Spheres8& sp, SmemBinned& S, const BinArgs& a,
                                             int64_t s0, const float4 org, int count, int slot,
                                             bool active, bool owner) {
  const float INF = __int_as_float(0x7f800000);
  sp.real = 0;
  sp.base = slot * kS;
#pragma unroll
  for (int i = 0; i < kS; i += 2) {
    float kx[2], ky[2], kz[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = sp.base + i + h;
      sp.mn[i + h] = INF;
      kx[h] = ky[h] = kz[h] = 0.f;
      if (active && e < count) {
        sp.real |= 1u << (i + h);
        const float4 rc = a.lrec[a.perm[s0 + e]];
        const float ax = rc.x - org.x, ay = rc.y - org.y, az = rc.z - org.z;
        const float aa = fmaf(az, az, fmaf(ay, ay, ax * ax));
        const float r2 = rc.w * rc.w;
        kx[h] = -2.f * ax;
        ky[h] = -2.f * ay;
        kz[h] = -2.f * az;
        if (owner) {
          const float thr = r2 - aa, band = kBand * (aa + org.w + r2);
          S.lim_lo[e] = thr - band;
          S.lim_hi[e] = thr + band;
        }
      }
    }
    sp.Kx[i / 2] = pack2(kx[0], kx[1]);
    sp.Ky[i / 2] = pack2(ky[0], ky[1]);
    sp.Kz[i / 2] = pack2(kz[0], kz[1]);
  }
}

__device__ __forceinline__ uint32_t definite_hits(const Spheres8& sp, const float* lim_lo) {
  uint32_t h = 0;
#pragma unroll
  for (int i = 0; i < kS; ++i)
    if ((sp.real >> i) & 1u) h |= uint32_t(sp.mn[i] <= lim_lo[sp.base + i]) << i;
  return h;
}

// One point pair (2u, 2u+1) against the thread's 8 spheres: 12 FFMA2 + 8 FMNMX3.
__device__ __forceinline__ void test_pair(Spheres8& sp, const ulonglong2* sA, const ulonglong2* sB,
                                          int u) {
  const ulonglong2 A0 = sA[2 * u], B0 = sB[2 * u];
  const ulonglong2 A1 = sA[2 * u + 1], B1 = sB[2 * u + 1];
#pragma unroll
  for (int q = 0; q < kS / 2; ++q) {
    unsigned long long t0 = ffma2(A0.x, sp.Kx[q], B0.y);
    t0 = ffma2(A0.y, sp.Ky[q], t0);
    t0 = ffma2(B0.x, sp.Kz[q], t0);
    unsigned long long t1 = ffma2(A1.x, sp.Kx[q], B1.y);
    t1 = ffma2(A1.y, sp.Ky[q], t1);
    t1 = ffma2(B1.x, sp.Kz[q], t1);
    float t0l, t0h, t1l, t1h;
    unpack2(t0, t0l, t0h);
    unpack2(t1, t1l, t1h);
    sp.mn[2 * q] = fmin3(sp.mn[2 * q], t0l, t1l);
    sp.mn[2 * q + 1] = fmin3(sp.mn[2 * q + 1], t0h, t1h);
  }
}

// Pairs u = 4g .. 4g+3 for g = ph, ph + P, ...  (chunks are padded to a
// multiple of 8 points with w = +inf rows, so groups are always full).  Stops
// early once every sphere of the slot is a definite hit (hitmask shared by
// the phases).
__device__ __forceinline__ void scan_pairs(Spheres8& sp, const ulonglong2* sA,
                                           const ulonglong2* sB, int npairs, int ph, int P,
                                           uint32_t* hitmask, const float* lim_lo) {
  const int ngroups = npairs / 4;
  int it = 0;
  for (int g = ph; g < ngroups; g += P) {
#pragma unroll
    for (int o = 0; o < 4; ++o) test_pair(sp, sA, sB, 4 * g + o);
    if ((++it & 7) == 0) {
      uint32_t h = definite_hits(sp, lim_lo);
      if (P > 1) {
        if (h) atomicOr(hitmask, h);
        h |= *reinterpret_cast<volatile uint32_t*>(hitmask);
      }
      if ((h & sp.real) == sp.real) break;
    }
  }
  const uint32_t h = definite_hits(sp, lim_lo);
  if (h) atomicOr(hitmask, h);
}

// Chunk staging, split so the loads of a tile's first chunk can be issued
// before the sphere gathers and stored after them.  Rows i >= len (up to the
// padded length) and non-finite rows become w = +inf: never a hit.
constexpr int kStageU = kChunk / kBT;  // rows per thread per chunk
struct StagedRows {
  float x[kStageU], y[kStageU], z[kStageU];
};
__device__ __forceinline__ void stage_load(StagedRows& r, const float* xs, uint32_t m4,
                                           uint32_t c0, uint32_t len) {
  const float INF = __int_as_float(0x7f800000);
#pragma unroll
  for (int u = 0; u < kStageU; ++u) {
    const uint32_t i = threadIdx.x + u * kBT;
    r.x[u] = r.y[u] = r.z[u] = INF;
    if (i < len) {
      r.x[u] = __ldg(xs + c0 + i);
      r.y[u] = __ldg(xs + m4 + c0 + i);
      r.z[u] = __ldg(xs + 2 * m4 + c0 + i);
    }
  }
}
__device__ __forceinline__ void stage_store(const StagedRows& r, ulonglong2* sA, ulonglong2* sB,
                                            uint32_t len8, const float4 org) {
  const float INF = __int_as_float(0x7f800000);
#pragma unroll
  for (int u = 0; u < kStageU; ++u) {
    const uint32_t i = threadIdx.x + u * kBT;
    if (i >= len8) break;
    float bx = 0.f, by = 0.f, bz = 0.f, w = INF;
    if (isfinite(r.x[u]) && isfinite(r.y[u]) && isfinite(r.z[u])) {
      bx = r.x[u] - org.x;
      by = r.y[u] - org.y;
      bz = r.z[u] - org.z;
      w = fmaf(bz, bz, fmaf(by, by, bx * bx));
    }
    sA[i] = make_ulonglong2(pack2(bx, bx), pack2(by, by));
    sB[i] = make_ulonglong2(pack2(bz, bz), pack2(w, w));
  }
}

// Final decision for a slot's spheres: definite hit -> verdict byte, definite
// miss -> nothing, inside the error band -> exact float64 path (k_slow).
__device__ __forceinline__ void decide(const Spheres8& sp, const SmemBinned& S, const BinArgs& a,
                                       int64_t s0, int64_t leaf, uint32_t hm, bool combined) {
#pragma unroll
  for (int i = 0; i < kS; ++i) {
    if (!((sp.real >> i) & 1u)) continue;
    const int e = sp.base + i;
    const float mv = combined ? okey_inv(S.minkey[e]) : sp.mn[i];
    // hits are flagged by list index (the slot's permutation entry); the
    // sphere id is gathered only for the rare ambiguous spheres
    if (((hm >> i) & 1u) || mv <= S.lim_lo[e]) {
      a.lhit[a.perm[s0 + e]] = 1;  // mapped back to the sphere by K6
    } else if (!(mv > S.lim_hi[e])) {
      const int q = a.lmeta[a.perm[s0 + e]].x;
      const unsigned j = atomicAdd(a.slow_n, 1u);
      a.slow[j] = make_int2(q, int(leaf));
      atomicAdd(a.n_refined, 1u);
    }
  }
}

// FFMA K5 min CTAs per SM: 6 (85 regs) beats 7 (spills) and 5
#ifndef CAPT_K5_MINB
#define CAPT_K5_MINB 6
#endif
__global__ void __launch_bounds__(kBT, CAPT_K5_MINB) k_binned_scan(BinArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmemBinned& S = *reinterpret_cast<SmemBinned*>(smem_raw);
  ulonglong2* const sA = S.A;
  ulonglong2* const sB = S.B;
  const DevTree& t = a.t;
  const int tid = threadIdx.x;
  const int n_tiles = int(*a.n_tiles);
  if (tid == 0) S.tile = int(atomicAdd(a.tile_ctr, 1u));
  __syncthreads();
  while (true) {
    const int tile = S.tile;
    if (tile >= n_tiles) break;
    // the next tile is drawn now (by warp 1, off warp 0's path); its index is
    // published after the tile's decision barrier
    int next = 0;
    if (tid == 32) next = int(atomicAdd(a.tile_ctr, 1u));
    const TileMeta tm = a.tiles[tile];
    const int64_t leaf = tm.leaf;
    const int64_t s0 = tm.s0;
    const int cnt = tm.cnt;
    const uint2 st = make_uint2(tm.setx, tm.m);
    const float4 org = tm.org;
    const uint32_t m = st.y;
    const uint32_t m4 = (m + 3u) & ~3u;
    const float* xs = reinterpret_cast<const float*>(t.data + st.x);

    // thread -> (sphere slot of kS spheres, phase over the point pairs)
    const int nslot = (cnt + kS - 1) / kS;
    const int P = max(1, kBT / nslot);
    const bool active = tid < nslot * P;
    const int slot = tid % nslot;
    const int ph = tid / nslot;
    // the first chunk's rows are loaded before the sphere gathers so that
    // both latencies overlap; the previous tile's final barrier freed sA/sB
    StagedRows rows;
    stage_load(rows, xs, m4, 0, min(uint32_t(kChunk), m));
    Spheres8 sp;
    load_spheres(sp, S, a, s0, org, cnt, slot, active, active && ph == 0);
    for (int e = tid; e < nslot * kS; e += kBT) S.minkey[e] = 0xffffffffu;
    for (int e = tid; e < nslot; e += kBT) S.hitmask[e] = 0;
    stage_store(rows, sA, sB, (min(uint32_t(kChunk), m) + 7u) & ~7u, org);

    // stream the set through shared memory in chunks of kChunk points
    bool done = sp.real == 0;
    for (uint32_t c0 = 0; c0 < m; c0 += kChunk) {
      const uint32_t len = min(uint32_t(kChunk), m - c0);
      const uint32_t len8 = (len + 7u) & ~7u;
      if (c0) {
        __syncthreads();  // previous chunk consumed
        stage_load(rows, xs, m4, c0, len);
        stage_store(rows, sA, sB, len8, org);
      }
      __syncthreads();  // chunk staged; inits and limits visible
      if (!done) {
        scan_pairs(sp, sA, sB, int(len8 / 2), ph, P, &S.hitmask[slot], S.lim_lo);
        uint32_t h = definite_hits(sp, S.lim_lo);
        if (P > 1) h |= *reinterpret_cast<volatile uint32_t*>(&S.hitmask[slot]);
        done = (h & sp.real) == sp.real;
      }
    }
    // combine the phases' minima, then each slot's owner decides
    if (P > 1 && active) {
#pragma unroll
      for (int i = 0; i < kS; ++i)
        if ((sp.real >> i) & 1u) atomicMin(&S.minkey[sp.base + i], okey(sp.mn[i]));
    }
    __syncthreads();
    if (tid == 32) S.tile = next;  // every thread has read S.tile by now
    if (active && ph == 0) decide(sp, S, a, s0, leaf, S.hitmask[slot], P > 1);
    __syncthreads();  // tile state (minkey, hitmask, smem points) free for the next tile
  }
}

// ---------------------------------------------------------------------------
// K5 on the tensor cores (tcgen05, kind::tf32).  For a tile of <= 512 spheres
// of one leaf and a chunk of <= 128 points of its set:
//     D[s][p] = w_p + (-2 a_s) . b_p     (a = c - o, b = p - o, w = |b|^2)
// as ONE 128 x N x 16 product per 128-sphere block, with every fp32 operand
// split into tf32 hi + lo parts (K = 16: Kh.bh + Kl.bh + Kh.bl + wh + wl;
// the dropped Kl.bl and the truncations are < 3 * 2^-20 |K||b|, tf32 products
// are exact, accumulation is fp32).  The accumulator lives in TMEM; each warp
// reads its 32 spheres' rows (tcgen05.ld) and keeps the running minimum.  A
// sphere collides iff min_p D <= r^2 - |a|^2; the decision band is
// kBandTc (|a|^2 + max|b|^2 + r^2), 16x the FFMA kernel's, so definite
// verdicts stay provably the reference's and the rest go to the exact queue.
// CTA: 128 threads; thread i owns row i of every 128-sphere block.
// ---------------------------------------------------------------------------
constexpr int kTcNc = CAPT_TC_NC;        // points per chunk
constexpr int kTcMb = kTsTc / 128;        // 128-sphere blocks per tile
constexpr float kBandTc = 0x1p-14f;
constexpr int kTcCols = kTcMb * kTcNc;    // TMEM columns: every block of a chunk at once

struct __align__(1024) SmemTc {
  unsigned char A[kTsTc * 64];   // sphere rows, K-major canonical layout
  unsigned char B[kTcNc * 64];   // point rows
  uint64_t mbar;
  uint32_t tmem;
  int tile;
};

__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// one operand row: 16 tf32 values at row r of a K-major tile
__device__ __forceinline__ void put_row(unsigned char* base, int r, const float (&v)[16]) {
#pragma unroll
  for (int k = 0; k < 16; k += 4)
    *reinterpret_cast<float4*>(base + tc::kmaj_off(r, k)) = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
}

constexpr int kTcThreads = 128 * kTcMb;  // one sphere row per thread
__global__ void __launch_bounds__(kTcThreads) k_binned_scan_tc(BinArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  SmemTc& S = *reinterpret_cast<SmemTc*>(smem_raw);
  const DevTree& t = a.t;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  if (tid == 0) tc::mbar_init(&S.mbar, 1);
  if (warp == 0) tc::tmem_alloc<kTcCols>(&S.tmem);
  // (TMEM and the barrier are set up while K3 drains; tiles, records and the
  // permutation come from K2/K3)
  pdl_wait();
  const int n_tiles = int(*a.n_tiles);
  if (tid == 0) S.tile = int(atomicAdd(a.tile_ctr, 1u));
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = S.tmem;
  // thread -> (128-sphere block tb, row): a warp reads the TMEM lanes of its
  // quadrant (warp % 4) in its block's columns
  const int tb = tid >> 7, row_id = tid & 127;
  const uint32_t taddr = tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(tb * kTcNc);
  uint32_t phase = 0;
  const float INF = __int_as_float(0x7f800000);
  while (true) {
    const int tile = S.tile;
    if (tile >= n_tiles) break;
    int next = 0;
    if (tid == 32) next = int(atomicAdd(a.tile_ctr, 1u));
    const TileMeta tm = a.tiles[tile];
    const int cnt = tm.cnt;
    const float4 org = tm.org;
    const uint32_t m4 = (tm.m + 3u) & ~3u;
    const uint32_t m = tm.m;
    const float* xs = reinterpret_cast<const float*>(t.data + tm.setx);
    const int nb = (cnt + 127) >> 7;  // sphere blocks in this tile
    // thread i < kTcNc stages row i of every chunk; the next chunk's point is
    // loaded while the current chunk's product runs (one chunk ahead), the
    // first one beside the sphere gathers
    static_assert(kTcNc <= kTcThreads, "one staged row per thread");
    float qx = INF, qy = INF, qz = INF;
    if (tid < kTcNc && uint32_t(tid) < m) {
      qx = __ldg(xs + tid);
      qy = __ldg(xs + m4 + tid);
      qz = __ldg(xs + 2 * m4 + tid);
    }
    // this thread's sphere: row row_id of block tb
    const int e = tb * 128 + row_id;
    float mn = INF, lim_lo = -INF, lim_hi = -INF;  // padding rows: never decided
    if (tb < nb) {
      float row[16];
      if (e < cnt) {
        const float4 rc = a.lrec[a.perm[tm.s0 + e]];
        const float ax = rc.x - org.x, ay = rc.y - org.y, az = rc.z - org.z;
        const float aa = fmaf(az, az, fmaf(ay, ay, ax * ax));
        const float r2 = rc.w * rc.w;
        const float thr = r2 - aa, band = kBandTc * (aa + org.w + r2);
        lim_lo = thr - band;
        lim_hi = thr + band;
        const float K[3] = {-2.f * ax, -2.f * ay, -2.f * az};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const float h = tf32_hi(K[d]);
          row[d] = h;
          row[3 + d] = tf32_hi(K[d] - h);
          row[6 + d] = h;
        }
        row[9] = 1.f;
        row[10] = 1.f;
      } else {
#pragma unroll
        for (int k = 0; k < 11; ++k) row[k] = 0.f;
      }
#pragma unroll
      for (int k = 11; k < 16; ++k) row[k] = 0.f;
      put_row(S.A, e, row);
    }
    bool done = false;
    for (uint32_t c0 = 0; c0 < m && !done; c0 += kTcNc) {
      const uint32_t len = min(uint32_t(kTcNc), m - c0);
      const uint32_t nc = (len + 31u) & ~31u;  // MMA N (multiple of 16) = whole TMEM loads
      // stage the chunk's point rows (w = +inf for padding / non-finite rows)
      if (uint32_t(tid) < nc) {
        const uint32_t i = tid;
        const float px = qx, py = qy, pz = qz;
        float row[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) row[k] = 0.f;
        if (isfinite(px) && isfinite(py) && isfinite(pz)) {
          const float bv[3] = {px - org.x, py - org.y, pz - org.z};
          const float w = fmaf(bv[2], bv[2], fmaf(bv[1], bv[1], bv[0] * bv[0]));
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const float h = tf32_hi(bv[d]);
            row[d] = h;
            row[3 + d] = h;
            row[6 + d] = tf32_hi(bv[d] - h);
          }
          const float wh = tf32_hi(w);
          row[9] = wh;
          row[10] = tf32_hi(w - wh);
        } else {
          row[9] = INF;
        }
        put_row(S.B, int(i), row);
      }
      tc::fence_async_smem();
      __syncthreads();
      {
        const uint32_t j = c0 + kTcNc + tid;  // next chunk's row for this thread
        qx = qy = qz = INF;
        if (tid < kTcNc && j < m) {
          qx = __ldg(xs + j);
          qy = __ldg(xs + m4 + j);
          qz = __ldg(xs + 2 * m4 + j);
        }
      }
      // every block's product for this chunk in one batch, one commit
      if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t idesc = tc::idesc_tf32(128, int(nc));
        const uint32_t sb = tc::smem_u32(S.B);
        for (int b = 0; b < nb; ++b) {
          const uint32_t sa = tc::smem_u32(S.A) + uint32_t(b) * 16u * tc::kRowBlockBytes;
          const uint32_t d = tmem + uint32_t(b * kTcNc);
          tc::mma_tf32(d, tc::make_desc(sa), tc::make_desc(sb), idesc, 0u);
          tc::mma_tf32(d, tc::make_desc(sa + 2 * tc::kCoreBytes), tc::make_desc(sb + 2 * tc::kCoreBytes),
                       idesc, 1u);
        }
        tc::commit(&S.mbar);
      }
      tc::mbar_wait(&S.mbar, phase);
      phase ^= 1u;
      tc::fence_after_sync();
      if (tb < nb) {  // warp-uniform (tb is per warp)
        float bm = INF;
        for (uint32_t c = 0; c < nc; c += 32) {
          uint32_t v[32];
          tc::tmem_ld32(taddr + c, v);
          tc::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; j += 2)
            bm = fmin3(bm, __uint_as_float(v[j]), __uint_as_float(v[j + 1]));
        }
        mn = fminf(mn, bm);
      }
      tc::fence_before_sync();
      done = __syncthreads_and(tb >= nb || e >= cnt || mn <= lim_lo);
    }
    // decision (thread-owned sphere)
    if (tb < nb && e < cnt) {
      if (mn <= lim_lo) {
        a.lhit[a.perm[tm.s0 + e]] = 1;
      } else if (!(mn > lim_hi)) {
        const int q = a.lmeta[a.perm[tm.s0 + e]].x;
        const unsigned j = atomicAdd(a.slow_n, 1u);
        a.slow[j] = make_int2(q, tm.leaf);
        atomicAdd(a.n_refined, 1u);
      }
    }
    if (tid == 32) S.tile = next;
    __syncthreads();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0) tc::tmem_free<kTcCols>(tmem);
  pdl_trigger();
}

// Exact float64 path, one warp per queued sphere: lanes split the set,
// query.py:96-99 arithmetic (fp64, no FMA), ballot OR.
template <typename InT>
__global__ void k_slow(BinArgs a) {
  pdl_wait();
  // K5's hits, flagged by list index -> the spheres' verdict bytes
  {
    const uint32_t nl = *a.list_n;
    // 8 entries per thread, strided by the grid so that every load coalesces
    constexpr int kU = 8;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t j0 = blockIdx.x * blockDim.x + threadIdx.x; j0 < nl; j0 += kU * stride) {
      uint8_t f[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t j = j0 + u * stride;
        f[u] = j < nl ? __ldcs(a.lhit + j) : 0;
      }
      int q[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) q[u] = f[u] ? __ldcs(&a.lmeta[j0 + u * stride].x) : -1;
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (q[u] >= 0) a.verdict[q[u]] = 1;
    }
  }
  const unsigned n = *a.slow_n;
  const int lane = threadIdx.x & 31;
  const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
  const DevTree& t = a.t;
  for (unsigned i = warp; i < n; i += nwarps) {
    const int2 e = a.slow[i];
    double c64[3], r64;
    load_sphere<InT>(a.centers, a.radii, e.x, t.k, c64, r64);
    const uint2 st = t.set[e.y];
    const float* base = reinterpret_cast<const float*>(t.data + st.x);
    const uint32_t m4 = (st.y + 3u) & ~3u;
    // fp32 first pass in the direct form (relative error < 5u, band TAU as in
    // the direct kernels): most spheres the binned scan left ambiguous (its
    // band is wider) are decided here; the rest take the float64 pass
    {
      const float cf[3] = {float(c64[0]), float(c64[1]), float(c64[2])};
      const float rf = float(r64), r2 = rf * rf;
      const bool fast = double(cf[0]) == c64[0] && double(cf[1]) == c64[1] &&
                        double(cf[2]) == c64[2] && double(rf) == r64 && isfinite(cf[0]) &&
                        isfinite(cf[1]) && isfinite(cf[2]) && r2 >= kR2Min && r2 <= kR2Max;
      if (fast && t.k == 3) {
        const float loB = r2 * (1.0f - kTau), hiB = r2 * (1.0f + kTau);
        bool h32 = false, amb = false;
        for (uint32_t j0 = 0; j0 < st.y && !__any_sync(0xffffffffu, h32); j0 += 128) {
          float px[4], py[4], pz[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t j = j0 + u * 32 + lane;
            const bool in = j < m4;
            px[u] = in ? __ldg(base + j) : __int_as_float(0x7f800000);
            py[u] = in ? __ldg(base + m4 + j) : 0.f;
            pz[u] = in ? __ldg(base + 2 * m4 + j) : 0.f;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float dx = cf[0] - px[u], dy = cf[1] - py[u], dz = cf[2] - pz[u];
            const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
            h32 |= d2 <= loB;
            amb |= d2 < hiB;
          }
        }
        if (__any_sync(0xffffffffu, h32)) {
          if (lane == 0) a.verdict[e.x] = 1;
          continue;
        }
        if (!__any_sync(0xffffffffu, amb)) continue;  // definite miss
      }
    }
    const double R = __dmul_rn(r64, r64);
    bool hit = false;
    // 4 rows per lane per step: the loads of 128 points are in flight at once
    for (uint32_t j0 = 0; j0 < st.y && !__any_sync(0xffffffffu, hit); j0 += 128) {
      float p[4][kMaxK];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t j = j0 + u * 32 + lane;
#pragma unroll
        for (int d = 0; d < kMaxK; ++d)
          p[u][d] = (j < st.y && d < t.k) ? __ldg(base + d * m4 + j) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j0 + u * 32 + lane >= st.y) continue;
        double sum = 0.0;
#pragma unroll
        for (int d = 0; d < kMaxK; ++d) {
          if (d >= t.k) break;
          const double x = __dsub_rn(c64[d], double(p[u][d]));
          const double sq = __dmul_rn(x, x);
          sum = d == 0 ? sq : __dadd_rn(sum, sq);
        }
        hit |= sum <= R;
      }
    }
    if (__any_sync(0xffffffffu, hit) && lane == 0) a.verdict[e.x] = 1;
  }
  pdl_trigger();
}

// One thread per lane group: its L verdict bytes in one vector load (L <= 8:
// 1/2/4/8 bytes; larger L: several 8-byte loads), coalesced across the warp;
// the warp ballot is the verdict word.  The verdict array is padded to a
// multiple of 8 bytes past n.
__global__ void k_pack(int64_t n_groups, int L, const uint8_t* __restrict__ v,
                       uint32_t* __restrict__ bits, int64_t n_words) {
  pdl_wait();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t n_thr = n_words * 32;
  for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < n_thr; g += stride) {
    bool any = false;
    if (g < n_groups) {
      const uint8_t* p = v + g * L;
      switch (L) {
        case 1: any = p[0] != 0; break;
        case 2: any = *reinterpret_cast<const uint16_t*>(p) != 0; break;
        case 4: any = *reinterpret_cast<const uint32_t*>(p) != 0; break;
        case 8: any = *reinterpret_cast<const uint64_t*>(p) != 0; break;
        default: {
          const uint64_t* q = reinterpret_cast<const uint64_t*>(p);
          uint64_t acc = 0;
          for (int k = 0; k < L / 8; ++k) acc |= q[k];
          any = acc != 0;
        }
      }
    }
    const uint32_t word = __ballot_sync(0xffffffffu, any);
    if ((threadIdx.x & 31) == 0) bits[g >> 5] = word;
  }
}

struct Arena {
  cudaStream_t s;
  void* ptrs[24];
  int np = 0;
  template <class T>
  T* get(size_t count) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, (count ? count : 1) * sizeof(T), s) != cudaSuccess) return nullptr;
    ptrs[np++] = p;
    return static_cast<T*>(p);
  }
  ~Arena() {
    for (int i = 0; i < np; ++i) cudaFreeAsync(ptrs[i], s);
  }
};

}  // namespace

__global__ void k_zero(uint32_t* __restrict__ p, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = 0u;
  pdl_trigger();
}

// launch with programmatic stream serialisation (see pdl_wait)
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem,
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

bool binned_preferred(const DevTree& t, int64_t n, uint32_t flags) {
  if (flags & CAPT_STATS) return false;
  if (flags & (CAPT_MODE_DIRECT | CAPT_MODE_THREAD)) return false;
  if (n >= (int64_t(1) << 31)) return false;
  if (flags & CAPT_MODE_BINNED) return true;
  // measured: the hybrid unbinned kernel wins below ~1 M spheres (config-4
  // sweep: 5.7 vs 2.8 G q/s at 256 K, a tie at 1 M, 13 vs 26 at 4 M); with
  // large sets (config 3, mean 1.8 k points) the binned pipeline already wins
  // 2x at 1 M spheres, whatever the leaf count
  return n >= (int64_t(1) << 20);
}

int launch_binned(const DevTree& t, const void* centers, const void* radii, int64_t n, int L,
                  const uint8_t* mask, uint32_t flags, uint32_t* bits, int64_t n_words,
                  unsigned long long* first_bad, cudaStream_t s) {
  constexpr int V = kK1V;
  struct Setup {
    int sms = 0, occ = 0, occ_tc = 0;
  };
  static DeviceOnce once;
  static Setup setup[kMaxDevices];
  {
    const int rc = per_device_once(once, [&](int dev) {
      Setup& u = setup[dev];
      CAPT_CUDA(cudaFuncSetAttribute(k_binned_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(SmemBinned))));
      CAPT_CUDA(cudaFuncSetAttribute(k_bin_count3<V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(float) * kSmemNodes3)));
      CAPT_CUDA(cudaFuncSetAttribute(k_binned_scan_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(SmemTc))));
      CAPT_CUDA(cudaDeviceGetAttribute(&u.sms, cudaDevAttrMultiProcessorCount, dev));
      CAPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&u.occ, k_binned_scan, kBT,
                                                              sizeof(SmemBinned)));
      if (u.occ < 1) u.occ = 1;
      u.occ_tc = 512 / kTcCols;  // TMEM columns per SM
      if (u.occ_tc > 8) u.occ_tc = 8;
      return CAPT_OK;
    });
    if (rc) return rc;
  }
  int dev = 0;
  CAPT_CUDA(cudaGetDevice(&dev));
  const Setup& u = setup[dev];
  Arena A;
  A.s = s;
  BinArgs a;
  memset(&a, 0, sizeof(a));
  a.t = t;
  a.centers = centers;
  a.radii = radii;
  a.n = n;
  a.L = L;
  a.mask = mask;
  a.flags = flags;
  a.first_bad = first_bad;
  const int64_t nl = t.n;
  // everything that must start at zero, in one block (one memset):
  // counters (slow_n, n_tiles, tile_ctr, n_refined, list_n) | counts | cursor | bcursor
  const int64_t zero_words = 8 + 2 * nl + kBuckets;
  uint32_t* ctr = A.get<uint32_t>(zero_words);
  a.counts = ctr ? ctr + 8 : nullptr;
  a.cursor = ctr ? ctr + 8 + nl : nullptr;
  a.bcursor = ctr ? ctr + 8 + 2 * nl : nullptr;
  a.start = A.get<uint32_t>(nl);
  a.tstart = A.get<uint32_t>(nl);
  // K5 on the tensor cores unless CAPT_K5_FFMA selects the CUDA-core kernel
  const bool use_tc = !(flags & CAPT_K5_FFMA);
  a.ts = use_tc ? uint32_t(kTsTc) : uint32_t(kTS);
  a.tiles = A.get<TileMeta>(nl + n / a.ts + 1);
  a.perm = A.get<uint32_t>(n);
  a.verdict = A.get<uint8_t>(n + 8);
  a.slow = A.get<int2>(n);
  a.lrec = A.get<float4>(n);
  a.lmeta = A.get<int2>(n);
  a.lhit = A.get<uint8_t>(n);
  a.part = A.get<int2>(n);
  a.bshift = 0;
  while ((nl >> a.bshift) > kBuckets) ++a.bshift;
  if (!a.part || !a.bcursor || !ctr || !a.counts || !a.start || !a.tstart || !a.tiles || !a.perm ||
      !a.verdict || !a.slow || !a.lrec || !a.lmeta || !a.lhit || !a.cursor)
    return fail(CAPT_ENOMEM, "binned scratch allocation");
  {
    float lo = float(t.r_min), hi = float(t.r_max);
    if (double(lo) < t.r_min) lo = nextafterf(lo, INFINITY);
    if (double(hi) > t.r_max) hi = nextafterf(hi, -INFINITY);
    a.rlo_f = lo;
    a.rhi_f = hi;
  }
  a.slow_n = ctr;
  a.n_tiles = ctr + 1;
  a.tile_ctr = ctr + 2;
  a.n_refined = ctr + 3;
  a.list_n = ctr + 4;
  // (verdict bytes need no clearing: K1 writes one for every sphere)
  k_zero<<<grid_for(zero_words, 256, 4), 256, 0, s>>>(ctr, zero_words);
  const bool f64 = flags & CAPT_INPUT_F64;
  const int G = grid_for(n, 256, 8);
  const int G4 = grid_for((n + V - 1) / V, 256, 8);
  if (f64) k_bin_count<double><<<G, 256, 0, s>>>(a);
  else if (t.k == 3) {
    CAPT_CUDA(launch_pdl(k_bin_count3<V>, G4, 256, sizeof(float) * kSmemNodes3, s, a));
  }
  else k_bin_count<float><<<G, 256, 0, s>>>(a);
  // per-leaf starts and tiles
  if (nl <= kScanSingleMax) {
    CAPT_CUDA(launch_pdl(k_scan_tiles, 1, kScanT, 0, s, a));
  } else {
    uint32_t* tc = A.get<uint32_t>(nl);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, a.counts, a.start, nl, s);
    void* tmp = A.get<char>(tb);
    if (!tc || !tmp) return fail(CAPT_ENOMEM, "binned scratch allocation");
    CAPT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, a.counts, a.start, nl, s));
    k_tile_counts<<<grid_for(nl, 256, 8), 256, 0, s>>>(a, tc);
    CAPT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, tc, a.tstart, nl, s));
    k_tile_total<<<1, 1, 0, s>>>(a, tc);
    note_launches(6);
  }
  {
    const int Gp = grid_for((n + kPartItems - 1) / kPartItems * 256, 256, 4);
    CAPT_CUDA(launch_pdl(k_part_bucket, Gp, 256, 0, s, a));
    CAPT_CUDA(launch_pdl(k_part_leaf, Gp, 256, 0, s, a));
  }
  if (use_tc) {
    CAPT_CUDA(launch_pdl(k_binned_scan_tc, u.sms * u.occ_tc, kTcThreads, sizeof(SmemTc), s, a));
  } else {
    k_binned_scan<<<u.sms * u.occ, kBT, sizeof(SmemBinned), s>>>(a);
  }
  if (f64) CAPT_CUDA(launch_pdl(k_slow<double>, u.sms * 8, 128, 0, s, a));
  else CAPT_CUDA(launch_pdl(k_slow<float>, u.sms * 8, 128, 0, s, a));
  CAPT_CUDA(launch_pdl(k_pack, grid_for(n_words * 32, 256, 8), 256, 0, s, n / L, L,
                         static_cast<const uint8_t*>(a.verdict), bits, n_words));
  CAPT_CUDA(cudaGetLastError());
  note_launches(8);  // zero, count, scan+tiles, 2 partition passes, scan, slow, pack
  return CAPT_OK;
}

}  // namespace capt
