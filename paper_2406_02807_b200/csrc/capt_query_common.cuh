// Device helpers shared by the direct and binned query kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "capt_internal.cuh"

namespace capt {

// one 256-bit load (sm_100): a leaf's probe record
__device__ __forceinline__ void ld_v8(const float* p, float (&v)[8]) {
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
        "=f"(v[7])
      : "l"(p));
}
// two fp16 values packed in a float's bits -> float2
__device__ __forceinline__ float2 h2f2(float bits) {
  const unsigned u = __float_as_uint(bits);
  return __half22float2(*reinterpret_cast<const __half2*>(&u));
}
// shared-memory load at an absolute shared-window address
__device__ __forceinline__ float lds_f32(unsigned addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

// Top 12 levels of the Eytzinger split array live in shared memory (16 KB).
constexpr int kSmemNodes = 4095;

// Relative decision band: the fp32 distance has relative error < 5u
// (u = 2^-24: one rounded difference per axis, one product, two rounded
// fused adds), r^2 one more u; TAU = 2^-19 = 32u leaves a wide margin.
constexpr float kTau = 0x1p-19f;
constexpr float kR2Min = 0x1p-100f;  // outside [kR2Min, kR2Max] -> float64 path
constexpr float kR2Max = 0x1p100f;

// c[ax] without dynamic indexing (keeps the centre in registers)
template <typename C>
__device__ __forceinline__ C pick3(const C c[3], int ax) {
  return ax == 0 ? c[0] : (ax == 1 ? c[1] : c[2]);
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// np.maximum: NaN-propagating
__device__ __forceinline__ double np_max(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a >= b ? a : b;
}

// leaf_indices (tree.py:266-273): i = 2i + 1 + (x[step % k] > T[i]).
// The reference compares fp32 values upcast to float64 -> identical to an
// fp32 compare for fp32 inputs; float64 inputs compare in float64.
template <typename C>
__device__ __forceinline__ int64_t descend_t(const DevTree& t, const float* sT, int n_smem,
                                             const C c[3]) {
  int64_t i = 0;
  int ax = 0;
  for (int s = 0; s < t.depth; ++s) {
    const float tv = (i < n_smem) ? sT[i] : __ldg(t.T + i);
    i = 2 * i + 1 + (pick3(c, ax) > C(tv) ? 1 : 0);
    ax = (ax + 1 == t.k) ? 0 : ax + 1;
  }
  return i - (t.n - 1);
}

__device__ __forceinline__ int64_t descend(const DevTree& t, const float* sT, int n_smem,
                                           const double c64[3]) {
  return descend_t<double>(t, sT, n_smem, c64);
}

// Exact reference AABB prefilter (query.py:202-208): fp64 copies of the fp32
// box, res = max(max(lo - c, 0), c - hi), ((r0^2 + r1^2) + r2^2) <= r^2.
__device__ __forceinline__ bool aabb_keep64(int k, const float4 lo, const float4 hi,
                                            const double c[3], double R) {
  const double l[3] = {lo.x, lo.y, lo.z};
  const double h[3] = {hi.x, hi.y, hi.z};
  double s = 0.0;
#pragma unroll
  for (int d = 0; d < kMaxK; ++d) {
    if (d >= k) break;
    double r = np_max(__dsub_rn(l[d], c[d]), 0.0);
    r = np_max(r, __dsub_rn(c[d], h[d]));
    const double sq = __dmul_rn(r, r);
    s = (d == 0) ? sq : __dadd_rn(s, sq);
  }
  return s <= R;
}

// Exact reference scan of one affordance set (query.py:96-99, 214-218).
static __device__ __noinline__ bool scan_f64(const DevTree& t, uint2 set, const double c[3],
                                      double r64, bool* boundary) {
  const float* base = reinterpret_cast<const float*>(t.data + set.x);
  const uint32_t m4 = (set.y + 3u) & ~3u;
  const double R = __dmul_rn(r64, r64);
  bool hit = false;
  for (uint32_t i = 0; i < set.y; ++i) {
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < kMaxK; ++d) {
      if (d >= t.k) break;
      const double x = __dsub_rn(c[d], double(__ldg(base + d * m4 + i)));
      const double sq = __dmul_rn(x, x);
      s = (d == 0) ? sq : __dadd_rn(s, sq);
    }
    if (s <= R) {
      hit = true;
      if (!boundary) break;
    }
    if (boundary && fabs(s - R) < 1e-6) *boundary = true;
  }
  return hit;
}

// Shared per-sphere setup.  Returns ST_FALSE (0) when the verdict is false
// (non-finite centre, AABB reject), ST_SCAN (2) for the fp32 scan, ST_SLOW (3)
// for the exact float64 scan (radius outside the safe fp32 range, or a
// float64 input that is not exactly representable in fp32).
__device__ __forceinline__ int classify(const DevTree& t, int64_t leaf, const double c64[3],
                                        double r64, bool prefilter, float& cx, float& cy,
                                        float& cz, float& r2, float& loB, float& hiB) {
  bool cfin = true;
#pragma unroll
  for (int d = 0; d < kMaxK; ++d) cfin &= d >= t.k || isfinite(c64[d]);
  // +-inf / NaN centres give inf or NaN distances: never a collision unless
  // r^2 itself overflows to inf (then the exact path decides)
  if (!cfin && __dmul_rn(r64, r64) <= 1.7976931348623157e308) return 0;
  const float cf0 = float(c64[0]), cf1 = float(c64[1]), cf2 = float(c64[2]);
  const float rf = float(r64);
  const bool exact = double(cf0) == c64[0] && double(cf1) == c64[1] && double(cf2) == c64[2] &&
                     double(rf) == r64;
  r2 = rf * rf;
  const bool fast = cfin && exact && r2 >= kR2Min && r2 <= kR2Max;
  cx = cf0;
  cy = cf1;
  cz = cf2;
  loB = r2 * (1.0f - kTau);
  hiB = r2 * (1.0f + kTau);
  if (prefilter) {
    const float4 lo = __ldg(t.box + 2 * leaf);
    const float4 hi = __ldg(t.box + 2 * leaf + 1);
    bool exact_check = !fast;
    if (fast) {
      const float rx = fmaxf(fmaxf(lo.x - cx, 0.f), cx - hi.x);
      const float ry = fmaxf(fmaxf(lo.y - cy, 0.f), cy - hi.y);
      const float rz = fmaxf(fmaxf(lo.z - cz, 0.f), cz - hi.z);
      const float s = fmaf(rz, rz, fmaf(ry, ry, rx * rx));
      if (s > hiB) return 0;
      if (s >= loB) exact_check = true;
    }
    if (exact_check && !aabb_keep64(t.k, lo, hi, c64, __dmul_rn(r64, r64))) return 0;
  }
  return fast ? 2 : 3;
}

// fp32 test of 4 points (SoA float4 of x, y, z).
__device__ __forceinline__ void test4(const float4 px, const float4 py, const float4 pz,
                                      float cx, float cy, float cz, float r2, float loB,
                                      float hiB, bool& hit, bool& amb, bool& bnd, bool stats) {
  const float xs[4] = {px.x, px.y, px.z, px.w};
  const float ys[4] = {py.x, py.y, py.z, py.w};
  const float zs[4] = {pz.x, pz.y, pz.z, pz.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float dx = cx - xs[i], dy = cy - ys[i], dz = cz - zs[i];
    const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    hit |= d2 <= loB;
    amb |= d2 < hiB;
    if (stats)
      bnd |= isfinite(d2) && fabsf(d2 - r2) <= 1.001e-6f + 0x1p-17f * fmaxf(d2, r2);
  }
}

// fp32 cooperative scan: 0 = no point within the band, 1 = definite hit,
// 2 = some point inside the error band (decide exactly).
__device__ __forceinline__ int warp_scan_f32(const DevTree& t, uint2 set, float cx, float cy,
                                             float cz, float loB, float hiB, int lane) {
  const float* xs = reinterpret_cast<const float*>(t.data + set.x);
  const uint32_t m4 = (set.y + 3u) & ~3u;
  bool amb = false;
  for (uint32_t p0 = 0; p0 < set.y; p0 += 128) {
    float x[4], y[4], z[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t p = p0 + j * 32 + lane;
      x[j] = y[j] = z[j] = __int_as_float(0x7f800000);
      if (p < m4) {
        x[j] = __ldg(xs + p);
        y[j] = __ldg(xs + m4 + p);
        z[j] = __ldg(xs + 2 * m4 + p);
      }
    }
    bool hit = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float dx = cx - x[j], dy = cy - y[j], dz = cz - z[j];
      const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      hit |= d2 <= loB;
      amb |= d2 < hiB;
    }
    if (__any_sync(0xffffffffu, hit)) return 1;
  }
  return __any_sync(0xffffffffu, amb) ? 2 : 0;
}

// Exact reference scan (query.py:96-99), one point per lane per step.
// Exact scan of rows [0, rows) of a set stored SoA with stride m4 from base:
// 128 rows per step (4 per lane, all loads in flight), warp vote per step.
__device__ __forceinline__ bool warp_scan_f64_rows(const float* base, uint32_t m4, uint32_t rows,
                                                   int k, const double c[3], double R, int lane) {
  for (uint32_t p0 = 0; p0 < rows; p0 += 128) {
    float v[4][kMaxK];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t p = p0 + 32 * u + lane;
      const uint32_t pc = p < rows ? p : 0u;
#pragma unroll
      for (int d = 0; d < kMaxK; ++d) v[u][d] = d < k ? __ldg(base + d * m4 + pc) : 0.f;
    }
    bool hit = false;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (p0 + 32 * u + lane >= rows) continue;
      double s = 0.0;
#pragma unroll
      for (int d = 0; d < kMaxK; ++d) {
        if (d >= k) break;
        const double x = __dsub_rn(c[d], double(v[u][d]));
        const double sq = __dmul_rn(x, x);
        s = (d == 0) ? sq : __dadd_rn(s, sq);
      }
      hit |= s <= R;
    }
    if (__any_sync(0xffffffffu, hit)) return true;
  }
  return false;
}

__device__ __forceinline__ bool warp_scan_f64(const DevTree& t, uint2 set, const double c[3],
                                              double r64, int lane) {
  const float* base = reinterpret_cast<const float*>(t.data + set.x);
  const uint32_t m4 = (set.y + 3u) & ~3u;
  return warp_scan_f64_rows(base, m4, set.y, t.k, c, __dmul_rn(r64, r64), lane);
}

// Warp-cooperative descent (tree.py:266-273): 5 Eytzinger levels per L1/L2
// round trip -- lane j loads node j of the 31-node subtree under the current
// node, the path is then walked with shuffles.
template <typename C>
__device__ __forceinline__ int64_t warp_descend(const DevTree& t, const C c[3], int lane) {
  int64_t i = 0;
  int ax = 0;
  for (int s = 0; s < t.depth;) {
    const int lv = min(5, t.depth - s);
    const int nodes = (1 << lv) - 1;
    float tv = 0.f;
    if (lane < nodes) {
      const int lvl = 31 - __clz(lane + 1);
      const int64_t g = ((i + 1) << lvl) - 1 + (lane + 1 - (1 << lvl));
      tv = __ldg(t.T + g);
    }
    int j = 0;
    for (int r = 0; r < lv; ++r) {
      const float v = __shfl_sync(0xffffffffu, tv, j);
      j = 2 * j + 1 + (pick3(c, ax) > C(v) ? 1 : 0);
      ax = (ax + 1 == t.k) ? 0 : ax + 1;
    }
    i = ((i + 1) << lv) - 1 + (j + 1 - (1 << lv));
    s += lv;
  }
  return i - (t.n - 1);
}

}  // namespace capt
