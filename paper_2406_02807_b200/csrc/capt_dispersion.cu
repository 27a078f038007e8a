// Nearest-neighbour distances of a cloud (the dispersion proxy of
// oracle.py:141-158, which queries a float64 cKDTree with k=2 and keeps the
// second hit: the nearest OTHER point, duplicates at distance 0).
//
// Exact brute force in float64: every point is compared with every other one,
// the squared distance accumulated axis by axis as ((d0^2 + d1^2) + d2^2)
// without contraction, the minimum taken over the squares and one correctly
// rounded sqrt at the end -- the same value a float64 k-d tree returns.  The
// candidate points stream through shared memory in tiles; one thread owns one
// query point.  O(n^2) fp64 work (a 300 k-point cloud is ~10^11 pair tests, a
// few tens of ms); the mean/median/p95 are taken on the host with numpy, as in
// the reference.
#include <cuda_runtime.h>

#include <cfloat>

#include "capt_internal.cuh"

namespace capt {
namespace {

constexpr int kNnT = 256;
constexpr int kNnTile = 1024;

__global__ void __launch_bounds__(kNnT) k_nn(const float* __restrict__ pts, int64_t n, int k,
                                           double* __restrict__ out) {
  __shared__ float tile[kNnTile * kMaxK];
  const int64_t i = int64_t(blockIdx.x) * kNnT + threadIdx.x;
  double p[kMaxK] = {0.0, 0.0, 0.0};
  if (i < n)
    for (int d = 0; d < k; ++d) p[d] = double(pts[i * k + d]);
  double best = DBL_MAX;
  for (int64_t t0 = 0; t0 < n; t0 += kNnTile) {
    const int len = int(min(int64_t(kNnTile), n - t0));
    __syncthreads();
    for (int e = threadIdx.x; e < len * k; e += kNnT) tile[e] = pts[t0 * k + e];
    __syncthreads();
    if (i < n) {
      if (k == 3) {
        for (int j = 0; j < len; ++j) {
          const double x = __dsub_rn(double(tile[3 * j]), p[0]);
          const double y = __dsub_rn(double(tile[3 * j + 1]), p[1]);
          const double z = __dsub_rn(double(tile[3 * j + 2]), p[2]);
          const double s = __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z));
          if (t0 + j != i && s < best) best = s;
        }
      } else {
        for (int j = 0; j < len; ++j) {
          double s = 0.0;
          for (int d = 0; d < k; ++d) {
            const double x = __dsub_rn(double(tile[k * j + d]), p[d]);
            s = d == 0 ? __dmul_rn(x, x) : __dadd_rn(s, __dmul_rn(x, x));
          }
          if (t0 + j != i && s < best) best = s;
        }
      }
    }
  }
  if (i < n) out[i] = __dsqrt_rn(best);
}

}  // namespace
}  // namespace capt

using namespace capt;

extern "C" int capt_nn_distances(int device, int k, const float* points, int64_t n,
                                 uint32_t flags, double* out, void* stream) {
  if (k < 1 || k > kMaxK) return fail(CAPT_EINVAL, "k must be 1..3");
  if (n < 2) return fail(CAPT_EINVAL, "dispersion needs at least 2 points");
  if (!points || !out) return fail(CAPT_EINVAL, "NULL argument");
  CAPT_CUDA(cudaSetDevice(device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool host = flags & CAPT_HOST_IO;
  const float* d_pts = points;
  double* d_out = out;
  if (host) {
    float* dp = nullptr;
    double* dq = nullptr;
    CAPT_CUDA(cudaMallocAsync(&dp, sizeof(float) * k * n, s));
    CAPT_CUDA(cudaMallocAsync(&dq, sizeof(double) * n, s));
    CAPT_CUDA(cudaMemcpyAsync(dp, points, sizeof(float) * k * n, cudaMemcpyHostToDevice, s));
    d_pts = dp;
    d_out = dq;
  }
  k_nn<<<int((n + kNnT - 1) / kNnT), kNnT, 0, s>>>(d_pts, n, k, d_out);
  CAPT_CUDA(cudaGetLastError());
  note_launches(1);
  if (host) {
    CAPT_CUDA(cudaMemcpyAsync(out, d_out, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(const_cast<float*>(d_pts), s);
    cudaFreeAsync(d_out, s);
    CAPT_CUDA(cudaStreamSynchronize(s));
  }
  return CAPT_OK;
}
