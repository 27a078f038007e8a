// Diagnostic: one 128 x 256 x 16 tf32 tcgen05 product through the operand
// layout / descriptor helpers of capt_tc.cuh, checked on the host.  Used by
// tests/test_gpu_tc.py to pin the layout before the binned scan relies on it.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "capt_internal.cuh"
#include "capt_tc.cuh"

namespace capt {
namespace {

constexpr int kM = 128, kN = 256;

__global__ void __launch_bounds__(128) k_tc_selftest(const float* __restrict__ A,
                                                     const float* __restrict__ B,
                                                     float* __restrict__ D) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sa = smem;                                   // kM rows x 64 B
  unsigned char* sb = smem + kM * 64;                         // kN rows x 64 B
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + (kM + kN) * 64);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(mbar + 1);
  const int tid = threadIdx.x;
  for (int i = tid; i < kM * tc::kTcK; i += blockDim.x) {
    const int r = i / tc::kTcK, k = i % tc::kTcK;
    *reinterpret_cast<float*>(sa + tc::kmaj_off(r, k)) = A[i];
  }
  for (int i = tid; i < kN * tc::kTcK; i += blockDim.x) {
    const int r = i / tc::kTcK, k = i % tc::kTcK;
    *reinterpret_cast<float*>(sb + tc::kmaj_off(r, k)) = B[i];
  }
  if (tid == 0) tc::mbar_init(mbar, 1);
  if (tid < 32) tc::tmem_alloc<256>(tbase);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tbase;
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_tf32(kM, kN);
    const uint32_t a0 = tc::smem_u32(sa), b0 = tc::smem_u32(sb);
    tc::mma_tf32(tmem, tc::make_desc(a0), tc::make_desc(b0), idesc, 0u);
    tc::mma_tf32(tmem, tc::make_desc(a0 + 2 * tc::kCoreBytes), tc::make_desc(b0 + 2 * tc::kCoreBytes),
                 idesc, 1u);
    tc::commit(mbar);
  }
  tc::mbar_wait(mbar, 0);
  tc::fence_after_sync();
  const int warp = tid >> 5;
  for (int c0 = 0; c0 < kN; c0 += 32) {
    uint32_t v[32];
    tc::tmem_ld32(tmem + (uint32_t(32 * warp) << 16) + uint32_t(c0), v);
    tc::tmem_wait_ld();
    for (int j = 0; j < 32; ++j) D[tid * kN + c0 + j] = __uint_as_float(v[j]);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (tid < 32) tc::tmem_free<256>(tmem);
}

}  // namespace
}  // namespace capt

using namespace capt;

extern "C" int capt_tc_selftest(int device, double* max_rel_err) {
  if (!max_rel_err) return fail(CAPT_EINVAL, "NULL argument");
  CAPT_CUDA(cudaSetDevice(device));
  std::vector<float> A(kM * tc::kTcK), B(kN * tc::kTcK), D(kM * kN);
  uint32_t s = 12345u;
  auto rnd = [&]() {
    s = s * 1664525u + 1013904223u;
    float f = float((s >> 8) & 0xFFFF) / 65536.0f - 0.5f;
    uint32_t u;
    memcpy(&u, &f, 4);
    u &= 0xFFFFE000u;  // exactly representable in tf32
    memcpy(&f, &u, 4);
    return f;
  };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  float *dA = nullptr, *dB = nullptr, *dD = nullptr;
  CAPT_CUDA(cudaMalloc(&dA, 4 * A.size()));
  CAPT_CUDA(cudaMalloc(&dB, 4 * B.size()));
  CAPT_CUDA(cudaMalloc(&dD, 4 * D.size()));
  CAPT_CUDA(cudaMemcpy(dA, A.data(), 4 * A.size(), cudaMemcpyHostToDevice));
  CAPT_CUDA(cudaMemcpy(dB, B.data(), 4 * B.size(), cudaMemcpyHostToDevice));
  const int smem = (kM + kN) * 64 + 64;
  CAPT_CUDA(cudaFuncSetAttribute(k_tc_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_tc_selftest<<<1, 128, smem>>>(dA, dB, dD);
  CAPT_CUDA(cudaGetLastError());
  CAPT_CUDA(cudaDeviceSynchronize());
  CAPT_CUDA(cudaMemcpy(D.data(), dD, 4 * D.size(), cudaMemcpyDeviceToHost));
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  double worst = 0.0;
  for (int i = 0; i < kM; ++i)
    for (int j = 0; j < kN; ++j) {
      double ref = 0.0, mag = 0.0;
      for (int k = 0; k < tc::kTcK; ++k) {
        ref += double(A[i * tc::kTcK + k]) * double(B[j * tc::kTcK + k]);
        mag += std::fabs(double(A[i * tc::kTcK + k]) * double(B[j * tc::kTcK + k]));
      }
      const double e = std::fabs(double(D[i * kN + j]) - ref) / (mag > 0 ? mag : 1.0);
      if (!(e <= worst)) worst = e;  // NaN-propagating
    }
  *max_rel_err = worst;
  return CAPT_OK;
}
