// Measurement helper: FP32 FFMA throughput of the device (roofline
// denominator for the distance scan).
#include "capt_internal.cuh"

namespace capt {

// 8 independent FMA chains per thread, 1024 iterations each.
__global__ void k_ffma_peak(float* out, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5f) out[0] = s;  // keep the chains alive
}

}  // namespace capt

extern "C" int capt_measure_fp32_peak(int device, double* tflops) {
  using namespace capt;
  if (!tflops) return fail(CAPT_EINVAL, "NULL tflops");
  CAPT_CUDA(cudaSetDevice(device));
  int sms = 0;
  CAPT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  float* d = nullptr;
  CAPT_CUDA(cudaMalloc(&d, 4));
  const int block = 256, per_sm = 8, iters = 4096;
  const int grid = sms * per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_ffma_peak<<<grid, block>>>(d, iters, 0.999f, 1e-3f);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) k_ffma_peak<<<grid, block>>>(d, iters, 0.999f, 1e-3f);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "ffma peak");
  const double flops = 2.0 * 8.0 * iters * double(grid) * block * reps;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return CAPT_OK;
}
