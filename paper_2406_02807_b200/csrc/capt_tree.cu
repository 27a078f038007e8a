// Tree handles: error plumbing, upload from the reference layout
// (Capt.__init__ tree.py:74-97), export back to it, slab replication.
#include <cub/cub.cuh>
#include <cuda_fp16.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <vector>

#include "capt_internal.cuh"

namespace capt {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void note_launches(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

void ensure_pool(int device) {
  static std::atomic<uint64_t> done{0};
  if (device < 0 || device >= 64 || (done.load() >> device) & 1ull) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.fetch_or(1ull << device);
}

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  char buf[512];
  snprintf(buf, sizeof(buf), "CUDA error %d (%s) in %s", int(e), cudaGetErrorString(e), what);
  g_last_error = buf;
  cudaGetLastError();  // clear sticky-free errors
  return e == cudaErrorMemoryAllocation ? CAPT_ENOMEM : CAPT_ECUDA;
}

int alloc_slab(capt_tree** out, int device, SlabHeader h) {
  capt_tree* t = new capt_tree();
  t->h = h;
  t->device = device;
  t->slab = nullptr;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&t->slab), size_t(h.bytes));
  if (e != cudaSuccess) {
    delete t;
    return cuda_fail(e, "cudaMalloc(tree slab)");
  }
  *out = t;
  return CAPT_OK;
}

// --------------------------------------------------------------------------
// upload: reference layout -> padded device layout
// --------------------------------------------------------------------------

// One warp per leaf: copy the SoA coordinates of set j from the reference's
// compact layout (values[off*k + d*m + i]) to the padded per-set layout,
// +inf padding rows, zeros for unused dims.
__global__ void k_pack_sets(int k, int64_t n, const int64_t* __restrict__ offs,
                            const float* __restrict__ vals, const uint2* __restrict__ set,
                            float4* __restrict__ data) {
  int lane = threadIdx.x & 31;
  int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = warp; j < n; j += nwarps) {
    int64_t a = offs[j];
    int64_t m = offs[j + 1] - a;
    int64_t m4 = (m + 3) & ~int64_t(3);
    float* dst = reinterpret_cast<float*>(data + set[j].x);
    for (int d = 0; d < kMaxK; ++d) {
      for (int64_t i = lane; i < m4; i += 32) {
        float v;
        if (d >= k) v = 0.f;
        else if (i < m) v = vals[a * k + d * m + i];
        else v = __int_as_float(0x7f800000);
        dst[d * m4 + i] = v;
      }
    }
  }
}

__global__ void k_pack_boxes(int k, int64_t n, const float* __restrict__ lo,
                             const float* __restrict__ hi, float4* __restrict__ box) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    float l[3] = {0.f, 0.f, 0.f}, h[3] = {0.f, 0.f, 0.f};
    for (int d = 0; d < k; ++d) {
      l[d] = lo[j * k + d];
      h[d] = hi[j * k + d];
    }
    box[2 * j] = make_float4(l[0], l[1], l[2], 0.f);
    box[2 * j + 1] = make_float4(h[0], h[1], h[2], 0.f);
  }
}

// Inverse of k_pack_sets (export).
__global__ void k_unpack_sets(int k, int64_t n, const int64_t* __restrict__ offs,
                              const uint2* __restrict__ set, const float4* __restrict__ data,
                              float* __restrict__ vals) {
  int lane = threadIdx.x & 31;
  int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = warp; j < n; j += nwarps) {
    int64_t a = offs[j];
    int64_t m = offs[j + 1] - a;
    int64_t m4 = (m + 3) & ~int64_t(3);
    const float* src = reinterpret_cast<const float*>(data + set[j].x);
    for (int d = 0; d < k; ++d)
      for (int64_t i = lane; i < m; i += 32) vals[a * k + d * m + i] = src[d * m4 + i];
  }
}

__global__ void k_unpack_boxes(int k, int64_t n, const float4* __restrict__ box,
                               float* __restrict__ lo, float* __restrict__ hi) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    float4 l = box[2 * j], h = box[2 * j + 1];
    float lv[3] = {l.x, l.y, l.z}, hv[3] = {h.x, h.y, h.z};
    for (int d = 0; d < k; ++d) {
      lo[j * k + d] = lv[d];
      hi[j * k + d] = hv[d];
    }
  }
}

// One warp per leaf: centre of the finite points' box and the largest fp32
// |fl(p - o)|^2, evaluated exactly as the binned scan stages the set.
__global__ void k_origins(DevTree t) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = warp; j < t.n; j += nwarps) {
    const uint2 st = t.set[j];
    const uint32_t m4 = (st.y + 3u) & ~3u;
    const float* base = reinterpret_cast<const float*>(t.data + st.x);
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (uint32_t i = lane; i < st.y; i += 32) {
      const float p[3] = {base[i], base[m4 + i], base[2 * m4 + i]};
      if (!isfinite(p[0]) || !isfinite(p[1]) || !isfinite(p[2])) continue;
      for (int d = 0; d < 3; ++d) {
        lo[d] = fminf(lo[d], p[d]);
        hi[d] = fmaxf(hi[d], p[d]);
      }
    }
    float o[3];
    for (int d = 0; d < 3; ++d) {
      for (int s = 16; s > 0; s >>= 1) {
        lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], s));
        hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], s));
      }
      o[d] = lo[d] <= hi[d] ? 0.5f * lo[d] + 0.5f * hi[d] : 0.f;
    }
    float bb = 0.f;
    for (uint32_t i = lane; i < st.y; i += 32) {
      const float p[3] = {base[i], base[m4 + i], base[2 * m4 + i]};
      if (!isfinite(p[0]) || !isfinite(p[1]) || !isfinite(p[2])) continue;
      const float bx = p[0] - o[0], by = p[1] - o[1], bz = p[2] - o[2];
      bb = fmaxf(bb, fmaf(bz, bz, fmaf(by, by, bx * bx)));
    }
    for (int s = 16; s > 0; s >>= 1) bb = fmaxf(bb, __shfl_xor_sync(0xffffffffu, bb, s));
    if (lane == 0) {
      const_cast<float4*>(t.org)[j] = make_float4(o[0], o[1], o[2], bb);
      const float4 rp = make_float4(base[0], base[m4], base[2 * m4], 0.f);
      const_cast<float4*>(t.rep)[j] = rp;
      const float4 lo = t.box[2 * j], hi = t.box[2 * j + 1];
      const __half2 h0 = __halves2half2(__float2half_rd(lo.x), __float2half_rd(lo.y));
      const __half2 h1 = __halves2half2(__float2half_rd(lo.z), __float2half_ru(hi.x));
      const __half2 h2 = __halves2half2(__float2half_ru(hi.y), __float2half_ru(hi.z));
      float4* pr = reinterpret_cast<float4*>(const_cast<float*>(t.probe) + 8 * j);
      pr[0] = make_float4(rp.x, rp.y, rp.z, __uint_as_float(*reinterpret_cast<const unsigned*>(&h0)));
      pr[1] = make_float4(__uint_as_float(*reinterpret_cast<const unsigned*>(&h1)),
                          __uint_as_float(*reinterpret_cast<const unsigned*>(&h2)), 0.f, 0.f);
    }
  }
}

__global__ void k_order_keys(DevTree t, uint32_t* keys, int* ids) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < t.n;
       j += int64_t(gridDim.x) * blockDim.x) {
    keys[j] = t.set[j].y;
    ids[j] = int(j);
  }
}

int compute_origins(const DevTree& t, cudaStream_t s, bool with_origins) {
  if (with_origins) {
    k_origins<<<grid_for(t.n * 32, 256), 256, 0, s>>>(t);
    CAPT_CUDA(cudaGetLastError());
  }
  // leaves by descending set size (stable: equal sizes keep leaf order)
  uint32_t *keys = nullptr, *keys_out = nullptr;
  int* ids = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  const int n = int(t.n);
  cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, keys, keys_out, ids,
                                            const_cast<int*>(t.order), n, 0, 32, s);
  CAPT_CUDA(cudaMallocAsync(&keys, 4 * size_t(n), s));
  CAPT_CUDA(cudaMallocAsync(&keys_out, 4 * size_t(n), s));
  CAPT_CUDA(cudaMallocAsync(&ids, 4 * size_t(n), s));
  CAPT_CUDA(cudaMallocAsync(&tmp, tb ? tb : 1, s));
  k_order_keys<<<grid_for(t.n, 256), 256, 0, s>>>(t, keys, ids);
  CAPT_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, tb, keys, keys_out, ids,
                                                      const_cast<int*>(t.order), n, 0, 32, s));
  cudaFreeAsync(keys, s);
  cudaFreeAsync(keys_out, s);
  cudaFreeAsync(ids, s);
  cudaFreeAsync(tmp, s);
  CAPT_CUDA(cudaGetLastError());
  note_launches(3);
  return CAPT_OK;
}

}  // namespace capt

using namespace capt;

extern "C" {

const char* capt_last_error(void) { return g_last_error.c_str(); }

int capt_version(void) { return 1; }

int64_t capt_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

int capt_tree_create(int device, int k, int64_t n, int64_t n_points, double r_min,
                     double r_max, const float* tests, const float* aff_lo,
                     const float* aff_hi, const int64_t* offsets, const float* aff_values,
                     capt_tree** out) {
  if (!out) return fail(CAPT_EINVAL, "out is NULL");
  *out = nullptr;
  if (k < 1 || k > kMaxK) return fail(CAPT_EINVAL, "k must be 1..3 on the device path");
  if (n < 1 || (n & (n - 1))) return fail(CAPT_EINVAL, "leaf count is not a power of two");
  if (!aff_lo || !aff_hi || !offsets || (n > 1 && !tests))
    return fail(CAPT_EINVAL, "missing tree array");
  if (offsets[0] != 0) return fail(CAPT_EINVAL, "offsets[0] must be 0");
  CAPT_CUDA(cudaSetDevice(device));
  SlabHeader h;
  memset(&h, 0, sizeof(h));
  h.magic = kSlabMagic;
  h.version = kSlabVersion;
  h.k = k;
  h.n = n;
  h.depth = depth_of(n);
  h.n_points = n_points;
  h.r_min = r_min;
  h.r_max = r_max;
  std::vector<uint2> set(static_cast<size_t>(n));
  int64_t f4 = 0, maxm = 0;
  for (int64_t j = 0; j < n; ++j) {
    int64_t m = offsets[j + 1] - offsets[j];
    if (m < 1) return fail(CAPT_EINVAL, "every affordance set holds at least its representative");
    if (m > 0xffffffffll) return fail(CAPT_EINVAL, "affordance set too large");
    int64_t m4 = (m + 3) & ~int64_t(3);
    set[j] = make_uint2(unsigned(f4), unsigned(m));
    f4 += 3 * m4 / 4;
    if (f4 > 0xffffffffll) return fail(CAPT_EINVAL, "tree too large for 32-bit float4 offsets");
    if (m > maxm) maxm = m;
  }
  h.total = offsets[n];
  h.max_aff = maxm;
  layout_slab(h, f4);
  int rc = alloc_slab(out, device, h);
  if (rc) return rc;
  capt_tree* t = *out;
  cudaStream_t s = 0;
  float* d_vals = nullptr;
  float* d_lo = nullptr;
  float* d_hi = nullptr;
  cudaError_t e = cudaSuccess;
#define UPCHK(x)                                  \
  do {                                            \
    e = (x);                                      \
    if (e != cudaSuccess) {                       \
      cudaFree(d_vals); cudaFree(d_lo); cudaFree(d_hi); \
      capt_tree_destroy(t); *out = nullptr;       \
      return cuda_fail(e, #x);                    \
    }                                             \
  } while (0)
  UPCHK(cudaMemcpy(t->slab, &h, sizeof(h), cudaMemcpyHostToDevice));
  if (n > 1)
    UPCHK(cudaMemcpy(t->slab + h.off_T, tests, sizeof(float) * (n - 1), cudaMemcpyHostToDevice));
  UPCHK(cudaMemcpy(t->slab + h.off_set, set.data(), sizeof(uint2) * n, cudaMemcpyHostToDevice));
  UPCHK(cudaMemcpy(t->slab + h.off_offs, offsets, sizeof(int64_t) * (n + 1),
                   cudaMemcpyHostToDevice));
  UPCHK(cudaMalloc(&d_vals, sizeof(float) * (h.total * k + 1)));
  UPCHK(cudaMalloc(&d_lo, sizeof(float) * n * k));
  UPCHK(cudaMalloc(&d_hi, sizeof(float) * n * k));
  UPCHK(cudaMemcpy(d_vals, aff_values, sizeof(float) * h.total * k, cudaMemcpyHostToDevice));
  UPCHK(cudaMemcpy(d_lo, aff_lo, sizeof(float) * n * k, cudaMemcpyHostToDevice));
  UPCHK(cudaMemcpy(d_hi, aff_hi, sizeof(float) * n * k, cudaMemcpyHostToDevice));
  DevTree v = view(t);
  k_pack_sets<<<grid_for(n * 32, 256), 256, 0, s>>>(k, n, v.offs, d_vals, v.set,
                                                    const_cast<float4*>(v.data));
  k_pack_boxes<<<grid_for(n, 256), 256, 0, s>>>(k, n, d_lo, d_hi, const_cast<float4*>(v.box));
  UPCHK(cudaGetLastError());
  if (compute_origins(v, s)) {
    cudaFree(d_vals); cudaFree(d_lo); cudaFree(d_hi);
    capt_tree_destroy(t);
    *out = nullptr;
    return CAPT_ECUDA;
  }
  UPCHK(cudaDeviceSynchronize());
  cudaFree(d_vals);
  cudaFree(d_lo);
  cudaFree(d_hi);
#undef UPCHK
  rc = build_field(t, s);
  if (rc) {
    capt_tree_destroy(t);
    *out = nullptr;
  }
  return rc;
}

int capt_tree_info_get(const capt_tree* t, capt_tree_info* info) {
  if (!t || !info) return fail(CAPT_EINVAL, "NULL argument");
  memset(info, 0, sizeof(*info));
  info->k = t->h.k;
  info->depth = t->h.depth;
  info->n_leaves = t->h.n;
  info->n_points = t->h.n_points;
  info->total_stored = t->h.total;
  info->max_affordance = t->h.max_aff;
  info->r_min = t->h.r_min;
  info->r_max = t->h.r_max;
  info->device_bytes = t->h.bytes;
  info->device = t->device;
  info->n_ties = t->h.n_ties;
  return CAPT_OK;
}

int capt_tree_export(const capt_tree* t, float* tests, float* aff_lo, float* aff_hi,
                     int64_t* offsets, float* aff_values) {
  if (!t) return fail(CAPT_EINVAL, "NULL tree");
  CAPT_CUDA(cudaSetDevice(t->device));
  const SlabHeader& h = t->h;
  DevTree v = view(t);
  int k = h.k;
  int64_t n = h.n;
  if (tests && n > 1)
    CAPT_CUDA(cudaMemcpy(tests, v.T, sizeof(float) * (n - 1), cudaMemcpyDeviceToHost));
  if (offsets) CAPT_CUDA(cudaMemcpy(offsets, v.offs, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
  if (aff_lo || aff_hi) {
    float *d_lo = nullptr, *d_hi = nullptr;
    CAPT_CUDA(cudaMalloc(&d_lo, sizeof(float) * n * k));
    CAPT_CUDA(cudaMalloc(&d_hi, sizeof(float) * n * k));
    k_unpack_boxes<<<grid_for(n, 256), 256>>>(k, n, v.box, d_lo, d_hi);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess && aff_lo) e = cudaMemcpy(aff_lo, d_lo, sizeof(float) * n * k, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && aff_hi) e = cudaMemcpy(aff_hi, d_hi, sizeof(float) * n * k, cudaMemcpyDeviceToHost);
    cudaFree(d_lo);
    cudaFree(d_hi);
    if (e != cudaSuccess) return cuda_fail(e, "export boxes");
  }
  if (aff_values && h.total > 0) {
    float* d_vals = nullptr;
    CAPT_CUDA(cudaMalloc(&d_vals, sizeof(float) * h.total * k));
    k_unpack_sets<<<grid_for(n * 32, 256), 256>>>(k, n, v.offs, v.set, v.data, d_vals);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess)
      e = cudaMemcpy(aff_values, d_vals, sizeof(float) * h.total * k, cudaMemcpyDeviceToHost);
    cudaFree(d_vals);
    if (e != cudaSuccess) return cuda_fail(e, "export values");
  }
  return CAPT_OK;
}

void capt_tree_destroy(capt_tree* t) {
  if (!t) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(t->device);
  if (t->owns_slab) cudaFree(t->slab);
  else cudaDeviceSynchronize();  // (cudaFree's implicit sync: no query still reads the borrowed slab)
  if (t->field_mem) cudaFree(t->field_mem);
  cudaSetDevice(cur);
  delete t;
}

int capt_tree_slab(const capt_tree* t, const void** dev_ptr, int64_t* bytes) {
  if (!t || !dev_ptr || !bytes) return fail(CAPT_EINVAL, "NULL argument");
  *dev_ptr = t->slab;
  *bytes = t->h.bytes;
  return CAPT_OK;
}

int capt_tree_from_slab(int device, const void* dev_slab, int64_t bytes, uint32_t flags,
                        void* stream, capt_tree** out) {
  if (!out || !dev_slab) return fail(CAPT_EINVAL, "NULL argument");
  *out = nullptr;
  CAPT_CUDA(cudaSetDevice(device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SlabHeader h;
  CAPT_CUDA(cudaMemcpyAsync(&h, dev_slab, sizeof(h), cudaMemcpyDeviceToHost, s));
  CAPT_CUDA(cudaStreamSynchronize(s));
  if (h.magic != kSlabMagic || h.version != kSlabVersion || h.bytes != bytes)
    return fail(CAPT_EINVAL, "not a capt_b200 tree slab");
  int rc = CAPT_OK;
  cudaError_t e = cudaSuccess;
  if (flags & CAPT_SLAB_BORROW) {
    // adopt the caller's buffer (a replica received by broadcast): no copy
    *out = new capt_tree();
    (*out)->h = h;
    (*out)->device = device;
    (*out)->slab = static_cast<char*>(const_cast<void*>(dev_slab));
    (*out)->owns_slab = false;
  } else {
    rc = alloc_slab(out, device, h);
    if (rc) return rc;
    e = cudaMemcpyAsync((*out)->slab, dev_slab, size_t(bytes), cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  if (e != cudaSuccess) {
    capt_tree_destroy(*out);
    *out = nullptr;
    return cuda_fail(e, "copy slab");
  }
  rc = build_field(*out, s);
  if (rc) {
    capt_tree_destroy(*out);
    *out = nullptr;
  }
  return rc;
}

}  // extern "C"
