// probe.cu -- traffic-pattern speed of light for the config-4 kernel.
//
// ks_probe_widen streams n int32 in and n int64 out (sign-extended): exactly
// the compulsory HBM traffic of the lanes kernel (4 B duration read + 8 B
// start write per (task, scenario) update) with no recurrence, so bench.py can
// report how close the simulator gets to what this read/write mix allows on
// the device, next to the copy peak in MEASURED_PEAKS.json.
#include "ddsim_internal.h"

namespace ddsim {

// thread t of a warp reads int2 t (8 B) and writes longlong2 t (16 B): the
// 256 B in / 512 B out per warp-step shape of the lanes kernel's V = 2 tiles;
// four independent steps in flight per thread.
__global__ void __launch_bounds__(256) probe_widen_kernel(const int2* __restrict__ src,
                                                          longlong2* __restrict__ dst,
                                                          long long n2) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    int2 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldcs(src + i + k * stride);
#pragma unroll
    for (int k = 0; k < 4; ++k) __stcs(dst + i + k * stride, make_longlong2(v[k].x, v[k].y));
  }
  for (; i < n2; i += stride) {
    const int2 v = __ldcs(src + i);
    __stcs(dst + i, make_longlong2(v.x, v.y));
  }
}

// variants (DDSIM_PROBE_VARIANT, config-4 size, 1x B200): default 32 CTAs per SM
// 6.21 TB/s; 8 = 8 CTAs per SM 5.97; 4 = 4 per SM 5.79; 5 = 16 per SM 6.08;
// 6 = 16 per SM, eight steps in flight 6.17; 1 = 8 per SM, eight in flight 6.08;
// 2 = write-back (non-streaming) stores 5.93; 3 = TMA bulk stores of 8 KB shared
// tiles 5.43. The default is the ceiling bench.py reports (pattern_copy_gbs).
template <int K, bool CS>
__global__ void __launch_bounds__(256) probe_widen_var(const int2* __restrict__ src,
                                                       longlong2* __restrict__ dst, long long n2) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + (K - 1) * stride < n2; i += K * stride) {
    int2 v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = __ldcs(src + i + k * stride);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (CS)
        __stcs(dst + i + k * stride, make_longlong2(v[k].x, v[k].y));
      else
        dst[i + k * stride] = make_longlong2(v[k].x, v[k].y);
    }
  }
  for (; i < n2; i += stride) {
    const int2 v = __ldcs(src + i);
    __stcs(dst + i, make_longlong2(v.x, v.y));
  }
}

// 256 threads widen 512 int2 -> 512 longlong2 (8 KB) into shared memory, one
// thread bulk-stores the tile; two tiles alternate (bulk_group wait before reuse)
__global__ void __launch_bounds__(256) probe_widen_tma(const int2* __restrict__ src,
                                                       longlong2* __restrict__ dst, long long n2) {
  __shared__ __align__(128) longlong2 tile[2][512];
  const long long tiles = n2 / 512;
  int buf = 0;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const long long base = t * 512;
    const int2 a = __ldcs(src + base + threadIdx.x);
    const int2 b = __ldcs(src + base + 256 + threadIdx.x);
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    tile[buf][threadIdx.x] = make_longlong2(a.x, a.y);
    tile[buf][256 + threadIdx.x] = make_longlong2(b.x, b.y);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(&tile[buf][0]);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + base), "r"(sa),
                   "r"(512 * 16)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    buf ^= 1;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  for (long long i = tiles * 512 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2;
       i += (long long)gridDim.x * blockDim.x) {
    const int2 v = src[i];
    dst[i] = make_longlong2(v.x, v.y);
  }
}

__global__ void probe_widen_tail(const int* src, long long* dst, long long from, long long n) {
  const long long i = from + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}

}  // namespace ddsim

extern "C" int ks_probe_widen(const int32_t* src, int64_t* dst, int64_t n, void* stream) {
  using namespace ddsim;
  if (n < 0 || (n > 0 && (!src || !dst))) return KS_ERR_INVALID;
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % 16 != 0)
    return KS_ERR_INVALID;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long n2 = n / 2;
  if (n2 > 0) {
    const int2* s2 = reinterpret_cast<const int2*>(src);
    longlong2* d2 = reinterpret_cast<longlong2*>(dst);
    const char* var = getenv("DDSIM_PROBE_VARIANT");
    const int v = var ? atoi(var) : 0;
    if (v == 1)
      probe_widen_var<8, true><<<nsm * 8, 256, 0, st>>>(s2, d2, n2);
    else if (v == 2)
      probe_widen_var<4, false><<<nsm * 8, 256, 0, st>>>(s2, d2, n2);
    else if (v == 3)
      probe_widen_tma<<<nsm * 8, 256, 0, st>>>(s2, d2, n2);
    else if (v == 4)
      probe_widen_kernel<<<nsm * 4, 256, 0, st>>>(s2, d2, n2);
    else if (v == 5)
      probe_widen_kernel<<<nsm * 16, 256, 0, st>>>(s2, d2, n2);
    else if (v == 6)
      probe_widen_var<8, true><<<nsm * 16, 256, 0, st>>>(s2, d2, n2);
    else if (v == 7)
      probe_widen_kernel<<<nsm * 32, 256, 0, st>>>(s2, d2, n2);
    else if (v == 8)
      probe_widen_kernel<<<nsm * 8, 256, 0, st>>>(s2, d2, n2);
    else  // default: the fastest measured shape (6.21 TB/s vs 5.97 at 8 CTAs per SM)
      probe_widen_kernel<<<nsm * 32, 256, 0, st>>>(s2, d2, n2);
    note_launch();
  }
  if (n % 2) {
    probe_widen_tail<<<1, 1, 0, st>>>(src, reinterpret_cast<long long*>(dst), n2 * 2, n);
    note_launch();
  }
  return cudaGetLastError() == cudaSuccess ? KS_OK : KS_ERR_CUDA;
}
