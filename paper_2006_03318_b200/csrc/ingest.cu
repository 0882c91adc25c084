// Trace ingest on the device: build_graph + link_syncs + compute_gaps
// (pkg/src/kernsim/graph.py:189-312), check_lane_overlaps (trace.py:255-265)
// and map_tasks_to_layers (layers.py:30-81) over columnar event records.
//
// Shape: segmented sorts (CUB radix sort, stable, LSD over the key fields)
// plus hand-written gather / join / binary-search / emit kernels.  All rules
// are per-event independent once the sorted views exist, so every kernel is
// one thread per event (or per candidate edge).  Quirks reproduced exactly:
//   * lane order by (start, id) for edges, (start, end, id) for the overlap
//     check;
//   * correlation join: the LAST CPU-kind event of a correlation launches
//     (dict overwrite, graph.py:192-194);
//   * memcpy_dtoh lookup: the FIRST GPU-kind event of the correlation in
//     document order (graph.py:289-292), then the newest launched GPU task on
//     its stream before the call, skipping the memcpy itself (graph.py:295);
//   * device-wide syncs wait on every GPU lane present in the trace.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <string>
#include <vector>

#include "ddsim_internal.h"

namespace ddsim {
namespace {

struct IngestError {
  int code;
  std::string msg;
};
#define ICUDA(x)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) throw IngestError{KS_ERR_CUDA, std::string(#x) + ": " + \
                                                              cudaGetErrorString(e_)}; \
  } while (0)

constexpr int TPB = 256;
inline int blocks_for(long long n) {
  long long b = (n + TPB - 1) / TPB;
  return (int)std::max(1LL, std::min(b, 148LL * 64));
}

__device__ __forceinline__ bool is_cpu_kind(int k) { return k == 0 || k == 1 || k == 4 || k == 6; }
__device__ __forceinline__ bool is_gpu_kind(int k) { return k == 2 || k == 3; }

// Pool of stream-ordered device allocations freed together.
struct Pool {
  cudaStream_t st;
  std::vector<void*> ptrs;
  template <class T>
  T* get(size_t n) {
    T* p = nullptr;
    ICUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st));
    ptrs.push_back(p);
    return p;
  }
  template <class T>
  T* up(const T* h, size_t n) {
    T* p = get<T>(n);
    if (n && h) ICUDA(cudaMemcpyAsync(p, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
    return p;
  }
  ~Pool() {
    for (void* p : ptrs)
      if (p) cudaFreeAsync(p, st);
  }
};

// ---------------------------------------------------------------- kernels
__global__ void iota_k(int* a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = (int)i;
}
template <class T>
__global__ void gather_k(const T* src, const int* idx, T* dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}
__global__ void end_k(const long long* s, const long long* d, long long* e, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    e[i] = s[i] + d[i];
}

// lane edges + CPU gaps over the (lane, start, id) order
__global__ void lane_edges_k(const int* perm, const int* lane, const long long* start,
                             const long long* dur, const unsigned char* lane_class, long long n,
                             int* esrc, int* edst, unsigned char* ekind, unsigned char* eflag,
                             long long* gap) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int a = perm[i];
    const int la = lane[a];
    bool has_next = false;
    int b = -1;
    if (i + 1 < n) {
      b = perm[i + 1];
      has_next = lane[b] == la;
    }
    const int cls = lane_class[la];
    eflag[i] = has_next ? 1 : 0;
    if (has_next) {
      esrc[i] = a;
      edst[i] = b;
      ekind[i] = cls == 0 ? KS_EDGE_LANE_SEQ_CPU : (cls == 1 ? KS_EDGE_LANE_SEQ_GPU : KS_EDGE_COMM_ORDER);
    }
    long long g = 0;
    if (cls == 0 && has_next) {
      const long long d = start[b] - (start[a] + dur[a]);
      g = d > 0 ? d : 0;
    }
    gap[a] = g;
  }
}

__global__ void lane_bounds_k(const int* perm, const int* lane, long long n, int* lptr_first,
                              int* lptr_last) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int l = lane[perm[i]];
    if (i == 0 || lane[perm[i - 1]] != l) lptr_first[l] = (int)i;
    if (i + 1 == n || lane[perm[i + 1]] != l) lptr_last[l] = (int)i + 1;
  }
}

// correlation keys: CPU-kind (launch side) and GPU-kind (memcpy side)
__global__ void corr_keys_k(const unsigned char* kind, const long long* corr, long long n,
                            long long* cpu_key, long long* gpu_key) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = kind[i];
    const long long c = corr[i];
    cpu_key[i] = (is_cpu_kind(k) && c >= 0) ? c : LLONG_MAX;
    gpu_key[i] = (is_gpu_kind(k) && c >= 0) ? c : LLONG_MAX;
  }
}

__device__ __forceinline__ long long lower_bound_ll(const long long* a, long long lo, long long hi,
                                                    long long x) {
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (a[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
__device__ __forceinline__ long long upper_bound_ll(const long long* a, long long lo, long long hi,
                                                    long long x) {
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (a[mid] <= x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// rule 3: launcher = last CPU-kind event of the correlation
__global__ void launch_join_k(const unsigned char* kind, const long long* corr, long long n,
                              const long long* cpu_sorted_key, const int* cpu_sorted_idx,
                              long long n_cpu, int* launcher, int* esrc, int* edst,
                              unsigned char* ekind, unsigned char* eflag,
                              unsigned long long* orphan_min) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int L = -1;
    if (is_gpu_kind(kind[i]) && corr[i] >= 0) {
      const long long p = upper_bound_ll(cpu_sorted_key, 0, n_cpu, corr[i]) - 1;
      if (p >= 0 && cpu_sorted_key[p] == corr[i]) L = cpu_sorted_idx[p];
      if (L < 0) atomicMin(orphan_min, (unsigned long long)i);
    }
    launcher[i] = L;
    eflag[i] = L >= 0 ? 1 : 0;
    if (L >= 0) {
      esrc[i] = L;
      edst[i] = (int)i;
      ekind[i] = KS_EDGE_LAUNCH_CORRELATION;
    }
  }
}

// stream-task sort keys: (lane, launch start, id); non-entries -> lane = L
__global__ void stream_keys_k(const unsigned char* kind, const int* lane, const long long* start,
                              const int* launcher, long long n, int n_lanes, int* skey_lane,
                              long long* skey_ls) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const bool entry = is_gpu_kind(kind[i]) && launcher[i] >= 0;
    skey_lane[i] = entry ? lane[i] : n_lanes;
    skey_ls[i] = entry ? start[launcher[i]] : LLONG_MAX;
  }
}

// rule 4 (syncs + blocking dtoh): one candidate per (event, target lane slot)
__global__ void sync_src_flag_k(const unsigned char* kind, const unsigned char* is_dtoh,
                                const long long* corr, long long n, unsigned char* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = kind[i];
    flag[i] = (k == KS_KIND_SYNC) || (is_cpu_kind(k) && is_dtoh[i] && corr[i] >= 0);
  }
}

__global__ void sync_link_k(const unsigned char* kind, const long long* start, const long long* corr,
                            const int* sync_target, const unsigned char* is_dtoh, const int* lane,
                            const int* srcs, long long n_src, const int* gpu_lanes, int n_gpu,
                            const int* seg_first, const int* seg_last, const long long* st_ls,
                            const int* st_idx, const long long* gpu_sorted_key,
                            const int* gpu_sorted_idx, long long n_gpu_keyed, int* esrc, int* edst,
                            unsigned char* ekind, unsigned char* eflag) {
  const long long total = n_src * (long long)(n_gpu + 1);
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < total;
       c += (long long)gridDim.x * blockDim.x) {
    const long long e = srcs[c / (n_gpu + 1)];
    const int slot = (int)(c % (n_gpu + 1));
    eflag[c] = 0;
    const int k = kind[e];
    int tl = -1;
    long long exclude = -1;
    if (k == KS_KIND_SYNC) {
      if (slot == n_gpu) continue;
      if (sync_target[e] >= 0) {
        if (slot != 0) continue;
        tl = sync_target[e];
      } else {
        tl = gpu_lanes[slot];
      }
    } else if (is_cpu_kind(k) && is_dtoh[e] && corr[e] >= 0) {
      if (slot != n_gpu) continue;
      const long long p = lower_bound_ll(gpu_sorted_key, 0, n_gpu_keyed, corr[e]);
      if (p >= n_gpu_keyed || gpu_sorted_key[p] != corr[e]) continue;
      const int m = gpu_sorted_idx[p];  // first GPU-kind event with the correlation
      tl = lane[m];
      exclude = m;
    } else {
      continue;
    }
    const int f = seg_first[tl], l = seg_last[tl];
    if (f >= l) continue;
    long long p = lower_bound_ll(st_ls, f, l, start[e]) - 1;  // newest launch before the call
    if (p >= f && st_idx[p] == exclude) --p;
    if (p < f) continue;
    esrc[c] = st_idx[p];
    edst[c] = (int)e;
    ekind[c] = KS_EDGE_SYNC_BLOCK;
    eflag[c] = 1;
  }
}

__global__ void overlap_k(const int* perm, const int* lane, const long long* start,
                          const long long* endv, long long n, const long long* first_seen,
                          unsigned long long* best) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i + 1 < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int a = perm[i], b = perm[i + 1];
    if (lane[a] != lane[b]) continue;
    if (endv[a] > start[b]) {
      const unsigned long long key =
          (unsigned long long)first_seen[lane[a]] * (unsigned long long)(n + 1) + (unsigned long long)i;
      atomicMin(best, key);
    }
  }
}

__global__ void first_seen_k(const int* lane, long long n, long long* first_seen) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    atomicMin((unsigned long long*)&first_seen[lane[i]], (unsigned long long)i);
}

// stable LSD sort of an index permutation by successive keys
template <class K>
void sort_by_key(Pool& P, const K* key_of_event, int* perm, long long n) {
  K* k_in = P.get<K>(n);
  K* k_out = P.get<K>(n);
  int* v_out = P.get<int>(n);
  gather_k<K><<<blocks_for(n), TPB, 0, P.st>>>(key_of_event, perm, k_in, n);
  note_launch();
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, k_in, k_out, perm, v_out, (int)n, 0, sizeof(K) * 8,
                                  P.st);
  void* t = P.get<unsigned char>(tmp);
  ICUDA(cub::DeviceRadixSort::SortPairs(t, tmp, k_in, k_out, perm, v_out, (int)n, 0,
                                        sizeof(K) * 8, P.st));
  note_launch(4);
  ICUDA(cudaMemcpyAsync(perm, v_out, sizeof(int) * n, cudaMemcpyDeviceToDevice, P.st));
}

// sort (key, idx) pairs, both outputs kept
void sort_pairs_ll(Pool& P, const long long* key, long long n, long long* key_sorted,
                   int* idx_sorted) {
  int* idx = P.get<int>(n);
  iota_k<<<blocks_for(n), TPB, 0, P.st>>>(idx, n);
  note_launch();
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, key_sorted, idx, idx_sorted, (int)n, 0, 64,
                                  P.st);
  void* t = P.get<unsigned char>(tmp);
  ICUDA(cub::DeviceRadixSort::SortPairs(t, tmp, key, key_sorted, idx, idx_sorted, (int)n, 0, 64,
                                        P.st));
  note_launch(4);
}

long long compact_edges(Pool& P, const int* s, const int* d, const unsigned char* k,
                        const unsigned char* f, long long n, int* os, int* od, unsigned char* ok) {
  int* cnt = P.get<int>(1);
  size_t tmp = 0;
  cub::DeviceSelect::Flagged(nullptr, tmp, s, f, os, cnt, (int)n, P.st);
  void* t = P.get<unsigned char>(tmp);
  ICUDA(cub::DeviceSelect::Flagged(t, tmp, s, f, os, cnt, (int)n, P.st));
  ICUDA(cub::DeviceSelect::Flagged(t, tmp, d, f, od, cnt, (int)n, P.st));
  ICUDA(cub::DeviceSelect::Flagged(t, tmp, k, f, ok, cnt, (int)n, P.st));
  note_launch(3);
  int h = 0;
  ICUDA(cudaMemcpyAsync(&h, cnt, sizeof(int), cudaMemcpyDeviceToHost, P.st));
  ICUDA(cudaStreamSynchronize(P.st));
  return h;
}

// ---------------------------------------------------------------- layers
__global__ void layer_map_k(const unsigned char* kind, const int* lane, const long long* start,
                            const long long* dur, long long n, const int* mseg_first,
                            const int* mseg_last, int n_lanes, const long long* m_start,
                            const long long* m_end, const int* m_tag, const int* m_orig,
                            const long long* mx, int levels, long long M, int* tag_out,
                            unsigned long long* ambiguous) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    tag_out[i] = -1;
    const int l = lane[i];
    if (l < 0 || l >= n_lanes || !is_cpu_kind(kind[i])) continue;
    const long long s = start[i], e = start[i] + dur[i];
    const long long f = mseg_first[l], last = mseg_last[l];
    if (f >= last) continue;
    // last marker (in start order) with start <= s
    long long pos = upper_bound_ll(m_start, f, last, s) - 1;
    long long b_len = LLONG_MAX, s_len = LLONG_MAX;
    int b_tag = INT_MAX, s_tag = INT_MAX, b_orig = INT_MAX, s_orig = INT_MAX;
    long long b_pos = -1, s_pos = -1;
    while (pos >= f) {
      if (m_end[pos] >= e) {
        const long long len = m_end[pos] - m_start[pos];
        const int tg = m_tag[pos], og = m_orig[pos];
        const bool better_b = len < b_len || (len == b_len && (tg < b_tag || (tg == b_tag && og < b_orig)));
        if (better_b) {
          s_len = b_len; s_tag = b_tag; s_orig = b_orig; s_pos = b_pos;
          b_len = len; b_tag = tg; b_orig = og; b_pos = pos;
        } else {
          const bool better_s = len < s_len || (len == s_len && (tg < s_tag || (tg == s_tag && og < s_orig)));
          if (better_s) {
            s_len = len; s_tag = tg; s_orig = og; s_pos = pos;
          }
        }
        --pos;
        continue;
      }
      // skip the longest run [pos-2^k+1, pos] whose max end < e
      int k = 0;
      for (int q = levels - 1; q >= 1; --q) {
        if (pos - (1LL << q) + 1 >= f && mx[(long long)q * M + pos] < e) {
          k = q;
          break;
        }
      }
      pos -= (1LL << k);
    }
    if (b_pos < 0) continue;
    if (s_pos >= 0) {
      const bool nested = m_start[s_pos] <= m_start[b_pos] && m_end[b_pos] <= m_end[s_pos];
      if (!nested) atomicMin(ambiguous, (unsigned long long)i);
    }
    tag_out[i] = b_tag;
  }
}

__global__ void sparse_level_k(const int* mlane, const int* mseg_first, long long* mx, long long M,
                               int q) {
  const long long half = 1LL << (q - 1);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < M;
       i += (long long)gridDim.x * blockDim.x) {
    const long long a = mx[(long long)(q - 1) * M + i];
    long long v = a;
    if (i - half >= mseg_first[mlane[i]]) {
      const long long b = mx[(long long)(q - 1) * M + i - half];
      v = a > b ? a : b;
    }
    mx[(long long)q * M + i] = v;
  }
}

__global__ void inherit_k(const unsigned char* kind, const int* launcher, long long n, int* tag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (!is_gpu_kind(kind[i])) continue;
    const int u = launcher[i];
    if (u >= 0 && tag[u] >= 0) tag[i] = tag[u];
  }
}

__global__ void fill_ll_k(long long* a, long long v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = v;
}
__global__ void fill_i_k(int* a, int v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = v;
}

}  // namespace
void set_last_error(const std::string& msg);
}  // namespace ddsim

using namespace ddsim;

// DDSIM_INGEST_TIMING=1: synchronize and print the wall time of each stage
struct StageTimer {
  const char* what;
  cudaStream_t st;
  bool on;
  std::chrono::steady_clock::time_point t0;
  StageTimer(const char* w, cudaStream_t s)
      : what(w), st(s), on(std::getenv("DDSIM_INGEST_TIMING") != nullptr),
        t0(std::chrono::steady_clock::now()) {}
  void mark(const char* stage) {
    if (!on) return;
    cudaStreamSynchronize(st);
    auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[%s] %-12s %8.3f ms\n", what, stage,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};

// Keep freed stream-ordered memory in the device pool between calls (the
// default release threshold returns it to the driver at every synchronize).
static void keep_pool(int device) { keep_device_pool(device); }

void ddsim::IngestDev::release() {
  void* p[] = {lane, start, dur, gap, src, dst, ekind, lane_order};
  for (void* x : p)
    if (x) cudaFree(x);
  lane = nullptr;
  start = dur = gap = nullptr;
  src = dst = lane_order = nullptr;
  ekind = nullptr;
}

// keep != nullptr: the edges, lane order, gaps and the per-event lane / start /
// duration columns stay on the device in *keep (ks_ingest_keep)
static int ingest_impl(const ks_trace_cols* tc, int device, int check_overlaps,
                       ks_ingest_out* out, IngestDev* keep) {
  if (!tc || !out) return KS_ERR_INVALID;
  cudaSetDevice(device);
  keep_pool(device);
  const long long n = tc->n;
  const int L = tc->n_lanes;
  out->n_edges = 0;
  out->bad_a = out->bad_b = -1;
  if (n == 0) {
    for (int l = 0; l <= L; ++l) out->lane_order_ptr[l] = 0;
    return KS_OK;
  }
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return KS_ERR_CUDA;
  int rc = KS_OK;
  StageTimer T_("ks_ingest", st);
  try {
    Pool P{st};
    long long* d_id = P.up(reinterpret_cast<const long long*>(tc->id), n);
    unsigned char* d_kind = P.up(tc->kind, n);
    int* d_lane = P.up(tc->lane, n);
    long long* d_start = P.up(reinterpret_cast<const long long*>(tc->start), n);
    long long* d_dur = P.up(reinterpret_cast<const long long*>(tc->duration), n);
    long long* d_corr = P.up(reinterpret_cast<const long long*>(tc->correlation), n);
    int* d_st = P.up(tc->sync_target, n);
    unsigned char* d_dtoh = P.up(tc->is_dtoh, n);
    unsigned char* d_lclass = P.up(tc->lane_class, (size_t)L);
    T_.mark("upload");
    long long* d_end = P.get<long long>(n);
    end_k<<<blocks_for(n), TPB, 0, st>>>(d_start, d_dur, d_end, n);
    note_launch();

    // ---- overlap check: order (lane, start, end, id) ---------------------------
    if (check_overlaps) {
      int* perm = P.get<int>(n);
      iota_k<<<blocks_for(n), TPB, 0, st>>>(perm, n);
      note_launch();
      sort_by_key(P, d_id, perm, n);
      sort_by_key(P, d_end, perm, n);
      sort_by_key(P, d_start, perm, n);
      sort_by_key(P, d_lane, perm, n);
      long long* fs = P.get<long long>(L);
      fill_ll_k<<<blocks_for(L), TPB, 0, st>>>(fs, LLONG_MAX, L);
      first_seen_k<<<blocks_for(n), TPB, 0, st>>>(d_lane, n, fs);
      unsigned long long* best = P.get<unsigned long long>(1);
      ICUDA(cudaMemsetAsync(best, 0xff, sizeof(unsigned long long), st));
      overlap_k<<<blocks_for(n), TPB, 0, st>>>(perm, d_lane, d_start, d_end, n, fs, best);
      note_launch(3);
      unsigned long long hb = ~0ull;
      ICUDA(cudaMemcpyAsync(&hb, best, 8, cudaMemcpyDeviceToHost, st));
      ICUDA(cudaStreamSynchronize(st));
      if (hb != ~0ull) {
        const long long pos = (long long)(hb % (unsigned long long)(n + 1));
        int pa = 0, pb = 0;
        ICUDA(cudaMemcpy(&pa, perm + pos, sizeof(int), cudaMemcpyDeviceToHost));
        ICUDA(cudaMemcpy(&pb, perm + pos + 1, sizeof(int), cudaMemcpyDeviceToHost));
        out->bad_a = tc->id[pa];
        out->bad_b = tc->id[pb];
        throw IngestError{KS_ERR_OVERLAP, "lane overlap"};
      }
    }

    T_.mark("overlap");
    // ---- rules 1, 2, 5: lane order (lane, start, id) + gaps ---------------------
    int* perm = P.get<int>(n);
    iota_k<<<blocks_for(n), TPB, 0, st>>>(perm, n);
    note_launch();
    sort_by_key(P, d_id, perm, n);
    sort_by_key(P, d_start, perm, n);
    sort_by_key(P, d_lane, perm, n);
    int* lane_first = P.get<int>(L);
    int* lane_last = P.get<int>(L);
    fill_i_k<<<blocks_for(L), TPB, 0, st>>>(lane_first, 0, L);
    fill_i_k<<<blocks_for(L), TPB, 0, st>>>(lane_last, 0, L);
    lane_bounds_k<<<blocks_for(n), TPB, 0, st>>>(perm, d_lane, n, lane_first, lane_last);
    note_launch(3);

    T_.mark("lane-sort");
    // lanes that carry events (lane_bounds of the sorted view), GPU ones in index order
    std::vector<int> lf(L), ll(L);
    ICUDA(cudaMemcpyAsync(lf.data(), lane_first, sizeof(int) * L, cudaMemcpyDeviceToHost, st));
    ICUDA(cudaMemcpyAsync(ll.data(), lane_last, sizeof(int) * L, cudaMemcpyDeviceToHost, st));
    // rule-4 sources: Sync events and CPU memcpy_dtoh launches (compacted list)
    int* ssrc = P.get<int>(n);
    int* d_ns = P.get<int>(1);
    {
      unsigned char* sflag = P.get<unsigned char>(n);
      sync_src_flag_k<<<blocks_for(n), TPB, 0, st>>>(d_kind, d_dtoh, d_corr, n, sflag);
      int* all = P.get<int>(n);
      iota_k<<<blocks_for(n), TPB, 0, st>>>(all, n);
      note_launch(2);
      size_t tmp = 0;
      cub::DeviceSelect::Flagged(nullptr, tmp, all, sflag, ssrc, d_ns, (int)n, st);
      void* t = P.get<unsigned char>(tmp);
      ICUDA(cub::DeviceSelect::Flagged(t, tmp, all, sflag, ssrc, d_ns, (int)n, st));
      note_launch();
    }
    int ns = 0;
    ICUDA(cudaMemcpyAsync(&ns, d_ns, sizeof(int), cudaMemcpyDeviceToHost, st));
    ICUDA(cudaStreamSynchronize(st));
    std::vector<int> gpu_lanes_h;
    for (int l = 0; l < L; ++l)
      if (tc->lane_class[l] == 1 && ll[l] > lf[l]) gpu_lanes_h.push_back(l);
    const int G = (int)gpu_lanes_h.size();
    // candidate edge buffers: [lane n][launch n][sync ns*(G+1)]
    const long long c_lane = n, c_launch = n, c_sync = (long long)ns * (G + 1);
    const long long C = c_lane + c_launch + c_sync;
    int* esrc = P.get<int>(C);
    int* edst = P.get<int>(C);
    unsigned char* ekind = P.get<unsigned char>(C);
    unsigned char* eflag = P.get<unsigned char>(C);
    long long* d_gap = P.get<long long>(n);
    lane_edges_k<<<blocks_for(n), TPB, 0, st>>>(perm, d_lane, d_start, d_dur, d_lclass, n, esrc, edst,
                                                ekind, eflag, d_gap);
    note_launch();

    T_.mark("lane-edges");
    // ---- rule 3: launch correlation ---------------------------------------------
    long long* cpu_key = P.get<long long>(n);
    long long* gpu_key = P.get<long long>(n);
    corr_keys_k<<<blocks_for(n), TPB, 0, st>>>(d_kind, d_corr, n, cpu_key, gpu_key);
    note_launch();
    long long* cpu_sk = P.get<long long>(n);
    int* cpu_si = P.get<int>(n);
    long long* gpu_sk = P.get<long long>(n);
    int* gpu_si = P.get<int>(n);
    sort_pairs_ll(P, cpu_key, n, cpu_sk, cpu_si);
    sort_pairs_ll(P, gpu_key, n, gpu_sk, gpu_si);
    int* d_launcher = P.get<int>(n);
    unsigned long long* orphan = P.get<unsigned long long>(1);
    ICUDA(cudaMemsetAsync(orphan, 0xff, sizeof(unsigned long long), st));
    // sentinel keys (LLONG_MAX) sort last: searches run over the full arrays,
    // a real correlation never equals LLONG_MAX
    launch_join_k<<<blocks_for(n), TPB, 0, st>>>(d_kind, d_corr, n, cpu_sk, cpu_si, n, d_launcher,
                                                 esrc + c_lane, edst + c_lane, ekind + c_lane,
                                                 eflag + c_lane, orphan);
    note_launch();
    if (tc->strict) {
      unsigned long long ho = ~0ull;
      ICUDA(cudaMemcpyAsync(&ho, orphan, 8, cudaMemcpyDeviceToHost, st));
      ICUDA(cudaStreamSynchronize(st));
      if (ho != ~0ull) {
        out->bad_a = tc->id[ho];
        throw IngestError{KS_ERR_ORPHAN, "GPU task without CPU launch"};
      }
    }

    T_.mark("launch-join");
    // ---- rule 4: stream tasks sorted by (lane, launch start, id) ------------------
    int* skl = P.get<int>(n);
    long long* skls = P.get<long long>(n);
    stream_keys_k<<<blocks_for(n), TPB, 0, st>>>(d_kind, d_lane, d_start, d_launcher, n, L, skl, skls);
    note_launch();
    int* sperm = P.get<int>(n);
    iota_k<<<blocks_for(n), TPB, 0, st>>>(sperm, n);
    note_launch();
    sort_by_key(P, d_id, sperm, n);
    sort_by_key(P, skls, sperm, n);
    sort_by_key(P, skl, sperm, n);
    // sorted views
    long long* st_ls = P.get<long long>(n);
    gather_k<long long><<<blocks_for(n), TPB, 0, st>>>(skls, sperm, st_ls, n);
    int* st_lane = P.get<int>(n);
    gather_k<int><<<blocks_for(n), TPB, 0, st>>>(skl, sperm, st_lane, n);
    note_launch(2);
    int* seg_first = P.get<int>(L + 1);
    int* seg_last = P.get<int>(L + 1);
    fill_i_k<<<blocks_for(L + 1), TPB, 0, st>>>(seg_first, 0, L + 1);
    fill_i_k<<<blocks_for(L + 1), TPB, 0, st>>>(seg_last, 0, L + 1);
    lane_bounds_k<<<blocks_for(n), TPB, 0, st>>>(sperm, skl, n, seg_first,
                                                 seg_last);
    note_launch(3);
    T_.mark("stream-sort");
    int* d_gl = G > 0 ? P.up(gpu_lanes_h.data(), (size_t)G) : P.get<int>(1);
    sync_link_k<<<blocks_for(c_sync), TPB, 0, st>>>(
        d_kind, d_start, d_corr, d_st, d_dtoh, d_lane, ssrc, ns, d_gl, G, seg_first, seg_last, st_ls,
        sperm, gpu_sk, gpu_si, n, esrc + c_lane + c_launch, edst + c_lane + c_launch,
        ekind + c_lane + c_launch, eflag + c_lane + c_launch);
    note_launch();

    T_.mark("sync-link");
    // ---- compact + copy back ------------------------------------------------------
    int* os = P.get<int>(C);
    int* od = P.get<int>(C);
    unsigned char* ok = P.get<unsigned char>(C);
    const long long m = compact_edges(P, esrc, edst, ekind, eflag, C, os, od, ok);
    if (!keep && m > out->edge_cap) throw IngestError{KS_ERR_INVALID, "edge capacity too small"};
    T_.mark("compact");
    if (keep) {
      // hand the buffers over (the pool frees everything else)
      auto take = [&](void* ptr) {
        for (auto& q : P.ptrs)
          if (q == ptr) q = nullptr;
      };
      keep->device = device;
      keep->n = n;
      keep->m = m;
      keep->L = L;
      keep->lane = d_lane;
      keep->start = d_start;
      keep->dur = d_dur;
      keep->gap = d_gap;
      keep->src = os;
      keep->dst = od;
      keep->ekind = ok;
      keep->lane_order = perm;
      for (void* q : {(void*)d_lane, (void*)d_start, (void*)d_dur, (void*)d_gap, (void*)os,
                      (void*)od, (void*)ok, (void*)perm})
        take(q);
      keep->lane_class.assign(tc->lane_class, tc->lane_class + L);
    } else {
      ICUDA(cudaMemcpyAsync(out->edge_src, os, sizeof(int) * m, cudaMemcpyDeviceToHost, st));
      ICUDA(cudaMemcpyAsync(out->edge_dst, od, sizeof(int) * m, cudaMemcpyDeviceToHost, st));
      ICUDA(cudaMemcpyAsync(out->edge_kind, ok, m, cudaMemcpyDeviceToHost, st));
      ICUDA(cudaMemcpyAsync(out->lane_order, perm, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
      ICUDA(cudaMemcpyAsync(out->gap, d_gap, sizeof(long long) * n, cudaMemcpyDeviceToHost, st));
    }
    ICUDA(cudaMemcpyAsync(out->launcher, d_launcher, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    ICUDA(cudaStreamSynchronize(st));
    // lane_order_ptr: lanes appear in index order in the sorted view
    int pos = 0;
    for (int l = 0; l < L; ++l) {
      out->lane_order_ptr[l] = pos;
      if (ll[l] > lf[l]) pos = ll[l];
    }
    out->lane_order_ptr[L] = pos;
    out->n_edges = m;
    if (keep) keep->lane_order_ptr.assign(out->lane_order_ptr, out->lane_order_ptr + L + 1);
    T_.mark("copy-back");
  } catch (const IngestError& e) {
    set_last_error(e.msg);
    rc = e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    rc = KS_ERR_INVALID;
  } catch (...) {
    rc = KS_ERR_INVALID;
  }
  T_.mark("release");
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (rc != KS_OK) cudaGetLastError();  // do not leave a non-sticky error for later calls
  return rc;
}

extern "C" int ks_ingest(const ks_trace_cols* tc, int device, int check_overlaps,
                         ks_ingest_out* out) {
  return ingest_impl(tc, device, check_overlaps, out, nullptr);
}

extern "C" int ks_ingest_keep(const ks_trace_cols* tc, int device, int check_overlaps,
                              ks_ingest_out* out, ks_ingest_dev** dev_out) {
  if (!dev_out) return KS_ERR_INVALID;
  *dev_out = nullptr;
  ks_ingest_dev* h = new ks_ingest_dev;
  const int rc = ingest_impl(tc, device, check_overlaps, out, &h->d);
  if (rc != KS_OK) {
    h->d.release();
    delete h;
    return rc;
  }
  *dev_out = h;
  return KS_OK;
}

extern "C" int ks_ingest_dev_copy(const ks_ingest_dev* h, int32_t* edge_src, int32_t* edge_dst,
                                  uint8_t* edge_kind, int32_t* lane_order, int64_t* gap) {
  if (!h) return KS_ERR_INVALID;
  const IngestDev& I = h->d;
  cudaSetDevice(I.device);
  cudaError_t e = cudaSuccess;
  if (edge_src && I.m) e = cudaMemcpy(edge_src, I.src, sizeof(int) * I.m, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && edge_dst && I.m)
    e = cudaMemcpy(edge_dst, I.dst, sizeof(int) * I.m, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && edge_kind && I.m)
    e = cudaMemcpy(edge_kind, I.ekind, I.m, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && lane_order && I.n)
    e = cudaMemcpy(lane_order, I.lane_order, sizeof(int) * I.n, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && gap && I.n)
    e = cudaMemcpy(gap, I.gap, sizeof(long long) * I.n, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    set_last_error(cudaGetErrorString(e));
    return KS_ERR_CUDA;
  }
  return KS_OK;
}

extern "C" void ks_ingest_dev_free(ks_ingest_dev* h) {
  if (!h) return;
  cudaSetDevice(h->d.device);
  h->d.release();
  delete h;
}

extern "C" int ks_map_layers(const ks_trace_cols* tc, const int32_t* launcher,
                             const ks_marker_cols* mc, int device, int32_t* tag_out,
                             int64_t* bad_event) {
  if (!tc || !mc || !tag_out) return KS_ERR_INVALID;
  cudaSetDevice(device);
  keep_pool(device);
  const long long n = tc->n, M = mc->n;
  const int L = tc->n_lanes;
  if (bad_event) *bad_event = -1;
  if (n == 0) return KS_OK;
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return KS_ERR_CUDA;
  int rc = KS_OK;
  try {
    Pool P{st};
    unsigned char* d_kind = P.up(tc->kind, n);
    int* d_lane = P.up(tc->lane, n);
    long long* d_start = P.up(reinterpret_cast<const long long*>(tc->start), n);
    long long* d_dur = P.up(reinterpret_cast<const long long*>(tc->duration), n);
    int* d_launch = P.up(launcher, n);
    int* d_tag = P.get<int>(n);
    unsigned long long* amb = P.get<unsigned long long>(1);
    ICUDA(cudaMemsetAsync(amb, 0xff, 8, st));
    if (M > 0) {
      // markers sorted by (lane, start), stable on the original order
      int* ml = P.up(mc->lane, M);
      long long* ms = P.up(reinterpret_cast<const long long*>(mc->start), M);
      long long* me = P.up(reinterpret_cast<const long long*>(mc->end), M);
      int* mt = P.up(mc->tag, M);
      int* mperm = P.get<int>(M);
      iota_k<<<blocks_for(M), TPB, 0, st>>>(mperm, M);
      note_launch();
      sort_by_key(P, ms, mperm, M);
      sort_by_key(P, ml, mperm, M);
      long long* s_ms = P.get<long long>(M);
      long long* s_me = P.get<long long>(M);
      int* s_mt = P.get<int>(M);
      int* s_ml = P.get<int>(M);
      gather_k<long long><<<blocks_for(M), TPB, 0, st>>>(ms, mperm, s_ms, M);
      gather_k<long long><<<blocks_for(M), TPB, 0, st>>>(me, mperm, s_me, M);
      gather_k<int><<<blocks_for(M), TPB, 0, st>>>(mt, mperm, s_mt, M);
      gather_k<int><<<blocks_for(M), TPB, 0, st>>>(ml, mperm, s_ml, M);
      note_launch(4);
      int* mf = P.get<int>(L);
      int* mlst = P.get<int>(L);
      fill_i_k<<<blocks_for(L), TPB, 0, st>>>(mf, 0, L);
      fill_i_k<<<blocks_for(L), TPB, 0, st>>>(mlst, 0, L);
      lane_bounds_k<<<blocks_for(M), TPB, 0, st>>>(mperm, ml, M, mf, mlst);
      note_launch(3);
      int levels = 1;
      while ((1LL << levels) <= M) ++levels;
      long long* mx = P.get<long long>((size_t)levels * M);
      ICUDA(cudaMemcpyAsync(mx, s_me, sizeof(long long) * M, cudaMemcpyDeviceToDevice, st));
      for (int q = 1; q < levels; ++q) {
        sparse_level_k<<<blocks_for(M), TPB, 0, st>>>(s_ml, mf, mx, M, q);
        note_launch();
      }
      layer_map_k<<<blocks_for(n), TPB, 0, st>>>(d_kind, d_lane, d_start, d_dur, n, mf, mlst, L, s_ms,
                                                 s_me, s_mt, mperm, mx, levels, M, d_tag, amb);
      note_launch();
    } else {
      fill_i_k<<<blocks_for(n), TPB, 0, st>>>(d_tag, -1, n);
      note_launch();
    }
    inherit_k<<<blocks_for(n), TPB, 0, st>>>(d_kind, d_launch, n, d_tag);
    note_launch();
    unsigned long long ha = ~0ull;
    ICUDA(cudaMemcpyAsync(&ha, amb, 8, cudaMemcpyDeviceToHost, st));
    ICUDA(cudaMemcpyAsync(tag_out, d_tag, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    ICUDA(cudaStreamSynchronize(st));
    if (ha != ~0ull) {
      if (bad_event) *bad_event = tc->id[ha];
      throw IngestError{KS_ERR_AMBIGUOUS, "ambiguous marker"};
    }
  } catch (const IngestError& e) {
    set_last_error(e.msg);
    rc = e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    rc = KS_ERR_INVALID;
  } catch (...) {
    rc = KS_ERR_INVALID;
  }
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (rc != KS_OK) cudaGetLastError();  // do not leave a non-sticky error for later calls
  return rc;
}
