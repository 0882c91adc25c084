// freeze: the frozen graph of an ingested trace, compiled on the device.
//
// Reference: DependencyGraph construction and verify_acyclic
// (pkg/src/kernsim/graph.py:75-148, 198-245).  ks_ingest (ingest.cu) leaves
// its outputs on the device (IngestDev); this file turns them into the parts
// of a frozen graph every kernel path needs, without a host round trip:
//
//   unique edges      radix sort of (u << 32 | v) + unique           (CUB)
//   predecessor CSR   radix sort of (v << 32 | u)                    (CUB)
//   topological order potentials relaxed from the trace start times until
//                     key(v) >= key(u) + 1 on every edge: a segmented (max,+)
//                     scan along each lane's order and an atomicMax pass over
//                     the cross-lane edges per round (a synthetic or clock-
//                     skewed trace records some synchronisations before the
//                     kernels they wait for; rounds ~ the longest chain of
//                     such corrections); sorted by (key, id rank) and checked
//                     on every edge.  No fixed point within the round cap (a
//                     cycle) -> the host compiler (depth-first Kahn, its
//                     CycleDetected) runs instead
//   frozen rows       row r = order[r]; per-row lane / duration / gap / rank /
//                     flags arrays gathered in row order
//   list-scheduler    multiset child CSR over rows: radix sort of
//   CSR               (row(u) << 32 | row(v)), in-degrees by histogram
//
// The kernel programs (lane-register, dense, general records) are built on
// the host on first use from copies of these arrays (graph.cu,
// ensure_programs), as for a host-compiled graph.
#include "ddsim_internal.h"

#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <string>
#include <vector>

namespace ddsim {
namespace {

struct FreezeError {
  std::string msg;
};
#define FCUDA(x)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) throw FreezeError{std::string(#x) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

constexpr int TPB = 256;
inline int blocks_for(long long n) {
  long long b = (n + TPB - 1) / TPB;
  return (int)std::max(1LL, std::min(b, 148LL * 64));
}

// stream-ordered temporaries freed together
struct Tmp {
  cudaStream_t st;
  std::vector<void*> ptrs;
  template <class T>
  T* get(size_t n) {
    T* p = nullptr;
    FCUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st));
    ptrs.push_back(p);
    return p;
  }
  ~Tmp() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};
template <class T>
T* persist(size_t n) {  // owned by the graph (cudaFree in free_graph)
  T* p = nullptr;
  FCUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  return p;
}

#define GRID_STRIDE(i, n) \
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (n); \
       i += (long long)gridDim.x * blockDim.x)

__global__ void edge_keys_k(const int* src, const int* dst, long long m, unsigned long long* k) {
  GRID_STRIDE(i, m) k[i] = ((unsigned long long)(unsigned)src[i] << 32) | (unsigned)dst[i];
}
__global__ void swap_keys_k(const unsigned long long* a, long long m, unsigned long long* b) {
  GRID_STRIDE(i, m) b[i] = (a[i] << 32) | (a[i] >> 32);
}
// Potential relaxation (longest-path style, unit weights) from the trace
// start times: key(v) >= key(u) + 1 on every cross-lane edge (atomicMax) and
// along every lane (segmented (max,+) scan), until nothing moves.  Starts are
// already nearly consistent in a trace, so few rounds fix the edges they
// violate (a synchronisation recorded before the kernels it waits for).
// edges the lane scan does not enforce: all but lane-order successors
__global__ void cross_edges_k(const unsigned long long* uk, long long m, const int* lane,
                              const int* lpos, unsigned char* flag) {
  GRID_STRIDE(i, m) {
    const int u = (int)(uk[i] >> 32), v = (int)(uk[i] & 0xffffffffu);
    flag[i] = !(lane[u] == lane[v] && lpos[v] == lpos[u] + 1);
  }
}
__global__ void relax_edges_k(const unsigned long long* ce, long long mc, long long* key,
                              int* changed) {
  GRID_STRIDE(i, mc) {
    const int u = (int)(ce[i] >> 32), v = (int)(ce[i] & 0xffffffffu);
    const long long nv = key[u] + 1;
    if (nv > key[v] && atomicMax(reinterpret_cast<long long*>(key + v), nv) < nv) *changed = 1;
  }
}
__global__ void lane_vals_k(const int* lo, long long n, const long long* key, long long* val) {
  GRID_STRIDE(i, n) val[i] = key[lo[i]] - i;
}
__global__ void lane_apply_k(const int* lo, long long n, const long long* mx, long long* key,
                             int* changed) {
  GRID_STRIDE(i, n) {
    const long long nk = mx[i] + i;
    if (nk > key[lo[i]]) {
      key[lo[i]] = nk;
      *changed = 1;
    }
  }
}
__global__ void gather_i_k(const int* src, const int* idx, long long n, int* dst) {
  GRID_STRIDE(i, n) dst[i] = src[idx[i]];
}
__global__ void gather_ll_k(const long long* src, const int* idx, long long n, long long* dst) {
  GRID_STRIDE(i, n) dst[i] = src[idx[i]];
}
struct MaxOp {
  __device__ __forceinline__ long long operator()(long long a, long long b) const {
    return a > b ? a : b;
  }
};
__global__ void iota_k(int* a, long long n) {
  GRID_STRIDE(i, n) a[i] = (int)i;
}
__global__ void pos_k(const int* order, long long n, int* pos) {
  GRID_STRIDE(i, n) pos[order[i]] = (int)i;
}
__global__ void verify_k(const unsigned long long* uk, long long m, const int* pos,
                         unsigned long long* bad) {
  GRID_STRIDE(i, m) {
    const int u = (int)(uk[i] >> 32), v = (int)(uk[i] & 0xffffffffu);
    if (pos[u] >= pos[v]) atomicMin(bad, (unsigned long long)i);
  }
}
__global__ void rows_k(const int* order, long long n, const int* lane, const long long* dur,
                       const long long* gap, const int* rank, const unsigned char* flags,
                       int* lane_r, long long* dur_r, long long* gap_r, int* rank_r,
                       unsigned char* flags_r) {
  GRID_STRIDE(r, n) {
    const int t = order[r];
    lane_r[r] = lane[t];
    dur_r[r] = dur[t];
    gap_r[r] = gap[t];
    rank_r[r] = rank ? rank[t] : t;
    flags_r[r] = flags ? flags[t] : 0;
  }
}
__global__ void row_edge_keys_k(const int* src, const int* dst, long long m, const int* pos,
                                unsigned long long* k) {
  GRID_STRIDE(i, m)
  k[i] = ((unsigned long long)(unsigned)pos[src[i]] << 32) | (unsigned)pos[dst[i]];
}
__global__ void csr_k(const unsigned long long* k, long long m, int* count_hi, int* count_lo,
                      int* lo) {
  GRID_STRIDE(i, m) {
    const unsigned long long x = k[i];
    if (count_hi) atomicAdd(&count_hi[(int)(x >> 32) + 1], 1);
    if (count_lo) atomicAdd(&count_lo[(int)(x & 0xffffffffu)], 1);
    if (lo) lo[i] = (int)(x & 0xffffffffu);
  }
}

int key_bits(long long n) {  // bits of a dense index
  int b = 1;
  while ((1LL << b) < n) ++b;
  return b;
}

void sort_u64(Tmp& T, const unsigned long long* in, unsigned long long* out, long long m, int bits) {
  size_t tmp = 0;
  FCUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, in, out, (int)m, 0, bits, T.st));
  void* t = T.get<unsigned char>(tmp);
  FCUDA(cub::DeviceRadixSort::SortKeys(t, tmp, in, out, (int)m, 0, bits, T.st));
  note_launch();
}

}  // namespace

void free_device_freeze(DeviceFreeze& F) {
  void* p[] = {F.child_ptr, F.child, F.indeg, F.lane_r, F.rank_r, F.prio_r, F.dur_r, F.gap_r,
               F.ready_r, F.flags_r, F.group_r, F.ukeys, F.pkeys, F.order_d};
  for (void* x : p)
    if (x) cudaFree(x);
  F = DeviceFreeze{};
}

int freeze_from_ingest(const IngestDev& I, const int32_t* id_rank_h, const uint8_t* flags_h,
                       DeviceFreeze& F, std::string& err) {
  const long long n = I.n, m = I.m;
  F = DeviceFreeze{};
  F.n = n;
  if (n <= 0) return KS_OK;
  cudaSetDevice(I.device);
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return KS_ERR_CUDA;
  int rc = KS_OK;
  try {
    Tmp T{st};
    const int bits = key_bits(n);
    // ---- unique edges, sorted by (u, v) ---------------------------------------
    unsigned long long* ek = T.get<unsigned long long>(m);
    edge_keys_k<<<blocks_for(m), TPB, 0, st>>>(I.src, I.dst, m, ek);
    note_launch();
    unsigned long long* sk = T.get<unsigned long long>(m);
    sort_u64(T, ek, sk, m, 32 + bits);
    F.ukeys = persist<unsigned long long>(m);
    int* d_nu = T.get<int>(1);
    {
      size_t tmp = 0;
      FCUDA(cub::DeviceSelect::Unique(nullptr, tmp, sk, F.ukeys, d_nu, (int)m, st));
      void* t = T.get<unsigned char>(tmp);
      FCUDA(cub::DeviceSelect::Unique(t, tmp, sk, F.ukeys, d_nu, (int)m, st));
      note_launch();
    }
    int nu = 0;
    FCUDA(cudaMemcpyAsync(&nu, d_nu, sizeof(int), cudaMemcpyDeviceToHost, st));
    FCUDA(cudaStreamSynchronize(st));
    F.m_unique = nu;
    // ---- predecessor keys, sorted by (v, u) -----------------------------------
    unsigned long long* swp = T.get<unsigned long long>(nu);
    swap_keys_k<<<blocks_for(nu), TPB, 0, st>>>(F.ukeys, nu, swp);
    note_launch();
    F.pkeys = persist<unsigned long long>(nu);
    sort_u64(T, swp, F.pkeys, nu, 32 + bits);
    // ---- topological order: relaxed trace-time potentials ------------------------
    long long* pot = T.get<long long>(n);
    FCUDA(cudaMemcpyAsync(pot, I.start, sizeof(long long) * n, cudaMemcpyDeviceToDevice, st));
    unsigned long long* ce = T.get<unsigned long long>(nu);
    int* d_nc = T.get<int>(1);
    {
      unsigned char* cf = T.get<unsigned char>(nu);
      int* lpos = T.get<int>(n);
      pos_k<<<blocks_for(n), TPB, 0, st>>>(I.lane_order, n, lpos);
      cross_edges_k<<<blocks_for(nu), TPB, 0, st>>>(F.ukeys, nu, I.lane, lpos, cf);
      note_launch(2);
      size_t tmp = 0;
      FCUDA(cub::DeviceSelect::Flagged(nullptr, tmp, F.ukeys, cf, ce, d_nc, (int)nu, st));
      void* t = T.get<unsigned char>(tmp);
      FCUDA(cub::DeviceSelect::Flagged(t, tmp, F.ukeys, cf, ce, d_nc, (int)nu, st));
      note_launch();
    }
    int nc = 0;
    FCUDA(cudaMemcpyAsync(&nc, d_nc, sizeof(int), cudaMemcpyDeviceToHost, st));
    FCUDA(cudaStreamSynchronize(st));
    int* seg = T.get<int>(n);  // lane of each lane-order position
    gather_i_k<<<blocks_for(n), TPB, 0, st>>>(I.lane, I.lane_order, n, seg);
    note_launch();
    long long* val = T.get<long long>(n);
    long long* mx = T.get<long long>(n);
    size_t scan_tmp = 0;
    FCUDA(cub::DeviceScan::InclusiveScanByKey(nullptr, scan_tmp, seg, val, mx, MaxOp(), (int)n,
                                              cub::Equality(), st));
    void* scan_t = T.get<unsigned char>(scan_tmp);
    int* changed = T.get<int>(1);
    int* h_changed = nullptr;
    FCUDA(cudaMallocHost(&h_changed, sizeof(int)));
    int rounds = 0;
    const int max_rounds = getenv("DDSIM_FREEZE_ROUNDS") ? atoi(getenv("DDSIM_FREEZE_ROUNDS")) : 4096;
    bool settled = false;
    for (; rounds < max_rounds; ++rounds) {
      FCUDA(cudaMemsetAsync(changed, 0, sizeof(int), st));
      lane_vals_k<<<blocks_for(n), TPB, 0, st>>>(I.lane_order, n, pot, val);
      FCUDA(cub::DeviceScan::InclusiveScanByKey(scan_t, scan_tmp, seg, val, mx, MaxOp(), (int)n,
                                                cub::Equality(), st));
      lane_apply_k<<<blocks_for(n), TPB, 0, st>>>(I.lane_order, n, mx, pot, changed);
      if (nc > 0) relax_edges_k<<<blocks_for(nc), TPB, 0, st>>>(ce, nc, pot, changed);
      note_launch(nc > 0 ? 4 : 3);
      FCUDA(cudaMemcpyAsync(h_changed, changed, sizeof(int), cudaMemcpyDeviceToHost, st));
      FCUDA(cudaStreamSynchronize(st));
      if (*h_changed == 0) {
        settled = true;
        break;
      }
    }
    cudaFreeHost(h_changed);
    F.rounds = rounds;
    int* rank = nullptr;
    int* by_rank = T.get<int>(n);  // tasks in id-rank order
    if (id_rank_h) {
      rank = T.get<int>(n);
      FCUDA(cudaMemcpyAsync(rank, id_rank_h, sizeof(int) * n, cudaMemcpyHostToDevice, st));
      int* seq = T.get<int>(n);
      iota_k<<<blocks_for(n), TPB, 0, st>>>(seq, n);
      int* rs = T.get<int>(n);
      size_t tmp = 0;
      FCUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, rank, rs, seq, by_rank, (int)n, 0, bits,
                                            st));
      void* t = T.get<unsigned char>(tmp);
      FCUDA(cub::DeviceRadixSort::SortPairs(t, tmp, rank, rs, seq, by_rank, (int)n, 0, bits, st));
      note_launch(2);
    } else {
      iota_k<<<blocks_for(n), TPB, 0, st>>>(by_rank, n);
      note_launch();
    }
    long long* key = T.get<long long>(n);
    gather_ll_k<<<blocks_for(n), TPB, 0, st>>>(pot, by_rank, n, key);
    note_launch();
    long long* key_s = T.get<long long>(n);
    F.order_d = persist<int>(n);
    {
      size_t tmp = 0;  // stable: ties keep the id-rank order
      FCUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, key_s, by_rank, F.order_d, (int)n,
                                            0, 64, st));
      void* t = T.get<unsigned char>(tmp);
      FCUDA(cub::DeviceRadixSort::SortPairs(t, tmp, key, key_s, by_rank, F.order_d, (int)n, 0, 64,
                                            st));
      note_launch();
    }
    int* pos = T.get<int>(n);
    pos_k<<<blocks_for(n), TPB, 0, st>>>(F.order_d, n, pos);
    unsigned long long* bad = T.get<unsigned long long>(1);
    FCUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
    verify_k<<<blocks_for(nu), TPB, 0, st>>>(F.ukeys, nu, pos, bad);
    note_launch(2);
    unsigned long long hb = 0;
    FCUDA(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, st));
    F.order.resize(n);
    FCUDA(cudaMemcpyAsync(F.order.data(), F.order_d, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    FCUDA(cudaStreamSynchronize(st));
    F.ok = settled && hb == ~0ull;
    if (!F.ok) {
      // not a trace-time consistent graph: the host compiler orders it
      rc = KS_OK;
      throw FreezeError{"__fallback__"};
    }
    // ---- frozen rows: per-row arrays --------------------------------------------
    unsigned char* flags = nullptr;
    if (flags_h) {
      flags = T.get<unsigned char>(n);
      FCUDA(cudaMemcpyAsync(flags, flags_h, n, cudaMemcpyHostToDevice, st));
    }
    F.lane_r = persist<int>(n);
    F.dur_r = persist<long long>(n);
    F.gap_r = persist<long long>(n);
    F.rank_r = persist<int>(n);
    F.flags_r = persist<unsigned char>(n);
    F.prio_r = persist<int>(n);
    F.ready_r = persist<long long>(n);
    F.group_r = persist<unsigned>(n);
    rows_k<<<blocks_for(n), TPB, 0, st>>>(F.order_d, n, I.lane, I.dur, I.gap, rank, flags, F.lane_r,
                                          F.dur_r, F.gap_r, F.rank_r, F.flags_r);
    note_launch();
    FCUDA(cudaMemsetAsync(F.prio_r, 0, sizeof(int) * n, st));
    FCUDA(cudaMemsetAsync(F.ready_r, 0, sizeof(long long) * n, st));
    FCUDA(cudaMemsetAsync(F.group_r, 0, sizeof(unsigned) * n, st));
    // ---- list-scheduler CSR over rows (multiset edges, children ascending) -------
    unsigned long long* rk = T.get<unsigned long long>(m);
    row_edge_keys_k<<<blocks_for(m), TPB, 0, st>>>(I.src, I.dst, m, pos, rk);
    note_launch();
    unsigned long long* rks = T.get<unsigned long long>(m);
    sort_u64(T, rk, rks, m, 32 + bits);
    F.child_ptr = persist<int>(n + 1);
    F.child = persist<int>(m);
    F.indeg = persist<int>(n);
    int* cnt = T.get<int>(n + 1);
    FCUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * (n + 1), st));
    FCUDA(cudaMemsetAsync(F.indeg, 0, sizeof(int) * n, st));
    csr_k<<<blocks_for(m), TPB, 0, st>>>(rks, m, cnt, F.indeg, F.child);
    note_launch();
    {
      size_t tmp = 0;
      FCUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt, F.child_ptr, (int)(n + 1), st));
      void* t = T.get<unsigned char>(tmp);
      FCUDA(cub::DeviceScan::InclusiveSum(t, tmp, cnt, F.child_ptr, (int)(n + 1), st));
      note_launch();
    }
    FCUDA(cudaStreamSynchronize(st));
  } catch (const FreezeError& e) {
    if (e.msg != "__fallback__") {
      err = e.msg;
      rc = KS_ERR_CUDA;
    }
  }
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (rc != KS_OK || !F.ok) {
    std::vector<int> keep_order;
    if (rc == KS_OK) keep_order.swap(F.order);
    const bool ok = F.ok;
    free_device_freeze(F);
    F.ok = ok;
    F.order.swap(keep_order);
    cudaGetLastError();
  }
  return rc;
}

}  // namespace ddsim
