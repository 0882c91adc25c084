// Graph compiler + C-ABI of libddsim.
//
// ks_graph_create freezes a kernsim DependencyGraph (pkg/src/kernsim/graph.py:
// 75-126) into device-resident arrays:
//   * the lane-chaining check that licenses the max-plus path (every task in
//     its lane's lane_order chain, consecutive pairs joined by an edge; see
//     sim.py:113-130 -- lane exclusivity then never binds);
//   * a topological order of the (deduplicated) edge set, depth-first so that
//     a produced value is consumed soon after (Kahn with a LIFO frontier,
//     lane successors pushed before cross-lane children);
//   * value-slot allocation: every task whose rel = start+dur+gap is read by a
//     later task gets a slot for its live range (linear scan); short ranges go
//     to shared memory, long ones to a global spill area;
//   * the multiset CSR + in-degrees the list scheduler needs (sim.py:95-106).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <deque>
#include <chrono>
#include <cstdio>
#include <functional>
#include <numeric>
#include <queue>
#include <string>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>
#include <cstdlib>

#include "ddsim_internal.h"

namespace ddsim {

static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }
static std::atomic<long long> g_launches{0};
void note_launch(int n) { g_launches.fetch_add(n); }

void keep_device_pool(int device) {
  static std::atomic<unsigned> done{0};
  if (device < 0 || device >= 32 || (done.load() >> device) & 1u) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.fetch_or(1u << device);
}

struct KsError {
  int code;
  std::string msg;
};

static void fail(int code, const std::string& msg) { throw KsError{code, msg}; }

#define CUDA_TRY(expr)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      fail(e_ == cudaErrorMemoryAllocation ? KS_ERR_OOM : KS_ERR_CUDA,                 \
           std::string(#expr) + ": " + cudaGetErrorString(e_));                        \
  } while (0)

// DDSIM_COMPILE_ONLY=1: run the graph compiler without a device (CPU tests of
// the compiler itself); such handles cannot simulate.
static bool g_compile_only = false;

template <class V>
static auto dev_upload(const V& v) -> typename V::value_type* {
  using T = typename V::value_type;
  if (v.empty() || g_compile_only) return nullptr;
  T* p = nullptr;
  CUDA_TRY(cudaMalloc(&p, v.size() * sizeof(T)));
  CUDA_TRY(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

// Split [0, n) over the host cores (independent iterations only).
template <class F>
static void host_parallel_for(long long n, F f) {
  unsigned hw = std::thread::hardware_concurrency();
  long long K = std::max(1LL, std::min<long long>(hw ? hw : 1, n / 262144));
  if (K <= 1) {
    f(0LL, n);
    return;
  }
  std::vector<std::thread> th;
  const long long step = (n + K - 1) / K;
  for (long long k = 0; k < K; ++k) {
    const long long b = k * step, e = std::min(n, b + step);
    if (b < e) th.emplace_back(f, b, e);
  }
  for (auto& t : th) t.join();
}

// Independent compile sections on their own threads (the CUDA device is
// per-thread state: set it in each); the first exception is rethrown on join.
struct ConcurrentSections {
  int device;
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err;
  std::mutex mu;
  explicit ConcurrentSections(int dev) : device(dev) {}
  template <class F>
  void run(const char* name, F f) {
    th.emplace_back([this, f, name]() mutable {
      try {
        if (device >= 0 && !g_compile_only) cudaSetDevice(device);
        const auto t0 = std::chrono::steady_clock::now();
        f();
        if (std::getenv("DDSIM_INGEST_TIMING"))
          std::fprintf(stderr, "[compile_graph]   %-11s %8.3f ms (concurrent)\n", name,
                       std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                           .count());
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        err.push_back(std::current_exception());
      }
    });
  }
  void join() {
    for (auto& t : th) t.join();
    th.clear();
    if (!err.empty()) std::rethrow_exception(err.front());
  }
  ~ConcurrentSections() {
    for (auto& t : th)
      if (t.joinable()) t.join();
  }
};

// Free slot ids, smallest first (the order a min-heap gives, so slot
// assignments are unchanged): a three-level 64-ary bitmap, O(1) per level.
struct MinFreeSet {
  std::vector<unsigned long long> b0, b1, b2;
  size_t cnt = 0;
  bool empty() const { return cnt == 0; }
  void push(int x) {
    const size_t i0 = (size_t)x >> 6, i1 = i0 >> 6, i2 = i1 >> 6;
    if (i0 >= b0.size()) {
      b0.resize(std::max(i0 + 1, b0.size() * 2));
      b1.resize((b0.size() + 63) / 64);
      b2.resize((b1.size() + 63) / 64);
    }
    b0[i0] |= 1ull << (x & 63);
    b1[i1] |= 1ull << (i0 & 63);
    b2[i2] |= 1ull << (i1 & 63);
    ++cnt;
  }
  int top() const {
    size_t i2 = 0;
    while (!b2[i2]) ++i2;
    const size_t i1 = i2 * 64 + __builtin_ctzll(b2[i2]);
    const size_t i0 = i1 * 64 + __builtin_ctzll(b1[i1]);
    return (int)(i0 * 64 + __builtin_ctzll(b0[i0]));
  }
  void pop() {
    const int x = top();
    const size_t i0 = (size_t)x >> 6, i1 = i0 >> 6, i2 = i1 >> 6;
    b0[i0] &= ~(1ull << (x & 63));
    if (!b0[i0]) {
      b1[i1] &= ~(1ull << (i0 & 63));
      if (!b1[i1]) b2[i2] &= ~(1ull << (i1 & 63));
    }
    --cnt;
  }
};

constexpr int kSmemSlotsMax = 24;
constexpr int kShortRange = 48;

}  // namespace ddsim

using namespace ddsim;

// What build_programs reads: owned copies of the descriptor arrays it uses
// (the caller's arrays need only live until ks_graph_create returns) and the
// compile_graph intermediates (unique edges, predecessor lists, record order).
struct LazyPrograms {
  int n = 0, L = 0, NC = 0, R = 0;
  long long E = 0;
  bool chained = false;
  ks_graph_desc desc;
  hvec<int64_t> duration, gap, ready;
  hvec<int32_t> lane, lane_order_ptr, lane_order, chain_ptr, chain_member, chain_head, chain_tail;
  hvec<uint32_t> group;
  hvec<unsigned long long> keys;
  hvec<int> optr, pptr, padj, corder, rec_first_row, ch_lane, tail_of, cptr, cadj;
  // graphs frozen on the device (ks_graph_create_from_ingest): the host arrays
  // above are filled from these on first use (materialize_from_device)
  bool from_device = false;
  unsigned long long* d_ukeys = nullptr;  // (u << 32 | v) unique, ascending
  unsigned long long* d_pkeys = nullptr;  // (v << 32 | u) unique, ascending
  int* d_lane_order = nullptr;
  long long m_unique = 0;
  ~LazyPrograms() {
    if (d_ukeys) cudaFree(d_ukeys);
    if (d_pkeys) cudaFree(d_pkeys);
    if (d_lane_order) cudaFree(d_lane_order);
  }
};
struct ks_graph {
  int device = 0;
  std::once_flag programs_once;
  std::unique_ptr<LazyPrograms> lazy;  // until build_programs
  int n = 0, L = 0;
  int n_ordered = 0;
  int n_edges_unique = 0;
  bool chained = false;
  int n_slots = 0, ksm = 0, kglob = 0;
  int n_rec = 0;
  int n_levels = 0;
  long long dur_abs_max = -1;  // max |base duration| (build_programs; -1: unknown)
  int n_chains = 0;
  int perm_ld = 0;
  bool rows_are_records = true;  // no chains: record i writes row i
  hvec<int> order;        // frozen row -> input index
  hvec<int> row_of;       // input index -> frozen row
  hvec<int> level;        // per frozen row
  hvec<int> rank_row;     // id rank per frozen row
  // lane-register program (chained, <= 4 lanes, no chains)
  bool has_lanes = false;
  int ln_rec = 0;          // lanes records (= frozen rows)
  int lksm = 0, lkglob = 0;
  std::vector<int> lane_codes;  // handler codes in decreasing frequency
  // segment-parallel evaluation (SegParams, lanes_body.cuh): chunk-aligned rows
  // where no slot value is live and no chain is split, and the prefix sums of
  // the records' base weights max(dur, 0) + gap (chain records: their members')
  std::vector<int> lane_cuts;
  std::vector<long long> lane_wt_prefix;
  std::vector<long long> lane_gap_prefix;  // prefix sums of the records' gaps
  // carries: global-slot values live across the cuts before the chain segment
  // [seg_c0, seg_c1) (the one permutable chain's record and its neighbours,
  // replayed numerically); the scan evaluates each carry from its producing
  // segment's transfer coefficients (lanes_seg.cuh)
  int seg_c0 = -1, seg_c1 = -1;
  std::vector<int> carry_rows, carry_gid;  // producer row (ascending), global slot id
  bool lane_ready = false;      // some record has a ready floor
  LaneRec* d_lprog = nullptr;
  int* d_lside_off = nullptr;
  int* d_lside_slots = nullptr;
  long long* d_lside_ready = nullptr;
  LaneChainDev* d_lchains = nullptr;    // permutable chains on the lanes path
  LaneMemberDev* d_lmembers = nullptr;
  int* d_lpreds = nullptr;
  // dense-duration program (no chains, <= 255 lanes)
  bool has_dense = false;
  int dksm = 0, dkglob = 0;
  DenseRec* d_dprog = nullptr;
  int* d_side_off = nullptr;
  int* d_side_slots = nullptr;
  long long* d_side_ready = nullptr;
  // device
  NodeRec* d_prog = nullptr;
  int* d_extra = nullptr;
  ChainDesc* d_chains = nullptr;
  NodeRec* d_members = nullptr;
  int* d_child_ptr = nullptr;
  int* d_child = nullptr;
  int* d_indeg = nullptr;
  int* d_lane = nullptr;
  long long* d_dur = nullptr;
  long long* d_gap = nullptr;
  long long* d_ready = nullptr;
  int* d_rank = nullptr;
  int* d_prio = nullptr;
  unsigned char* d_flags = nullptr;
  unsigned* d_group = nullptr;
  // breakdown geometry (chained graphs): per-lane static row sequences and
  // where each permutable chain sits in its lane
  bool bd_ok = false;
  bool gap_nonneg = true;
  int* d_bd_ptr = nullptr;
  int* d_bd_rows = nullptr;
  int* d_bd_lane_chain = nullptr;
  BdChain* d_bd_chains = nullptr;
  int* d_bd_member_rows = nullptr;
  // rows per lane of any graph (list-scheduled breakdown: per-scenario lane
  // sequences come from the dispatch order)
  int* d_bd_all_ptr = nullptr;
  // toposort_lanes_kernel requirements per row: (lane, emitted prefix length)
  bool topo_req = false;
  std::once_flag topo_once;
  TopoRec* d_topo_rec = nullptr;
  int* d_req_lane = nullptr;
  int* d_req_pos = nullptr;
};

namespace {

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// LSD radix sort of 64-bit keys, 16-bit digits; digits that are constant
// across all keys are skipped (edge keys are (u << 32 | v) with u, v < n).
static void radix_sort_u64(hvec<unsigned long long>& a) {
  const size_t n = a.size();
  if (n < 4096) {
    std::sort(a.begin(), a.end());
    return;
  }
  unsigned long long all_or = 0, all_and = ~0ull;
  for (unsigned long long x : a) { all_or |= x; all_and &= x; }
  hvec<unsigned long long> b(n);
  std::vector<size_t> cnt(65536);
  for (int sh = 0; sh < 64; sh += 16) {
    if ((((all_or ^ all_and) >> sh) & 0xffffull) == 0) continue;  // digit constant
    std::fill(cnt.begin(), cnt.end(), 0);
    for (unsigned long long x : a) ++cnt[(x >> sh) & 0xffff];
    size_t o = 0;
    for (size_t& c : cnt) { size_t t = c; c = o; o += t; }
    for (unsigned long long x : a) b[cnt[(x >> sh) & 0xffff]++] = x;
    a.swap(b);
  }
}

struct HostTimer {  // DDSIM_INGEST_TIMING=1: wall time of compile_graph's sections
  bool on = std::getenv("DDSIM_INGEST_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[compile_graph] %-13s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};

void ensure_programs(const ks_graph* g);

void compile_graph(const ks_graph_desc* d, ks_graph* g) {
  HostTimer gt;
  const int n = d->n_tasks;
  const int L = d->n_lanes;
  if (n < 0 || L < 0) fail(KS_ERR_INVALID, "negative sizes");
  if (n > 0 && (!d->duration || !d->gap || !d->lane || !d->id_rank))
    fail(KS_ERR_INVALID, "missing task arrays");
  for (int i = 0; i < n; ++i)
    if (d->lane[i] < 0 || d->lane[i] >= L) fail(KS_ERR_INVALID, "lane index out of range");
  const long long E = d->n_edges;
  for (long long k = 0; k < E; ++k) {
    const int u = d->edge_src[k], v = d->edge_dst[k];
    if (u < 0 || u >= n || v < 0 || v >= n) fail(KS_ERR_INVALID, "edge endpoint out of range");
  }
  g->n = n;
  g->L = L;

  // ---- chains (inserted-task table) ---------------------------------------
  const int NC = d->n_chains;
  hvec<int> chain_of(n, -1);
  hvec<int> ch_lane(NC, -1);
  for (int c = 0; c < NC; ++c) {
    for (int k = d->chain_ptr[c]; k < d->chain_ptr[c + 1]; ++k) {
      const int m = d->chain_member[k];
      if (m < 0 || m >= n || chain_of[m] >= 0) fail(KS_ERR_INVALID, "bad chain member");
      chain_of[m] = c;
      if (ch_lane[c] < 0) ch_lane[c] = d->lane[m];
      if (d->lane[m] != ch_lane[c]) fail(KS_ERR_INVALID, "chain members must share a lane");
    }
    if (d->chain_ptr[c + 1] <= d->chain_ptr[c]) fail(KS_ERR_INVALID, "empty chain");
  }

  gt.mark("chains");
  // ---- unique edges ----------------------------------------------------------
  // sorted unique (u << 32 | v): counting sort by u, then each (short) out list by v.
  // Threads own disjoint u ranges: each scans all edges but counts / scatters
  // only its own sources (no shared counters), then dedupes its range.
  hvec<unsigned long long> keys(E);
  {
    unsigned hw = std::thread::hardware_concurrency();
    int T = (int)std::max<long long>(1, std::min<long long>(hw ? hw : 1, E / (1 << 20)));
    T = std::min(T, std::max(1, n));
    hvec<int> ulo(T + 1);
    for (int t = 0; t <= T; ++t) ulo[t] = (int)((long long)n * t / T);
    hvec<long long> cnt((size_t)n + 1, 0);
    auto run = [&](auto fn) {
      if (T == 1) { fn(0); return; }
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t) th.emplace_back(fn, t);
      for (auto& x : th) x.join();
    };
    run([&](int t) {
      const int lo = ulo[t], hi = ulo[t + 1];
      for (long long k = 0; k < E; ++k) {
        const int u = d->edge_src[k];
        if (u >= lo && u < hi) cnt[(size_t)u + 1]++;
      }
    });
    for (int i = 0; i < n; ++i) cnt[(size_t)i + 1] += cnt[(size_t)i];
    hvec<long long> kept(T, 0);
    run([&](int t) {
      const int lo = ulo[t], hi = ulo[t + 1];
      hvec<long long> fill(cnt.begin() + lo, cnt.begin() + hi);
      for (long long k = 0; k < E; ++k) {
        const int u = d->edge_src[k];
        if (u >= lo && u < hi)
          keys[(size_t)fill[(size_t)(u - lo)]++] =
              ((unsigned long long)(unsigned)u << 32) | (unsigned)d->edge_dst[k];
      }
      long long o = cnt[(size_t)lo];  // dedupe in place within the range
      for (int u = lo; u < hi; ++u) {
        auto b = keys.begin() + cnt[(size_t)u], e = keys.begin() + cnt[(size_t)u + 1];
        if (e - b > 1) std::sort(b, e);
        for (auto it = b; it != e; ++it)
          if (it == b || *it != *(it - 1)) keys[(size_t)o++] = *it;
      }
      kept[t] = o - cnt[(size_t)lo];
    });
    size_t o = (size_t)kept[0];  // compact the ranges (range 0 is in place)
    for (int t = 1; t < T; ++t) {
      const size_t from = (size_t)cnt[(size_t)ulo[t]];
      if (from != o) std::memmove(&keys[o], &keys[from], (size_t)kept[t] * sizeof(keys[0]));
      o += (size_t)kept[t];
    }
    keys.resize(o);
  }
  g->n_edges_unique = (int)keys.size();
  hvec<int> optr(n + 1, 0);  // out-edge ranges of the sorted unique keys
  for (unsigned long long k : keys) optr[(k >> 32) + 1]++;
  for (int i = 0; i < n; ++i) optr[i + 1] += optr[i];
  auto has_edge = [&](int u, int v) {
    const unsigned long long k = ((unsigned long long)(unsigned)u << 32) | (unsigned)v;
    return std::binary_search(keys.begin() + optr[u], keys.begin() + optr[u + 1], k);
  };

  gt.mark("unique-edges");
  // ---- lane chaining check ---------------------------------------------------
  bool chained = d->lane_order_ptr != nullptr;
  hvec<int> lane_succ(n, -1);
  if (chained) {
    // every position of the lane lists independently: a task passes the lane
    // test only in its own lane's list, so `seen` is written per lane (the
    // exchange catches a task listed twice in that list)
    for (int l = 0; l < L && chained; ++l)
      if (d->lane_order_ptr[l] > d->lane_order_ptr[l + 1] || d->lane_order_ptr[l] < 0) chained = false;
    const long long K0 = chained && L > 0 ? d->lane_order_ptr[0] : 0;
    const long long K = chained && L > 0 ? d->lane_order_ptr[L] : 0;
    hvec<char> seen(n, 0);
    hvec<int> lane_at;  // lane of each list position
    if (K > K0) {
      lane_at.resize(K - K0);
      for (int l = 0; l < L; ++l)
        std::fill(lane_at.begin() + (d->lane_order_ptr[l] - K0),
                  lane_at.begin() + (d->lane_order_ptr[l + 1] - K0), l);
    }
    std::atomic<bool> ok{chained};
    host_parallel_for(K - K0, [&](long long b, long long e) {
      bool good = true;
      for (long long k = K0 + b; k < K0 + e && good; ++k) {
        const int l = lane_at[k - K0];
        const int t = d->lane_order[k];
        if (t < 0 || t >= n || d->lane[t] != l || chain_of[t] >= 0 ||
            __atomic_exchange_n(&seen[t], (char)1, __ATOMIC_RELAXED)) {
          good = false;
          break;
        }
        if (k > d->lane_order_ptr[l]) {
          const int prev = d->lane_order[k - 1];
          if (prev < 0 || prev >= n || !has_edge(prev, t)) {
            good = false;
            break;
          }
          lane_succ[prev] = t;
        }
      }
      if (!good) ok.store(false);
    });
    chained = ok.load();
    for (int i = 0; i < n && chained; ++i)
      if (!seen[i] && chain_of[i] < 0) chained = false;
  }
  if (NC > 0 && !chained)
    fail(KS_ERR_UNSUPPORTED, "permutable chains need an otherwise lane-chained graph");
  g->chained = chained;
  g->n_chains = NC;

  gt.mark("chain-check");
  // ---- unique preds per task (for records) -----------------------------------
  // transpose of the unique edges: parallel atomic count / scatter, then each
  // (short) list sorted -- the same ascending-source lists a sequential
  // scatter of the (u, v)-sorted keys gives
  hvec<int> pptr(n + 1, 0), padj(keys.size());
  const long long KE = (long long)keys.size();
  host_parallel_for(KE, [&](long long b, long long e) {
    for (long long q = b; q < e; ++q) __atomic_fetch_add(&pptr[(keys[q] & 0xffffffffu) + 1], 1, __ATOMIC_RELAXED);
  });
  for (int i = 0; i < n; ++i) pptr[i + 1] += pptr[i];
  {
    hvec<int> fill(pptr.begin(), pptr.end() - 1);
    host_parallel_for(KE, [&](long long b, long long e) {
      for (long long q = b; q < e; ++q) {
        const int v = (int)(keys[q] & 0xffffffffu);
        padj[__atomic_fetch_add(&fill[v], 1, __ATOMIC_RELAXED)] = (int)(keys[q] >> 32);
      }
    });
    host_parallel_for(n, [&](long long b, long long e) {
      for (long long v = b; v < e; ++v)
        if (pptr[v + 1] - pptr[v] > 1) std::sort(padj.begin() + pptr[v], padj.begin() + pptr[v + 1]);
    });
  }
  hvec<int> tail_of(n, -1);  // task -> chain whose tail it is
  for (int c = 0; c < NC; ++c) {
    const int t = d->chain_tail ? d->chain_tail[c] : -1;
    if (t >= 0) tail_of[t] = c;
  }

  gt.mark("preds");
  // ---- contracted graph (chain -> one node) ---------------------------------
  const int NN = n + NC;
  auto X = [&](int t) { return chain_of[t] >= 0 ? n + chain_of[t] : t; };
  hvec<unsigned long long> ckeys;  // without chains the contracted graph is `keys`
  if (NC > 0) ckeys.reserve(keys.size() + 2 * NC);
  for (size_t q = 0; NC > 0 && q < keys.size(); ++q) {
    const unsigned long long k = keys[q];
    const int u = (int)(k >> 32), v = (int)(k & 0xffffffffu);
    const int xu = X(u), xv = X(v);
    if (xu == xv) {
      if (u == v) {
        ckeys.push_back(((unsigned long long)xu << 32) | (unsigned)xv);  // self loop: cycle
        continue;
      }
      fail(KS_ERR_INVALID, "edge between members of one chain");
    }
    ckeys.push_back(((unsigned long long)xu << 32) | (unsigned)xv);
  }
  for (int c = 0; c < NC; ++c) {
    const int h = d->chain_head ? d->chain_head[c] : -1;
    const int t = d->chain_tail ? d->chain_tail[c] : -1;
    if (h >= 0) {
      if (h >= n || chain_of[h] >= 0 || d->lane[h] != ch_lane[c])
        fail(KS_ERR_INVALID, "bad chain head");
      ckeys.push_back(((unsigned long long)h << 32) | (unsigned)(n + c));
    }
    if (t >= 0) {
      if (t >= n || chain_of[t] >= 0 || d->lane[t] != ch_lane[c])
        fail(KS_ERR_INVALID, "bad chain tail");
      ckeys.push_back(((unsigned long long)(n + c) << 32) | (unsigned)t);
    }
  }
  if (NC > 0) {
    radix_sort_u64(ckeys);
    ckeys.erase(std::unique(ckeys.begin(), ckeys.end()), ckeys.end());
  }
  const hvec<unsigned long long>& CK = NC > 0 ? ckeys : keys;  // sorted by (u, v)
  hvec<int> cptr, cadj(CK.size()), cindeg;
  if (NC == 0) {  // the contracted graph is the unique-edge graph: reuse its ranges
    cptr.assign(optr.begin(), optr.end());
    cindeg.resize(NN);
    host_parallel_for(NN, [&](long long b, long long e) {
      for (long long i = b; i < e; ++i) cindeg[i] = pptr[i + 1] - pptr[i];
    });
    host_parallel_for((long long)CK.size(), [&](long long b, long long e) {
      for (long long q = b; q < e; ++q) cadj[q] = (int)(CK[q] & 0xffffffffu);
    });
  } else {
    cptr.assign(NN + 1, 0);
    cindeg.assign(NN, 0);
    for (size_t q = 0; q < CK.size(); ++q) {
      const unsigned long long k = CK[q];
      cptr[(k >> 32) + 1]++;
      cindeg[k & 0xffffffffu]++;
      cadj[q] = (int)(k & 0xffffffffu);
    }
    for (int i = 0; i < NN; ++i) cptr[i + 1] += cptr[i];
  }
  // rank of contracted nodes (tie-break for the initial stack)
  hvec<int> crank(NN);
  for (int i = 0; i < n; ++i) crank[i] = d->id_rank[i];
  for (int c = 0; c < NC; ++c) {
    int r = INT32_MAX;
    for (int k = d->chain_ptr[c]; k < d->chain_ptr[c + 1]; ++k)
      r = std::min(r, d->id_rank[d->chain_member[k]]);
    crank[n + c] = r;
  }
  auto clane = [&](int x) { return x < n ? d->lane[x] : ch_lane[x - n]; };

  gt.mark("contract");
  // ---- depth-first Kahn (LIFO frontier) --------------------------------------
  hvec<int> corder;
  corder.reserve(NN);
  {
    hvec<int> indeg = cindeg;
    hvec<int> init;
    for (int i = 0; i < NN; ++i)  // chain members are represented by their chain node
      if (indeg[i] == 0 && !(i < n && chain_of[i] >= 0)) init.push_back(i);
    std::sort(init.begin(), init.end(), [&](int a, int b) { return crank[a] > crank[b]; });
    hvec<int> stack(init);
    hvec<int> cross;
    while (!stack.empty()) {
      const int x = stack.back();
      stack.pop_back();
      corder.push_back(x);
      cross.clear();
      int same = -1;
      for (int k = cptr[x]; k < cptr[x + 1]; ++k) {
        const int y = cadj[k];
        if (--indeg[y] == 0) {
          if (same < 0 && clane(y) == clane(x))
            same = y;
          else
            cross.push_back(y);
        }
      }
      if (same >= 0) stack.push_back(same);
      std::sort(cross.begin(), cross.end(), [&](int a, int b) { return crank[a] > crank[b]; });
      for (int y : cross) stack.push_back(y);
    }
  }
  const int R = (int)corder.size();  // records

  gt.mark("toposort");
  // ---- frozen rows ----------------------------------------------------------
  g->order.clear();
  g->order.reserve(n);
  hvec<int> rec_first_row(R);
  hvec<char> placed(n, 0);
  for (int i = 0; i < R; ++i) {
    const int x = corder[i];
    rec_first_row[i] = (int)g->order.size();
    if (x < n) {
      g->order.push_back(x);
      placed[x] = 1;
    } else {
      const int c = x - n;
      for (int k = d->chain_ptr[c]; k < d->chain_ptr[c + 1]; ++k) {
        g->order.push_back(d->chain_member[k]);
        placed[d->chain_member[k]] = 1;
      }
    }
  }
  g->n_ordered = (int)g->order.size();
  {
    hvec<int> rest;
    for (int i = 0; i < n; ++i)
      if (!placed[i]) rest.push_back(i);
    std::sort(rest.begin(), rest.end(),
              [&](int a, int b) { return d->id_rank[a] < d->id_rank[b]; });
    for (int t : rest) g->order.push_back(t);
  }
  g->row_of.resize(n);
  g->rank_row.resize(n);
  host_parallel_for(n, [&](long long b, long long e) {  // order is a permutation
    for (int r = (int)b; r < (int)e; ++r) {
      g->row_of[g->order[r]] = r;
      g->rank_row[r] = d->id_rank[g->order[r]];
    }
  });
  g->rows_are_records = (NC == 0);

  gt.mark("rows");
  // ---- list-scheduler arrays and per-row device arrays (eager: every path) --
  {

  // ---- list-scheduler arrays (frozen rows, multiset edges) -------------------
  hvec<int> ch_ptr(n + 1, 0), ch_adj(E), indeg(n, 0);
  hvec<int> lane_r(n), rank_r(n), prio_r(n);
  hvec<long long> dur_r(n), gap_r(n), ready_r(n);
  hvec<unsigned char> flags_r(n);
  hvec<unsigned> group_r(n);
  hvec<int> esr(E), edr(E);  // edge endpoints as frozen rows
  host_parallel_for(E, [&](long long b, long long e) {
    for (long long k = b; k < e; ++k) {
      esr[k] = g->row_of[d->edge_src[k]];
      edr[k] = g->row_of[d->edge_dst[k]];
    }
  });
  // multiset CSR by parallel atomic count / scatter; each child list is then
  // sorted so the layout is deterministic (the schedulers pick by key, not by
  // list position)
  host_parallel_for(E, [&](long long b, long long e) {
    for (long long k = b; k < e; ++k) {
      __atomic_fetch_add(&ch_ptr[esr[k] + 1], 1, __ATOMIC_RELAXED);
      __atomic_fetch_add(&indeg[edr[k]], 1, __ATOMIC_RELAXED);
    }
  });
  for (int i = 0; i < n; ++i) ch_ptr[i + 1] += ch_ptr[i];
  {
    hvec<int> fill(ch_ptr.begin(), ch_ptr.end() - 1);
    host_parallel_for(E, [&](long long b, long long e) {
      for (long long k = b; k < e; ++k) ch_adj[__atomic_fetch_add(&fill[esr[k]], 1, __ATOMIC_RELAXED)] = edr[k];
    });
    host_parallel_for(n, [&](long long b, long long e) {
      for (long long r = b; r < e; ++r)
        if (ch_ptr[r + 1] - ch_ptr[r] > 1) std::sort(ch_adj.begin() + ch_ptr[r], ch_adj.begin() + ch_ptr[r + 1]);
    });
  }
  host_parallel_for(n, [&](long long b, long long e) {
  for (int r = (int)b; r < (int)e; ++r) {
    const int t = g->order[r];
    lane_r[r] = d->lane[t];
    rank_r[r] = d->id_rank[t];
    prio_r[r] = d->priority ? d->priority[t] : 0;
    dur_r[r] = d->duration[t];
    gap_r[r] = d->gap[t];
    ready_r[r] = d->ready_time ? d->ready_time[t] : 0;
    flags_r[r] = d->flags ? d->flags[t] : 0;
    group_r[r] = d->group ? d->group[t] : 0u;
  }
  });

  g->d_child_ptr = dev_upload(ch_ptr);
  g->d_child = dev_upload(ch_adj);
  g->d_indeg = dev_upload(indeg);
  g->d_lane = dev_upload(lane_r);
  g->d_dur = dev_upload(dur_r);
  g->d_gap = dev_upload(gap_r);
  g->d_ready = dev_upload(ready_r);
  g->d_rank = dev_upload(rank_r);
  g->d_prio = dev_upload(prio_r);
  g->d_flags = dev_upload(flags_r);
  g->d_group = dev_upload(group_r);
  
  }
  gt.mark("row arrays");
  // ---- what the program builders read, kept for build_programs -----------------
  {
    auto st = std::make_unique<LazyPrograms>();
    LazyPrograms& S = *st;
    S.n = n;
    S.L = L;
    S.E = E;
    S.NC = NC;
    S.R = R;
    S.chained = chained;
    auto own = [&](auto& dst, const auto* src, size_t cnt) {
      if (!src) return;
      dst.resize(cnt);
      host_parallel_for((long long)cnt, [&](long long b, long long e) {
        std::copy(src + b, src + e, dst.begin() + b);
      });
    };
    own(S.duration, d->duration, (size_t)n);
    own(S.gap, d->gap, (size_t)n);
    bool any_ready = false;
    for (int i = 0; i < n && d->ready_time && !any_ready; ++i) any_ready = d->ready_time[i] != 0;
    if (any_ready) own(S.ready, d->ready_time, (size_t)n);
    own(S.lane, d->lane, (size_t)n);
    if (d->group) own(S.group, d->group, (size_t)n);
    if (d->lane_order_ptr) {
      own(S.lane_order_ptr, d->lane_order_ptr, (size_t)L + 1);
      const long long K0 = L > 0 ? d->lane_order_ptr[0] : 0, K = L > 0 ? d->lane_order_ptr[L] : 0;
      S.lane_order.resize((size_t)std::max(0LL, K));
      if (K > K0) std::copy(d->lane_order + K0, d->lane_order + K, S.lane_order.begin() + K0);
    }
    if (NC > 0) {
      own(S.chain_ptr, d->chain_ptr, (size_t)NC + 1);
      own(S.chain_member, d->chain_member, (size_t)S.chain_ptr[NC]);
      if (d->chain_head) own(S.chain_head, d->chain_head, (size_t)NC);
      if (d->chain_tail) own(S.chain_tail, d->chain_tail, (size_t)NC);
    }
    memset(&S.desc, 0, sizeof(S.desc));
    S.desc.n_tasks = n;
    S.desc.n_lanes = L;
    S.desc.duration = S.duration.data();
    S.desc.gap = S.gap.data();
    S.desc.ready_time = S.ready.empty() ? nullptr : S.ready.data();
    S.desc.lane = S.lane.data();
    S.desc.group = S.group.empty() ? nullptr : S.group.data();
    S.desc.lane_order_ptr = S.lane_order_ptr.empty() ? nullptr : S.lane_order_ptr.data();
    S.desc.lane_order = S.lane_order.data();
    S.desc.n_chains = NC;
    S.desc.chain_ptr = S.chain_ptr.data();
    S.desc.chain_member = S.chain_member.data();
    S.desc.chain_head = S.chain_head.empty() ? nullptr : S.chain_head.data();
    S.desc.chain_tail = S.chain_tail.empty() ? nullptr : S.chain_tail.data();
    S.keys = std::move(keys);
    S.optr = std::move(optr);
    S.pptr = std::move(pptr);
    S.padj = std::move(padj);
    S.corder = std::move(corder);
    S.rec_first_row = std::move(rec_first_row);
    S.ch_lane = std::move(ch_lane);
    S.tail_of = std::move(tail_of);
    S.cptr = std::move(cptr);
    S.cadj = std::move(cadj);
    g->lazy = std::move(st);
  }
  gt.mark("keep");
  if (getenv("DDSIM_EAGER_PROGRAMS") != nullptr) ensure_programs(g);
}

// The kernel programs of a frozen graph -- general records (maxplus.cu),
// dense register-forwarding program (maxplus_dense.cu), lane-register program
// (maxplus_lanes.cu), breakdown lane sequences -- are built on the first call
// that needs them (ensure_programs), from the graph compile_graph kept.
void build_programs(ks_graph* g, LazyPrograms& S) {
  HostTimer gt;
  const ks_graph_desc* d = &S.desc;
  const int n = S.n, L = S.L, NC = S.NC, R = S.R;
  const long long E = S.E;
  (void)E;
  const bool chained = S.chained;
  const int NN = n + NC;
  (void)NN;
  auto& keys = S.keys;
  auto& optr = S.optr;
  auto& pptr = S.pptr;
  auto& padj = S.padj;
  auto& corder = S.corder;
  auto& rec_first_row = S.rec_first_row;
  auto& ch_lane = S.ch_lane;
  auto& tail_of = S.tail_of;
  auto& cptr = S.cptr;
  auto& cadj = S.cadj;
  {  // bounds the expanded duration matrix (int32 when it fits, simulate_impl)
    long long mx = 0;
    for (int t = 0; t < n; ++t) {
      const long long v = d->duration[t];
      mx = std::max(mx, v == LLONG_MIN ? LLONG_MAX : (v < 0 ? -v : v));
    }
    g->dur_abs_max = mx;
  }
  // ---- levels ------------------------------------------------------------------
  // Without chains: pull form in record space -- level(i) = 1 + max over the
  // record's predecessors, which are recent records (cache-resident); the
  // record-space predecessor lists are built in parallel and reused by the
  // records builder. With chains: push form over the contracted graph.
  hvec<int> rp_ptr, rp;  // record-space predecessors (NC == 0)
  if (NC == 0) {
    hvec<int> rec_of(n, -1);
    host_parallel_for(R, [&](long long b, long long e) {
      for (int i = (int)b; i < (int)e; ++i) rec_of[corder[i]] = i;
    });
    rp_ptr.assign(R + 1, 0);
    host_parallel_for(R, [&](long long b, long long e) {
      for (int i = (int)b; i < (int)e; ++i) rp_ptr[i + 1] = pptr[corder[i] + 1] - pptr[corder[i]];
    });
    for (int i = 0; i < R; ++i) rp_ptr[i + 1] += rp_ptr[i];
    rp.resize(rp_ptr[R]);
    host_parallel_for(R, [&](long long b, long long e) {
      for (int i = (int)b; i < (int)e; ++i) {
        const int x = corder[i];
        for (int k = pptr[x], o = rp_ptr[i]; k < pptr[x + 1]; ++k, ++o) rp[o] = rec_of[padj[k]];
      }
    });
    hvec<int> lv(R);
    int maxl = 0;
    for (int i = 0; i < R; ++i) {
      int m = 0;
      for (int q = rp_ptr[i]; q < rp_ptr[i + 1]; ++q) m = std::max(m, lv[rp[q]]);
      lv[i] = m + 1;
      maxl = std::max(maxl, m + 1);
    }
    g->n_levels = maxl;
    g->level.assign(n, -1);
    host_parallel_for(R, [&](long long b, long long e) {  // rows are records without chains
      for (int i = (int)b; i < (int)e; ++i) g->level[i] = lv[i] - 1;
    });
  } else {
    hvec<int> clevel(NN, 0);
    int maxl = 0;
    for (int i = 0; i < R; ++i) {
      const int x = corder[i];
      const int lv = clevel[x] + 1;
      clevel[x] = lv;
      maxl = std::max(maxl, lv);
      for (int k = cptr[x]; k < cptr[x + 1]; ++k) clevel[cadj[k]] = std::max(clevel[cadj[k]], lv);
    }
    g->n_levels = maxl;
    g->level.assign(n, -1);
    for (int i = 0; i < R; ++i) {
      const int x = corder[i];
      if (x < n)
        g->level[rec_first_row[i]] = clevel[x] - 1;
      else
        for (int k = 0; k < d->chain_ptr[x - n + 1] - d->chain_ptr[x - n]; ++k)
          g->level[rec_first_row[i] + k] = clevel[x] - 1;
    }
  }

  gt.mark("levels");
  // ---- the four builders below (general records, dense program, lane program,
  // list-scheduler arrays) read only the shared graph above: run concurrently
  hvec<NodeRec> members;
  hvec<ChainDesc> chains(NC);
  bool nonneg = true;
  for (int i = 0; i < n && nonneg; ++i)
    if (d->gap[i] < 0 || (d->ready_time && d->ready_time[i] < 0)) nonneg = false;
  // (each builder allocates its own arrays: first-touch page faults then run
  // on the builders' threads instead of serially here)
  ConcurrentSections sect(g->device);
  sect.run("records", [&] {
  HostTimer rt_;
  uvec<NodeRec> prog(R);
  hvec<int> extra;
  // ---- value live ranges -------------------------------------------------------
  // values: task t (0..n-1) -> rel(t); chain tail value n + c.
  const int NV = n + NC;
  hvec<int> rec_of_task(n, -1), rec_of_chain(NC, -1);
  host_parallel_for(R, [&](long long b, long long e) {  // corder: distinct nodes
    for (int i = (int)b; i < (int)e; ++i) {
      const int x = corder[i];
      if (x < n)
        rec_of_task[x] = i;
      else
        rec_of_chain[x - n] = i;
    }
  });
  hvec<int> last_use;
  // inputs of each record (flat CSR: rin_ptr / rin)
  hvec<int> rin_ptr, rin;
  if (NC > 0) {
    last_use.assign(NV, -1);
    rin_ptr.assign(R + 1, 0);
    rin.reserve(keys.size() + 2 * (size_t)NC);
  }
  hvec<int> in;
  for (int i = 0; i < R && NC > 0; ++i) {
    const int x = corder[i];
    in.clear();
    auto add_task_preds = [&](int t) {
      for (int k = pptr[t]; k < pptr[t + 1]; ++k) in.push_back(padj[k]);
    };
    if (x < n) {
      add_task_preds(x);
      if (tail_of[x] >= 0) in.push_back(n + tail_of[x]);
    } else {
      const int c = x - n;
      for (int k = d->chain_ptr[c]; k < d->chain_ptr[c + 1]; ++k) add_task_preds(d->chain_member[k]);
      const int h = d->chain_head ? d->chain_head[c] : -1;
      if (h >= 0) in.push_back(h);
    }
    if (in.size() > 1) {
      std::sort(in.begin(), in.end());
      in.erase(std::unique(in.begin(), in.end()), in.end());
    }
    for (int v : in) last_use[v] = std::max(last_use[v], i);
    rin.insert(rin.end(), in.begin(), in.end());
    rin_ptr[i + 1] = (int)rin.size();
  }

  rt_.mark(" rec:last-use");
  // ---- slot allocation (linear scan, allocate-then-free) ----------------------
  hvec<int> slot(NV, -1);
  hvec<char> in_glob(NV, 0);
  MinFreeSet free_s, free_g;
  int next_s = 0, next_g = 0;
  // value v defined by record i, last read by record lu
  auto alloc_at = [&](int lu, int i, int& sl, char& gl) {
    if (lu < 0) return;  // nobody reads it
    const bool short_range = (lu - i) <= kShortRange;
    if (short_range) {
      if (!free_s.empty()) {
        sl = free_s.top();
        free_s.pop();
        return;
      }
      if (next_s < kSmemSlotsMax) {
        sl = next_s++;
        return;
      }
    }
    gl = 1;
    if (!free_g.empty()) {
      sl = free_g.top();
      free_g.pop();
    } else {
      sl = next_g++;
    }
  };
  if (NC == 0) {
    // Record space: without chains every record defines exactly one value, so
    // the scan reads its arrays sequentially and the predecessors it releases
    // are recent records (cache-resident); last use and the record-space
    // predecessor lists are built in parallel. Same scan, same slots.
    hvec<int> lu_r(R);
    host_parallel_for(R, [&](long long b, long long e) {
      for (int i = (int)b; i < (int)e; ++i) {
        const int x = corder[i];
        int m = -1;
        for (int k = optr[x]; k < optr[x + 1]; ++k)
          m = std::max(m, rec_of_task[(int)(keys[k] & 0xffffffffu)]);
        lu_r[i] = m;
      }
    });
    const hvec<int>& rptr = rp_ptr;  // record-space predecessors from the levels pass
    rt_.mark(" rec:rspace");
    hvec<int> slot_r(R, -1);
    hvec<char> glob_r(R, 0);
    for (int i = 0; i < R; ++i) {
      alloc_at(lu_r[i], i, slot_r[i], glob_r[i]);
      for (int q = rptr[i]; q < rptr[i + 1]; ++q)
        if (const int j = rp[q]; lu_r[j] == i && slot_r[j] >= 0) (glob_r[j] ? free_g : free_s).push(slot_r[j]);
    }
    rt_.mark(" rec:scan");
    host_parallel_for(R, [&](long long b, long long e) {
      for (int i = (int)b; i < (int)e; ++i) {
        slot[corder[i]] = slot_r[i];
        in_glob[corder[i]] = glob_r[i];
      }
    });
  }
  for (int i = 0; i < R && NC > 0; ++i) {
    const int x = corder[i];
    if (x < n) {
      alloc_at(last_use[x], i, slot[x], in_glob[x]);
    } else {
      const int c = x - n;
      for (int k = d->chain_ptr[c]; k < d->chain_ptr[c + 1]; ++k) {
        const int m = d->chain_member[k];
        alloc_at(last_use[m], i, slot[m], in_glob[m]);
      }
      if (d->chain_tail && d->chain_tail[c] >= 0) alloc_at(last_use[n + c], i, slot[n + c], in_glob[n + c]);
    }
    for (int q = rin_ptr[i]; q < rin_ptr[i + 1]; ++q)
      if (const int v = rin[q]; last_use[v] == i && slot[v] >= 0) (in_glob[v] ? free_g : free_s).push(slot[v]);
  }
  rt_.mark(" rec:slots");
  g->ksm = next_s;
  g->kglob = next_g;
  g->n_slots = next_s + next_g;
  auto final_slot = [&](int v) { return slot[v] < 0 ? -1 : (in_glob[v] ? g->ksm + slot[v] : slot[v]); };

  // ---- records -----------------------------------------------------------------
  auto make_task_rec = [&](int t, const hvec<int>& preds) {
    NodeRec r;
    memset(&r, 0, sizeof(r));
    r.dur = d->duration[t];
    r.gap = d->gap[t];
    r.ready = d->ready_time ? d->ready_time[t] : 0;
    r.out_slot = final_slot(t);
    const size_t np = preds.size();
    r.pred0 = np > 0 ? final_slot(preds[0]) : -1;
    r.pred1 = np > 1 ? final_slot(preds[1]) : -1;
    r.extra_off = 0;
    r.nextra = np > 2 ? (int)np - 2 : 0;
    if (r.nextra) {
      r.extra_off = (int)extra.size();
      for (size_t k = 2; k < np; ++k) extra.push_back(final_slot(preds[k]));
    }
    r.group = d->group ? d->group[t] : 0u;
    r.ovr_row = -1;
    r.lane = d->lane[t];
    r.row = g->row_of[t];
    r.kind = 0;
    return r;
  };
  int perm_off = 0;
  hvec<int> preds;
  if (NC == 0) {  // no chains: records are independent -> fill them in parallel
    hvec<int> eoff(R + 1, 0);
    for (int i = 0; i < R; ++i) {
      const int x = corder[i];
      eoff[i + 1] = eoff[i] + std::max(0, pptr[x + 1] - pptr[x] - 2);
    }
    extra.resize(eoff[R]);
    host_parallel_for(R, [&](long long b, long long e) {
      for (int i = (int)b; i < (int)e; ++i) {
        const int t = corder[i];
        NodeRec r;
        memset(&r, 0, sizeof(r));
        r.dur = d->duration[t];
        r.gap = d->gap[t];
        r.ready = d->ready_time ? d->ready_time[t] : 0;
        r.out_slot = final_slot(t);
        const int p0 = pptr[t], np = pptr[t + 1] - p0;
        r.pred0 = np > 0 ? final_slot(padj[p0]) : -1;
        r.pred1 = np > 1 ? final_slot(padj[p0 + 1]) : -1;
        r.nextra = np > 2 ? np - 2 : 0;
        r.extra_off = r.nextra ? eoff[i] : 0;
        for (int k = 2; k < np; ++k) extra[eoff[i] + k - 2] = final_slot(padj[p0 + k]);
        r.group = d->group ? d->group[t] : 0u;
        r.ovr_row = -1;
        r.lane = d->lane[t];
        r.row = g->row_of[t];
        r.kind = 0;
        prog[i] = r;
      }
    });
  }
  for (int i = 0; i < R && NC > 0; ++i) {
    const int x = corder[i];
    if (x < n) {
      preds.clear();
      for (int k = pptr[x]; k < pptr[x + 1]; ++k) preds.push_back(padj[k]);
      if (tail_of[x] >= 0) preds.push_back(n + tail_of[x]);
      prog[i] = make_task_rec(x, preds);
    } else {
      const int c = x - n;
      NodeRec r;
      memset(&r, 0, sizeof(r));
      r.kind = 1;
      r.row = c;
      r.out_slot = r.pred0 = r.pred1 = -1;
      r.ovr_row = -1;
      prog[i] = r;
      ChainDesc& ch = chains[c];
      ch.first_row = rec_first_row[i];
      ch.B = d->chain_ptr[c + 1] - d->chain_ptr[c];
      const int h = d->chain_head ? d->chain_head[c] : -1;
      ch.head_slot = h >= 0 ? final_slot(h) : -1;
      ch.tail_slot = (d->chain_tail && d->chain_tail[c] >= 0) ? final_slot(n + c) : -1;
      ch.member_off = (int)members.size();
      ch.perm_off = perm_off;
      ch.lane = ch_lane[c];
      ch.pad = 0;
      perm_off += ch.B;
      for (int k = d->chain_ptr[c]; k < d->chain_ptr[c + 1]; ++k) {
        const int m = d->chain_member[k];
        preds.clear();
        for (int q = pptr[m]; q < pptr[m + 1]; ++q) preds.push_back(padj[q]);
        members.push_back(make_task_rec(m, preds));
      }
    }
  }
  rt_.mark(" rec:fill");
  g->perm_ld = perm_off;
  g->n_rec = R;
  g->d_prog = dev_upload(prog);  // uploads overlap the other builders
  g->d_extra = dev_upload(extra);
  g->d_chains = dev_upload(chains);
  g->d_members = dev_upload(members);

  });
  sect.run("dense-prog", [&] {
  // ---- dense program: register forwarding for the two previous records ----
  if (NC == 0 && L <= 127 && nonneg) {
    hvec<int> pos(n, -1);
    host_parallel_for(R, [&](long long b, long long e) {
      for (int i = (int)b; i < (int)e; ++i) pos[corder[i]] = i;
    });
    hvec<int> far_use(n, -1);  // last consumer more than 2 records later (per source)
    host_parallel_for(n, [&](long long b, long long e) {
      for (int u = (int)b; u < (int)e; ++u) {
        if (pos[u] < 0) continue;
        int m = -1;
        for (int k = optr[u]; k < optr[u + 1]; ++k) {
          const int i = pos[(int)(keys[k] & 0xffffffffu)];
          if (i - pos[u] > 2) m = std::max(m, i);
        }
        far_use[u] = m;
      }
    });
    hvec<int> dslot(n, -1);
    hvec<char> dglob(n, 0);
    MinFreeSet fs, fg;
    int ns = 0, ngl = 0;
    hvec<int> fa_ptr(R + 1, 0), fa;  // values freed after record i (CSR)
    for (int i = 0; i < R; ++i)
      if (far_use[corder[i]] >= 0) fa_ptr[far_use[corder[i]] + 1]++;
    for (int i = 0; i < R; ++i) fa_ptr[i + 1] += fa_ptr[i];
    fa.resize(fa_ptr[R]);
    {
      hvec<int> fill(fa_ptr.begin(), fa_ptr.end() - 1);
      for (int i = 0; i < R; ++i)
        if (far_use[corder[i]] >= 0) fa[fill[far_use[corder[i]]]++] = corder[i];
    }
    for (int i = 0; i < R; ++i) {
      const int v = corder[i];
      if (far_use[v] >= 0) {
        const bool shrt = far_use[v] - i <= kShortRange;
        if (shrt && !fs.empty()) {
          dslot[v] = fs.top();
          fs.pop();
        } else if (shrt && ns < kSmemSlotsMax) {
          dslot[v] = ns++;
        } else {
          dglob[v] = 1;
          if (!fg.empty()) {
            dslot[v] = fg.top();
            fg.pop();
          } else {
            dslot[v] = ngl++;
          }
        }
      }
      for (int q = fa_ptr[i]; q < fa_ptr[i + 1]; ++q) (dglob[fa[q]] ? fg : fs).push(dslot[fa[q]]);
    }
    g->dksm = ns;
    g->dkglob = ngl;
    hvec<int> lane_last(L, -1);
    for (int i = 0; i < R; ++i) lane_last[d->lane[corder[i]]] = i;
    uvec<DenseRec> dprog(R);
    hvec<int> side_off(R + 1, 0);
    hvec<int> side_slots;
    hvec<long long> side_ready;
    bool ok = ns + ngl < 32000;
    // records are independent given the slots: encode in parallel, side lists
    // by count / prefix / fill
    auto encode = [&](int i, DenseRec* out, int* side) {
      const int v = corder[i];
      DenseRec r;
      memset(&r, 0, sizeof(r));
      r.gap = d->gap[v];
      r.lane = (unsigned char)(d->lane[v] | (r.gap != 0 ? DLANE_GAP : 0));
      unsigned op = 0;
      if (!chained || lane_last[d->lane[v]] == i) op |= DOP_MS;
      if (dslot[v] >= 0) {
        op |= dglob[v] ? DOP_OUT_GLOBAL : DOP_OUT_SMEM;
        r.out = (short)(dglob[v] ? ns + dslot[v] : dslot[v]);
      }
      int nsm_pred = 0, nside = 0;
      for (int k = pptr[v]; k < pptr[v + 1]; ++k) {
        const int u = padj[k];
        const int dist = i - pos[u];
        if (dist == 1) {
          op |= DOP_PREV;
        } else if (dist == 2) {
          op |= DOP_PREV2;
        } else if (!dglob[u] && nsm_pred == 0) {
          op |= DOP_S0;
          r.s0 = (short)dslot[u];
          ++nsm_pred;
        } else if (!dglob[u] && nsm_pred == 1) {
          op |= DOP_S1;
          r.s1 = (short)dslot[u];
          ++nsm_pred;
        } else {
          op |= DOP_SLOW;
          if (side) side[nside] = dglob[u] ? ns + dslot[u] : dslot[u];
          ++nside;
        }
      }
      if (d->ready_time && d->ready_time[v] != 0) op |= DOP_SLOW;
      r.op = (unsigned char)op;
      if (out) *out = r;
      return nside;
    };
    if (ok) {
      host_parallel_for(R, [&](long long b, long long e) {
        for (int i = (int)b; i < (int)e; ++i) side_off[i + 1] = encode(i, nullptr, nullptr);
      });
      for (int i = 0; i < R; ++i) side_off[i + 1] += side_off[i];
      side_slots.resize(side_off[R]);
      host_parallel_for(R, [&](long long b, long long e) {
        for (int i = (int)b; i < (int)e; ++i) encode(i, &dprog[i], side_slots.data() + side_off[i]);
      });
    }
    bool any_ready = false;
    for (int i = 0; i < R && ok && d->ready_time && !any_ready; ++i)
      any_ready = d->ready_time[corder[i]] != 0;
    if (ok) {
      if (any_ready) {
        side_ready.resize(R);
        for (int i = 0; i < R; ++i) side_ready[i] = d->ready_time[corder[i]];
      }
      g->has_dense = true;
      g->d_dprog = dev_upload(dprog);
      if (!side_slots.empty()) {
        g->d_side_off = dev_upload(side_off);
        g->d_side_slots = dev_upload(side_slots);
      }
      g->d_side_ready = dev_upload(side_ready);
    }
  }

  });
  sect.run("lanes-prog", [&] {
  // ---- lane-register program (maxplus_lanes.cu) ------------------------------
  // One emitted record per frozen row: a task, or for a permutable chain a
  // chain record on its first member row followed by B-1 no-op rows (so the
  // duration tiles of 16 rows stay aligned with 16 records).  Chain members
  // read all their predecessors from slots and publish their values to slots;
  // the chain's last value becomes the lane head of its lane (the tail task
  // reads it as its own lane).
  if (chained && L <= 4 && nonneg && g->n_ordered == n && NC < 32768) {
    const int RE = n;  // emitted records == frozen rows
    hvec<int> ekind(RE, 0), eid(RE, -1);  // 0 task, 1 chain (eid = chain), 2 no-op
    for (int i = 0; i < R; ++i) {
      const int x = corder[i];
      const int r0 = rec_first_row[i];
      if (x < n) {
        eid[r0] = x;
      } else {
        const int c = x - n;
        ekind[r0] = 1;
        eid[r0] = c;
        for (int k = 1; k < d->chain_ptr[c + 1] - d->chain_ptr[c]; ++k) ekind[r0 + k] = 2;
      }
    }
    // Chain members read every predecessor from a slot.  Among predecessors
    // on one lane only the latest (highest row) matters: rel is non-decreasing
    // along a lane when durations and gaps are >= 0 (gaps host-checked,
    // durations device-checked: a negative one reruns the exact general
    // kernel, which keeps every edge).
    auto member_preds = [&](int m, hvec<int>& out) {
      out.clear();
      for (int q = pptr[m]; q < pptr[m + 1]; ++q) {
        const int u = padj[q];
        bool keep = true;
        for (int& w : out)
          if (d->lane[w] == d->lane[u]) {
            if (g->row_of[u] > g->row_of[w]) w = u;
            keep = false;
            break;
          }
        if (keep) out.push_back(u);
      }
    };
    hvec<int> mp;
    // which predecessor reads are lane heads at read time?
    hvec<int> head(L, -1);          // task id, or -2 - c after chain c
    hvec<int> far_use(n, -1);       // last slot read of each task value
    hvec<int> near_use(n, INT32_MAX);  // first slot read
    hvec<unsigned> hmask(RE, 0);
    hvec<int> sp_ptr(RE + 1, 0), sp_list;  // slot-read predecessors per record (CSR)
    for (int r = 0; r < RE; ++r) {
      if (ekind[r] == 0) {
        const int v = eid[r];
        const int l = d->lane[v];
        unsigned mask = 0;
        for (int k = pptr[v]; k < pptr[v + 1]; ++k) {
          const int u = padj[k];
          const int m = d->lane[u];
          if (head[m] == u) {
            if (m != l) mask |= 1u << m;
          } else {
            sp_list.push_back(u);
            far_use[u] = std::max(far_use[u], r);
            near_use[u] = std::min(near_use[u], r);
          }
        }
        hmask[r] = mask;
        head[l] = v;
      } else if (ekind[r] == 1) {
        const int c = eid[r];
        for (int k = d->chain_ptr[c]; k < d->chain_ptr[c + 1]; ++k) {
          member_preds(d->chain_member[k], mp);
          for (int u : mp) {
            far_use[u] = std::max(far_use[u], r);
            near_use[u] = std::min(near_use[u], r);
          }
        }
        head[ch_lane[c]] = -2 - c;
      }
      sp_ptr[r + 1] = (int)sp_list.size();
    }
    hvec<int> lslot(n, -1);
    hvec<char> lglob(n, 0);
    MinFreeSet fs, fg;
    int ns = 0, ngl = 0;
    auto for_values = [&](int r, auto fn) {  // task values produced by record r
      if (ekind[r] == 0) {
        fn(eid[r]);
      } else if (ekind[r] == 1) {
        const int c = eid[r];
        for (int k = d->chain_ptr[c]; k < d->chain_ptr[c + 1]; ++k) fn(d->chain_member[k]);
      }
    };
    hvec<int> fa_ptr(RE + 1, 0), fa;  // values freed after record r (CSR)
    for (int r = 0; r < RE; ++r)
      for_values(r, [&](int v) { if (far_use[v] >= 0) fa_ptr[far_use[v] + 1]++; });
    for (int r = 0; r < RE; ++r) fa_ptr[r + 1] += fa_ptr[r];
    fa.resize(fa_ptr[RE]);
    {
      hvec<int> fill(fa_ptr.begin(), fa_ptr.end() - 1);
      for (int r = 0; r < RE; ++r)
        for_values(r, [&](int v) { if (far_use[v] >= 0) fa[fill[far_use[v]]++] = v; });
    }
    for (int r = 0; r < RE; ++r) {
      for_values(r, [&](int v) {
        if (far_use[v] < 0) return;
        const bool shrt = far_use[v] - r <= kShortRange;
        if (shrt && !fs.empty()) {
          lslot[v] = fs.top();
          fs.pop();
        } else if (shrt && ns < kSmemSlotsMax) {
          lslot[v] = ns++;
        } else {
          lglob[v] = 1;
          if (!fg.empty()) {
            lslot[v] = fg.top();
            fg.pop();
          } else {
            lslot[v] = ngl++;
          }
        }
      });
      for (int q = fa_ptr[r]; q < fa_ptr[r + 1]; ++q) (lglob[fa[q]] ? fg : fs).push(lslot[fa[q]]);
    }
    auto code_of = [&](int u) { return lglob[u] ? ns + lslot[u] : lslot[u]; };
    hvec<int> lane_last(L, -1);
    for (int r = 0; r < RE; ++r)
      if (ekind[r] == 0) lane_last[d->lane[eid[r]]] = r;
    hvec<LaneRec> lprog(RE);
    hvec<int> lside_off(RE + 1, 0), lside_slots;
    hvec<LaneChainDev> lchains(NC);
    hvec<int> lperm(NC, 0);  // chain offsets in the permutation rows (record order, as
    {                        // the records builder assigns them; not read from it: concurrent)
      int o = 0;
      for (int i = 0; i < R; ++i)
        if (corder[i] >= n) {
          const int c = corder[i] - n;
          lperm[c] = o;
          o += d->chain_ptr[c + 1] - d->chain_ptr[c];
        }
    }
    hvec<LaneMemberDev> lmembers;
    hvec<int> lpreds;
    bool any_ready = false;
    int cur_chain_lane = 0;
    for (int r = 0; r < RE; ++r) {
      LaneRec rec;
      memset(&rec, 0, sizeof(rec));
      if (ekind[r] == 1) cur_chain_lane = ch_lane[eid[r]];
      if (ekind[r] == 2) rec.h = (unsigned char)cur_chain_lane;  // member row: the chain's lane
      if (ekind[r] != 0) {
        rec.rare = (unsigned char)(ekind[r] == 1 ? LREC_CHAIN : LREC_NOP);
        if (ekind[r] == 1) {
          const int c = eid[r];
          rec.s0 = (short)c;
          rec.h = (unsigned char)ch_lane[c];
          LaneChainDev& lc = lchains[c];
          lc.lane = ch_lane[c];
          lc.B = d->chain_ptr[c + 1] - d->chain_ptr[c];
          lc.mem_off = (int)lmembers.size();
          lc.perm_off = lperm[c];
          for (int k = d->chain_ptr[c]; k < d->chain_ptr[c + 1]; ++k) {
            const int m = d->chain_member[k];
            LaneMemberDev md;
            memset(&md, 0, sizeof(md));
            md.gap = d->gap[m];
            md.pred_off = (int)lpreds.size();
            member_preds(m, mp);
            for (int u : mp) lpreds.push_back(code_of(u));
            md.npred = (int)lpreds.size() - md.pred_off;
            md.out = lslot[m] >= 0 ? code_of(m) : -1;
            if (d->ready_time && d->ready_time[m] != 0) any_ready = true;
            lmembers.push_back(md);
          }
        }
        lside_off[r + 1] = (int)lside_slots.size();
        lprog[r] = rec;
        continue;
      }
      const int v = eid[r];
      rec.gap = d->gap[v];
      unsigned rare = 0;
      int nsm_pred = 0;
      for (int q = sp_ptr[r]; q < sp_ptr[r + 1]; ++q) {
        const int u = sp_list[q];
        if (!lglob[u] && nsm_pred == 0) {
          rare |= LREC_S0;
          rec.s0 = (short)lslot[u];
          ++nsm_pred;
        } else if (!lglob[u] && nsm_pred == 1) {
          rare |= LREC_S1;
          rec.s1 = (short)lslot[u];
          ++nsm_pred;
        } else {
          rare |= LREC_SIDE;
          lside_slots.push_back(code_of(u));
        }
      }
      lside_off[r + 1] = (int)lside_slots.size();
      const long long rt = d->ready_time ? d->ready_time[v] : 0;
      if (rt != 0) {
        rare |= LREC_SIDE;
        any_ready = true;
      }
      unsigned mask = hmask[r];
      if (rare & LREC_PRE) mask |= 16u;  // temp lane carries the rare predecessors
      if (lane_last[d->lane[v]] == r) rare |= LREC_MS;
      if (lslot[v] >= 0) {
        rare |= lglob[v] ? LREC_OUT_GLOBAL : LREC_OUT_SMEM;
        rec.out = (short)lslot[v];
      }
      rec.rare = (unsigned char)rare;
      rec.h = (unsigned char)((unsigned)d->lane[v] | (mask << 2) | (rec.gap != 0 ? 128u : 0u));
      lprog[r] = rec;
    }
    // segment cuts: boundaries b (multiples of the 16-record chunk) with no
    // slot value live across them (produced before b, read at or after b)
    // and not inside a chain's no-op rows
    std::vector<int> cuts;
    std::vector<int> carry_rows, carry_gid;
    int seg_c0 = -1, seg_c1 = -1;
    std::vector<long long> gpre(RE + 1, 0), gapre(RE + 1, 0);
    {
      hvec<int> delta(RE + 2, 0);
      hvec<int> prod(n, -1);  // producer row of each value
      for (int r = 0; r < RE; ++r)
        for_values(r, [&](int v) {
          prod[v] = r;
          if (far_use[v] > r) {
            delta[r + 1]++;
            delta[far_use[v] + 1]--;
          }
        });
      hvec<int> live_at(RE + 1, 0);  // values live across row boundary b
      {
        int live = 0;
        for (int b = 0; b <= RE; ++b) {
          live += delta[b];
          live_at[b] = live;
        }
      }
      // One permutable chain whose member predecessors live long (e.g. one
      // AllReduce per gradient bucket, read at the end of the backward pass):
      // the chain segment [c0, c1) is replayed numerically, and the values
      // live across c0 (all in global slots, all read inside the chain
      // segment) become carries, so the backward pass can still be cut.
      int rc = -1;
      for (int r = 0; r < RE && NC == 1; ++r)
        if (ekind[r] == 1) rc = r;
      if (rc >= 0) {
        int c1 = RE;
        for (int b = (rc / 16 + 1) * 16; b < RE; b += 16)
          if (live_at[b] == 0 && ekind[b] != 2) {
            c1 = b;
            break;
          }
        for (int c0 = rc / 16 * 16; c0 >= 16 && c0 >= rc / 16 * 16 - 64 * 16 && seg_c0 < 0;
             c0 -= 16) {
          if (ekind[c0] == 2) continue;
          bool ok = true;
          std::vector<int> cr;
          for (int v = 0; v < n && ok; ++v) {
            if (far_use[v] < 0) continue;
            const bool across = prod[v] < c0 && far_use[v] >= c0;
            if (across) {
              if (!lglob[v] || near_use[v] < c0 || far_use[v] >= c1) ok = false;
              else cr.push_back(v);
            } else if (lglob[v] && !(prod[v] >= c0 && far_use[v] < c1)) {
              // a global value outside the chain segment: no transfer form
              ok = false;
            }
          }
          if (ok && !cr.empty()) {
            seg_c0 = c0;
            seg_c1 = c1;
            std::sort(cr.begin(), cr.end(), [&](int a, int b) { return prod[a] < prod[b]; });
            for (int v : cr) {
              carry_rows.push_back(prod[v]);
              carry_gid.push_back(lslot[v]);
            }
          }
        }
      }
      hvec<int> cdelta(RE + 2, 0);  // carries live across b
      for (size_t q = 0; q < carry_rows.size(); ++q) {
        cdelta[carry_rows[q] + 1]++;
        cdelta[seg_c0 + 1]--;  // every carry is live across c0 and read at or after it
      }
      int clive = 0;
      for (int b = 0; b < RE; ++b) {
        clive += cdelta[b];
        if (b == 0 || b % 16 != 0 || ekind[b] == 2) continue;
        if (seg_c0 >= 0 && b > seg_c0 && b < seg_c1) continue;
        if (live_at[b] == 0 || (seg_c0 >= 0 && b <= seg_c0 && live_at[b] == clive)) cuts.push_back(b);
      }
      auto wt = [&](int t) { return std::max<long long>(d->duration[t], 0) + d->gap[t]; };
      for (int r = 0; r < RE; ++r) {
        long long w = 0;
        if (ekind[r] == 0) {
          w = wt(eid[r]);
        } else if (ekind[r] == 1) {
          const int c = eid[r];
          for (int k = d->chain_ptr[c]; k < d->chain_ptr[c + 1]; ++k) w += wt(d->chain_member[k]);
        }
        gpre[r + 1] = gpre[r] + w;
        long long gg = 0;
        if (ekind[r] == 0) {
          gg = d->gap[eid[r]];
        } else if (ekind[r] == 1) {
          const int c = eid[r];
          for (int k = d->chain_ptr[c]; k < d->chain_ptr[c + 1]; ++k) gg += d->gap[d->chain_member[k]];
        }
        gapre[r + 1] = gapre[r] + gg;
      }
    }
    // chain members with ready floors stay on the general kernel
    if (ns + ngl < 32000 && !(NC > 0 && any_ready)) {
      g->lane_cuts = std::move(cuts);
      g->seg_c0 = seg_c0;
      g->seg_c1 = seg_c1;
      g->carry_rows = std::move(carry_rows);
      g->carry_gid = std::move(carry_gid);
      g->lane_wt_prefix = std::move(gpre);
      g->lane_gap_prefix = std::move(gapre);
      g->lane_ready = any_ready;
      hvec<long long> freq(256, 0);
      for (int r = 0; r < RE; ++r)
        if (ekind[r] == 0) freq[lprog[r].h]++;
      g->lane_codes.clear();
      for (int c = 0; c < 256; ++c)
        if (freq[c]) g->lane_codes.push_back(c);
      std::stable_sort(g->lane_codes.begin(), g->lane_codes.end(),
                       [&](int a, int b) { return freq[a] > freq[b]; });
      hvec<long long> lready;
      if (any_ready) {
        lready.resize(RE);
        for (int r = 0; r < RE; ++r) lready[r] = ekind[r] == 0 ? d->ready_time[eid[r]] : 0;
      }
      g->has_lanes = true;
      g->ln_rec = RE;
      g->lksm = ns;
      g->lkglob = ngl;
      g->d_lprog = dev_upload(lprog);
      if (!lside_slots.empty()) {
        g->d_lside_off = dev_upload(lside_off);
        g->d_lside_slots = dev_upload(lside_slots);
      }
      g->d_lside_ready = dev_upload(lready);
      if (NC > 0) {
        g->d_lchains = dev_upload(lchains);
        g->d_lmembers = dev_upload(lmembers);
        g->d_lpreds = dev_upload(lpreds);
      }
    }
  }

  });
  sect.join();
  gt.mark("programs");
  // ---- breakdown geometry -------------------------------------------------------
  for (int i = 0; i < n; ++i)
    if (d->gap[i] < 0) g->gap_nonneg = false;
  if (L > 0) {
    hvec<int> aptr(L + 1, 0);
    for (int i = 0; i < n; ++i) aptr[d->lane[i] + 1]++;
    for (int l = 0; l < L; ++l) aptr[l + 1] += aptr[l];
    g->d_bd_all_ptr = dev_upload(aptr);
  }
  if (chained && L > 0) {
    hvec<int> bptr(L + 1, 0), brows, lane_chain(L, -1), pos_in_lane(n, -1);
    for (int l = 0; l < L; ++l) {
      for (int k = d->lane_order_ptr[l]; k < d->lane_order_ptr[l + 1]; ++k) {
        pos_in_lane[d->lane_order[k]] = (int)brows.size() - bptr[l];
        brows.push_back(g->row_of[d->lane_order[k]]);
      }
      bptr[l + 1] = (int)brows.size();
    }
    bool ok = true;
    hvec<BdChain> bch(NC);
    hvec<int> mrows(members.size());
    for (size_t k = 0; k < members.size(); ++k) mrows[k] = members[k].row;
    for (int c = 0; c < NC && ok; ++c) {
      const int l = ch_lane[c];
      if (lane_chain[l] >= 0) ok = false;  // one permutable chain per lane
      lane_chain[l] = c;
      const int h = d->chain_head ? d->chain_head[c] : -1;
      bch[c].lane = l;
      bch[c].pos = h >= 0 ? pos_in_lane[h] + 1 : 0;
      bch[c].B = chains[c].B;
      bch[c].member_off = chains[c].member_off;
      bch[c].perm_off = chains[c].perm_off;
      bch[c].pad = 0;
    }
    if (ok) {
      g->bd_ok = true;
      g->d_bd_ptr = dev_upload(bptr);
      g->d_bd_rows = dev_upload(brows);
      g->d_bd_lane_chain = dev_upload(lane_chain);
      g->d_bd_chains = dev_upload(bch);
      g->d_bd_member_rows = dev_upload(mrows);
    }
  }
}

// Host arrays of a device-frozen graph (no chains, rows == records): the
// descriptor columns from the per-row device arrays, the unique-edge and
// predecessor lists from the sorted device keys.
void materialize_from_device(ks_graph* g, LazyPrograms& S) {
  const int n = g->n, L = g->L;
  const long long nu = S.m_unique;
  auto down = [&](auto& h, const auto* d, size_t cnt) {
    h.resize(cnt);
    if (cnt) CUDA_TRY(cudaMemcpy(h.data(), d, cnt * sizeof(h[0]), cudaMemcpyDeviceToHost));
  };
  hvec<int64_t> dur_r, gap_r;
  hvec<int> lane_r, rank_r;
  down(dur_r, g->d_dur, (size_t)n);
  down(gap_r, g->d_gap, (size_t)n);
  down(lane_r, g->d_lane, (size_t)n);
  down(rank_r, g->d_rank, (size_t)n);
  down(S.keys, S.d_ukeys, (size_t)nu);
  hvec<unsigned long long> pk;
  down(pk, S.d_pkeys, (size_t)nu);
  down(S.lane_order, S.d_lane_order, (size_t)n);
  g->row_of.resize(n);
  g->rank_row.resize(n);
  S.duration.resize(n);
  S.gap.resize(n);
  S.lane.resize(n);
  host_parallel_for(n, [&](long long b, long long e) {
    for (int r = (int)b; r < (int)e; ++r) {
      const int t = g->order[r];
      g->row_of[t] = r;
      g->rank_row[r] = rank_r[r];
      S.duration[t] = dur_r[r];
      S.gap[t] = gap_r[r];
      S.lane[t] = lane_r[r];
    }
  });
  S.optr.assign(n + 1, 0);
  S.pptr.assign(n + 1, 0);
  for (long long q = 0; q < nu; ++q) {
    S.optr[(S.keys[q] >> 32) + 1]++;
    S.pptr[(pk[q] >> 32) + 1]++;
  }
  for (int i = 0; i < n; ++i) {
    S.optr[i + 1] += S.optr[i];
    S.pptr[i + 1] += S.pptr[i];
  }
  S.padj.resize(nu);
  S.cadj.resize(nu);
  host_parallel_for(nu, [&](long long b, long long e) {
    for (long long q = b; q < e; ++q) {
      S.padj[q] = (int)(pk[q] & 0xffffffffu);
      S.cadj[q] = (int)(S.keys[q] & 0xffffffffu);
    }
  });
  S.cptr = S.optr;
  S.corder.assign(g->order.begin(), g->order.end());
  S.rec_first_row.resize(n);
  std::iota(S.rec_first_row.begin(), S.rec_first_row.end(), 0);
  memset(&S.desc, 0, sizeof(S.desc));
  S.desc.n_tasks = n;
  S.desc.n_lanes = L;
  S.desc.duration = S.duration.data();
  S.desc.gap = S.gap.data();
  S.desc.lane = S.lane.data();
  S.desc.lane_order_ptr = S.lane_order_ptr.data();
  S.desc.lane_order = S.lane_order.data();
  S.from_device = false;
}

// verify_acyclic on the lane heads (toposort_lanes_req_kernel): a head is
// ready once every predecessor its lane order does not already put before it
// has been emitted, i.e. once the emitted prefix of that predecessor's lane is
// long enough.  Per row: (lane, prefix length) requirements, the largest per
// lane; built on the first ks_toposort call from the device CSR.
void ensure_topo_req(const ks_graph* gc) {
  ks_graph* g = const_cast<ks_graph*>(gc);
  std::call_once(g->topo_once, [g] {
    if (!g->bd_ok || g->n_chains > 0 || g->L > 32 || g->n == 0 || g->n >= (1 << 27)) return;
    DevGuard guard(g->device);
    const int n = g->n, L = g->L;
    hvec<int> bptr(L + 1), brows(n), cptr(n + 1), lane_r(n);
    CUDA_TRY(cudaMemcpy(bptr.data(), g->d_bd_ptr, 4 * (L + 1), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(brows.data(), g->d_bd_rows, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(cptr.data(), g->d_child_ptr, 4 * ((size_t)n + 1), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(lane_r.data(), g->d_lane, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    hvec<int> child(cptr[n]);
    if (cptr[n]) CUDA_TRY(cudaMemcpy(child.data(), g->d_child, 4 * (size_t)cptr[n], cudaMemcpyDeviceToHost));
    hvec<int> pos(n, 0);
    for (int l = 0; l < L; ++l)
      for (int k = bptr[l]; k < bptr[l + 1]; ++k) pos[brows[k]] = k - bptr[l];
    auto needed = [&](int u, int v) { return !(lane_r[u] == lane_r[v] && pos[u] < pos[v]); };
    hvec<int> cnt(n + 1, 0);
    for (int u = 0; u < n; ++u)
      for (int k = cptr[u]; k < cptr[u + 1]; ++k)
        if (needed(u, child[k])) cnt[child[k] + 1]++;
    for (int r = 0; r < n; ++r) cnt[r + 1] += cnt[r];
    hvec<int> cl(cnt[n]), cp(cnt[n]);
    {
      hvec<int> fill(cnt.begin(), cnt.end() - 1);
      for (int u = 0; u < n; ++u)
        for (int k = cptr[u]; k < cptr[u + 1]; ++k)
          if (needed(u, child[k])) {
            const int o = fill[child[k]]++;
            cl[o] = lane_r[u];
            cp[o] = pos[u] + 1;
          }
    }
    hvec<int> rptr(n + 1, 0), rl, rp;  // deduplicated per (row, lane): the largest prefix
    for (int v = 0; v < n; ++v) {
      const size_t b = rl.size();
      for (int k = cnt[v]; k < cnt[v + 1]; ++k) {
        bool merged = false;
        for (size_t q = b; q < rl.size(); ++q)
          if (rl[q] == cl[k]) {
            rp[q] = std::max(rp[q], cp[k]);
            merged = true;
            break;
          }
        if (!merged) {
          rl.push_back(cl[k]);
          rp.push_back(cp[k]);
        }
      }
      rptr[v + 1] = (int)rl.size();
    }
    hvec<int> rank_r(n);
    CUDA_TRY(cudaMemcpy(rank_r.data(), g->d_rank, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    hvec<TopoRec> recs(n);  // in lane order (brows)
    for (int k = 0; k < n; ++k) {
      const int r = brows[k];
      TopoRec& x = recs[k];
      memset(&x, 0, sizeof(x));
      x.row = r;
      x.rank = rank_r[r];
      x.r0 = rptr[r];
      x.rn = rptr[r + 1] - rptr[r];
      for (int q = 0; q < 4 && q < x.rn; ++q) {
        x.ml[q] = rl[x.r0 + q];
        x.mq[q] = rp[x.r0 + q];
      }
    }
    g->d_topo_rec = dev_upload(recs);
    g->d_req_lane = dev_upload(rl);
    g->d_req_pos = dev_upload(rp);
    g->topo_req = true;
  });
}

void ensure_programs(const ks_graph* gc) {
  ks_graph* g = const_cast<ks_graph*>(gc);
  std::call_once(g->programs_once, [g] {
    if (!g->lazy) return;
    DevGuard guard(g->device);
    HostTimer gt;
    if (g->lazy->from_device) {
      materialize_from_device(g, *g->lazy);
      gt.mark("materialize");
    }
    build_programs(g, *g->lazy);
    g->lazy.reset();
  });
}

void free_graph(ks_graph* g) {
  if (!g) return;
  void* dptrs[] = {g->d_dprog,   g->d_side_off,   g->d_side_slots,  g->d_side_ready,
                   g->d_lprog,   g->d_lside_off,  g->d_lside_slots, g->d_lside_ready,
                   g->d_bd_ptr,  g->d_bd_rows,    g->d_bd_lane_chain, g->d_bd_chains,
                   g->d_bd_member_rows, g->d_lchains, g->d_lmembers, g->d_lpreds,
                   g->d_bd_all_ptr, g->d_topo_rec, g->d_req_lane, g->d_req_pos};
  for (void* p : dptrs)
    if (p) cudaFree(p);
  void* ptrs[] = {g->d_prog,  g->d_extra, g->d_chains, g->d_members, g->d_child_ptr,
                  g->d_child, g->d_indeg, g->d_lane,   g->d_dur,     g->d_gap,
                  g->d_ready, g->d_rank,  g->d_prio,   g->d_flags,   g->d_group};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete g;
}

// ---- per-call scenario tables ---------------------------------------------------
// Device blocks of finished calls, per host thread, reused by the next call on
// the same stream (stream order makes the reuse safe, as it does for
// cudaFreeAsync + cudaMallocAsync): a small sweep's call otherwise spends ~8 us
// of host time in a dozen allocator calls.  Bounded; freed at thread exit.
struct ScratchPool {
  struct Blk {
    void* p;
    size_t bytes;
    cudaStream_t st;
  };
  std::vector<Blk> free_blks;
  size_t held = 0;
  static constexpr size_t kMaxHeld = 512ull << 20;
  static constexpr size_t kMaxBlks = 64;
  void* take(size_t bytes, cudaStream_t st) {
    int best = -1;
    for (int i = 0; i < (int)free_blks.size(); ++i) {
      const Blk& b = free_blks[i];
      if (b.st == st && b.bytes >= bytes && b.bytes <= 2 * bytes + 4096 &&
          (best < 0 || b.bytes < free_blks[best].bytes))
        best = i;
    }
    if (best < 0) return nullptr;
    void* p = free_blks[best].p;
    held -= free_blks[best].bytes;
    free_blks[best] = free_blks.back();
    free_blks.pop_back();
    return p;
  }
  void give(void* p, size_t bytes, cudaStream_t st) {
    if (held + bytes > kMaxHeld || free_blks.size() >= kMaxBlks) {
      cudaFreeAsync(p, st);
      return;
    }
    free_blks.push_back({p, bytes, st});
    held += bytes;
  }
  ~ScratchPool() {
    for (const Blk& b : free_blks) cudaFree(b.p);
  }
};
ScratchPool& scratch_pool() {
  static thread_local ScratchPool pool;
  return pool;
}

struct ScenTables {
  std::vector<std::pair<void*, size_t>> bufs;
  int* scale_ptr = nullptr;
  ScaleStepDev* scale = nullptr;
  long long* ovr = nullptr;
  int* ovr_map = nullptr;
  short* perm = nullptr;
  unsigned char* present = nullptr;
  int* vrank = nullptr;
  bool has_remove = false;  // a scale step removes tasks (KS_STEP_REMOVE)
  cudaStream_t st = nullptr;
  void* alloc(size_t bytes) {
    void* p = scratch_pool().take(bytes, st);
    if (p == nullptr) CUDA_TRY(cudaMallocAsync(&p, bytes, st));
    bufs.push_back({p, bytes});
    return p;
  }
  template <class T>
  T* up(const T* host, size_t count) {
    if (!host || count == 0) return nullptr;
    T* p = static_cast<T*>(alloc(count * sizeof(T)));
    CUDA_TRY(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, st));
    return p;
  }
  template <class T>
  T* scratch(size_t count) {
    if (count == 0) return nullptr;
    return static_cast<T*>(alloc(count * sizeof(T)));
  }
  ~ScenTables() {
    for (auto& b : bufs) scratch_pool().give(b.first, b.second, st);
  }
  // host staging must outlive async copies: keep vectors alive
  std::vector<std::vector<char>> keep;
};

void build_tables(const ks_graph* g, const ks_scenarios_desc* sc, ScenTables& T, bool need_ovr_map,
                  bool need_vrank) {
  const int S = sc->n_scenarios;
  if (sc->scale_ptr && sc->scale) {
    const int nsteps = sc->scale_ptr[S] - sc->scale_ptr[0];
    if (sc->scale_ptr[0] != 0) fail(KS_ERR_INVALID, "scale_ptr[0] must be 0");
    for (int k = 0; k < nsteps; ++k) {
      if (sc->scale[k].num == 0 && sc->scale[k].den == 0) {  // KS_STEP_REMOVE
        T.has_remove = true;
        continue;
      }
      if (sc->scale[k].num <= 0 || sc->scale[k].den <= 0)
        fail(KS_ERR_BAD_PIPELINE, "scale factor must be positive");
    }
    T.scale_ptr = T.up(sc->scale_ptr, (size_t)S + 1);
    // ks_scale_step and ScaleStepDev share layout (int,int,ll,ll)
    static_assert(sizeof(ks_scale_step) == sizeof(ScaleStepDev), "layout");
    T.scale = reinterpret_cast<ScaleStepDev*>(
        T.up(reinterpret_cast<const ScaleStepDev*>(sc->scale), (size_t)std::max(nsteps, 1)));
  }
  if (sc->n_overrides > 0) {
    T.ovr = T.up(reinterpret_cast<const long long*>(sc->override), (size_t)sc->n_overrides * S);
    if (need_ovr_map) {
      T.keep.emplace_back(sizeof(int) * (size_t)g->n);
      int* map = reinterpret_cast<int*>(T.keep.back().data());
      std::fill(map, map + g->n, -1);
      for (int k = 0; k < sc->n_overrides; ++k) {
        const int r = sc->override_task[k];
        if (r < 0 || r >= g->n) fail(KS_ERR_INVALID, "override row out of range");
        map[r] = k;
      }
      T.ovr_map = T.up(map, (size_t)g->n);
    }
  }
  if (g->n_chains > 0) {
    if (sc->chain_perm) {
      if (sc->perm_ld < g->perm_ld) fail(KS_ERR_INVALID, "perm_ld too small");
      T.perm = T.up(sc->chain_perm, (size_t)S * sc->perm_ld);
    }
    if (sc->chain_present) T.present = T.up(sc->chain_present, (size_t)S * g->n_chains);
  }
  if (need_vrank && sc->vdnn_rank) T.vrank = T.up(sc->vdnn_rank, (size_t)g->n);
}

}  // namespace

namespace ddsim {
__global__ void patch_ovr_kernel(NodeRec* prog, int n_rec, const int* ovr_map) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_rec; i += gridDim.x * blockDim.x) {
    NodeRec& r = prog[i];
    if (r.kind == 0) r.ovr_row = ovr_map[r.row];
  }
}
cudaError_t launch_patch_ovr(NodeRec* prog, int n_rec, const int* ovr_map, cudaStream_t st) {
  patch_ovr_kernel<<<std::min(148 * 4, (n_rec + 255) / 256), 256, 0, st>>>(prog, n_rec, ovr_map);
  note_launch();
  return cudaGetLastError();
}
}  // namespace ddsim

namespace {

// Segment rows for the segment-parallel lanes path, or empty to run the
// single-pass kernel.  Few scenarios leave most SMs idle (one thread walks
// every record of its scenario); K segments multiply the parallelism by K at
// the cost of a transfer pass.  Cuts come from the compiler's clean rows
// (no live slot value), near K evenly spaced targets.
// Upper bound of |duration| over every (row, scenario) a table derives: the
// base / override magnitude through each scenario's scale steps, each step
// ceil(b * num / den) + 1 (half-up rounds by at most one).  Host tables only.
bool expand_fits_int32(const ks_graph* g, const ks_scenarios_desc* sc) {
  if (g->dur_abs_max < 0) return false;
  const int S = sc->n_scenarios;
  long long b0 = g->dur_abs_max;
  if (sc->n_overrides > 0) {
    const long long cnt = (long long)sc->n_overrides * S;
    for (long long i = 0; i < cnt; ++i) {
      const long long v = sc->override[i];
      if (v == LLONG_MIN) return false;
      b0 = std::max(b0, v < 0 ? -v : v);
    }
  }
  const long long lim = INT_MAX;
  if (b0 > lim) return false;
  if (!sc->scale_ptr || !sc->scale) return true;
  for (int s = 0; s < S; ++s) {
    long long b = b0;
    for (int e = sc->scale_ptr[s]; e < sc->scale_ptr[s + 1]; ++e) {
      const ks_scale_step& st = sc->scale[e];
      if (st.num <= 0 || st.den <= 0) continue;  // removal steps
      const __int128 x = ((__int128)b * st.num + st.den - 1) / st.den + 1;
      if (x > lim) return false;
      b = std::max(b, (long long)x);  // steps on other groups leave b
    }
  }
  return true;
}

std::vector<int> pick_segments(const ks_graph* g, int S, int nsm) {
  std::vector<int> rows;
  if (getenv("DDSIM_NO_SEG") || !g->has_lanes || (g->lkglob > 0 && g->seg_c0 < 0) ||
      g->lane_ready || g->L < 1 ||
      g->L > 4 || g->lane_cuts.empty() || g->ln_rec < 512)
    return rows;
  // the single-pass kernel reaches the memory roofline once ~256 threads per
  // SM walk the records (measured: config 4 at 65,536 scenarios, V = 2)
  long long max_s = 256LL * nsm;
  if (const char* e = getenv("DDSIM_SEG_MAX_S")) max_s = atoll(e);
  if (S > max_s) return rows;
  // segments: enough for ~4,096 resident scenario-segments per SM (measured
  // best on configs 2 and 4), each >= 320 records, and short enough that the
  // base weights of a segment stay below 2^28 ns (int32 coefficients: the
  // device certificate is 2^30 per scenario; outside it the exact kernel reruns)
  long long tps = 4096;
  if (const char* e = getenv("DDSIM_SEG_TPS")) tps = std::max(32LL, atoll(e));
  // shorter segments only when a few scenarios must fill the GPU (config 1,
  // S = 2: 320 -> 96 -> 64 records per segment, 0.107 -> 0.074 -> 0.057 ms
  // with the block scan; config 2, S = 401: 320 -> 192, 0.143 -> 0.125 ms;
  // config 3, S = 4,000, is fastest at 320: fewer transfers and scan steps)
  long long min_len = S <= 256 ? 64 + 128 * (long long)S / 256
                      : S < 2048 ? 192 + 128 * ((long long)S - 256) / 1792 : 320;
  if (const char* e = getenv("DDSIM_SEG_MIN_LEN")) min_len = std::max(16LL, atoll(e));
  long long K = (tps * nsm + S - 1) / S;
  K = std::min<long long>(K, g->ln_rec / min_len);
  const long long total = g->lane_wt_prefix[g->ln_rec];
  K = std::max<long long>(K, (total >> 28) + 1);
  if (const char* e = getenv("DDSIM_SEG_K")) K = atoll(e);
  K = std::min<long long>(K, (long long)g->lane_cuts.size() + 1);
  if (K < 2) return rows;
  rows.push_back(0);
  for (long long k = 1; k < K; ++k) {
    const long long t = k * (long long)g->ln_rec / K;
    auto it = std::lower_bound(g->lane_cuts.begin(), g->lane_cuts.end(), (int)t);
    int best = -1;
    if (it != g->lane_cuts.end()) best = *it;
    if (it != g->lane_cuts.begin() && (best < 0 || t - *(it - 1) < best - t)) best = *(it - 1);
    if (best > rows.back()) rows.push_back(best);
  }
  rows.push_back(g->ln_rec);
  if (g->seg_c0 >= 0) {
    // the chain segment [c0, c1) is one segment
    std::vector<int> r2;
    for (int b : rows)
      if (b <= g->seg_c0 || b >= g->seg_c1) r2.push_back(b);
    r2.push_back(g->seg_c0);
    if (g->seg_c1 < g->ln_rec) r2.push_back(g->seg_c1);
    std::sort(r2.begin(), r2.end());
    r2.erase(std::unique(r2.begin(), r2.end()), r2.end());
    rows.swap(r2);
  }
  // coefficient entries are int32: a segment's base weights must leave room
  // (the chain segment has no transfer)
  for (size_t k = 0; k + 1 < rows.size(); ++k)
    if (rows[k] != g->seg_c0 &&
        g->lane_wt_prefix[rows[k + 1]] - g->lane_wt_prefix[rows[k]] >= (1LL << 29))
      return {};
  if (rows.size() < 3) return {};
  return rows;
}

int simulate_impl(const ks_graph* g, const ks_scenarios_desc* sc, int policy, int path,
                  const ks_sim_out* out, cudaStream_t stream) {
  if (!g || !sc || !out) fail(KS_ERR_INVALID, "null argument");
  if (g->device < 0) fail(KS_ERR_NO_DEVICE, "graph was compiled without a device");
  ensure_programs(g);
  const int S = sc->n_scenarios;
  if (S <= 0) fail(KS_ERR_INVALID, "n_scenarios must be positive");
  if (policy < 0 || policy > 2) fail(KS_ERR_INVALID, "unknown policy");
  // every path indexes dense[r * dense_ld + s] and start[r * start_ld + s]
  if (sc->dense_kind != 0 && sc->dense != nullptr && sc->dense_ld < S)
    fail(KS_ERR_INVALID, "dense_ld must be >= n_scenarios");
  if (out->start != nullptr && out->start_ld < S)
    fail(KS_ERR_INVALID, "start_ld must be >= n_scenarios");
  bool use_max = path == KS_PATH_MAXPLUS ||
                 (path == KS_PATH_AUTO && g->chained && out->schedule == nullptr);
  if (!use_max && g->n_chains > 0)
    fail(KS_ERR_UNSUPPORTED, "list scheduling of permutable chains is not supported");
  if (g->n_ordered < g->n) {
    // A cycle: Alg. 1 stalls with exactly the non-Kahn-reachable tasks left.
    fail(KS_ERR_DEADLOCK, std::to_string(g->n - g->n_ordered) + " tasks never became ready");
  }
  DevGuard guard(g->device);
  keep_device_pool(g->device);
  ScenTables T;
  T.st = stream;
  const bool dense = sc->dense_kind != 0 && sc->dense != nullptr;
  build_tables(g, sc, T, true, policy == KS_POLICY_VDNN);
  if (dense && (sc->scale_ptr || sc->n_overrides > 0))
    fail(KS_ERR_INVALID, "dense durations exclude overrides and scale steps");
  if (T.has_remove && !use_max)
    fail(KS_ERR_UNSUPPORTED,
         "removal steps need the max-plus path (lane-chained graph); apply remove_task structurally");

  // Derived durations on a lanes-eligible graph: expand them into a dense
  // int64 matrix (one thread per element; L2-resident at the sizes where the
  // derived path is used) and run the lanes kernel on it.
  ks_scenarios_desc expanded;
  const ks_scenarios_desc* orig_sc = sc;
  // Or the lanes kernels derive them per record (NVRTC kernels only): no
  // duration matrix in HBM.  Preferred unless the matrix would stay in L2 and
  // scale programs make the per-record derivation cost instructions on the
  // latency-bound path (measured: config 3, overrides only, 4,000 x 30k:
  // 2.43 -> 1.28 ms; config 2, scale programs, 401 x 30k (95 MB): 0.18 ms
  // expanded vs 0.28 ms derived).
  const bool l2_sized = (long long)g->n * S * 8 <= (96LL << 20);
  const bool derive = use_max && !dense && !T.has_remove && g->has_lanes && g->n_rec > 0 &&
                      (!(sc->scale_ptr && l2_sized) || getenv("DDSIM_FORCE_DERIVED") != nullptr) &&
                      getenv("DDSIM_NO_DERIVED") == nullptr && getenv("DDSIM_NO_LANES") == nullptr &&
                      getenv("DDSIM_NO_EXPAND") == nullptr && !g->lane_codes.empty() &&
                      g->lane_codes.size() <= 32 && jit_available();
  const bool expand = !derive && use_max && !dense && !T.has_remove && g->has_lanes &&
                      g->n_rec > 0 && (long long)g->n * S * 8 <= (8LL << 30) &&
                      getenv("DDSIM_NO_EXPAND") == nullptr && getenv("DDSIM_NO_LANES") == nullptr;
  if (expand) {
    // int32 elements when every derived duration provably fits: half the
    // bytes for the expansion and for each pass that reads it back (config 2)
    const bool narrow = expand_fits_int32(g, sc) && getenv("DDSIM_EXPAND64") == nullptr;
    // rows start on 128-byte lines (whole-sector stores; TMA needs 16 B)
    const long long eld = narrow ? (S + 31) / 32 * 32 : (S + 15) / 16 * 16;
    void* buf = nullptr;
    if (narrow) {
      int* b32 = T.scratch<int>((size_t)g->n * eld);
      CUDA_TRY(launch_expand_durations32(g->d_dur, g->d_group, T.ovr_map, T.ovr, T.scale_ptr,
                                         T.scale, g->n, S, eld, b32, stream));
      buf = b32;
    } else {
      long long* b64 = T.scratch<long long>((size_t)g->n * eld);
      CUDA_TRY(launch_expand_durations(g->d_dur, g->d_group, T.ovr_map, T.ovr, T.scale_ptr, T.scale,
                                       g->n, S, eld, b64, stream));
      buf = b64;
    }
    expanded = *sc;
    expanded.dense_kind = narrow ? 1 : 2;
    expanded.dense = buf;
    expanded.dense_ld = eld;
    expanded.n_overrides = 0;
    expanded.scale_ptr = nullptr;
    expanded.scale = nullptr;
    sc = &expanded;
  }
  // program / chain / override / scale tables of the general kernel's derived mode
  auto fill_general = [&](MaxplusParams& q) {
    q.n_rec = g->n_rec;
    q.prog = g->d_prog;
    if (T.ovr_map && g->n_rec > 0) {
      // per-call override rows: patch a copy of the program
      NodeRec* prog2 = T.scratch<NodeRec>(g->n_rec);
      CUDA_TRY(cudaMemcpyAsync(prog2, g->d_prog, sizeof(NodeRec) * g->n_rec,
                               cudaMemcpyDeviceToDevice, stream));
      CUDA_TRY(launch_patch_ovr(prog2, g->n_rec, T.ovr_map, stream));
      q.prog = prog2;
    }
    q.extra = g->d_extra;
    q.chains = g->d_chains;
    q.members = g->d_members;
    q.n_chains = g->n_chains;
    if (T.ovr_map && g->perm_ld > 0) {
      NodeRec* mem2 = T.scratch<NodeRec>(g->perm_ld);
      CUDA_TRY(cudaMemcpyAsync(mem2, g->d_members, sizeof(NodeRec) * g->perm_ld,
                               cudaMemcpyDeviceToDevice, stream));
      CUDA_TRY(launch_patch_ovr(mem2, g->perm_ld, T.ovr_map, stream));
      q.members = mem2;
    }
    q.ksm = g->ksm;
    q.kglob = g->kglob;
    q.ovr = T.ovr;
    q.scale_ptr = T.scale_ptr;
    q.scale = T.scale;
    q.perm = T.perm;
    q.perm_ld = orig_sc->perm_ld;
    q.present = T.present;
  };
  const bool dense_now = sc->dense_kind != 0 && sc->dense != nullptr;
  const bool tma_ok =
      dense_now && reinterpret_cast<uintptr_t>(sc->dense) % 16 == 0 &&
      (sc->dense_kind == 1 ? sc->dense_ld % 4 == 0 : sc->dense_ld % 2 == 0);
  // permutable chains run on the lanes path only for derived (expanded)
  // durations: the exact fallback for them is the general kernel's derived mode
  const bool lanes_ok = use_max && g->has_lanes && getenv("DDSIM_NO_LANES") == nullptr &&
                        (derive || (dense_now && tma_ok && sc->n_overrides == 0 && !sc->scale_ptr &&
                                    (g->n_chains == 0 || expand)));
  if (lanes_ok) {
    LaneParams p;
    memset(&p, 0, sizeof(p));
    p.prog = g->d_lprog;
    p.n_rec = g->ln_rec;
    p.side_off = g->d_lside_off;
    p.side_slots = g->d_lside_slots;
    p.side_ready = g->d_lside_ready;
    p.ksm = g->lksm;
    p.kglob = g->lkglob;
    p.S = S;
    p.L = g->L;
    const int dk = derive ? 0 : (sc->dense_kind == 1 ? 1 : 2);
    if (dk == 1 && (reinterpret_cast<uintptr_t>(sc->dense) % 16 != 0 || sc->dense_ld % 4 != 0))
      fail(KS_ERR_INVALID, "int32 dense durations need 16B alignment and dense_ld % 4 == 0");
    if (dk == 2) p.dense64 = reinterpret_cast<const long long*>(sc->dense);
    p.dense_ld = dk == 0 ? 0 : sc->dense_ld;
    LaneDerivedParams dpv;
    memset(&dpv, 0, sizeof(dpv));
    if (dk == 0) {
      LaneRowDur* rd = T.scratch<LaneRowDur>((size_t)g->n);
      CUDA_TRY(launch_build_rowdur(g->d_dur, g->d_group, T.ovr_map, g->n, rd, stream));
      dpv.rows = rd;
      dpv.ovr = T.ovr;
      dpv.scale_ptr = T.scale_ptr;
      dpv.scale = T.scale;
    }
    LaneChainParams cp;
    memset(&cp, 0, sizeof(cp));
    if (g->n_chains > 0) {
      cp.chains = g->d_lchains;
      cp.members = g->d_lmembers;
      cp.preds = g->d_lpreds;
      cp.perm = T.perm;
      cp.perm_ld = sc->perm_ld;
      cp.present = T.present;
      cp.n_chains = g->n_chains;
      if (dk == 1) cp.dense32 = reinterpret_cast<const int*>(sc->dense);
    }
    p.start = reinterpret_cast<long long*>(out->start);
    p.start_ld = out->start_ld;
    p.makespan = reinterpret_cast<long long*>(out->makespan);
    p.lane_busy = reinterpret_cast<long long*>(out->lane_busy);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device);
    const bool vec_ok = p.start == nullptr ||
                        (p.start_ld % 2 == 0 && reinterpret_cast<uintptr_t>(p.start) % 16 == 0);
    const int BD = maxplus_lanes_block_dim(S, nsm, dk, vec_ok);
    const int LV = maxplus_lanes_vec(S, dk, vec_ok);
    p.s_pad = (long long)((S + LV * BD - 1) / (LV * BD)) * LV * BD;
    if (p.kglob > 0) p.gslots = T.scratch<long long>((size_t)p.kglob * p.s_pad);
    int* flag = T.scratch<int>(1);
    CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), stream));
    p.neg_flag = flag;
    const int* d32 = dk == 1 ? reinterpret_cast<const int*>(sc->dense) : nullptr;
    bool seg_done = false;
    const std::vector<int> seg = pick_segments(g, S, nsm);
    if (!seg.empty() && jit_available()) {
      // one thread per scenario, blocks of <= 128 threads (multiple of 16)
      const int nb = (S + 127) / 128;
      const int BDs = std::max(32, ((S + nb - 1) / nb + 15) / 16 * 16);
      LaneSegParams sg;
      memset(&sg, 0, sizeof(sg));
      sg.K = (int)seg.size() - 1;
      sg.LN = g->L;
      sg.s_pad = (long long)((S + BDs - 1) / BDs) * BDs;
      sg.cuts = T.up(seg.data(), seg.size());
      {
        std::vector<long long> gs(sg.K);
        for (int k = 0; k < sg.K; ++k)
          gs[k] = g->lane_gap_prefix[seg[k + 1]] - g->lane_gap_prefix[seg[k]];
        sg.gapsum = T.up(gs.data(), gs.size());
      }
      sg.nb = (int)(sg.s_pad / BDs);
      sg.state = T.scratch<long long>((size_t)sg.K * sg.LN * sg.s_pad);
      sg.kc = -1;
      sg.replay_only = -1;
      for (int k = 0; k < sg.K && g->seg_c0 >= 0; ++k)
        if (seg[k] == g->seg_c0) sg.kc = k;
      if (g->seg_c0 >= 0 && sg.kc < 0) fail(KS_ERR_INVALID, "segment cuts miss the chain segment");
      if (sg.kc >= 0 && !g->carry_rows.empty()) {
        // carries: producing segment of each (rows ascending), their global
        // slots, and their transfer coefficients [kglob][LN][s_pad]
        std::vector<int> cptr(sg.K + 1, 0);
        for (int r : g->carry_rows) {
          const int k = (int)(std::upper_bound(seg.begin(), seg.end(), r) - seg.begin()) - 1;
          cptr[k + 1]++;
        }
        for (int k = 0; k < sg.K; ++k) cptr[k + 1] += cptr[k];
        sg.carry_ptr = T.up(cptr.data(), cptr.size());
        sg.carry_gid = T.up(g->carry_gid.data(), g->carry_gid.size());
        sg.carry_coef = T.scratch<int>((size_t)p.kglob * sg.LN * sg.s_pad);
      }
      // fused single pass (look-back) only on request: its publish chain costs
      // ~2.5 us per segment hop (config 2, K = 92: 0.35 vs 0.17 ms for the
      // transfer / scan / replay kernels; config 4 at 8,192: 2.68 vs 2.58 ms)
      if (getenv("DDSIM_SEG_FUSED") != nullptr && sg.kc < 0) {
        sg.ticket = T.scratch<int>(1 + (size_t)sg.K * sg.nb);
        sg.flags = sg.ticket + 1;
        CUDA_TRY(cudaMemsetAsync(sg.ticket, 0, sizeof(int) * (1 + (size_t)sg.K * sg.nb), stream));
      } else {
        sg.trans = T.scratch<int>((size_t)(sg.K - 1) * sg.LN * sg.LN * sg.s_pad);
      }
      LaneParams ps = p;
      ps.s_pad = sg.s_pad;
      if (ps.kglob > 0) ps.gslots = T.scratch<long long>((size_t)ps.kglob * sg.s_pad);
      if (ps.makespan) CUDA_TRY(cudaMemsetAsync(ps.makespan, 0, sizeof(long long) * S, stream));
      if (ps.lane_busy)
        CUDA_TRY(cudaMemsetAsync(ps.lane_busy, 0, sizeof(long long) * (size_t)S * g->L, stream));
      const cudaError_t e = launch_maxplus_lanes_seg(ps, g->n_chains > 0 ? &cp : nullptr, d32, dk,
                                                     g->lane_codes, sg, BDs, stream,
                                                     dk == 0 ? &dpv : nullptr);
      if (e == cudaSuccess) {
        seg_done = true;
      } else if (e != cudaErrorNotSupported) {
        CUDA_TRY(e);
      }
    }
    if (!seg_done)
      CUDA_TRY(launch_maxplus_lanes(p, g->n_chains > 0 ? &cp : nullptr, d32, dk, &g->lane_codes,
                                    stream, dk == 0 ? &dpv : nullptr));
    MaxplusParams q;
    memset(&q, 0, sizeof(q));
    q.prog = g->d_prog;
    q.n_rec = g->n_rec;
    q.extra = g->d_extra;
    q.ksm = g->ksm;
    q.kglob = g->kglob;
    q.S = S;
    q.L = g->L;
    q.dense_kind = dk;
    q.dense64 = p.dense64;
    q.dense_ld = sc->dense_ld;
    q.start = p.start;
    q.start_ld = p.start_ld;
    q.makespan = p.makespan;
    q.lane_busy = p.lane_busy;
    q.run_if = flag;
    if (g->n_chains > 0 || dk == 0) {  // exact rerun in derived mode (original tables)
      fill_general(q);
      q.dense_kind = 0;
      q.dense64 = nullptr;
    }
    const int BDq = maxplus_block_dim(S, q.dense_kind, nsm);
    q.s_pad = (long long)((S + BDq - 1) / BDq) * BDq;
    if (q.kglob > 0) q.gslots = T.scratch<long long>((size_t)q.kglob * q.s_pad);
    CUDA_TRY(launch_maxplus(q, dk == 1 ? reinterpret_cast<const int*>(sc->dense) : nullptr, stream));
    if (out->dispatched) CUDA_TRY(launch_fill_i32(out->dispatched, g->n, S, stream));
  } else if (use_max && dense_now && g->has_dense && sc->n_overrides == 0 && !sc->scale_ptr &&
             getenv("DDSIM_NO_DENSE") == nullptr) {
    DenseParams p;
    memset(&p, 0, sizeof(p));
    p.prog = g->d_dprog;
    p.n_rec = g->n_rec;
    p.side_off = g->d_side_off;
    p.side_slots = g->d_side_slots;
    p.V = (S % 2 == 0 && out->start_ld % 2 == 0 && sc->dense_ld % 2 == 0 &&
           reinterpret_cast<uintptr_t>(out->start) % 16 == 0) ? 2 : 1;
    p.side_ready = g->d_side_ready;
    p.ksm = g->dksm;
    p.kglob = g->dkglob;
    p.S = S;
    p.L = g->L;
    if (sc->dense_ld < S) fail(KS_ERR_INVALID, "dense_ld < n_scenarios");
    const int dk = sc->dense_kind == 1 ? 1 : 2;
    if (dk == 1 && (reinterpret_cast<uintptr_t>(sc->dense) % 16 != 0 || sc->dense_ld % 4 != 0))
      fail(KS_ERR_INVALID, "int32 dense durations need 16B alignment and dense_ld % 4 == 0");
    if (dk == 2) p.dense64 = reinterpret_cast<const long long*>(sc->dense);
    p.dense_ld = sc->dense_ld;
    p.start = reinterpret_cast<long long*>(out->start);
    p.start_ld = out->start_ld;
    p.makespan = reinterpret_cast<long long*>(out->makespan);
    p.lane_busy = reinterpret_cast<long long*>(out->lane_busy);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device);
    const int BD = maxplus_dense_block_dim(S, p.V, nsm);
    p.s_pad = (long long)((S + BD * p.V - 1) / (BD * p.V)) * BD * p.V;
    if (p.kglob > 0) p.gslots = T.scratch<long long>((size_t)p.kglob * p.s_pad);
    if (g->n_rec > 0) {
      int* flag = T.scratch<int>(1);
      CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), stream));
      p.neg_flag = flag;
      CUDA_TRY(launch_maxplus_dense(p, dk == 1 ? reinterpret_cast<const int*>(sc->dense) : nullptr,
                                    dk, stream));
      // exact rerun (general kernel, full int64 semantics) only if a negative
      // duration was seen: the CTAs of this launch exit at once otherwise
      MaxplusParams q;
      memset(&q, 0, sizeof(q));
      q.prog = g->d_prog;
      q.n_rec = g->n_rec;
      q.extra = g->d_extra;
      q.ksm = g->ksm;
      q.kglob = g->kglob;
      q.S = S;
      q.L = g->L;
      q.dense_kind = dk;
      q.dense64 = p.dense64;
      q.dense_ld = sc->dense_ld;
      q.start = p.start;
      q.start_ld = p.start_ld;
      q.makespan = p.makespan;
      q.lane_busy = p.lane_busy;
      q.run_if = flag;
      const int BDq = maxplus_block_dim(S, dk, nsm);
      q.s_pad = (long long)((S + BDq - 1) / BDq) * BDq;
      if (q.kglob > 0) q.gslots = T.scratch<long long>((size_t)q.kglob * q.s_pad);
      CUDA_TRY(launch_maxplus(q, dk == 1 ? reinterpret_cast<const int*>(sc->dense) : nullptr, stream));
    } else {
      if (out->makespan) CUDA_TRY(launch_fill_i64(p.makespan, 0, S, stream));
      if (out->lane_busy) CUDA_TRY(launch_fill_i64(p.lane_busy, 0, (long long)S * g->L, stream));
    }
    if (out->dispatched) CUDA_TRY(launch_fill_i32(out->dispatched, g->n, S, stream));
  } else if (use_max) {
    MaxplusParams p;
    memset(&p, 0, sizeof(p));
    fill_general(p);
    p.S = S;
    p.L = g->L;
    int dmode = 0;
    if (dense_now) {
      if (g->n_chains > 0) fail(KS_ERR_UNSUPPORTED, "dense durations with permutable chains");
      if (sc->dense_ld < S) fail(KS_ERR_INVALID, "dense_ld < n_scenarios");
      if (sc->dense_kind == 1) {
        const bool aligned = (reinterpret_cast<uintptr_t>(sc->dense) % 16 == 0) && (sc->dense_ld % 4 == 0);
        dmode = (aligned && g->n_rec > 0) ? 1 : -1;
        if (dmode < 0) fail(KS_ERR_INVALID, "int32 dense durations need 16B alignment and dense_ld % 4 == 0");
      } else {
        dmode = 2;
        p.dense64 = reinterpret_cast<const long long*>(sc->dense);
      }
      p.dense_ld = sc->dense_ld;
    }
    p.dense_kind = dmode;
    p.start = reinterpret_cast<long long*>(out->start);
    p.start_ld = out->start_ld;
    p.makespan = reinterpret_cast<long long*>(out->makespan);
    p.lane_busy = reinterpret_cast<long long*>(out->lane_busy);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device);
    const int BD = maxplus_block_dim(S, dmode, nsm);
    p.s_pad = (long long)((S + BD - 1) / BD) * BD;
    if (p.kglob > 0) p.gslots = T.scratch<long long>((size_t)p.kglob * p.s_pad);
    CUDA_TRY(launch_maxplus(p, dense_now && dmode == 1 ? reinterpret_cast<const int*>(sc->dense) : nullptr,
                            stream));
    if (out->dispatched) CUDA_TRY(launch_fill_i32(out->dispatched, g->n, S, stream));
  } else {
    ListParams p;
    memset(&p, 0, sizeof(p));
    p.N = g->n;
    p.L = g->L;
    p.S = S;
    p.child_ptr = g->d_child_ptr;
    p.child = g->d_child;
    p.indeg = g->d_indeg;
    p.lane = g->d_lane;
    p.dur = g->d_dur;
    p.gap = g->d_gap;
    p.ready = g->d_ready;
    p.id_rank = g->d_rank;
    p.prio = g->d_prio;
    p.flags = g->d_flags;
    p.group = g->d_group;
    p.vrank = T.vrank;
    p.policy = policy;
    p.zero_time = 0;
    if (dense_now) {
      if (sc->dense_kind == 1)
        p.dense32 = reinterpret_cast<const int*>(sc->dense);
      else
        p.dense64 = reinterpret_cast<const long long*>(sc->dense);
      p.dense_ld = sc->dense_ld;
    }
    p.ovr_row = T.ovr_map;
    p.ovr = T.ovr;
    p.scale_ptr = T.scale_ptr;
    p.scale = T.scale;
    const size_t N = std::max(g->n, 1);
    p.rdy = T.scratch<long long>(2 * N * S);
    p.rem = T.scratch<int>(N * S);
    p.front = T.scratch<int>(N * S);
    p.start = reinterpret_cast<long long*>(out->start);
    p.start_ld = out->start_ld;
    p.makespan = reinterpret_cast<long long*>(out->makespan);
    p.lane_busy = reinterpret_cast<long long*>(out->lane_busy);
    p.schedule = out->schedule;
    p.dispatched = out->dispatched;
    CUDA_TRY(launch_listsched(p, stream));
  }
  CUDA_TRY(cudaGetLastError());
  return KS_OK;
}

}  // namespace

extern "C" {

const char* ks_error_name(int code) {
  switch (code) {
    case KS_OK: return "OK";
    case KS_ERR_DEADLOCK: return "Deadlock";
    case KS_ERR_CYCLE: return "CycleDetected";
    case KS_ERR_INVALID: return "InvalidArgument";
    case KS_ERR_CUDA: return "CudaError";
    case KS_ERR_OOM: return "OutOfMemory";
    case KS_ERR_UNSUPPORTED: return "Unsupported";
    case KS_ERR_ORPHAN: return "OrphanKernel";
    case KS_ERR_AMBIGUOUS: return "AmbiguousMarker";
    case KS_ERR_OVERLAP: return "OverlapViolation";
    case KS_ERR_BAD_PIPELINE: return "BadPipeline";
    case KS_ERR_NO_DEVICE: return "NoDevice";
    case KS_ERR_MALFORMED: return "MalformedDocument";
    case KS_ERR_SCHEMA: return "SchemaViolation";
    default: return "KernsimError";
  }
}

const char* ks_last_error_detail(void) { return g_last_error.c_str(); }

const char* ks_version(void) { return "ddsim 0.1.0 sm_100a"; }

int64_t ks_launch_count(void) { return g_launches.load(); }

int ks_device_count(int* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (n) *n = (e == cudaSuccess) ? c : 0;
  if (e != cudaSuccess) {
    g_last_error = cudaGetErrorString(e);
    return KS_ERR_NO_DEVICE;
  }
  return KS_OK;
}

#define KS_GUARD_BEGIN try {
#define KS_GUARD_END                                              \
  }                                                               \
  catch (const KsError& e) {                                      \
    g_last_error = e.msg;                                         \
    cudaGetLastError();                                           \
    return e.code;                                                \
  }                                                               \
  catch (const std::bad_alloc&) {                                 \
    g_last_error = "host allocation failed";                      \
    return KS_ERR_OOM;                                            \
  }                                                               \
  catch (...) {                                                   \
    g_last_error = "unexpected exception";                        \
    return KS_ERR_INVALID;                                        \
  }

int ks_graph_create(const ks_graph_desc* desc, int device, ks_graph** out, int32_t* order_out) {
  KS_GUARD_BEGIN
  if (!desc || !out) fail(KS_ERR_INVALID, "null argument");
  g_compile_only = getenv("DDSIM_COMPILE_ONLY") != nullptr;
  if (g_compile_only) {
    ks_graph* g = new ks_graph();
    g->device = -1;
    try {
      compile_graph(desc, g);
    } catch (...) {
      free_graph(g);
      throw;
    }
    if (order_out) std::copy(g->order.begin(), g->order.end(), order_out);
    *out = g;
    return KS_OK;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) fail(KS_ERR_NO_DEVICE, "no CUDA device");
  if (device < 0 || device >= ndev) fail(KS_ERR_INVALID, "bad device");
  DevGuard guard(device);
  ks_graph* g = new ks_graph();
  g->device = device;
  try {
    compile_graph(desc, g);
  } catch (...) {
    free_graph(g);
    throw;
  }
  if (order_out) std::copy(g->order.begin(), g->order.end(), order_out);
  *out = g;
  return KS_OK;
  KS_GUARD_END
}

int ks_graph_create_from_ingest(const ks_ingest_dev* h, const int32_t* id_rank,
                                const uint8_t* flags, ks_graph** out, int32_t* order_out) {
  KS_GUARD_BEGIN
  if (!h || !out) fail(KS_ERR_INVALID, "null argument");
  const IngestDev& I = h->d;
  if (I.n > INT32_MAX - 1 || I.m > INT32_MAX - 1) fail(KS_ERR_UNSUPPORTED, "more than 2^31 events");
  DevGuard guard(I.device);
  keep_device_pool(I.device);
  HostTimer gt;
  const int n = (int)I.n, L = I.L;
  DeviceFreeze F;
  std::string err;
  const int rc = freeze_from_ingest(I, id_rank, flags, F, err);
  if (rc != KS_OK) fail(rc, err);
  gt.mark(F.ok ? "device freeze" : "device freeze (fallback)");
  if (gt.on) std::fprintf(stderr, "[compile_graph] relaxation rounds %d\n", F.rounds);
  if (!F.ok) {
    // no trace-time topological order: the host compiler (depth-first Kahn)
    hvec<int32_t> src(I.m), dst(I.m), lo(I.n), lane(I.n), rank(I.n), prio(I.n, 0);
    hvec<int64_t> dur(I.n), gap(I.n), ready(I.n, 0);
    CUDA_TRY(cudaMemcpy(src.data(), I.src, 4 * I.m, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(dst.data(), I.dst, 4 * I.m, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(lo.data(), I.lane_order, 4 * I.n, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(lane.data(), I.lane, 4 * I.n, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(dur.data(), I.dur, 8 * I.n, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(gap.data(), I.gap, 8 * I.n, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) rank[i] = id_rank ? id_rank[i] : i;
    ks_graph_desc d;
    memset(&d, 0, sizeof(d));
    d.n_tasks = n;
    d.n_lanes = L;
    d.duration = dur.data();
    d.gap = gap.data();
    d.ready_time = ready.data();
    d.lane = lane.data();
    d.id_rank = rank.data();
    d.priority = prio.data();
    d.flags = flags;
    d.n_edges = I.m;
    d.edge_src = src.data();
    d.edge_dst = dst.data();
    d.lane_order_ptr = I.lane_order_ptr.data();
    d.lane_order = lo.data();
    return ks_graph_create(&d, I.device, out, order_out);
  }
  ks_graph* g = new ks_graph();
  g->device = I.device;
  g->n = n;
  g->L = L;
  g->chained = true;  // ingest links every lane's events in lane order (rules 1, 2, 5)
  g->n_chains = 0;
  g->n_ordered = n;
  g->n_edges_unique = (int)F.m_unique;
  g->rows_are_records = true;
  g->order.assign(F.order.begin(), F.order.end());
  g->d_child_ptr = F.child_ptr;
  g->d_child = F.child;
  g->d_indeg = F.indeg;
  g->d_lane = F.lane_r;
  g->d_dur = F.dur_r;
  g->d_gap = F.gap_r;
  g->d_ready = F.ready_r;
  g->d_rank = F.rank_r;
  g->d_prio = F.prio_r;
  g->d_flags = F.flags_r;
  g->d_group = F.group_r;
  auto st = std::make_unique<LazyPrograms>();
  st->n = n;
  st->L = L;
  st->E = I.m;
  st->NC = 0;
  st->R = n;
  st->chained = true;
  st->from_device = true;
  st->d_ukeys = F.ukeys;
  st->d_pkeys = F.pkeys;
  st->m_unique = F.m_unique;
  st->lane_order_ptr.assign(I.lane_order_ptr.begin(), I.lane_order_ptr.end());
  if (I.n) {
    CUDA_TRY(cudaMalloc(&st->d_lane_order, sizeof(int) * I.n));
    CUDA_TRY(cudaMemcpy(st->d_lane_order, I.lane_order, sizeof(int) * I.n, cudaMemcpyDeviceToDevice));
  }
  if (F.order_d) cudaFree(F.order_d);
  g->lazy = std::move(st);
  if (order_out) std::copy(g->order.begin(), g->order.end(), order_out);
  *out = g;
  gt.mark("graph");
  if (getenv("DDSIM_EAGER_PROGRAMS") != nullptr) ensure_programs(g);
  return KS_OK;
  KS_GUARD_END
}

int ks_graph_shape(const ks_graph* g, int32_t* chained, int32_t* n_ordered) {
  if (!g) return KS_ERR_INVALID;
  if (chained) *chained = g->chained ? 1 : 0;
  if (n_ordered) *n_ordered = g->n_ordered;
  return KS_OK;
}

int ks_graph_get_info(const ks_graph* g, ks_graph_info* info) {
  if (!g || !info) return KS_ERR_INVALID;
  KS_GUARD_BEGIN
  ensure_programs(g);
  KS_GUARD_END
  info->n_tasks = g->n;
  info->n_lanes = g->L;
  info->n_edges_unique = g->n_edges_unique;
  info->chained = g->chained ? 1 : 0;
  info->n_ordered = g->n_ordered;
  info->n_slots = g->n_slots;
  info->n_slots_smem = g->ksm;
  info->n_levels = g->n_levels;
  info->has_lanes = g->has_lanes ? 1 : 0;
  info->n_lane_slots_smem = g->lksm;
  info->n_lane_slots_global = g->lkglob;
  info->n_lane_cuts = (int)g->lane_cuts.size();
  info->seg_chain_begin = g->seg_c0;
  info->seg_chain_end = g->seg_c1;
  info->n_carries = (int)g->carry_rows.size();
  return KS_OK;
}

int ks_graph_levels(const ks_graph* g, int32_t* level_out) {
  if (!g || !level_out) return KS_ERR_INVALID;
  KS_GUARD_BEGIN
  ensure_programs(g);
  KS_GUARD_END
  std::copy(g->level.begin(), g->level.end(), level_out);
  return KS_OK;
}

int ks_graph_destroy(ks_graph* g) {
  if (!g) return KS_OK;
  if (g->device < 0) {
    delete g;
    return KS_OK;
  }
  DevGuard guard(g->device);
  free_graph(g);
  return KS_OK;
}

int ks_simulate(const ks_graph* g, const ks_scenarios_desc* sc, int policy, int path,
                const ks_sim_out* out, void* stream) {
  KS_GUARD_BEGIN
  return simulate_impl(g, sc, policy, path, out, reinterpret_cast<cudaStream_t>(stream));
  KS_GUARD_END
}

int ks_toposort(const ks_graph* g, int32_t* order_out, int32_t* n_out) {
  KS_GUARD_BEGIN
  if (!g) fail(KS_ERR_INVALID, "null graph");
  ensure_programs(g);
  DevGuard guard(g->device);
  const int n = g->n;
  if (n == 0) {
    if (n_out) *n_out = 0;
    return KS_OK;
  }
  cudaStream_t st;
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  int rc = KS_OK;
  {
    ScenTables T;
    T.st = st;
    ListParams p;
    memset(&p, 0, sizeof(p));
    p.N = n;
    p.L = g->L;
    p.S = 1;
    p.child_ptr = g->d_child_ptr;
    p.child = g->d_child;
    p.indeg = g->d_indeg;
    p.lane = g->d_lane;
    p.dur = g->d_dur;
    p.gap = g->d_gap;
    p.ready = g->d_ready;
    p.id_rank = g->d_rank;
    p.prio = g->d_prio;
    p.flags = g->d_flags;
    p.group = g->d_group;
    p.policy = KS_POLICY_DEFAULT;
    p.zero_time = 1;
    p.schedule = T.scratch<int>(n);
    p.dispatched = T.scratch<int>(1);
    if (g->chained && g->n_chains == 0 && g->bd_ok && g->L <= 32 &&
        getenv("DDSIM_TOPO_LISTSCHED") == nullptr) {
      // lane-chained: the frontier is the set of lane heads (one warp, lanes in lanes)
      if (getenv("DDSIM_TOPO_INDEG") == nullptr) ensure_topo_req(g);
      if (g->topo_req && getenv("DDSIM_TOPO_INDEG") == nullptr) {
        CUDA_TRY(launch_toposort_lanes_req(n, g->L, g->d_bd_ptr, g->d_topo_rec, g->d_req_lane,
                                           g->d_req_pos, p.schedule, p.dispatched, st));
      } else {
        int* deg = (size_t)n * sizeof(int) > 200 * 1024 ? T.scratch<int>(n) : nullptr;
        CUDA_TRY(launch_toposort_lanes(n, g->L, g->d_bd_ptr, g->d_bd_rows, g->d_child_ptr,
                                       g->d_child, g->d_indeg, g->d_rank, deg, p.schedule,
                                       p.dispatched, st));
      }
    } else {
      p.rdy = T.scratch<long long>(2 * (size_t)n);
      p.rem = T.scratch<int>(n);
      p.front = T.scratch<int>(n);
      CUDA_TRY(launch_listsched(p, st));
    }
    std::vector<int> sched(n);
    int nd = 0;
    CUDA_TRY(cudaMemcpyAsync(sched.data(), p.schedule, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&nd, p.dispatched, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int k = 0; k < nd; ++k) order_out[k] = g->order[sched[k]];
    if (n_out) *n_out = nd;
    if (nd < n) {
      g_last_error = "dependency cycle";
      rc = KS_ERR_CYCLE;
    }
  }
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  return rc;
  KS_GUARD_END
}

}  // extern "C"

// ---- host-buffer entry point --------------------------------------------------
namespace {

// Per-thread reusable resources of ks_simulate_host (the drop-in path calls it
// once per simulate(): creating two streams, device buffers and a pinned
// staging buffer per call cost milliseconds).  Buffers up to kHostCacheMax
// bytes are kept and grown; larger ones are allocated for the call only.
constexpr size_t kHostCacheMax = 256u << 20;
struct HostCallCache {
  int device = -1;
  cudaStream_t st[2] = {nullptr, nullptr};
  void* dev[2][6] = {};
  size_t dev_cap[2][6] = {};
  char* staging[2] = {nullptr, nullptr};
  size_t staging_cap[2] = {0, 0};
  void release() {  // errors ignored (the runtime may already be unloading)
    if (device < 0) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    for (int k = 0; k < 2; ++k) {
      for (int j = 0; j < 6; ++j)
        if (dev[k][j]) cudaFree(dev[k][j]);
      if (staging[k]) cudaFreeHost(staging[k]);
      if (st[k]) cudaStreamDestroy(st[k]);
    }
    cudaSetDevice(prev);
    cudaGetLastError();
    *this = HostCallCache{};
  }
  // ks_simulate_host_multi runs each device's shard on a short-lived thread:
  // its cache goes with it
  ~HostCallCache() { release(); }
};
thread_local HostCallCache tl_host;

struct ChunkBufs {
  void* dense = nullptr;
  long long* start = nullptr;
  long long* makespan = nullptr;
  long long* lane_busy = nullptr;
  int* schedule = nullptr;
  int* dispatched = nullptr;
  char* staging = nullptr;  // pinned: small outputs bound for pageable memory
};

// Small per-chunk outputs (makespan, lane_busy, dispatched) headed for
// pageable host memory go through pinned staging and a stream-ordered host
// memcpy: a direct cudaMemcpyAsync into pageable memory blocks the issuing
// thread until the stream drains, which serialised the chunk pipeline.
struct HostCopy {
  void* dst;
  const void* src;
  size_t bytes;
};
void CUDART_CB host_copy_fn(void* p) {
  const HostCopy* c = static_cast<const HostCopy*>(p);
  memcpy(c->dst, c->src, c->bytes);
}
bool host_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

int simulate_host_impl(const ks_graph* g, const ks_scenarios_desc* sc, int policy, int path,
                       const ks_sim_out* out) {
  if (!g || !sc || !out) fail(KS_ERR_INVALID, "null argument");
  ensure_programs(g);
  const int S = sc->n_scenarios;
  if (S <= 0) fail(KS_ERR_INVALID, "n_scenarios must be positive");
  if (sc->dense_kind != 0 && sc->dense != nullptr && sc->dense_ld < S)
    fail(KS_ERR_INVALID, "dense_ld must be >= n_scenarios");
  if (out->start != nullptr && out->start_ld < S)
    fail(KS_ERR_INVALID, "start_ld must be >= n_scenarios");
  DevGuard guard(g->device);
  const long long N = std::max(g->n, 1);
  const bool dense = sc->dense_kind != 0 && sc->dense != nullptr;
  const size_t esz = dense ? (sc->dense_kind == 1 ? 4 : 8) : 0;
  // chunk so that dense-in + start-out of one chunk stay near 4 GiB
  const long long per_scen = N * ((long long)esz + (out->start ? 8 : 0)) + 64;
  // Chunk (dense in + start out) per buffer set: large chunks keep the kernel
  // count low (each launch is latency-bound at small S); two sets must fit in
  // ~60 % of free device memory.  Measured on B200: 4 GB -> 3.6, 16 GB -> 4.4
  // G updates/s end to end on config 4.
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  double chunk_gb = std::min(16.0, 0.3 * (double)free_b / (double)(1ll << 30));
  if (chunk_gb < 0.25) chunk_gb = 0.25;
  if (const char* e = getenv("DDSIM_CHUNK_GB")) chunk_gb = atof(e);
  long long sc_chunk = std::max<long long>(4, (long long)(chunk_gb * (1ll << 30)) / per_scen);
  sc_chunk = std::min<long long>(sc_chunk, S);
  sc_chunk = (sc_chunk + 3) / 4 * 4;
  // chunk boundaries: a 1/4 then a 1/2 chunk so the first D2H starts early and
  // the D2H queue never waits for a full-size H2D, then full chunks (two
  // device buffer sets, alternating streams)
  std::vector<long long> bounds{0};
  if (S > sc_chunk)
    for (long long part : {sc_chunk / 4, sc_chunk / 2}) {
      part = (part + 3) / 4 * 4;
      if (part >= 4 && bounds.back() + part < S) bounds.push_back(bounds.back() + part);
    }
  while (bounds.back() < S) bounds.push_back(std::min<long long>(S, bounds.back() + sc_chunk));
  const int nchunks = (int)bounds.size() - 1;
  HostCallCache& HC = tl_host;
  if (HC.device != g->device) {  // first call of this thread on this device
    HC.release();
    CUDA_TRY(cudaStreamCreateWithFlags(&HC.st[0], cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&HC.st[1], cudaStreamNonBlocking));
    HC.device = g->device;
  }
  cudaStream_t st[2] = {HC.st[0], HC.st[1]};
  std::vector<void*> temp_dev, temp_host;  // uncached (large) buffers of this call
  ChunkBufs buf[2];
  const long long ldc = sc_chunk;  // multiple of 4
  const size_t stage_bytes = (size_t)ldc * (8 + 8 * std::max(g->L, 1) + 4);
  const bool ms_pinned = !out->makespan || host_pinned(out->makespan);
  const bool lb_pinned = !out->lane_busy || host_pinned(out->lane_busy);
  const bool dp_pinned = !out->dispatched || host_pinned(out->dispatched);
  std::deque<HostCopy> copies;
  // D2H of n bytes from device src to host dst (staged at stage_off if dst is pageable)
  auto d2h = [&](void* dst, const void* src, size_t n, bool pinned, ChunkBufs& b, size_t stage_off,
                 cudaStream_t stream) {
    if (pinned) {
      CUDA_TRY(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, stream));
      return;
    }
    CUDA_TRY(cudaMemcpyAsync(b.staging + stage_off, src, n, cudaMemcpyDeviceToHost, stream));
    copies.push_back(HostCopy{dst, b.staging + stage_off, n});
    CUDA_TRY(cudaLaunchHostFunc(stream, host_copy_fn, &copies.back()));
  };
  auto dev_get = [&](int k, int slot, size_t bytes) -> void* {
    if (bytes > kHostCacheMax) {
      void* p = nullptr;
      CUDA_TRY(cudaMalloc(&p, bytes));
      temp_dev.push_back(p);
      return p;
    }
    if (HC.dev_cap[k][slot] < bytes) {
      if (HC.dev[k][slot]) cudaFree(HC.dev[k][slot]);
      HC.dev[k][slot] = nullptr;
      HC.dev_cap[k][slot] = 0;
      CUDA_TRY(cudaMalloc(&HC.dev[k][slot], bytes));
      HC.dev_cap[k][slot] = bytes;
    }
    return HC.dev[k][slot];
  };
  auto alloc = [&](ChunkBufs& b, int k) {
    if (dense) b.dense = dev_get(k, 0, esz * N * ldc);
    if (out->start) b.start = static_cast<long long*>(dev_get(k, 1, 8 * N * ldc));
    if (out->makespan) b.makespan = static_cast<long long*>(dev_get(k, 2, 8 * ldc));
    if (out->lane_busy)
      b.lane_busy = static_cast<long long*>(dev_get(k, 3, 8 * ldc * std::max(g->L, 1)));
    if (out->schedule) b.schedule = static_cast<int*>(dev_get(k, 4, 4 * N * ldc));
    if (out->dispatched) b.dispatched = static_cast<int*>(dev_get(k, 5, 4 * ldc));
    if (stage_bytes > kHostCacheMax) {
      CUDA_TRY(cudaHostAlloc(&b.staging, stage_bytes, cudaHostAllocDefault));
      temp_host.push_back(b.staging);
    } else {
      if (HC.staging_cap[k] < stage_bytes) {
        if (HC.staging[k]) cudaFreeHost(HC.staging[k]);
        HC.staging[k] = nullptr;
        HC.staging_cap[k] = 0;
        CUDA_TRY(cudaHostAlloc(&HC.staging[k], stage_bytes, cudaHostAllocDefault));
        HC.staging_cap[k] = stage_bytes;
      }
      b.staging = HC.staging[k];
    }
  };
  auto release = [&]() {
    for (void* p : temp_dev) cudaFree(p);
    for (void* p : temp_host) cudaFreeHost(p);
  };
  int rc = KS_OK;
  try {
    alloc(buf[0], 0);
    if (nchunks > 1) alloc(buf[1], 1);
    // DDSIM_HOST_TRACE=1: per-chunk event timeline on stderr (diagnostics)
    const bool trace = getenv("DDSIM_HOST_TRACE") != nullptr;
    std::vector<cudaEvent_t> ev;
    auto mark = [&](cudaStream_t s) {
      if (!trace) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, s);
      ev.push_back(e);
    };
    // per-chunk host slices of the scenario tables (kept alive to the end)
    std::vector<std::vector<int>> sptr(nchunks);
    std::vector<std::vector<long long>> ovr(nchunks);
    std::vector<std::vector<short>> perm(nchunks);
    std::vector<std::vector<unsigned char>> pres(nchunks);
    // Copies run FIFO per direction (chunk c's H2D after chunk c-1's, same for
    // D2H): concurrent same-direction copies would split the link, and both
    // buffer sets would drain at once instead of one refilling while the
    // other drains (measured on B200: H2D then overlaps D2H).
    cudaEvent_t h2d_done[2], d2h_done[2];
    for (int k = 0; k < 2; ++k) {
      CUDA_TRY(cudaEventCreateWithFlags(&h2d_done[k], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&d2h_done[k], cudaEventDisableTiming));
    }
    struct EvGuard {
      cudaEvent_t* a;
      ~EvGuard() {
        for (int k = 0; k < 4; ++k) cudaEventDestroy(a[k]);
      }
    };
    cudaEvent_t evs[4] = {h2d_done[0], h2d_done[1], d2h_done[0], d2h_done[1]};
    EvGuard evg{evs};
    for (int c = 0; c < nchunks; ++c) {
      const long long s0 = bounds[c];
      const int n_s = (int)(bounds[c + 1] - s0);
      ChunkBufs& b = buf[c & 1];
      cudaStream_t stream = st[c & 1];
      ks_scenarios_desc sub = *sc;
      sub.n_scenarios = n_s;
      mark(stream);
      if (c > 0) CUDA_TRY(cudaStreamWaitEvent(stream, h2d_done[(c - 1) & 1], 0));
      if (dense) {
        CUDA_TRY(cudaMemcpy2DAsync(b.dense, esz * ldc,
                                   static_cast<const char*>(sc->dense) + esz * s0, esz * sc->dense_ld,
                                   esz * n_s, g->n, cudaMemcpyHostToDevice, stream));
        sub.dense = b.dense;
        sub.dense_ld = ldc;
      }
      if (sc->scale_ptr && sc->scale) {
        sptr[c].resize(n_s + 1);
        for (int k = 0; k <= n_s; ++k) sptr[c][k] = sc->scale_ptr[s0 + k] - sc->scale_ptr[s0];
        sub.scale_ptr = sptr[c].data();
        sub.scale = sc->scale + sc->scale_ptr[s0];
      }
      if (sc->n_overrides > 0) {
        ovr[c].resize((size_t)sc->n_overrides * n_s);
        for (int k = 0; k < sc->n_overrides; ++k)
          memcpy(&ovr[c][(size_t)k * n_s], sc->override + (size_t)k * S + s0, 8 * (size_t)n_s);
        sub.override = reinterpret_cast<const int64_t*>(ovr[c].data());
      }
      if (sc->chain_perm) {
        perm[c].assign(sc->chain_perm + s0 * sc->perm_ld, sc->chain_perm + (s0 + n_s) * sc->perm_ld);
        sub.chain_perm = perm[c].data();
      }
      if (sc->chain_present && g->n_chains > 0) {
        pres[c].assign(sc->chain_present + s0 * g->n_chains,
                       sc->chain_present + (s0 + n_s) * g->n_chains);
        sub.chain_present = pres[c].data();
      }
      ks_sim_out o;
      o.start = reinterpret_cast<int64_t*>(b.start);
      o.start_ld = ldc;
      o.makespan = reinterpret_cast<int64_t*>(b.makespan);
      o.lane_busy = reinterpret_cast<int64_t*>(b.lane_busy);
      o.schedule = b.schedule;
      o.dispatched = b.dispatched;
      CUDA_TRY(cudaEventRecord(h2d_done[c & 1], stream));
      mark(stream);
      simulate_impl(g, &sub, policy, path, &o, stream);
      mark(stream);
      if (c > 0) CUDA_TRY(cudaStreamWaitEvent(stream, d2h_done[(c - 1) & 1], 0));
      mark(stream);
      if (out->start)
        CUDA_TRY(cudaMemcpy2DAsync(out->start + s0, 8 * out->start_ld, b.start, 8 * ldc, 8 * n_s,
                                   g->n, cudaMemcpyDeviceToHost, stream));
      if (out->makespan) d2h(out->makespan + s0, b.makespan, 8 * n_s, ms_pinned, b, 0, stream);
      if (out->lane_busy)
        d2h(out->lane_busy + s0 * g->L, b.lane_busy, 8 * (size_t)n_s * g->L, lb_pinned, b,
            8 * (size_t)ldc, stream);
      if (out->schedule)
        CUDA_TRY(cudaMemcpyAsync(out->schedule + s0 * g->n, b.schedule, 4 * (size_t)n_s * g->n,
                                 cudaMemcpyDeviceToHost, stream));
      if (out->dispatched)
        d2h(out->dispatched + s0, b.dispatched, 4 * n_s, dp_pinned, b,
            (size_t)ldc * (8 + 8 * std::max(g->L, 1)), stream);
      CUDA_TRY(cudaEventRecord(d2h_done[c & 1], stream));
      mark(stream);
    }
    CUDA_TRY(cudaStreamSynchronize(st[0]));
    CUDA_TRY(cudaStreamSynchronize(st[1]));
    if (trace && !ev.empty()) {
      fprintf(stderr, "ks_simulate_host: %d chunks of %lld scenarios\n", nchunks, sc_chunk);
      for (size_t k = 0; k + 4 < ev.size(); k += 5) {
        float t[5];
        for (int j = 0; j < 5; ++j) cudaEventElapsedTime(&t[j], ev[0], ev[k + j]);
        fprintf(stderr, "  chunk %zu: issue %.1f  h2d..%.1f  kernel..%.1f  d2h %.1f-%.1f ms\n",
                k / 5, t[0], t[1], t[2], t[3], t[4]);
      }
      for (auto e : ev) cudaEventDestroy(e);
    }
  } catch (...) {
    cudaStreamSynchronize(st[0]);
    cudaStreamSynchronize(st[1]);
    release();
    throw;
  }
  release();
  return rc;
}

}  // namespace

namespace {

int breakdown_impl(const ks_graph* g, const ks_scenarios_desc* sc, const int64_t* start,
                   int64_t start_ld, const int64_t* makespan, const ks_breakdown_desc* bd,
                   int64_t* parts, int64_t* layer_busy, cudaStream_t stream) {
  if (!g || !sc || !bd || !start || !makespan) fail(KS_ERR_INVALID, "null argument");
  ensure_programs(g);
  if (g->device < 0) fail(KS_ERR_NO_DEVICE, "graph was compiled without a device");
  const int S = sc->n_scenarios;
  if (S <= 0) fail(KS_ERR_INVALID, "n_scenarios must be positive");
  const bool sched = bd->schedule != nullptr;
  if (!g->bd_ok && !sched)
    fail(KS_ERR_UNSUPPORTED,
         "batched breakdown needs a lane-chained graph (at most one permutable chain per lane) "
         "or the list scheduler's dispatch order (ks_breakdown_desc.schedule)");
  if (sched && g->n_chains > 0)
    fail(KS_ERR_UNSUPPORTED, "permutable chains run on the max-plus path (no dispatch order)");
  if (g->L > 32) fail(KS_ERR_UNSUPPORTED, "batched breakdown supports at most 32 lanes");
  if (!g->gap_nonneg) fail(KS_ERR_UNSUPPORTED, "batched breakdown needs non-negative gaps");
  if (!bd->row_class) fail(KS_ERR_INVALID, "row_class is required");
  if (layer_busy && bd->row_layer) {
    for (int r = 0; r < g->n; ++r)
      if (bd->row_layer[r] < 0 || bd->row_layer[r] >= bd->n_layers)
        fail(KS_ERR_INVALID, "row_layer out of range");
  }
  DevGuard guard(g->device);
  ScenTables T;
  T.st = stream;
  build_tables(g, sc, T, true, false);
  BreakdownParams p;
  memset(&p, 0, sizeof(p));
  p.n = g->n;
  p.L = g->L;
  p.S = S;
  p.n_chains = g->n_chains;
  p.lane_ptr = sched ? g->d_bd_all_ptr : g->d_bd_ptr;
  p.lane_rows = sched ? nullptr : g->d_bd_rows;
  p.lane_chain = g->d_bd_lane_chain;
  p.chains = g->d_bd_chains;
  p.member_rows = g->d_bd_member_rows;
  p.perm = T.perm;
  p.perm_ld = sc->perm_ld;
  p.present = T.present;
  p.row_class = T.up(bd->row_class, (size_t)g->n);
  p.gap = g->d_gap;
  if (sc->dense_kind != 0 && sc->dense != nullptr) {
    if (sc->dense_ld < S) fail(KS_ERR_INVALID, "dense_ld < n_scenarios");
    p.dkind = sc->dense_kind == 1 ? 1 : 2;
    p.dur = sc->dense;
    p.dld = sc->dense_ld;
  } else {
    // derived durations (base, overrides, scale steps) materialised once
    long long* buf = T.scratch<long long>((size_t)g->n * S);
    CUDA_TRY(launch_expand_durations(g->d_dur, g->d_group, T.ovr_map, T.ovr, T.scale_ptr, T.scale,
                                     g->n, S, S, buf, stream));
    p.dkind = 2;
    p.dur = buf;
    p.dld = S;
  }
  if (start_ld < S) fail(KS_ERR_INVALID, "start_ld must be >= n_scenarios");
  p.start = reinterpret_cast<const long long*>(start);
  p.start_ld = start_ld;
  p.makespan = reinterpret_cast<const long long*>(makespan);
  p.comm_as_gpu = bd->comm_as_gpu;
  p.dataload_as_cpu = bd->dataload_as_cpu;
  p.gaps_as_cpu_busy = bd->gaps_as_cpu_busy;
  p.parts = reinterpret_cast<long long*>(parts);
  p.bad = T.scratch<int>((size_t)S);
  p.start_may_be_neg = (g->n_chains > 0 || T.has_remove) ? 1 : 0;
  {
    // time windows per scenario: (scenario, window) threads for ~4 waves of
    // the lean merge (measured at 65,536 x 100k: K = 5 / 10 / 20 -> 92 / 67 /
    // 76 ms), at least ~192 rows of work per window (config 3, 4,000 x 29.6k: 57 -> 152
    // windows 11.9 -> 10.2 ms) -- ~16 below 1,024
    // scenarios, where one thread's dependent walk is the whole latency
    // (one scenario: 10k rows 0.71 -> 0.26 ms, 100k rows 2.0 -> 1.0 ms with 16-row windows
    // and short per-layer chunks)
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device);
    const long long target = (long long)nsm * 4096;
    long long K = (target + S - 1) / S;
    K = std::min<long long>(K, std::max(1, g->n / (S >= 1024 ? 192 : 16)));
    p.K = (int)std::max<long long>(1, std::min<long long>(K, 65535));
    if (const char* e = getenv("DDSIM_BD_WINDOWS")) p.K = std::max(1, atoi(e));
    p.stream_loads = getenv("DDSIM_BD_STREAM") != nullptr;
    // row-order streaming sweep (lane-chained graphs): DDSIM_BD_SWEEP=1 forces
    // it, =-1 disables it; DDSIM_BD_SWEEP_DEPTH caps its pending runs per lane
    // packed per-row class / gap codes for both merges; the sweep also needs
    // the row lanes (lane-chained rows, no permutable chains, <= 4 lanes)
    p.rinfo = T.scratch<long long>((size_t)g->n);
    if (!sched && g->n_chains == 0 && g->L <= 4) {
      p.row_lane = g->d_lane;
      if (layer_busy && bd->row_layer) p.linfo = T.scratch<int>((size_t)g->n);
    }
    if (const char* e = getenv("DDSIM_BD_SWEEP")) p.stream_mode = atoi(e);
    if (const char* e = getenv("DDSIM_BD_SWEEP_DEPTH")) p.stream_depth = atoi(e);
  }
  if (layer_busy && bd->row_layer) {
    p.row_layer = T.up(bd->row_layer, (size_t)g->n);
    p.layer_busy = reinterpret_cast<long long*>(layer_busy);
    p.n_layers = bd->n_layers;
  }
  if (sched && g->n > 0) {
    // per-scenario lane sequences: the dispatch order split by lane (a lane
    // runs one task at a time, lane_progress = finish + gap, sim.py:128, so
    // each lane's intervals are sorted and disjoint in dispatch order)
    int* srows = T.scratch<int>((size_t)g->n * S);
    CUDA_TRY(launch_bd_sched_rows(bd->schedule, g->d_lane, g->d_bd_all_ptr, g->n, g->L, S, srows,
                                  stream));
    p.srows = srows;
  }
  if (g->n > 0) CUDA_TRY(launch_breakdown(p, stream));
  return KS_OK;
}

}  // namespace

extern "C" int ks_breakdown(const ks_graph* g, const ks_scenarios_desc* sc, const int64_t* start,
                            int64_t start_ld, const int64_t* makespan, const ks_breakdown_desc* bd,
                            int64_t* parts, int64_t* layer_busy, void* stream) {
  KS_GUARD_BEGIN
  return breakdown_impl(g, sc, start, start_ld, makespan, bd, parts, layer_busy,
                        static_cast<cudaStream_t>(stream));
  KS_GUARD_END
}

extern "C" int ks_simulate_host(const ks_graph* g, const ks_scenarios_desc* sc, int policy,
                                int path, const ks_sim_out* out) {
  KS_GUARD_BEGIN
  return simulate_host_impl(g, sc, policy, path, out);
  KS_GUARD_END
}

// Scenario shards over several devices (one host thread per device).  Each
// shard gets a sub-description whose per-scenario tables are sliced (scale
// programs rebased, overrides repacked) and whose outputs point into the
// caller's host buffers at the shard's offset.
extern "C" int ks_simulate_host_multi(const ks_graph* const* graphs, int n_graphs,
                                      const ks_scenarios_desc* sc, int policy, int path,
                                      const ks_sim_out* out) {
  using namespace ddsim;
  if (!graphs || n_graphs < 1 || !sc || !out) {
    set_last_error("ks_simulate_host_multi: bad arguments");
    return KS_ERR_INVALID;
  }
  for (int k = 0; k < n_graphs; ++k) {
    if (!graphs[k] || graphs[k]->n != graphs[0]->n || graphs[k]->L != graphs[0]->L ||
        graphs[k]->order != graphs[0]->order) {
      set_last_error("ks_simulate_host_multi: graphs differ (freeze the same description)");
      return KS_ERR_INVALID;
    }
  }
  const int S = sc->n_scenarios;
  const ks_graph* g0 = graphs[0];
  const int K = std::max(1, std::min(n_graphs, S));
  std::vector<int> bounds(K + 1, 0);
  for (int k = 0; k <= K; ++k) bounds[k] = (int)((long long)S * k / K);
  std::vector<int> rc(K, KS_OK);
  std::vector<std::string> msg(K);
  std::vector<std::thread> th;
  for (int k = 0; k < K; ++k) {
    th.emplace_back([&, k] {
      const int s0 = bounds[k], ns = bounds[k + 1] - bounds[k];
      if (ns == 0) return;
      ks_scenarios_desc sub = *sc;
      sub.n_scenarios = ns;
      std::vector<int64_t> ovr;
      std::vector<int32_t> sptr;
      if (sc->dense) {
        const size_t es = sc->dense_kind == 1 ? 4 : 8;
        sub.dense = static_cast<const char*>(sc->dense) + es * (size_t)s0;
      }
      if (sc->n_overrides > 0) {
        ovr.resize((size_t)sc->n_overrides * ns);
        for (int j = 0; j < sc->n_overrides; ++j)
          memcpy(&ovr[(size_t)j * ns], sc->override + (size_t)j * S + s0, 8 * (size_t)ns);
        sub.override = ovr.data();
      }
      if (sc->scale_ptr) {
        sptr.resize(ns + 1);
        for (int j = 0; j <= ns; ++j) sptr[j] = sc->scale_ptr[s0 + j] - sc->scale_ptr[s0];
        sub.scale_ptr = sptr.data();
        sub.scale = sc->scale + sc->scale_ptr[s0];
      }
      if (sc->chain_perm) sub.chain_perm = sc->chain_perm + (size_t)s0 * sc->perm_ld;
      if (sc->chain_present) sub.chain_present = sc->chain_present + (size_t)s0 * g0->n_chains;
      ks_sim_out o = *out;
      if (out->start) o.start = out->start + s0;
      if (out->makespan) o.makespan = out->makespan + s0;
      if (out->lane_busy) o.lane_busy = out->lane_busy + (size_t)s0 * g0->L;
      if (out->schedule) o.schedule = out->schedule + (size_t)s0 * g0->n;
      if (out->dispatched) o.dispatched = out->dispatched + s0;
      rc[k] = ks_simulate_host(graphs[k], &sub, policy, path, &o);
      if (rc[k] != KS_OK) msg[k] = ks_last_error_detail();
    });
  }
  for (auto& t : th) t.join();
  for (int k = 0; k < K; ++k)
    if (rc[k] != KS_OK) {
      set_last_error("device shard " + std::to_string(k) + ": " + msg[k]);
      return rc[k];
    }
  return KS_OK;
}
