// breakdown: batched runtime decomposition of max-plus results.
//
// Reference: kernsim.breakdown.compute_breakdown / per_layer_breakdown
// (pkg/src/kernsim/breakdown.py:42-111).  The reference sweeps the sorted set
// of interval endpoints of one schedule and classifies each elementary span of
// [0, makespan) as CPU-only, GPU-only, both, or idle.
//
// Device formulation: on a lane-chained graph every lane's tasks execute in
// lane order and never overlap (start(next) >= start + dur + gap with
// dur, gap >= 0), so each lane's non-empty intervals -- CPU tasks
// [start, end + gap) (gaps_as_cpu_busy), GPU/comm tasks [start, end) -- are
// already sorted and disjoint.  Merging the L lane sequences in time order
// with per-class active counters yields exactly the reference's
// classification without materialising or sorting the endpoint set.
//
// Parallelism: [0, makespan) of each scenario is cut into K time windows; a
// thread owns one (scenario, window), binary-searches every lane for the last
// interval starting at or before its window (lane starts are sorted), merges
// up to the window end and adds its four sums atomically.  Threads of a warp
// hold consecutive scenarios of the same window, so their rows stay close and
// loads mostly share sectors.  Scenarios with a negative duration (which can
// break the sortedness) are found first by a coalesced pass and reported as -1.
//
// Memory: per event one start (8 B) and one duration (4/8 B) read.
// per_layer_breakdown is a row-sequential kernel with run-length register
// accumulation and coalesced read-modify-write of [layer][class][S].
#include "ddsim_internal.h"

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <type_traits>

namespace ddsim {

constexpr int kBdMaxLanes = 32;
enum { BD_CPU = 0, BD_GPU = 1, BD_COMM = 2, BD_CPU_DATALOAD = 3 };

struct LaneCursor {
  int v, len;          // next virtual position to prefetch, sequence length
  long long a, b;      // current interval
  int cls;             // 0 cpu, 1 gpu; -1 exhausted
  bool active;
  bool chain_on;       // the lane's permutable chain is present in this scenario
  // prefetched next candidate (loads issued one interval ahead so their
  // latency overlaps the other lanes' merge steps)
  int nrow;            // -1: none
  int nrc;
  long long nst, nd, ngap;
};

__device__ __forceinline__ long long bd_dur(const BreakdownParams& p, int row, int s) {
  if (p.dkind == 1) return (long long)static_cast<const int*>(p.dur)[(long long)row * p.dld + s];
  return static_cast<const long long*>(p.dur)[(long long)row * p.dld + s];
}

// CH: the graph has permutable chains (otherwise a lane's v-th row is a plain lookup)
template <bool CH>
__device__ __forceinline__ int bd_row(const BreakdownParams& p, int l, int v, int s, bool chain_on) {
  const int base = p.lane_ptr[l];
  if (p.srows) return p.srows[(long long)s * p.n + base + v];
  if (!CH) return p.lane_rows[base + v];
  const int c = p.lane_chain[l];
  if (c < 0 || !chain_on) return p.lane_rows[base + v];
  const BdChain ch = p.chains[c];
  if (v < ch.pos) return p.lane_rows[base + v];
  if (v < ch.pos + ch.B) {
    const int k = v - ch.pos;
    const int m = p.perm ? (int)p.perm[(long long)s * p.perm_ld + ch.perm_off + k] : k;
    return p.member_rows[ch.member_off + m];
  }
  return p.lane_rows[base + v - ch.B];
}

template <bool CH>
__device__ __forceinline__ void bd_prefetch(const BreakdownParams& p, LaneCursor& c, int l, int s) {
  if (c.v >= c.len) {
    c.nrow = -1;
    return;
  }
  const int row = bd_row<CH>(p, l, c.v, s, c.chain_on);
  ++c.v;
  c.nrow = row;
  // default caching: the scenarios of a warp reach a row at slightly
  // different times (their seek positions differ), so each 32 B sector serves
  // 4 threads across a short interval; an evict-first load re-fetched it
  c.nst = p.stream_loads ? __ldcs(&p.start[(long long)row * p.start_ld + s])
                         : p.start[(long long)row * p.start_ld + s];
  c.nd = bd_dur(p, row, s);
  c.nrc = __ldg(&p.row_class[row]);
  c.ngap = __ldg(&p.gap[row]);
}

// advance lane l to its next non-empty interval (cls = -1 when exhausted)
template <bool CH>
__device__ __forceinline__ void bd_advance(const BreakdownParams& p, LaneCursor& c, int l, int s) {
  while (c.nrow >= 0) {
    const long long st = c.nst, d = c.nd, gp = c.ngap;
    const int rc = c.nrc;
    bd_prefetch<CH>(p, c, l, s);
    if (st < 0) continue;  // removed task / absent chain member (start -1)
    long long e = st + d;
    int cls;
    if (rc == BD_CPU || rc == BD_CPU_DATALOAD) {
      if (rc == BD_CPU_DATALOAD && !p.dataload_as_cpu) continue;
      if (p.gaps_as_cpu_busy) e += gp;
      cls = 0;
    } else if (rc == BD_GPU) {
      cls = 1;
    } else {
      cls = p.comm_as_gpu ? 1 : 0;
    }
    if (e <= st) continue;
    c.a = st;
    c.b = e;
    c.cls = cls;
    return;
  }
  c.cls = -1;
}

// start of the lane's v-th row, -1 for removed / absent tasks
template <bool CH>
__device__ __forceinline__ long long bd_key(const BreakdownParams& p, int l, int v, int s, bool on) {
  return p.start[(long long)bd_row<CH>(p, l, v, s, on) * p.start_ld + s];
}

// Position to start lane l's scan for a window beginning at T0: the last row
// whose start is <= T0 (earlier intervals end before it starts), 0 if none.
template <bool CH>
__device__ int bd_seek(const BreakdownParams& p, int l, int len, int s, bool on, long long T0) {
  int lo = 0, hi = len;  // first v with key(v) > T0 lies in [lo, hi]
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    int m2 = mid;
    long long k = bd_key<CH>(p, l, m2, s, on);
    while (k == -1 && m2 + 1 < hi) k = bd_key<CH>(p, l, ++m2, s, on);
    if (k == -1 || k > T0)
      hi = mid;
    else
      lo = m2 + 1;
  }
  int v = lo - 1;
  while (v > 0 && bd_key<CH>(p, l, v, s, on) == -1) --v;
  return v < 0 ? 0 : v;
}

__device__ __forceinline__ long long mul_div(long long a, long long k, long long K) {
  return (long long)(((__int128)a * k) / K);
}

// Pass 1: zero the outputs and the negative-duration flags; pass 2 flags
// scenarios with a negative duration, row chunks x scenarios in parallel
// (coalesced across the scenarios of a warp).
__global__ void bd_zero_kernel(const BreakdownParams p) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < p.S; s += gridDim.x * blockDim.x) {
    p.bad[s] = 0;
    long long* o = p.parts + (long long)s * 4;
    o[0] = o[1] = o[2] = o[3] = 0;
  }
}
constexpr int kBdNegRows = 1024;
__global__ void bd_negative_kernel(const BreakdownParams p) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= p.S) return;
  const int r0 = blockIdx.y * kBdNegRows, r1 = min(p.n, r0 + kBdNegRows);
  int bad = 0;
  if (p.dkind == 1) {
    const int* d = static_cast<const int*>(p.dur) + s;
#pragma unroll 8
    for (int row = r0; row < r1; ++row) bad |= __ldcs(d + (long long)row * p.dld);
    bad = bad < 0;
  } else {
    const long long* d = static_cast<const long long*>(p.dur) + s;
    long long b = 0;
#pragma unroll 8
    for (int row = r0; row < r1; ++row) b |= __ldcs(d + (long long)row * p.dld);
    bad = b < 0;
  }
  if (bad) atomicOr(p.bad + s, 1);
}

// LM: lane capacity (>= L), a compile-time bound so that the per-lane cursors
// live in registers (every access below is an unrolled loop over l); EXACT:
// LM == L (no per-lane bound checks); CH: permutable chains present.
template <int LM, bool EXACT, bool CH>
__global__ void __launch_bounds__(128) breakdown_kernel(const BreakdownParams p) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (s >= p.S) return;
  long long* o = p.parts + (long long)s * 4;
  if (p.bad[s]) {
    if (k == 0) o[0] = o[1] = o[2] = o[3] = -1;
    return;
  }
  const long long ms = p.makespan[s];
  const long long T0 = mul_div(ms, k, p.K), T1 = mul_div(ms, k + 1, p.K);
  if (T1 <= T0) return;
  LaneCursor cur[LM];
#pragma unroll
  for (int l = 0; l < LM; ++l) {
    LaneCursor& c = cur[l];
    c.cls = -1;
    c.active = false;
    c.nrow = -1;
    if (!EXACT && l >= p.L) continue;
    const int c_ix = CH ? p.lane_chain[l] : -1;
    bool chain_on = false;
    int len = p.lane_ptr[l + 1] - p.lane_ptr[l];
    if (CH && c_ix >= 0) {
      chain_on = p.present == nullptr || p.present[(long long)s * p.n_chains + c_ix] != 0;
      if (chain_on) len += p.chains[c_ix].B;
    }
    c.len = len;
    c.chain_on = chain_on;
    c.v = len > 0 && T0 > 0 ? bd_seek<CH>(p, l, len, s, chain_on, T0) : 0;
    bd_prefetch<CH>(p, c, l, s);
  }
#pragma unroll
  for (int l = 0; l < LM; ++l)
    if (EXACT || l < p.L) bd_advance<CH>(p, cur[l], l, s);
  long long acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;  // cpu_only, gpu_only, parallel, idle
  int cc = 0, gc = 0;
  long long t = T0;
  while (true) {
    int best = -1;
    long long ev = LLONG_MAX;
#pragma unroll
    for (int l = 0; l < LM; ++l) {
      if (cur[l].cls >= 0) {
        const long long e = cur[l].active ? cur[l].b : cur[l].a;
        if (e < ev) {
          ev = e;
          best = l;
        }
      }
    }
    const long long te = best < 0 ? T1 : min(ev, T1);
    if (te > t) {
      const long long span = te - t;
      if (cc > 0 && gc > 0)
        acc2 += span;
      else if (cc > 0)
        acc0 += span;
      else if (gc > 0)
        acc1 += span;
      else
        acc3 += span;
      t = te;
    }
    if (best < 0 || ev >= T1) break;
#pragma unroll
    for (int l = 0; l < LM; ++l) {
      // predicated per-lane copies keep the cursors in registers (a dynamic
      // cur[best] puts them in local memory: measured 1.35x slower)
      if (l != best) continue;
      LaneCursor& c = cur[l];
      if (c.active) {
        if (c.cls == 0) --cc; else --gc;
        c.active = false;
        bd_advance<CH>(p, c, l, s);
      } else {
        if (c.cls == 0) ++cc; else ++gc;
        c.active = true;
      }
    }
  }
  unsigned long long* u = reinterpret_cast<unsigned long long*>(o);
  if (acc0) atomicAdd(u + 0, (unsigned long long)acc0);
  if (acc1) atomicAdd(u + 1, (unsigned long long)acc1);
  if (acc2) atomicAdd(u + 2, (unsigned long long)acc2);
  if (acc3) atomicAdd(u + 3, (unsigned long long)acc3);
}

// Class of a row's interval under the call's options (0 cpu, 1 gpu, 3 not
// counted) and the gap it carries as CPU busy: one 8-byte row code when the
// row codes were built (bd_rowinfo_kernel), else from row_class / gap
__device__ __forceinline__ int bd_class(const BreakdownParams& p, int row, long long& gapx) {
  if (p.rinfo) {
    const long long info = __ldg(&p.rinfo[row]);
    if (info >= 0) {
      gapx = info >> 12;
      return (int)(info >> 8) & 3;
    }
  }
  const int rc = __ldg(&p.row_class[row]);
  gapx = 0;
  if (rc == BD_CPU || rc == BD_CPU_DATALOAD) {
    if (rc == BD_CPU_DATALOAD && !p.dataload_as_cpu) return 3;
    if (p.gaps_as_cpu_busy) gapx = __ldg(&p.gap[row]);
    return 0;
  }
  if (rc == BD_GPU) return 1;
  return p.comm_as_gpu ? 1 : 0;
}

// Lean merge (L <= 8): the per-lane cursor state lives in shared memory
// (structure of arrays, [lane][thread]) so an event touches its lane through a
// dynamic index -- one copy of the advance code per event instead of LM
// divergent copies.  Only the per-lane next event time and the prefetched next
// interval (start, duration) stay in registers, updated by predicated selects.
constexpr int kBdLeanBD = 128;
template <int LM>
struct BdLean {
  int v[LM][kBdLeanBD];        // next position to prefetch
  int len[LM][kBdLeanBD];
  int nrow[LM][kBdLeanBD];     // prefetched row (-1: none)
  int cls[LM][kBdLeanBD];      // class of the current interval (0 cpu, 1 gpu)
  int act[LM][kBdLeanBD];      // inside the current interval
  unsigned char on[LM][kBdLeanBD];  // the lane's chain is present
  long long b[LM][kBdLeanBD];  // end of the current interval
};

template <int LM, bool EXACT, bool CH>
__global__ void __launch_bounds__(kBdLeanBD) breakdown_lean_kernel(const BreakdownParams p) {
  __shared__ BdLean<LM> sh;
  const int tid = threadIdx.x;
  const int s = blockIdx.x * kBdLeanBD + tid;
  const int k = blockIdx.y;
  if (s >= p.S) return;
  long long* o = p.parts + (long long)s * 4;
  const int bad = p.bad[s];
  if (p.redo && bad != 2) return;  // only the scenarios the streaming sweep handed back
  if (bad & 1) {
    if (k == 0) o[0] = o[1] = o[2] = o[3] = -1;
    return;
  }
  const long long ms = p.makespan[s];
  const long long T0 = mul_div(ms, k, p.K), T1 = mul_div(ms, k + 1, p.K);
  if (T1 <= T0) return;
  long long e[LM], pst[LM], pd[LM];  // next event; prefetched next interval
#pragma unroll
  for (int l = 0; l < LM; ++l) e[l] = pst[l] = pd[l] = LLONG_MAX;

  // prefetch lane l's row at position v (into pst / pd of lane l)
  auto prefetch = [&](int l) {
    const int v = sh.v[l][tid];
    int row = -1;
    long long a = 0, d = 0;
    if (v < sh.len[l][tid]) {
      row = bd_row<CH>(p, l, v, s, sh.on[l][tid] != 0);
      a = p.stream_loads ? __ldcs(&p.start[(long long)row * p.start_ld + s])
                         : p.start[(long long)row * p.start_ld + s];
      d = bd_dur(p, row, s);
      sh.v[l][tid] = v + 1;
    }
    sh.nrow[l][tid] = row;
#pragma unroll
    for (int q = 0; q < LM; ++q)
      if (q == l) {
        pst[q] = a;
        pd[q] = d;
      }
  };
  // make the prefetched interval of lane l current (skipping removed / empty
  // ones) and prefetch the following; e[l] = its start, LLONG_MAX when done
  auto consume = [&](int l) {
    long long ne = LLONG_MAX;
    while (true) {
      const int row = sh.nrow[l][tid];
      if (row < 0) break;
      long long st = 0, d = 0;
#pragma unroll
      for (int q = 0; q < LM; ++q)
        if (q == l) {
          st = pst[q];
          d = pd[q];
        }
      prefetch(l);
      if (st < 0) continue;  // removed task / absent chain member (start -1)
      long long gapx;
      const int cls = bd_class(p, row, gapx);
      if (cls == 3) continue;
      long long end = st + d + gapx;
      if (end <= st) continue;
      // absorb the lane's following intervals while they continue this one
      // back to back with the same class ([a, b) + [b, c) = [a, c) for the
      // coverage counts): kernels queued on a stream and CPU calls separated
      // only by their gaps mostly do, so most intervals never reach the merge
      while (end < T1) {  // (past the window end the merge stops anyway)
        const int nr = sh.nrow[l][tid];
        if (nr < 0) break;
        long long nst = 0, nd = 0;
#pragma unroll
        for (int q = 0; q < LM; ++q)
          if (q == l) {
            nst = pst[q];
            nd = pd[q];
          }
        if (nst != end) break;
        long long gap2;
        const int cls2 = bd_class(p, nr, gap2);
        const long long end2 = nst + nd + gap2;
        if (cls2 != cls || end2 < end) break;
        end = end2;
        prefetch(l);
      }
      sh.cls[l][tid] = cls;
      sh.b[l][tid] = end;
      sh.act[l][tid] = 0;
      ne = st;
      break;
    }
#pragma unroll
    for (int q = 0; q < LM; ++q)
      if (q == l) e[q] = ne;
  };

#pragma unroll
  for (int l = 0; l < LM; ++l) {
    sh.v[l][tid] = 0;
    sh.len[l][tid] = 0;
    sh.nrow[l][tid] = -1;
    sh.act[l][tid] = 0;
    sh.on[l][tid] = 0;
    if (!EXACT && l >= p.L) continue;
    const int c_ix = CH ? p.lane_chain[l] : -1;
    bool chain_on = false;
    int len = p.lane_ptr[l + 1] - p.lane_ptr[l];
    if (CH && c_ix >= 0) {
      chain_on = p.present == nullptr || p.present[(long long)s * p.n_chains + c_ix] != 0;
      if (chain_on) len += p.chains[c_ix].B;
    }
    sh.len[l][tid] = len;
    sh.on[l][tid] = chain_on ? 1 : 0;
    sh.v[l][tid] = len > 0 && T0 > 0 ? bd_seek<CH>(p, l, len, s, chain_on, T0) : 0;
    prefetch(l);
    consume(l);
  }
  long long acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;  // cpu_only, gpu_only, parallel, idle
  int cc = 0, gc = 0;
  long long t = T0;
  while (true) {
    int best = 0;
    long long ev = e[0];
#pragma unroll
    for (int l = 1; l < LM; ++l)
      if (e[l] < ev) {
        ev = e[l];
        best = l;
      }
    const long long te = min(ev, T1);
    if (te > t) {
      const long long span = te - t;
      if (cc > 0 && gc > 0)
        acc2 += span;
      else if (cc > 0)
        acc0 += span;
      else if (gc > 0)
        acc1 += span;
      else
        acc3 += span;
      t = te;
    }
    if (ev >= T1) break;
    const int c = sh.cls[best][tid];
    if (sh.act[best][tid]) {  // the current interval of lane `best` ends
      if (c == 0) --cc; else --gc;
      consume(best);
    } else {                  // it starts
      if (c == 0) ++cc; else ++gc;
      sh.act[best][tid] = 1;
      const long long b = sh.b[best][tid];
#pragma unroll
      for (int q = 0; q < LM; ++q)
        if (q == best) e[q] = b;
    }
  }
  unsigned long long* u = reinterpret_cast<unsigned long long*>(o);
  if (acc0) atomicAdd(u + 0, (unsigned long long)acc0);
  if (acc1) atomicAdd(u + 1, (unsigned long long)acc1);
  if (acc2) atomicAdd(u + 2, (unsigned long long)acc2);
  if (acc3) atomicAdd(u + 3, (unsigned long long)acc3);
}

// per_layer_breakdown (breakdown.py:100-111): per layer, summed CPU and GPU
// task durations of the scheduled tasks, comm lanes excluded.
__device__ __forceinline__ void lb_flush(const BreakdownParams& p, int key, long long acc, int s) {
  // row chunks of one scenario run in different blocks: accumulate atomically
  if (key >= 0 && acc != 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(p.layer_busy + (long long)key * p.S + s),
              (unsigned long long)acc);
}
constexpr int kLbRowChunk = 2048;  // rows per block row (blockIdx.y), at most
// fewer rows per chunk when there are few scenarios: one thread walks a chunk
// of one scenario, so a single-scenario table (the drop-in Analysis.whatif)
// needs many short chunks to get past one thread's dependent walk
inline int lb_row_chunk(int n, int S) {
  const long long chunks = (148LL * 1024 + S - 1) / S;
  long long c = std::max<long long>(64, (n + chunks - 1) / chunks);
  c = std::min<long long>(c, kLbRowChunk);
  c = std::max<long long>(c, (n + 65534) / 65535);  // grid y limit
  return (int)c;
}

// NEG: start rows may hold -1 (dropped tasks) and must be read; otherwise
// only the durations are (a third of the bytes). A layer's CPU launches and GPU
// kernels interleave in row order, so both classes of the current layer are
// accumulated in registers and flushed when the layer changes (a flush per
// class change cost a read-modify-write of [layer][class][S] per row).
template <bool NEG>
__global__ void __launch_bounds__(128) layer_busy_kernel(const BreakdownParams p) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= p.S) return;
  // one layer run per class: the CPU thread launches layers ahead of the
  // streams running them, so in row order the two classes sit in different layers
  int lay_c = -1, lay_g = -1;
  long long acc_c = 0, acc_g = 0;
  constexpr int U = 8;  // rows in flight per thread
  const int rbeg = blockIdx.y * p.lb_chunk;
  const int rend = min(p.n, rbeg + p.lb_chunk);
  for (int r0 = rbeg; r0 < rend; r0 += U) {
    long long st[U], d[U];
    int ly[U], gpu[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int row = r0 + j;
      ly[j] = -1;
      gpu[j] = 0;
      st[j] = 0;
      d[j] = 0;
      if (row < rend) {
        const int rc = __ldg(&p.row_class[row]);
        if (rc != BD_COMM) {
          ly[j] = __ldg(&p.row_layer[row]);
          gpu[j] = rc == BD_GPU;
        }
        if (NEG) st[j] = __ldcs(&p.start[(long long)row * p.start_ld + s]);
        d[j] = bd_dur(p, row, s);
      }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (ly[j] < 0 || (NEG && st[j] < 0)) continue;
      if (gpu[j]) {
        if (ly[j] != lay_g) {
          if (lay_g >= 0) lb_flush(p, lay_g * 2 + 1, acc_g, s);
          lay_g = ly[j];
          acc_g = 0;
        }
        acc_g += d[j];
      } else {
        if (ly[j] != lay_c) {
          if (lay_c >= 0) lb_flush(p, lay_c * 2, acc_c, s);
          lay_c = ly[j];
          acc_c = 0;
        }
        acc_c += d[j];
      }
    }
  }
  if (lay_c >= 0) lb_flush(p, lay_c * 2, acc_c, s);
  if (lay_g >= 0) lb_flush(p, lay_g * 2 + 1, acc_g, s);
}

// Dispatch order [S][n] -> per-scenario lane sequences srows[s][lane_ptr[l] + k]
// (the k-th dispatched row of lane l); one thread per scenario, per-lane
// cursors in registers-or-local memory (L <= 32).
__global__ void bd_sched_rows_kernel(const int* __restrict__ schedule,
                                     const int* __restrict__ row_lane,
                                     const int* __restrict__ lane_ptr, int n, int L, int S,
                                     int* __restrict__ srows) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  int cur[kBdMaxLanes];
  for (int l = 0; l < L; ++l) cur[l] = lane_ptr[l];
  const int* sc = schedule + (long long)s * n;
  int* out = srows + (long long)s * n;
  for (int k = 0; k < n; ++k) {
    const int row = sc[k];
    out[cur[row_lane[row]]++] = row;
  }
}

cudaError_t launch_bd_sched_rows(const int* schedule, const int* row_lane, const int* lane_ptr,
                                 int n, int L, int S, int* srows, cudaStream_t stream) {
  if (L > kBdMaxLanes) return cudaErrorInvalidValue;
  bd_sched_rows_kernel<<<(S + 127) / 128, 128, 0, stream>>>(schedule, row_lane, lane_ptr, n, L, S,
                                                             srows);
  note_launch();
  return cudaGetLastError();
}

// Vectorised per-layer busy for int32 durations without dropped tasks: four
// consecutive scenarios per thread (one 16 B load per row), same run-length
// accumulation and flushes as layer_busy_kernel.
__global__ void __launch_bounds__(128) layer_busy4_kernel(const BreakdownParams p) {
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (s >= p.S) return;
  int lay_c = -1, lay_g = -1;  // one layer run per class (as layer_busy_kernel)
  long long ac[4] = {0, 0, 0, 0}, ag[4] = {0, 0, 0, 0};
  constexpr int U = 8;
  const int rbeg = blockIdx.y * p.lb_chunk;
  const int rend = min(p.n, rbeg + p.lb_chunk);
  const int* dur = static_cast<const int*>(p.dur);
  auto flush = [&](int lay, int c, const long long* a) {
    if (lay < 0) return;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (s + i < p.S) lb_flush(p, lay * 2 + c, a[i], s + i);
  };
  for (int r0 = rbeg; r0 < rend; r0 += U) {
    int4 d[U];
    int ly[U], gpu[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int row = r0 + j;
      ly[j] = -1;
      gpu[j] = 0;
      d[j] = make_int4(0, 0, 0, 0);
      if (row < rend) {
        const int rc = __ldg(&p.row_class[row]);
        if (rc != BD_COMM) {
          ly[j] = __ldg(&p.row_layer[row]);
          gpu[j] = rc == BD_GPU;
        }
        d[j] = __ldcs(reinterpret_cast<const int4*>(dur + (long long)row * p.dld + s));
      }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (ly[j] < 0) continue;
      const long long v[4] = {d[j].x, d[j].y, d[j].z, d[j].w};
      if (gpu[j]) {
        if (ly[j] != lay_g) {
          flush(lay_g, 1, ag);
          lay_g = ly[j];
#pragma unroll
          for (int i = 0; i < 4; ++i) ag[i] = 0;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) ag[i] += v[i];
      } else {
        if (ly[j] != lay_c) {
          flush(lay_c, 0, ac);
          lay_c = ly[j];
#pragma unroll
          for (int i = 0; i < 4; ++i) ac[i] = 0;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) ac[i] += v[i];
      }
    }
  }
  flush(lay_c, 0, ac);
  flush(lay_g, 1, ag);
}

// ---- row-order streaming sweep ------------------------------------------------
//
// The windowed merge above follows each lane through time, so its next load
// depends on which lane's event comes first: one dependent global load per
// interval.  On a lane-chained graph without permutable chains the frozen row
// order is a topological order in which every lane's rows appear in lane order,
// so one thread per scenario can instead stream the rows in row order -- the
// load addresses are data independent (batched, coalesced across the
// scenarios of a warp, the simulate kernel's own access pattern) -- and:
//   * grow each lane's open run: an interval that starts exactly where the
//     lane's open run ends, with the same class, extends it (coverage counts
//     cannot tell [a, b) + [b, c) from [a, c)); otherwise the open run is closed
//     into a small per-lane FIFO of pending runs and a new one opens;
//   * sweep time forward to F = min over unfinished lanes of the lane's
//     frontier (the end of its last interval: a lane's later intervals start at
//     or after it, start >= finish + gap, sim.py:128), merging the pending runs
//     of all lanes in time order with the same cpu / gpu coverage counters and
//     classification as the merge above (breakdown.py:42-97).
// A scenario whose lanes drift apart by more than the FIFO depth in row order
// hands itself back (bad[s] = 2) to the windowed merge, launched after the
// sweep for those scenarios only.
constexpr int kBsBD = 64;  // threads (scenarios) per block
constexpr int kBsD = 4;    // FIFO capacity (pending closed runs per lane)
constexpr int kBsU = 8;    // rows per staged batch (two batches in flight)
// auto mode: scenarios needed for the sweep.  Below one wave the sweep is
// latency-bound at ~21 ms per 100k rows whatever S (one thread per scenario),
// while the windowed merge scales with S (19.3 ms at 16,384, 36.7 at 32,768)
constexpr int kBsMinS = 22528;
constexpr long long kBsGapMax = 1LL << 50;  // gaps packed into the row code

// per-row code: bits 0-5 lane, 8-9 class (0 cpu, 1 gpu, 3 not counted), bit 10
// the lane's last row, bits 12.. the gap counted as CPU busy (0 unless the row
// is a CPU interval and gaps_as_cpu_busy); -1: a gap too large to pack (the
// sweep hands every scenario back)
__global__ void bd_rowinfo_kernel(const BreakdownParams p) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < p.n; r += gridDim.x * blockDim.x) {
    const int l = p.row_lane ? p.row_lane[r] : 0;
    const int rc = p.row_class[r];
    int cls;
    long long gap = 0;
    if (rc == BD_CPU || rc == BD_CPU_DATALOAD) {
      if (rc == BD_CPU_DATALOAD && !p.dataload_as_cpu) {
        cls = 3;
      } else {
        cls = 0;
        if (p.gaps_as_cpu_busy) gap = p.gap[r];
      }
    } else if (rc == BD_GPU) {
      cls = 1;
    } else {
      cls = p.comm_as_gpu ? 1 : 0;
    }
    const long long last = p.lane_rows && p.lane_rows[p.lane_ptr[l + 1] - 1] == r ? 1 : 0;
    p.rinfo[r] = gap >= kBsGapMax ? -1LL : (gap << 12) | (last << 10) | (cls << 8) | l;
    // per_layer_breakdown key (breakdown.py:100-111): layer * 2 + is-GPU,
    // -1 for comm rows (the reference skips comm lanes)
    if (p.linfo) p.linfo[r] = rc == BD_COMM ? -1 : p.row_layer[r] * 2 + (rc == BD_GPU ? 1 : 0);
  }
}

template <int DK>
struct BsStage {
  long long st[kBsU][kBsBD];
  typename std::conditional<DK == 1, int, long long>::type d[kBsU][kBsBD];
  long long info[kBsU];  // row codes, shared by the block
  int linfo[kBsU];       // per-layer busy keys, shared by the block
};
template <int LM, int DK>
struct BsSmem {
  BsStage<DK> stage[2];
  long long fs[LM][kBsD][kBsBD];  // pending run start
  long long fe[LM][kBsD][kBsBD];  // pending run end * 2 + class
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src));
}

template <int LM, int DK, bool LB>
__global__ void __launch_bounds__(kBsBD, 8) breakdown_stream_kernel(const BreakdownParams p) {
  __shared__ BsSmem<LM, DK> sh;
  const int tid = threadIdx.x;
  const int s = blockIdx.x * kBsBD + tid;
  const bool live = s < p.S;  // idle threads still take part in the block barriers
  constexpr long long INF = LLONG_MAX;
  const long long ms = live ? p.makespan[s] : 0;
  const int depth = p.stream_depth;
  // per-lane state in registers, always indexed by a compile-time lane (the
  // row's lane is the same for the whole warp: a uniform switch picks it)
  long long rs[LM], re[LM];  // open run [rs, re)
  int rc[LM];                // open run class, -1 none
  int hd[LM], cnt[LM];       // FIFO of closed runs not yet swept
  bool act[LM];              // the sweep is inside the lane's head run
  long long e[LM], fr[LM];   // next sweep event; lane frontier
#pragma unroll
  for (int l = 0; l < LM; ++l) {
    rs[l] = re[l] = 0;
    rc[l] = -1;
    hd[l] = cnt[l] = 0;
    act[l] = false;
    e[l] = INF;
    fr[l] = l < p.L && p.lane_ptr[l + 1] > p.lane_ptr[l] ? 0 : INF;
  }
  long long acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;  // cpu_only, gpu_only, parallel, idle
  int cc = 0, gc = 0;
  long long t = 0;
  // lane holding the smallest frontier: a row of any other lane leaves F (and
  // so the sweep limit) unchanged, and its new head run starts at or after its
  // own frontier >= F, so only rows of this lane can make a sweep due
  int fmin = 0;
  {
    long long f0 = fr[0];
#pragma unroll
    for (int l = 1; l < LM; ++l)
      if (fr[l] < f0) {
        f0 = fr[l];
        fmin = l;
      }
  }

  // one sweep event on lane q (its head run starts or ends)
  auto handle = [&](auto qc) {
    constexpr int q = decltype(qc)::value;
    if (act[q]) {  // the head run ends
      const int c = cnt[q] > 0 ? (int)(sh.fe[q][hd[q]][tid] & 1) : rc[q];
      if (c == 0) --cc; else --gc;
      act[q] = false;
      if (cnt[q] > 0) {
        hd[q] = hd[q] + 1 == kBsD ? 0 : hd[q] + 1;
        --cnt[q];
        e[q] = cnt[q] > 0 ? sh.fs[q][hd[q]][tid] : (rc[q] >= 0 ? rs[q] : INF);
      } else {  // a finished lane's open run
        rc[q] = -1;
        e[q] = INF;
      }
    } else {  // it starts
      long long b;
      int c;
      if (cnt[q] > 0) {
        const long long x = sh.fe[q][hd[q]][tid];
        b = x >> 1;
        c = (int)(x & 1);
      } else {
        b = re[q];
        c = rc[q];
      }
      if (c == 0) ++cc; else ++gc;
      act[q] = true;
      e[q] = b;
    }
  };
  // merge the known runs of all lanes up to lim (events at or after lim wait)
  auto sweep = [&](long long lim) {
    while (true) {
      int best = 0;
      long long ev = e[0];
#pragma unroll
      for (int l = 1; l < LM; ++l)
        if (e[l] < ev) {
          ev = e[l];
          best = l;
        }
      const long long te = min(ev, lim);
      if (te > t) {
        const long long span = te - t;
        if (cc > 0 && gc > 0)
          acc2 += span;
        else if (cc > 0)
          acc0 += span;
        else if (gc > 0)
          acc1 += span;
        else
          acc3 += span;
        t = te;
      }
      if (ev >= lim) break;
      switch (best) {
        case 0: handle(std::integral_constant<int, 0>()); break;
        case 1: if (LM > 1) handle(std::integral_constant<int, (LM > 1 ? 1 : 0)>()); break;
        case 2: if (LM > 2) handle(std::integral_constant<int, (LM > 2 ? 2 : 0)>()); break;
        default: if (LM > 3) handle(std::integral_constant<int, (LM > 3 ? 3 : 0)>()); break;
      }
    }
  };
  bool ovf = false;
  // one row of lane q: grow / close / open the lane's run, move its frontier
  auto step = [&](auto qc, long long st, long long d, long long info) {
    constexpr int q = decltype(qc)::value;
    if (st >= 0) {
      const long long end = st + d + (info >> 12);
      const int cls = (int)(info >> 8) & 3;
      if (cls != 3 && end > st) {
        if (rc[q] == cls && st == re[q]) {  // continues the open run
          re[q] = end;
          if (act[q] && cnt[q] == 0) e[q] = end;
        } else {
          if (rc[q] >= 0) {  // close the open run into the FIFO
            if (cnt[q] >= depth) {
              ovf = true;
              return;
            }
            int slot = hd[q] + cnt[q];
            if (slot >= kBsD) slot -= kBsD;
            sh.fs[q][slot][tid] = rs[q];
            sh.fe[q][slot][tid] = re[q] * 2 + rc[q];
            ++cnt[q];
          } else if (cnt[q] == 0) {  // the lane had no run: this one is its head
            e[q] = st;
          }
          rs[q] = st;
          re[q] = end;
          rc[q] = cls;
        }
        fr[q] = end;
      } else {
        fr[q] = max(fr[q], st);
      }
    }
    if ((info >> 10) & 1) fr[q] = INF;  // the lane's last row
  };

  const int n = p.n;
  const int nb = (n + kBsU - 1) / kBsU;
  // batch b's rows -> stage b & 1: each thread copies its own scenario's
  // start and duration, threads 0 .. kBsU-1 the block's row codes
  // the thread's start / duration pointers advance by one batch of rows per
  // issue (strides held in registers: no per-row 64-bit address products)
  using DT = typename std::conditional<DK == 1, int, long long>::type;
  const long long sld = p.start_ld, dld = p.dld;
  const long long* sp = p.start + (live ? s : 0);
  const DT* dp = static_cast<const DT*>(p.dur) + (live ? s : 0);
  auto issue = [&](int b) {
    BsStage<DK>& sg = sh.stage[b & 1];
    const int r0 = b * kBsU;
    if (live) {
      const long long* a = sp;
      const DT* q = dp;
      if (r0 + kBsU <= n) {
#pragma unroll
        for (int j = 0; j < kBsU; ++j) {
          cp_async8(&sg.st[j][tid], a);
          if (DK == 1) cp_async4(&sg.d[j][tid], q); else cp_async8(&sg.d[j][tid], q);
          a += sld;
          q += dld;
        }
      } else {
        for (int j = 0; r0 + j < n; ++j) {
          cp_async8(&sg.st[j][tid], a);
          if (DK == 1) cp_async4(&sg.d[j][tid], q); else cp_async8(&sg.d[j][tid], q);
          a += sld;
          q += dld;
        }
      }
      sp += sld * kBsU;
      dp += dld * kBsU;
    }
    if (tid < kBsU && r0 + tid < n) {
      cp_async8(&sg.info[tid], p.rinfo + r0 + tid);
      if (LB) cp_async4(&sg.linfo[tid], p.linfo + r0 + tid);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  long long neg = 0;  // OR of every duration (and row code): the negative check rides along
  // per-layer busy (LB): each class keeps its own current layer run in
  // registers (the CPU thread launches layers ahead of the streams running
  // them, so in row order the two classes sit in different layers); the thread
  // owns its scenario's column, so a flush is a plain coalesced
  // read-modify-write of [layer][class][S]
  int lay[2] = {-1, -1};
  long long lacc[2] = {0, 0};
  auto lflush = [&](int c) {
    if (lay[c] >= 0 && lacc[c]) p.layer_busy[((long long)lay[c] * 2 + c) * p.S + s] += lacc[c];
  };
  issue(0);
  for (int b = 0; b < nb; ++b) {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    // batch b has landed for every thread, and every thread is done with
    // batch b - 1, whose stage the next copy overwrites
    __syncthreads();
    if (b + 1 < nb) issue(b + 1);
    if (!live) continue;
    const BsStage<DK>& sg = sh.stage[b & 1];
    const int jn = min(kBsU, n - b * kBsU);
    for (int j = 0; j < jn; ++j) {
      const long long st = sg.st[j][tid];
      const long long d = sg.d[j][tid];
      const long long info = sg.info[j];
      neg |= d | info;
      if (LB) {
        const int lk = sg.linfo[j];
        if (lk >= 0 && st >= 0) {
          const int c = lk & 1;
#pragma unroll
          for (int q = 0; q < 2; ++q)  // static indices keep both runs in registers
            if (q == c) {
              if ((lk >> 1) != lay[q]) {
                lflush(q);
                lay[q] = lk >> 1;
                lacc[q] = 0;
              }
              lacc[q] += d;
            }
        }
      }
      if (ovf) continue;
      const int l = (int)info & 63;
      switch (l) {
        case 0: step(std::integral_constant<int, 0>(), st, d, info); break;
        case 1: if (LM > 1) step(std::integral_constant<int, (LM > 1 ? 1 : 0)>(), st, d, info); break;
        case 2: if (LM > 2) step(std::integral_constant<int, (LM > 2 ? 2 : 0)>(), st, d, info); break;
        default: if (LM > 3) step(std::integral_constant<int, (LM > 3 ? 3 : 0)>(), st, d, info); break;
      }
      if (l != fmin) continue;
      long long F = fr[0], ne = e[0];
      fmin = 0;
#pragma unroll
      for (int q = 1; q < LM; ++q) {
        if (fr[q] < F) {
          F = fr[q];
          fmin = q;
        }
        ne = min(ne, e[q]);
      }
      const long long lim = min(F, ms);
      if (ne < lim) sweep(lim);
    }
  }
  if (!live) return;
  if (LB) {
    lflush(0);
    lflush(1);
  }
  long long* o = p.parts + (long long)s * 4;
  if (neg < 0) {
    // a negative duration breaks the lane order (reported as -1, as the
    // windowed merge does); an unpackable gap hands the scenario back
    bool negdur = false;
    for (int r = 0; r < n && !negdur; ++r) {
      const long long d = DK == 1 ? (long long)static_cast<const int*>(p.dur)[(long long)r * p.dld + s]
                                  : static_cast<const long long*>(p.dur)[(long long)r * p.dld + s];
      negdur = d < 0;
    }
    if (negdur) {
      p.bad[s] = 1;
      o[0] = o[1] = o[2] = o[3] = -1;
      return;
    }
    ovf = true;
  }
  if (ovf) {
    p.bad[s] = 2;
    return;
  }
  sweep(ms);
  o[0] = acc0;
  o[1] = acc1;
  o[2] = acc2;
  o[3] = acc3;
}

cudaError_t launch_breakdown(const BreakdownParams& p, cudaStream_t stream) {
  if (p.S <= 0) return cudaSuccess;
  if (p.L > kBdMaxLanes) return cudaErrorInvalidValue;
  const int BD = 128;
  const int grid = (p.S + BD - 1) / BD;
  bool lb_fused = false;  // per-layer busy computed by the streaming sweep
  if (p.parts) {
    bd_zero_kernel<<<std::min(grid, 148 * 16), BD, 0, stream>>>(p);
    note_launch();
    if ((p.n + kBdNegRows - 1) / kBdNegRows > 65535) return cudaErrorInvalidValue;
    const dim3 g2(grid, p.K);
    const bool ch = p.n_chains > 0;
    static_assert(kBdLeanBD == 128, "lean kernel block = BD");
    // streaming sweep: lane-chained rows (no dispatch order, no permutable
    // chains), at most 4 lanes, enough scenarios to fill the SMs with one
    // thread each (below that the windowed merge splits time instead)
    const bool sweep_ok = p.row_lane != nullptr && p.rinfo != nullptr && p.srows == nullptr &&
                          p.n_chains == 0 && p.L <= 4;
    const bool sweep = sweep_ok && (p.stream_mode > 0 || (p.stream_mode == 0 && p.S >= kBsMinS));
    BreakdownParams q = p;
    if (p.rinfo) {  // packed per-row class / gap codes (both merges read them)
      bd_rowinfo_kernel<<<std::min((p.n + 255) / 256, 148 * 8), 256, 0, stream>>>(q);
      note_launch();
    }
    if (!sweep) {
      bd_negative_kernel<<<dim3(grid, (p.n + kBdNegRows - 1) / kBdNegRows), BD, 0, stream>>>(p);
      note_launch();
    } else {
      q.stream_depth = p.stream_depth <= 0 || p.stream_depth > kBsD ? kBsD : p.stream_depth;
      const int gs = (p.S + kBsBD - 1) / kBsBD;
      // per-layer busy rides along (durations are read once for both)
      lb_fused = p.layer_busy != nullptr && p.row_layer != nullptr && p.linfo != nullptr;
      if (lb_fused) {
        cudaError_t e = launch_fill_i64(p.layer_busy, 0, (long long)p.n_layers * 2 * p.S, stream);
        if (e != cudaSuccess) return e;
      } else {
        q.linfo = nullptr;
      }
#define BD_SWEEP(LM)                                                          \
  do {                                                                        \
    if (p.dkind == 1)                                                         \
      lb_fused ? breakdown_stream_kernel<LM, 1, true><<<gs, kBsBD, 0, stream>>>(q)   \
               : breakdown_stream_kernel<LM, 1, false><<<gs, kBsBD, 0, stream>>>(q); \
    else                                                                      \
      lb_fused ? breakdown_stream_kernel<LM, 2, true><<<gs, kBsBD, 0, stream>>>(q)   \
               : breakdown_stream_kernel<LM, 2, false><<<gs, kBsBD, 0, stream>>>(q); \
  } while (0)
      switch (p.L) {
        case 1: BD_SWEEP(1); break;
        case 2: BD_SWEEP(2); break;
        case 3: BD_SWEEP(3); break;
        default: BD_SWEEP(4);
      }
#undef BD_SWEEP
      note_launch();
      q.redo = 1;  // the windowed merge below recomputes the handed-back scenarios
    }
    if (p.L <= 8 && getenv("DDSIM_BD_OLD") == nullptr) {
#define BD_LEAN(LM, EX)                                                      \
  do {                                                                       \
    if (ch)                                                                  \
      breakdown_lean_kernel<LM, EX, true><<<g2, BD, 0, stream>>>(q);         \
    else                                                                     \
      breakdown_lean_kernel<LM, EX, false><<<g2, BD, 0, stream>>>(q);        \
  } while (0)
      switch (p.L) {
        case 1: BD_LEAN(1, true); break;
        case 2: BD_LEAN(2, true); break;
        case 3: BD_LEAN(3, true); break;
        case 4: BD_LEAN(4, true); break;
        default: BD_LEAN(8, false);
      }
#undef BD_LEAN
      note_launch();
      goto layers;
    }
#define BD_LAUNCH(LM, EX)                                                     \
  do {                                                                        \
    if (ch)                                                                   \
      breakdown_kernel<LM, EX, true><<<g2, BD, 0, stream>>>(p);               \
    else                                                                      \
      breakdown_kernel<LM, EX, false><<<g2, BD, 0, stream>>>(p);              \
  } while (0)
    switch (p.L) {
      case 1: BD_LAUNCH(1, true); break;
      case 2: BD_LAUNCH(2, true); break;
      case 3: BD_LAUNCH(3, true); break;
      case 4: BD_LAUNCH(4, true); break;
      default:
        if (p.L <= 8)
          BD_LAUNCH(8, false);
        else if (p.L <= 16)
          BD_LAUNCH(16, false);
        else
          BD_LAUNCH(32, false);
    }
#undef BD_LAUNCH
    note_launch();
  }
layers:
  if (p.layer_busy && p.row_layer && !lb_fused) {
    cudaError_t e = launch_fill_i64(p.layer_busy, 0, (long long)p.n_layers * 2 * p.S, stream);
    if (e != cudaSuccess) return e;
    BreakdownParams pl = p;
    pl.lb_chunk = lb_row_chunk(p.n, p.S);
    if ((p.n + pl.lb_chunk - 1) / pl.lb_chunk > 65535) return cudaErrorInvalidValue;
    const dim3 g3(grid, (p.n + pl.lb_chunk - 1) / pl.lb_chunk);
    const bool vec4 = !p.start_may_be_neg && p.dkind == 1 && p.dld % 4 == 0 &&
                      reinterpret_cast<uintptr_t>(p.dur) % 16 == 0 &&
                      getenv("DDSIM_BD_LB_SCALAR") == nullptr;
    if (vec4) {
      const int g4 = ((p.S + 3) / 4 + BD - 1) / BD;
      layer_busy4_kernel<<<dim3(g4, g3.y), BD, 0, stream>>>(pl);
    } else if (p.start_may_be_neg)
      layer_busy_kernel<true><<<g3, BD, 0, stream>>>(pl);
    else
      layer_busy_kernel<false><<<g3, BD, 0, stream>>>(pl);
    note_launch();
  }
  return cudaGetLastError();
}

}  // namespace ddsim
