// listsched_sim: exact Alg. 1 event loop (pkg/src/kernsim/sim.py:89-142) for
// graphs whose tasks are not all lane-chained (unsequenced inserts of
// p3 / vdnn / gist / dgc / blueconnect), and the dispatch order
// (schedule_trace) of any graph.
//
// One warp owns one scenario.  Each step the warp scans the frontier for the
// arg-min of (max(lane_progress[lane], ready), id) (SchedulePolicy.choose,
// sim.py:55-63) with a shuffle reduction; PrioritySchedule (sim.py:72-86) and
// VdnnPrefetchPolicy (scenarios.py:618-630) are extra reductions over the same
// frontier.  The frontier lives in shared memory (SoA, cached keys: a task's
// ready time is final once it enters the frontier) and spills to global
// memory past kFrontCap entries.  With zero_time set every key is 0 and the
// dispatch order is Kahn's smallest-id order (verify_acyclic, graph.py:129-148).
#include "ddsim_internal.h"

#include <climits>

namespace ddsim {

constexpr int kFrontCap = 2048;

__device__ __forceinline__ long long ls_scale(long long d, long long num, long long den) {
  const bool neg = d < 0;
  const unsigned long long a = neg ? (unsigned long long)(-d) : (unsigned long long)d;
  const unsigned __int128 x = (unsigned __int128)a * (unsigned long long)num * 2u + (unsigned long long)den;
  const unsigned long long q = (unsigned long long)(x / ((unsigned __int128)(unsigned long long)den * 2u));
  return neg ? -(long long)q : (long long)q;
}

struct Front {
  long long* rdy;
  int* v;
  int* rank;
  int* lane;
  // global spill (index >= kFrontCap)
  long long* g_rdy;
  int* g_v;
  __device__ __forceinline__ void get(int i, const ListParams& p, long long& r, int& vv, int& rk,
                                      int& ln) const {
    if (i < kFrontCap) {
      r = rdy[i];
      vv = v[i];
      rk = rank[i];
      ln = lane[i];
    } else {
      r = g_rdy[i - kFrontCap];
      vv = g_v[i - kFrontCap];
      rk = p.id_rank[vv];
      ln = p.lane[vv];
    }
  }
  __device__ __forceinline__ void put(int i, const ListParams& p, long long r, int vv) const {
    if (i < kFrontCap) {
      rdy[i] = r;
      v[i] = vv;
      rank[i] = p.id_rank[vv];
      lane[i] = p.lane[vv];
    } else {
      g_rdy[i - kFrontCap] = r;
      g_v[i - kFrontCap] = vv;
    }
  }
};

__device__ __forceinline__ void argmin_reduce(long long& e, int& r, int& pos) {
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const long long oe = __shfl_xor_sync(0xffffffffu, e, off);
    const int orr = __shfl_xor_sync(0xffffffffu, r, off);
    const int op = __shfl_xor_sync(0xffffffffu, pos, off);
    if (oe < e || (oe == e && orr < r)) {
      e = oe;
      r = orr;
      pos = op;
    }
  }
}

// arg-max of (key, -rank)
__device__ __forceinline__ void argmax_reduce(int& key, int& r, int& pos) {
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const int ok = __shfl_xor_sync(0xffffffffu, key, off);
    const int orr = __shfl_xor_sync(0xffffffffu, r, off);
    const int op = __shfl_xor_sync(0xffffffffu, pos, off);
    if (ok > key || (ok == key && orr < r)) {
      key = ok;
      r = orr;
      pos = op;
    }
  }
}

__global__ void __launch_bounds__(32) listsched_kernel(const ListParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x;
  const int s = blockIdx.x;
  Front fr;
  fr.rdy = reinterpret_cast<long long*>(smem);
  fr.v = reinterpret_cast<int*>(fr.rdy + kFrontCap);
  fr.rank = fr.v + kFrontCap;
  fr.lane = fr.rank + kFrontCap;
  long long* lp = reinterpret_cast<long long*>(fr.lane + kFrontCap);  // [L]
  long long* lb = lp + p.L;                                            // [L]
  __shared__ int Fsh;

  const long long N = p.N;
  long long* rdy = p.rdy + (long long)s * N;
  int* rem = p.rem + (long long)s * N;
  fr.g_rdy = p.rdy + (long long)p.S * N + (long long)s * N;  // spill: second half
  fr.g_v = p.front + (long long)s * N;
  int e0 = 0, e1 = 0;
  if (p.scale_ptr) {
    e0 = p.scale_ptr[s];
    e1 = p.scale_ptr[s + 1];
  }
  if (lane == 0) Fsh = 0;
  __syncwarp();
  for (int v = lane; v < p.N; v += 32) {
    const int d = p.indeg[v];
    rem[v] = d;
    const long long r0 = p.zero_time ? 0 : p.ready[v];
    rdy[v] = r0;
    if (d == 0) fr.put(atomicAdd(&Fsh, 1), p, r0, v);
  }
  for (int l = lane; l < p.L; l += 32) {
    lp[l] = 0;
    lb[l] = 0;
  }
  __syncwarp();

  int nd = 0;
  long long ms = 0;
  const bool vdnn = p.policy == KS_POLICY_VDNN;
  for (;;) {
    const int F = *((volatile int*)&Fsh);
    if (F == 0) break;
    int elig = -1;
    if (vdnn) {
      // eligible malloc: max (conv rank, -id) among frontier mallocs
      int bk = INT_MIN, br = INT_MAX, bpos = -1;
      for (int i = lane; i < F; i += 32) {
        long long r;
        int vv, rk, ln;
        fr.get(i, p, r, vv, rk, ln);
        if (!(p.flags[vv] & KS_TASK_VDNN_MALLOC)) continue;
        const int key = p.vrank ? p.vrank[vv] : -1;
        if (key > bk || (key == bk && rk < br)) {
          bk = key;
          br = rk;
          bpos = i;
        }
      }
      argmax_reduce(bk, br, bpos);
      if (bpos >= 0) {
        long long r;
        int rk, ln;
        fr.get(bpos, p, r, elig, rk, ln);
      }
    }
    long long be = LLONG_MAX;
    int br = INT_MAX, bpos = -1;
    for (int i = lane; i < F; i += 32) {
      long long r;
      int vv, rk, ln;
      fr.get(i, p, r, vv, rk, ln);
      if (vdnn && (p.flags[vv] & KS_TASK_VDNN_MALLOC) && vv != elig) continue;
      const long long eff = p.zero_time ? 0 : max(lp[ln], r);
      if (eff < be || (eff == be && rk < br)) {
        be = eff;
        br = rk;
        bpos = i;
      }
    }
    argmin_reduce(be, br, bpos);
    if (p.policy == KS_POLICY_PRIORITY) {
      long long r0;
      int v0, rk0, ln0;
      fr.get(bpos, p, r0, v0, rk0, ln0);
      if (p.flags[v0] & KS_TASK_COMM) {
        int bk = INT_MIN, br2 = INT_MAX, bpos2 = -1;
        for (int i = lane; i < F; i += 32) {
          long long r;
          int vv, rk, ln;
          fr.get(i, p, r, vv, rk, ln);
          if (!(p.flags[vv] & KS_TASK_COMM)) continue;
          const long long eff = max(lp[ln], r);
          if (eff != be) continue;
          const int key = p.prio[vv];
          if (key > bk || (key == bk && rk < br2)) {
            bk = key;
            br2 = rk;
            bpos2 = i;
          }
        }
        argmax_reduce(bk, br2, bpos2);
        bpos = bpos2;
      }
    }
    long long rv;
    int v, rk, ln;
    fr.get(bpos, p, rv, v, rk, ln);
    __syncwarp();
    long long d = 0, g = 0, st = 0;
    if (!p.zero_time) {
      if (p.dense32)
        d = p.dense32[(long long)v * p.dense_ld + s];
      else if (p.dense64)
        d = p.dense64[(long long)v * p.dense_ld + s];
      else
        d = p.dur[v];
      if (p.ovr_row && p.ovr_row[v] >= 0) d = p.ovr[(long long)p.ovr_row[v] * p.S + s];
      const unsigned grp = p.group ? p.group[v] : 0u;
      if (grp != 0u)
        for (int e = e0; e < e1; ++e) {
          const ScaleStepDev sd = p.scale[e];
          if (grp >= (unsigned)sd.lo && grp <= (unsigned)sd.hi) d = ls_scale(d, sd.num, sd.den);
        }
      g = p.gap[v];
      st = max(lp[ln], rv);
    }
    const long long fin = st + d;
    const long long rel = fin + g;
    __syncwarp();  // every lane has read lp[ln] before lane 0 updates it (racecheck)
    if (lane == 0) {
      if (bpos != F - 1) {
        long long r2;
        int v2, rk2, ln2;
        fr.get(F - 1, p, r2, v2, rk2, ln2);
        fr.put(bpos, p, r2, v2);
      }
      Fsh = F - 1;
      lp[ln] = rel;
      lb[ln] += d;
      if (p.start) p.start[(long long)v * p.start_ld + s] = st;
      if (p.schedule) p.schedule[(long long)s * N + nd] = v;
    }
    ms = max(ms, fin);
    ++nd;
    __syncwarp();
    const int c0 = p.child_ptr[v], c1 = p.child_ptr[v + 1];
    for (int j = c0 + lane; j < c1; j += 32) {
      const int c = p.child[j];
      const long long old = atomicMax(&rdy[c], rel);
      if (atomicSub(&rem[c], 1) == 1) fr.put(atomicAdd(&Fsh, 1), p, max(old, rel), c);
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (p.makespan) p.makespan[s] = ms;
    if (p.dispatched) p.dispatched[s] = nd;
  }
  if (p.lane_busy)
    for (int l = lane; l < p.L; l += 32) p.lane_busy[(long long)s * p.L + l] = lb[l];
}

cudaError_t launch_listsched(const ListParams& p, cudaStream_t stream) {
  const size_t smem = (size_t)kFrontCap * (8 + 4 + 4 + 4) + (size_t)p.L * 16;
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  cudaError_t err = cudaFuncSetAttribute(listsched_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  listsched_kernel<<<p.S, 32, smem, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ddsim

namespace ddsim {

// verify_acyclic (graph.py:129-148) on a lane-chained graph: a task becomes
// ready only after its lane predecessor, so the Kahn frontier is a subset of
// the lane heads.  One warp, one lane per thread: each thread keeps its head's
// id rank and child range in registers (with the next head prefetched); a
// step is a warp arg-min over the ready heads' ranks (smallest id first), the
// winner's children decrement their in-degrees (shared memory when the graph
// fits, global otherwise) and its lane advances.
__global__ void __launch_bounds__(32) toposort_lanes_kernel(
    int N, int L, const int* __restrict__ lane_ptr, const int* __restrict__ lane_rows,
    const int* __restrict__ child_ptr, const int* __restrict__ child,
    const int* __restrict__ indeg, const int* __restrict__ rank, int* deg_g, int* out, int* count) {
  extern __shared__ int sdeg[];
  int* deg = deg_g ? deg_g : sdeg;
  const int t = threadIdx.x;
  for (int i = t; i < N; i += 32) deg[i] = indeg[i];
  __threadfence_block();
  __syncwarp();
  const bool own = t < L;
  const int len = own ? lane_ptr[t + 1] - lane_ptr[t] : 0;
  const int* lr = lane_rows + (own ? lane_ptr[t] : 0);
  int pos = 0;
  // current head and the prefetched next head: row, id rank, child range and
  // the first two children (most tasks have one or two)
  int head = -1, hr = INT_MAX, c0 = 0, c1 = 0, k0 = -1, k1 = -1;
  int nh = -1, nr = INT_MAX, n0 = 0, n1 = 0, m0 = -1, m1 = -1;
  auto fetch = [&](int r, int& rr, int& a, int& b, int& x, int& y) {
    rr = rank[r];
    a = child_ptr[r];
    b = child_ptr[r + 1];
    x = a < b ? child[a] : -1;
    y = a + 1 < b ? child[a + 1] : -1;
  };
  if (len > 0) {
    head = lr[0];
    fetch(head, hr, c0, c1, k0, k1);
  }
  if (len > 1) {
    nh = lr[1];
    fetch(nh, nr, n0, n1, m0, m1);
  }
  int step = 0;
  for (; step < N; ++step) {
    const bool ready = head >= 0 && *((volatile int*)&deg[head]) == 0;
    int key = ready ? hr : INT_MAX;
    int who = t;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const int ok = __shfl_xor_sync(0xffffffffu, key, off);
      const int ow = __shfl_xor_sync(0xffffffffu, who, off);
      if (ok < key || (ok == key && ow < who)) {
        key = ok;
        who = ow;
      }
    }
    if (key == INT_MAX) break;  // nothing ready: a cycle
    const int v = __shfl_sync(0xffffffffu, head, who);
    const int a = __shfl_sync(0xffffffffu, c0, who);
    const int b = __shfl_sync(0xffffffffu, c1, who);
    const int x = __shfl_sync(0xffffffffu, k0, who);
    const int y = __shfl_sync(0xffffffffu, k1, who);
    if (t == 0) {
      out[step] = v;
      if (x >= 0) atomicSub(&deg[x], 1);
    } else if (t == 1) {
      if (y >= 0) atomicSub(&deg[y], 1);
    }
    for (int k = a + 2 + t; k < b; k += 32) atomicSub(&deg[child[k]], 1);
    if (t == who) {  // advance the lane; prefetch the head after next
      ++pos;
      head = nh;
      hr = nr;
      c0 = n0;
      c1 = n1;
      k0 = m0;
      k1 = m1;
      nh = -1;
      nr = INT_MAX;
      if (pos + 1 < len) {
        nh = lr[pos + 1];
        fetch(nh, nr, n0, n1, m0, m1);
      }
    }
    if (deg_g) __threadfence_block();
    __syncwarp();
  }
  if (t == 0) *count = step;
}

// verify_acyclic on lane-chained graphs without in-degree counters: lane l's
// head is ready when every predecessor its lane order does not already place
// before it has been emitted -- for each requirement (lane m, q): the emitted
// prefix of lane m is >= q.  The emitted prefix lengths live in shared memory
// (one word per lane, written only by the lane that advances).  Each lane's
// heads are 48-byte records in lane order (row, id rank, requirements), kept
// kTopoRing ahead in a shared-memory ring by cp.async (no dependent global
// loads on the step).  A step: every thread checks its head, a warp arg-min
// of the ready heads' id ranks (smallest id first, graph.py:129-148), the
// winner's lane advances and refills its ring.
constexpr int kTopoRing = 8;
__device__ __forceinline__ void topo_cp16(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void topo_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void topo_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(kTopoRing - 1) : "memory");
}

__global__ void __launch_bounds__(32) toposort_lanes_req_kernel(
    int N, int L, const int* __restrict__ lane_ptr, const TopoRec* __restrict__ recs,
    const int* __restrict__ req_lane, const int* __restrict__ req_pos, int* out, int* count) {
  __shared__ int done[32];  // emitted prefix length per lane
  __shared__ __align__(16) TopoRec ring[32][kTopoRing];
  const int t = threadIdx.x;
  done[t] = 0;
  const bool own = t < L;
  const int len = own ? lane_ptr[t + 1] - lane_ptr[t] : 0;
  const TopoRec* base = recs + (own ? lane_ptr[t] : 0);
  auto issue = [&](int k) {  // record k of this lane -> its ring slot (one group)
    if (k < len) {
      const char* src = reinterpret_cast<const char*>(base + k);
      char* dst = reinterpret_cast<char*>(&ring[t][k % kTopoRing]);
      topo_cp16(dst, src);
      topo_cp16(dst + 16, src + 16);
      topo_cp16(dst + 32, src + 32);
    }
    topo_commit();
  };
  for (int k = 0; k < kTopoRing; ++k) issue(k);
  topo_wait();
  __syncwarp();
  int pos = 0;
  int step = 0;
  for (; step < N; ++step) {
    bool ready = pos < len;
    // (id rank, lane) in one word: a single warp min-reduction picks the
    // smallest ready id (ranks < 2^27, host-checked)
    unsigned key = 0xffffffffu;
    if (ready) {
      const TopoRec& h = ring[t][pos % kTopoRing];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < h.rn && done[h.ml[k]] < h.mq[k]) ready = false;
      for (int k = 4; ready && k < h.rn; ++k)
        if (done[req_lane[h.r0 + k]] < req_pos[h.r0 + k]) ready = false;
      if (ready) key = ((unsigned)h.rank << 5) | (unsigned)t;
    }
    key = __reduce_min_sync(0xffffffffu, key);
    if (key == 0xffffffffu) break;  // nothing ready: a cycle
    const int who = (int)(key & 31u);
    if (t == who) {
      out[step] = ring[t][pos % kTopoRing].row;
      ++pos;
      done[t] = pos;
      issue(pos + kTopoRing - 1);  // refills the slot just consumed
      topo_wait();                 // record pos has landed
    }
    __syncwarp();
  }
  if (t == 0) *count = step;
}

cudaError_t launch_toposort_lanes_req(int N, int L, const int* lane_ptr, const TopoRec* recs,
                                      const int* req_lane, const int* req_pos, int* out,
                                      int* count, cudaStream_t st) {
  if (L > 32) return cudaErrorInvalidValue;
  toposort_lanes_req_kernel<<<1, 32, 0, st>>>(N, L, lane_ptr, recs, req_lane, req_pos, out, count);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_toposort_lanes(int N, int L, const int* lane_ptr, const int* lane_rows,
                                  const int* child_ptr, const int* child, const int* indeg,
                                  const int* rank, int* deg_scratch, int* out, int* count,
                                  cudaStream_t st) {
  if (L > 32) return cudaErrorInvalidValue;
  const size_t smem = (size_t)N * sizeof(int);
  const bool in_smem = smem <= 200 * 1024;
  if (in_smem) {
    cudaError_t e = cudaFuncSetAttribute(toposort_lanes_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  toposort_lanes_kernel<<<1, 32, in_smem ? smem : 0, st>>>(N, L, lane_ptr, lane_rows, child_ptr,
                                                          child, indeg, rank,
                                                          in_smem ? nullptr : deg_scratch, out, count);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ddsim
