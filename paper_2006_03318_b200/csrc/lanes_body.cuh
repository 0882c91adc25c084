// Device body of the maxplus_lanes kernel, shared by the statically compiled
// kernel (maxplus_lanes.cu, 256-way switch dispatch) and the per-graph
// NVRTC-specialised kernel (jit.cu, if-chain over the handler codes the graph
// uses, in frequency order).  Self-contained: NVRTC compiles it without any
// host header.  See maxplus_lanes.cu for the algorithm.
#pragma once

#ifndef DDSIM_LANES_NO_STD_TYPES
#include <climits>
#endif

namespace ddsim_lanes {

// 16-byte program record.  h = own lane (2 bits) | predecessor-lane mask
// (5 bits; bit 4 = temp lane holding the rare predecessors) << 2 | gap!=0 << 7.
struct alignas(16) Rec {
  long long gap;
  short s0, s1;   // smem slots of rare predecessors (R_S0 / R_S1)
  short out;      // slot receiving rel (R_OUT_SMEM: smem id, R_OUT_GLOBAL: global id)
  unsigned char rare;
  unsigned char h;
};
enum {
  R_S0 = 1, R_S1 = 2, R_SIDE = 4, R_MS = 8, R_OUT_SMEM = 16, R_OUT_GLOBAL = 32,
  R_CHAIN = 64, R_NOP = 128, R_PRE = 7, R_POST = 56
};

struct Chain {
  int lane, B, mem_off, perm_off;
};
struct Member {
  long long gap;
  int pred_off, npred;
  int out;
  int pad;
};

struct Params {
  const Rec* prog;
  int n_rec;
  const int* side_off;
  const int* side_slots;  // < ksm: smem slot, else global slot + ksm
  const long long* side_ready;
  int ksm, kglob;
  long long* gslots;
  long long s_pad;
  int S, L;
  const long long* dense64;
  long long dense_ld;
  long long* start;
  long long start_ld;
  long long* makespan;
  long long* lane_busy;
  int* neg_flag;
};

// Permutable-chain tables: a separate kernel parameter of the chain variant
// only (growing Params changes the hot loop's code generation).
struct ChainParams {
  const Chain* chains;
  const Member* members;
  const int* preds;
  const short* perm;
  const unsigned char* present;
  const int* dense32;
  int perm_ld;
  int n_chains;
};

// Derived durations (DK = 0): no per-scenario duration matrix.  A record's
// duration is its row's base duration, or the row's per-scenario override,
// then the scenario's half-up Shrink steps on the row's group
// (scale_durations, transform.py:174-183) -- what expand_durations_kernel
// would have materialised, computed where it is consumed.  Rows are staged
// per chunk by bulk copy like the records.
struct alignas(16) RowDur {
  long long base;
  unsigned group;  // 0: no scale step applies
  int ovr;         // override row, -1 none
};
struct ScaleStep {
  int lo, hi;
  long long num, den;
};
struct DerivedParams {
  const RowDur* rows;      // [n_rec]
  const long long* ovr;    // [n_ovr][S]
  const int* scale_ptr;    // [S+1] or null
  const ScaleStep* scale;
};
constexpr int kProgRegs = 2;  // scale steps kept in registers per scenario
// NVRTC defines DDSIM_DERIVED_SCALE 0 when a derived-duration table has no
// scale programs (overrides only): the program registers and checks vanish
#ifndef DDSIM_DERIVED_SCALE
#define DDSIM_DERIVED_SCALE 1
#endif
struct Prog {
  int n, e0;
  int lo[kProgRegs], hi[kProgRegs];
  long long num[kProgRegs], den[kProgRegs];
};

// round_half_up(d * num / den) (transform.py:174-183), 128-bit when needed;
// out of line so the divisions do not hold registers in the record loops
__device__ __noinline__ long long lscale_half_up(long long d, long long num, long long den) {
  const bool neg = d < 0;
  const unsigned long long a = neg ? (unsigned long long)(-d) : (unsigned long long)d;
  const unsigned long long un = (unsigned long long)num, ud = (unsigned long long)den;
  unsigned long long q;
  if (a < (1ull << 40) && un < (1ull << 21) && ud < (1ull << 40)) {
    q = (2ull * a * un + ud) / (2ull * ud);
  } else {
    const unsigned __int128 x = (unsigned __int128)a * un * 2u + ud;
    q = (unsigned long long)(x / ((unsigned __int128)ud * 2u));
  }
  return neg ? -(long long)q : (long long)q;
}

__device__ __forceinline__ void prog_load(const DerivedParams* dp, long long s, bool act, Prog& P) {
  P.n = 0;
  P.e0 = 0;
  if (!DDSIM_DERIVED_SCALE) return;
#pragma unroll
  for (int q = 0; q < kProgRegs; ++q) {
    P.lo[q] = 1;
    P.hi[q] = 0;
    P.num[q] = 1;
    P.den[q] = 1;
  }
  if (dp == nullptr || dp->scale_ptr == nullptr || !act) return;
  P.e0 = dp->scale_ptr[s];
  P.n = dp->scale_ptr[s + 1] - P.e0;
#pragma unroll
  for (int q = 0; q < kProgRegs; ++q)
    if (q < P.n) {
      const ScaleStep st = dp->scale[P.e0 + q];
      P.lo[q] = st.lo;
      P.hi[q] = st.hi;
      P.num[q] = st.num;
      P.den[q] = st.den;
    }
}

__device__ __forceinline__ long long derived_dur(const DerivedParams* dp, long long base,
                                                 unsigned group, int ovr, long long s, int S,
                                                 bool act, const Prog& P) {
  long long d = base;
  if (ovr >= 0 && act) d = dp->ovr[(long long)ovr * S + s];
  if (DDSIM_DERIVED_SCALE && group != 0u && P.n > 0) {
    if (P.n <= kProgRegs) {
#pragma unroll
      for (int q = 0; q < kProgRegs; ++q)
        if (q < P.n && group >= (unsigned)P.lo[q] && group <= (unsigned)P.hi[q] && P.num[q] != 0)
          d = lscale_half_up(d, P.num[q], P.den[q]);
    } else {
      for (int e = P.e0; e < P.e0 + P.n; ++e) {
        const ScaleStep st = dp->scale[e];
        if (group >= (unsigned)st.lo && group <= (unsigned)st.hi && st.num != 0)
          d = lscale_half_up(d, st.num, st.den);
      }
    }
  }
  return d;
}

// Segment-parallel evaluation (small scenario counts): the record stream is
// cut into K segments at rows where no slot value is live, so a segment's
// input is the L lane heads only.  seg_transfer (lanes_seg.cuh) computes each
// segment's (max,+) transfer matrix per scenario, seg_scan composes them into
// every segment's input lane heads, and the replay (lanes_body<..., SEG>)
// re-walks each segment from its true input writing the start times.
struct SegParams {
  const int* cuts;           // [K+1] segment row boundaries (multiples of kChunkL)
  int K;
  int LN;                    // lanes in the transfer matrices (graph lane count)
  int* trans;                // [K-1][LN*LN][s_pad]: entry (j, i) = longest path weight
                             // from input lane head i to output lane head j, < 0 = none
  long long* state;          // [K][LN][s_pad]: lane heads at segment starts (seg_scan)
  long long s_pad;
  int* ticket;               // fused kernel: CTA work order (zeroed per launch)
  int* flags;                // fused kernel: [K][nb] "state of (segment, block) published"
  int nb;                    // scenario blocks
  int pad;
  const long long* gapsum;   // [K] gaps of each segment's records (host)
  // Chain segment kc (-1: none): one permutable chain whose member
  // predecessors live across cuts.  It has no transfer: its replay runs
  // between two scans and exports its output lane heads to state[kc + 1].
  // The values live across its first row ("carries", global slots) are
  // produced in earlier segments; the transfer pass writes their
  // coefficients, the scan their values (gslots) before the chain replay.
  int kc;
  int replay_only;           // replay launch: >= 0 replays only that segment,
                             // -1 every segment except kc
  const int* carry_ptr;      // [K+1] carries produced per segment
  const int* carry_gid;      // their global slot ids
  int* carry_coef;           // [kglob][LN][s_pad] coefficients on the producing
                             // segment's input lane heads (< 0 = none)
};

// CUtensorMap-compatible opaque kernel parameter (128 B, 64 B aligned)
struct alignas(64) Tmap {
  unsigned long long w[16];
};

constexpr int kChunkL = 16;
#ifndef DDSIM_STAGES
#define DDSIM_STAGES 4
#endif
constexpr int kStagesL = DDSIM_STAGES;  // TMA pipeline depth (chunks in flight)
constexpr int NLANE = 4;  // register lanes; index 4 = temp (rare predecessors)

__device__ __forceinline__ unsigned su32l(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void l_mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32l(bar)) : "memory");
}
__device__ __forceinline__ void l_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32l(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void l_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(su32l(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void l_bulk(void* dst, const void* src, unsigned bytes,
                                       unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(su32l(dst)), "l"(src), "r"(bytes), "r"(su32l(bar)) : "memory");
}
__device__ __forceinline__ void l_tile(void* dst, const Tmap* map, int x, int y,
                                       unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32l(dst)), "l"(map), "r"(x), "r"(y), "r"(su32l(bar))
      : "memory");
}
__device__ __forceinline__ long long lmax(long long a, long long b) { return a > b ? a : b; }

template <int V>
struct St {
  long long lv[NLANE + 1][V];  // lane heads' rel (+ temp), V scenarios
  long long lb[NLANE][V];      // lane busy
};

template <int OWN, int MASK, int GAP, int V>
__device__ __forceinline__ void hstep(St<V>& S, long long d0, long long d1, long long gap,
                                      long long*& sp, long long ld, bool store) {
  long long a = S.lv[OWN][0], b = S.lv[OWN][V - 1];
#pragma unroll
  for (int m = 0; m <= NLANE; ++m)
    if (((MASK >> m) & 1) && m != OWN) {
      a = lmax(a, S.lv[m][0]);
      if (V == 2) b = lmax(b, S.lv[m][V - 1]);
    }
  if (store) {
    // V = 2: one 16-byte streaming store of the two adjacent scenarios (the
    // host picks V = 2 only for 16-byte aligned start rows of even pitch)
    if (V == 2)
      __stcs(reinterpret_cast<longlong2*>(sp), make_longlong2(a, b));
    else
      __stcs(sp, a);
    sp += ld;
  }
  a += d0;
  if (V == 2) b += d1;
  if (GAP) {
    a += gap;
    if (V == 2) b += gap;
  }
  S.lv[OWN][0] = a;
  S.lb[OWN][0] += d0;
  if (V == 2) {
    S.lv[OWN][V - 1] = b;
    S.lb[OWN][V - 1] += d1;
  }
}

// Branch-free handler for latency-bound launches (few scenarios, so few warps
// per SM): own lane and predecessor-lane mask are data, not code, so a record
// costs a balanced max tree + add + predicated write-back instead of a chain of
// compare-and-branch through the handler if-chain.  All values are >= 0 on
// this path (device-checked), so 0 is the identity of max.
template <int V>
__device__ __forceinline__ void hstep_dyn(St<V>& S, unsigned h, long long d0, long long d1,
                                          long long gap, long long*& sp, long long ld,
                                          bool store) {
  const unsigned own = h & 3u;
  const unsigned m = ((h >> 2) & 31u) | (1u << own);
  long long a[NLANE + 1], b[NLANE + 1];
#pragma unroll
  for (int l = 0; l <= NLANE; ++l) {
    a[l] = (m >> l) & 1u ? S.lv[l][0] : 0;
    b[l] = (m >> l) & 1u ? S.lv[l][V - 1] : 0;
  }
  long long x = lmax(lmax(lmax(a[0], a[1]), lmax(a[2], a[3])), a[4]);
  long long y = lmax(lmax(lmax(b[0], b[1]), lmax(b[2], b[3])), b[4]);
  if (store) {
    if (V == 2)
      __stcs(reinterpret_cast<longlong2*>(sp), make_longlong2(x, y));
    else
      __stcs(sp, x);
    sp += ld;
  }
  x += d0 + gap;
  y += d1 + gap;
#pragma unroll
  for (int l = 0; l < NLANE; ++l) {
    const bool mine = own == (unsigned)l;
    S.lv[l][0] = mine ? x : S.lv[l][0];
#ifndef DDSIM_NO_LB
    S.lb[l][0] += mine ? d0 : 0;
#endif
    if (V == 2) {
      S.lv[l][V - 1] = mine ? y : S.lv[l][V - 1];
#ifndef DDSIM_NO_LB
      S.lb[l][V - 1] += mine ? d1 : 0;
#endif
    }
  }
}

template <int V>
__device__ __forceinline__ long long own_get(const St<V>& S, int own, int i) {
  switch (own) {
    case 0: return S.lv[0][i];
    case 1: return S.lv[1][i];
    case 2: return S.lv[2][i];
    default: return S.lv[3][i];
  }
}

template <int V>
__device__ __forceinline__ void own_set(St<V>& S, int own, int i, long long v) {
  switch (own) {
    case 0: S.lv[0][i] = v; break;
    case 1: S.lv[1][i] = v; break;
    case 2: S.lv[2][i] = v; break;
    default: S.lv[3][i] = v; break;
  }
}
template <int V>
__device__ __forceinline__ void busy_add(St<V>& S, int own, int i, long long v) {
  switch (own) {
    case 0: S.lb[0][i] += v; break;
    case 1: S.lb[1][i] += v; break;
    case 2: S.lb[2][i] += v; break;
    default: S.lb[3][i] += v; break;
  }
}

__device__ __forceinline__ int4 l_lds128(unsigned a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ int2 l_lds64i(unsigned a) {
  int2 v;
  asm volatile("ld.shared.v2.s32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ longlong2 l_lds128ll(unsigned a) {
  longlong2 v;
  asm volatile("ld.shared.v2.s64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void l_sts128ll(unsigned a, long long x, long long y) {
  asm volatile("st.shared.v2.s64 [%0], {%1,%2};" ::"r"(a), "l"(x), "l"(y) : "memory");
}

// Load / store the V values of one slot column.
template <int V>
__device__ __forceinline__ void slot_ld(unsigned a, long long& x0, long long& x1) {
  if (V == 2) {
    const longlong2 v = l_lds128ll(a);
    x0 = v.x;
    x1 = v.y;
  } else {
    asm volatile("ld.shared.s64 %0, [%1];" : "=l"(x0) : "r"(a));
    x1 = x0;
  }
}
template <int V>
__device__ __forceinline__ void slot_st(unsigned a, long long x0, long long x1) {
  if (V == 2)
    l_sts128ll(a, x0, x1);
  else
    asm volatile("st.shared.s64 [%0], %1;" ::"r"(a), "l"(x0) : "memory");
}

// Permutable chain (inserted-task table, e.g. AllReduce buckets in a
// per-scenario order): members run back to back on the chain's lane in the
// scenario's order; every member predecessor is read from a slot; member k
// writes frozen row `row + k`.  An absent chain leaves no start (-1), its
// consumers see 0 (the identity of max here) and its lane head unchanged.
// Only instantiated for graphs with chains (lanes_body<..., CH = true>).
template <int DK, int V>
__device__ __forceinline__ void chain_record(const Params& p, const ChainParams& cp, St<V>& S,
                                             int cid, int row,
                                             long long s, bool act, bool store, long long* sp,
                                             long long ld, unsigned slot_s, unsigned slot_pitch,
                                             unsigned col, long long& ms0, long long& ms1,
                                             int& neg, const DerivedParams* dp, const Prog& P,
                                             const Prog& P2) {
  const int ksm = p.ksm;
  auto slot_addr = [&](int code, int i) { return slot_s + (unsigned)code * slot_pitch + col + 8u * i; };
  const Chain ch = cp.chains[cid];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const long long sc = s + i;
    const bool pres = !act || cp.present == nullptr || cp.present[sc * cp.n_chains + cid] != 0;
    long long prev = own_get<V>(S, ch.lane, i);
    long long lbadd = 0, msv = 0;
    // The member order, the member records and their durations do not depend
    // on the lane head: they are loaded one member ahead (the order two ahead),
    // so a member waits for its slot reads only, not for ~4 dependent global
    // loads (perm -> member; duration row -> override value).  Config 3's
    // chain segment replay: 113 -> 78 us.  (Reading the next member's
    // predecessor values ahead as well measured no further gain.)
    auto member_at = [&](int q) {
      return (cp.perm != nullptr && act) ? (int)cp.perm[sc * cp.perm_ld + ch.perm_off + q] : q;
    };
    auto dur_of = [&](int k) -> long long {
      if (DK == 0) {
        const RowDur rd = dp->rows[row + k];
        return derived_dur(dp, rd.base, rd.group, rd.ovr, sc, p.S, act, i == 0 ? P : P2);
      } else if (act) {
        const long long at = (long long)(row + k) * p.dense_ld + sc;
        return DK == 1 ? (long long)cp.dense32[at] : p.dense64[at];
      }
      return 0;
    };
    int kn = ch.B > 0 ? member_at(0) : 0;
    int kn2 = ch.B > 1 ? member_at(1) : 0;
    Member Mn = cp.members[ch.mem_off + kn];
    long long dn = pres && ch.B > 0 ? dur_of(kn) : 0;
    for (int q = 0; q < ch.B; ++q) {
      const int k = kn;
      const Member M = Mn;
      const long long d = dn;
      if (q + 1 < ch.B) {
        kn = kn2;
        kn2 = q + 2 < ch.B ? member_at(q + 2) : 0;
        Mn = cp.members[ch.mem_off + kn];
        if (pres) dn = dur_of(kn);
      }
      long long val = -1;  // start written for member k
      if (pres) {
        long long x = prev;
        for (int e = 0; e < M.npred; ++e) {
          const int code = cp.preds[M.pred_off + e];
          long long v = 0;
          if (code < ksm)
            asm volatile("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(slot_addr(code, i)));
          else if (act)
            v = p.gslots[(long long)(code - ksm) * p.s_pad + sc];
          x = lmax(x, v);
        }
        neg |= (int)(d >> 32);
        val = x;
        const long long fin = x + d;
        prev = fin + M.gap;
        msv = lmax(msv, fin);
        lbadd += d;
      }
      if (store) __stcs(sp + (long long)k * ld + i, val);
      if (M.out >= 0) {
        const long long o = pres ? prev : 0;
        if (M.out < ksm)
          asm volatile("st.shared.s64 [%0], %1;" ::"r"(slot_addr(M.out, i)), "l"(o) : "memory");
        else if (act)
          p.gslots[(long long)(M.out - ksm) * p.s_pad + sc] = o;
      }
    }
    if (pres) {
      own_set<V>(S, ch.lane, i, prev);
      busy_add<V>(S, ch.lane, i, lbadd);
      if (i == 0) ms0 = lmax(ms0, msv);
      else ms1 = lmax(ms1, msv);
    }
  }
}

// The kernel body; DDSIM_DISPATCH(h) must expand to the handler dispatch
// (it sees S, d0, d1, gap, sp, ld, store and the template parameter V).
// Each thread owns V consecutive scenarios (V = 1 or 2).
// CH: the graph has permutable chains (chain / no-op records).  Without them
// the chain code is compiled out, so the hot loop keeps its registers.
// SEG: replay of segment seg_k (rows cuts[k] .. cuts[k+1]) of scenario block
// blk from the input lane heads `init`; makespan / lane busy accumulate with
// atomics into outputs zeroed by the launcher.  Its mbarriers sit at smem + 64
// so a kernel may run it after another pipelined pass (lanes_seg.cuh).
template <int DK, int V, bool CH = false, bool SEG = false>
__device__ __forceinline__ void lanes_body(const Tmap* tmap, const Params& p,
                                           const ChainParams* cpp = nullptr,
                                           const SegParams* sgp = nullptr, int seg_k = 0,
                                           int blk = 0, const long long* init = nullptr,
                                           const DerivedParams* dp = nullptr) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int BD = blockDim.x;
  const int W = BD * V;  // scenarios per CTA
  const int tid = threadIdx.x;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + (SEG ? 64 : 0));
  Rec* pst = reinterpret_cast<Rec*>(smem + 128);
  unsigned sbase = su32l(smem);
  asm volatile("" : "+r"(sbase));  // keep in a register (no per-record rematerialisation)
  const unsigned prog_s = sbase + 128;
  const unsigned tile_s = prog_s + kStagesL * kChunkL * (unsigned)sizeof(Rec);
  constexpr unsigned ES = DK == 1 ? 4u : 8u;  // tile element bytes (int32 / int64 durations)
  // DK 0: the tile area holds the chunk's RowDur entries (16 B per row)
  const unsigned tile_all = DK == 0 ? (unsigned)(kStagesL * kChunkL * 16)
                                    : (unsigned)(kStagesL * kChunkL * W) * ES;
  const unsigned slot_s = tile_s + tile_all;                  // [ksm][BD] x (8 V) B
  const unsigned col = (unsigned)(tid * 8 * V);
  const unsigned slot_pitch = (unsigned)(BD * 8 * V);
  int* tst = reinterpret_cast<int*>(smem + (tile_s - sbase));
  const int s0 = (SEG ? blk : (int)blockIdx.x) * W;
  const int s = s0 + tid * V;
  const bool act = s < p.S;  // S % V == 0 (host)
  int r_end = p.n_rec, c_begin = 0;
  if constexpr (SEG) {
    c_begin = sgp->cuts[seg_k] / kChunkL;
    r_end = sgp->cuts[seg_k + 1];
  }
  const int nchunks = (r_end + kChunkL - 1) / kChunkL;
  const unsigned tile_bytes = (unsigned)(kChunkL * W) * ES;
  auto issue = [&](int c) {
    const int st = (c - c_begin) % kStagesL;
    const int nrec = min(kChunkL, r_end - c * kChunkL);
    const unsigned pb = (unsigned)(nrec * sizeof(Rec));
    if (DK == 0) {
      l_expect(&bars[st], 2 * pb);
      l_bulk(pst + st * kChunkL, p.prog + (long long)c * kChunkL, pb, &bars[st]);
      l_bulk(reinterpret_cast<unsigned char*>(tst) + (size_t)st * kChunkL * 16,
             dp->rows + (long long)c * kChunkL, pb, &bars[st]);
      return;
    }
    l_expect(&bars[st], pb + tile_bytes);
    l_bulk(pst + st * kChunkL, p.prog + (long long)c * kChunkL, pb, &bars[st]);
    l_tile(reinterpret_cast<unsigned char*>(tst) + (size_t)st * kChunkL * W * ES, tmap, s0,
           c * kChunkL, &bars[st]);
  };
  if (tid == 0) {
    for (int i = 0; i < kStagesL; ++i) l_mbar_init(&bars[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int c = c_begin; c < min(c_begin + kStagesL, nchunks); ++c) issue(c);

  St<V> S;
#pragma unroll
  for (int l = 0; l <= NLANE; ++l)
#pragma unroll
    for (int i = 0; i < V; ++i) S.lv[l][i] = 0;
  if constexpr (SEG) {  // init: [lane][V]
#pragma unroll
    for (int l = 0; l < NLANE; ++l)
#pragma unroll
      for (int i = 0; i < V; ++i) S.lv[l][i] = init[l * V + i];
  }
#pragma unroll
  for (int l = 0; l < NLANE; ++l)
#pragma unroll
    for (int i = 0; i < V; ++i) S.lb[l][i] = 0;
  long long ms0 = 0, ms1 = 0;
  int neg = 0;
  const long long ld = p.start_ld;
  const bool store = act && p.start != nullptr;
  long long* sp = store ? p.start + (long long)c_begin * kChunkL * ld + s : nullptr;
  const unsigned row_pitch = DK == 0 ? 16u : (unsigned)W * ES;
  const int ksm = p.ksm;
  Prog P, P2;  // derived durations: the scale program of each scenario
  if (DK == 0) prog_load(dp, s, act, P);
  if (DK == 0 && V == 2) prog_load(dp, s + 1, act, P2);

  for (int c = c_begin; c < nchunks; ++c) {
    const int st = (c - c_begin) % kStagesL;
    l_wait(&bars[st], (unsigned)(((c - c_begin) / kStagesL) & 1));
    const unsigned rec0 = prog_s + (unsigned)(st * kChunkL * sizeof(Rec));
    const unsigned t0 = DK == 0 ? tile_s + (unsigned)(st * kChunkL) * 16u
                                : tile_s + (unsigned)(st * kChunkL) * row_pitch + (unsigned)tid * ES * V;
    const int nrec = min(kChunkL, r_end - c * kChunkL);
    int4 raw = l_lds128(rec0);
    // prefetched durations of the next record: int32 pair (DK 1) / int64 pair (DK 2)
    int2 dd = make_int2(0, 0);
    longlong2 dq = make_longlong2(0, 0);
    auto load_d = [&](unsigned ta) {
      if (DK == 0) {
        const int4 rd = l_lds128(ta);
        const long long b = ((long long)rd.y << 32) | (unsigned)rd.x;
        dq.x = derived_dur(dp, b, (unsigned)rd.z, rd.w, s, p.S, act, P);
        if (V == 2) dq.y = derived_dur(dp, b, (unsigned)rd.z, rd.w, s + 1, p.S, act, P2);
      } else if (DK == 1) {
        if (V == 2)
          dd = l_lds64i(ta);
        else
          asm volatile("ld.shared.s32 %0, [%1];" : "=r"(dd.x) : "r"(ta));
      } else {
        if (V == 2)
          dq = l_lds128ll(ta);
        else
          asm volatile("ld.shared.s64 %0, [%1];" : "=l"(dq.x) : "r"(ta));
      }
    };
    load_d(t0);
    auto record = [&](int j) {
      const int4 r = raw;
      long long d0, d1 = 0;
      if (DK == 1) {
        d0 = (unsigned)dd.x;
        if (V == 2) d1 = (unsigned)dd.y;
        neg |= dd.x | dd.y;
      } else {
        d0 = dq.x;
        if (V == 2) d1 = dq.y;
        neg |= (int)((d0 | d1) >> 32);
      }
      if (j + 1 < nrec) {  // prefetch the next record and durations
        raw = l_lds128(rec0 + (unsigned)(j + 1) * 16u);
        load_d(t0 + (unsigned)(j + 1) * row_pitch);
      }
      const long long gap = ((long long)(unsigned)r.y << 32) | (unsigned)r.x;
      const unsigned w = (unsigned)r.w;
      const unsigned h = w >> 24;
      const unsigned rare = (w >> 16) & 0xffu;
      if constexpr (CH) {
        if (rare & (R_CHAIN | R_NOP)) {
          if (rare & R_CHAIN)
            chain_record<DK, V>(p, *cpp, S, (int)(short)(r.z & 0xffff), c * kChunkL + j, s, act,
                                store, sp, ld, slot_s, slot_pitch, col, ms0, ms1, neg, dp, P, P2);
          if (store) sp += ld;
          return;
        }
      }
      if (rare & R_PRE) {
        // predecessors that are no longer lane heads (+ ready floor) -> temp lane
        long long x0 = 0, x1 = 0, y0, y1;
        const int row = c * kChunkL + j;
        if (rare & R_S0) {
          slot_ld<V>(slot_s + (unsigned)((r.z << 16) >> 16) * slot_pitch + col, y0, y1);
          x0 = lmax(x0, y0);
          x1 = lmax(x1, y1);
        }
        if (rare & R_S1) {
          slot_ld<V>(slot_s + (unsigned)(r.z >> 16) * slot_pitch + col, y0, y1);
          x0 = lmax(x0, y0);
          x1 = lmax(x1, y1);
        }
        if (rare & R_SIDE) {
          if (p.side_ready) {
            x0 = lmax(x0, p.side_ready[row]);
            x1 = lmax(x1, p.side_ready[row]);
          }
          if (p.side_off)
            for (int k = p.side_off[row]; k < p.side_off[row + 1]; ++k) {
              const int code = p.side_slots[k];
              if (code < ksm) {
                slot_ld<V>(slot_s + (unsigned)code * slot_pitch + col, y0, y1);
                x0 = lmax(x0, y0);
                x1 = lmax(x1, y1);
              } else if (act) {
                const long long* g = p.gslots + (long long)(code - ksm) * p.s_pad + s;
                x0 = lmax(x0, g[0]);
                x1 = lmax(x1, g[V - 1]);
              }
            }
        }
        S.lv[NLANE][0] = x0;
        S.lv[NLANE][V - 1] = V == 2 ? x1 : x0;
      }
      DDSIM_DISPATCH(h)
      if (rare & R_POST) {
        const int own = (int)(h & 3);
        const long long r0 = own_get<V>(S, own, 0), r1 = own_get<V>(S, own, V - 1);
        if (rare & R_MS) {
          const long long g2 = (h >> 7) & 1 ? gap : 0;
          ms0 = lmax(ms0, r0 - g2);
          ms1 = lmax(ms1, r1 - g2);
        }
        if (rare & R_OUT_SMEM) {
          slot_st<V>(slot_s + (unsigned)((w << 16) >> 16) * slot_pitch + col, r0, r1);
        } else if ((rare & R_OUT_GLOBAL) && act) {
          long long* g = p.gslots + (long long)((int)(w << 16) >> 16) * p.s_pad + s;
          g[0] = r0;
          if (V == 2) g[1] = r1;
        }
      }
    };
#ifdef DDSIM_UNROLL
    if (nrec == kChunkL) {
#pragma unroll DDSIM_UNROLL
      for (int j = 0; j < kChunkL; ++j) record(j);
    } else {
#pragma unroll 1
      for (int j = 0; j < nrec; ++j) record(j);
    }
#else
#pragma unroll 1
    for (int j = 0; j < nrec; ++j) record(j);
#endif
    __syncthreads();
    if (tid == 0 && c + kStagesL < nchunks) issue(c + kStagesL);
  }
  if constexpr (SEG) {
    if (act) {
      // the transfer's int32 coefficients are exact when the segment's
      // durations + gaps stay below 2^30 (lanes_seg.cuh); the replay holds the
      // duration sums anyway (lane busy), so it certifies the transfer, and a
      // negative duration voids the fast path for both passes
      bool over = false;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        long long wsum = sgp->gapsum[seg_k];
#pragma unroll
        for (int q = 0; q < NLANE; ++q) wsum += S.lb[q][i];
        over |= wsum >= (1LL << 30);
      }
      if ((neg < 0 || (over && seg_k != sgp->kc)) && p.neg_flag) atomicOr(p.neg_flag, 1);
      if (seg_k == sgp->kc && seg_k + 1 < sgp->K)
#pragma unroll
        for (int l = 0; l < NLANE; ++l)
#pragma unroll
          for (int i = 0; i < V; ++i)
            if (l < sgp->LN)
              sgp->state[((long long)(seg_k + 1) * sgp->LN + l) * sgp->s_pad + s + i] = S.lv[l][i];
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const long long m = i == 0 ? ms0 : ms1;  // >= 0 on this path
        if (p.makespan && m > 0)
          atomicMax(reinterpret_cast<unsigned long long*>(p.makespan + s + i),
                    (unsigned long long)m);
        if (p.lane_busy)
#pragma unroll
          for (int q = 0; q < NLANE; ++q)
            if (q < p.L && S.lb[q][i] != 0)
              atomicAdd(reinterpret_cast<unsigned long long*>(p.lane_busy +
                                                              (long long)(s + i) * p.L + q),
                        (unsigned long long)S.lb[q][i]);
      }
    }
    return;
  }
  if (act) {
    if (neg < 0 && p.neg_flag) atomicOr(p.neg_flag, 1);
    if (p.makespan) {
      p.makespan[s] = ms0;
      if (V == 2) p.makespan[s + 1] = ms1;
    }
    if (p.lane_busy)
      for (int l = 0; l < p.L; ++l) {
        long long v0 = 0, v1 = 0;
#pragma unroll
        for (int q = 0; q < NLANE; ++q)
          if (q == l) {
            v0 = S.lb[q][0];
            v1 = S.lb[q][V - 1];
          }
        p.lane_busy[(long long)s * p.L + l] = v0;
        if (V == 2) p.lane_busy[(long long)(s + 1) * p.L + l] = v1;
      }
  }
}

}  // namespace ddsim_lanes
