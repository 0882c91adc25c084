// Segment transfer body (NVRTC source, compiled after lanes_body.cuh): the
// (max,+) transfer matrix of one segment of the lane-register program, per
// scenario.  See SegParams in lanes_body.cuh for the three-pass scheme.
//
// Recurrence (sim.py:89-142 on lane-chained graphs == synthetic.py:35-48):
//     rel(v) = max_{u->v} rel(u) + dur(v) + gap(v),   start(v) = max_{u->v} rel(u).
// Within a segment every value is a (max,+) affine function of the input lane
// heads h_0 .. h_{L-1}:  rel(v) = max_i (A_v,i + h_i).  A value is carried as
// its L coefficients; a record costs L maxes per predecessor lane and L adds.
// The constant term is dominated and dropped: every record reads its own lane
// head, whose coefficient on its own input is >= 0, and inputs are >= 0
// (durations >= 0 device-checked, gaps >= 0 and no ready floors host-checked).
//
// Coefficients are int32 with "none" = a negative number: entries are path
// weights within the segment, so they stay below 2^30 when the segment's
// durations + gaps sum below 2^30, and kNegSym + that sum stays negative.  The
// replay of the same segment checks that sum (and negative durations) per
// scenario from its lane-busy sums; otherwise the exact general kernel reruns
// the launch.
#pragma once

namespace ddsim_lanes {

constexpr int kNegSym = -(1 << 30);

template <int LN>
struct Sym {
  int v[NLANE + 1][LN];  // lane heads' coefficients (+ temp lane)
};

__device__ __forceinline__ int imax(int a, int b) { return a > b ? a : b; }

template <int OWN, int MASK, int GAP, int LN>
__device__ __forceinline__ void hsym(Sym<LN>& Y, int d, int gap) {
  int x[LN];
#pragma unroll
  for (int c = 0; c < LN; ++c) x[c] = Y.v[OWN][c];
#pragma unroll
  for (int m = 0; m <= NLANE; ++m)
    if (((MASK >> m) & 1) && m != OWN)
#pragma unroll
      for (int c = 0; c < LN; ++c) x[c] = imax(x[c], Y.v[m][c]);
  const int a = GAP ? d + gap : d;
#pragma unroll
  for (int c = 0; c < LN; ++c) Y.v[OWN][c] = x[c] + a;
}

// Slot columns hold 4 coefficients (16 B per thread) whatever LN is.
__device__ __forceinline__ void sym_slot_ld(unsigned a, int (&y)[4]) {
  asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(y[0]), "=r"(y[1]), "=r"(y[2]), "=r"(y[3]) : "r"(a));
}
__device__ __forceinline__ void sym_slot_st(unsigned a, const int (&y)[4]) {
  asm volatile("st.shared.v4.s32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(y[0]), "r"(y[1]),
               "r"(y[2]), "r"(y[3]) : "memory");
}

template <int LN>
__device__ __forceinline__ void sym_get(const Sym<LN>& Y, int lane, int (&y)[4]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) y[c] = kNegSym;
#pragma unroll
  for (int l = 0; l < NLANE; ++l)
    if (l == lane)
#pragma unroll
      for (int c = 0; c < LN; ++c) y[c] = Y.v[l][c];
}
template <int LN>
__device__ __forceinline__ void sym_set(Sym<LN>& Y, int lane, const int (&y)[4]) {
#pragma unroll
  for (int l = 0; l < NLANE; ++l)
    if (l == lane)
#pragma unroll
      for (int c = 0; c < LN; ++c) Y.v[l][c] = y[c];
}

// Permutable chain in coefficient form (chain_record in lanes_body.cuh):
// members in the scenario's order, predecessors from slots, an absent chain
// publishes "none" and leaves its lane head alone.
template <int DK, int LN>
__device__ __forceinline__ void chain_sym(const Params& p, const ChainParams& cp, Sym<LN>& Y,
                                          int cid, int row, long long s, bool act,
                                          unsigned slot_s, unsigned slot_pitch, unsigned col,
                                          const DerivedParams* dp, const Prog& P) {
  const Chain ch = cp.chains[cid];
  const bool pres = !act || cp.present == nullptr || cp.present[s * cp.n_chains + cid] != 0;
  int prev[4];
  sym_get<LN>(Y, ch.lane, prev);
  for (int q = 0; q < ch.B; ++q) {
    const int k = (cp.perm != nullptr && act) ? (int)cp.perm[s * cp.perm_ld + ch.perm_off + q] : q;
    const Member M = cp.members[ch.mem_off + k];
    if (pres) {
      int x[4] = {prev[0], prev[1], prev[2], prev[3]};
      for (int e = 0; e < M.npred; ++e) {
        int y[4];
        sym_slot_ld(slot_s + (unsigned)cp.preds[M.pred_off + e] * slot_pitch + col, y);
#pragma unroll
        for (int c = 0; c < 4; ++c) x[c] = imax(x[c], y[c]);
      }
      long long d = 0;
      if (DK == 0) {
        const RowDur rd = dp->rows[row + k];
        d = derived_dur(dp, rd.base, rd.group, rd.ovr, s, p.S, act, P);
      } else if (act) {
        const long long at = (long long)(row + k) * p.dense_ld + s;
        d = DK == 1 ? (long long)cp.dense32[at] : p.dense64[at];
      }
      const int a = (int)d + (int)M.gap;
#pragma unroll
      for (int c = 0; c < 4; ++c) prev[c] = x[c] + a;
    }
    if (M.out >= 0) {
      int o[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) o[c] = pres ? prev[c] : kNegSym;
      sym_slot_st(slot_s + (unsigned)M.out * slot_pitch + col, o);
    }
  }
  if (pres) sym_set<LN>(Y, ch.lane, prev);
}

// Transfer of segment `seg` for scenario block `blk` (one thread per
// scenario; the last segment's transfer is never needed): coef[j][i] = longest
// path weight from input lane head i to output lane head j (< 0 = none).
// DDSIM_SYM_DISPATCH(h) expands to the handler if-chain over the graph's codes
// (it sees Y, dv, gp and LN).
template <int DK, int LN, bool CH>
__device__ __forceinline__ void sym_pass(const Tmap* tmap, const Params& p, const SegParams& sg,
                                         const ChainParams* cpp, int seg, int blk,
                                         int (&coef)[LN][LN], const DerivedParams* dp) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int BD = blockDim.x;
  const int tid = threadIdx.x;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem);
  Rec* pst = reinterpret_cast<Rec*>(smem + 128);
  unsigned sbase = su32l(smem);
  asm volatile("" : "+r"(sbase));
  const unsigned prog_s = sbase + 128;
  const unsigned tile_s = prog_s + kStagesL * kChunkL * (unsigned)sizeof(Rec);
  constexpr unsigned ES = DK == 1 ? 4u : 8u;
  const unsigned tile_all = DK == 0 ? (unsigned)(kStagesL * kChunkL * 16)
                                    : (unsigned)(kStagesL * kChunkL * BD) * ES;
  const unsigned slot_s = tile_s + tile_all;  // [ksm][BD] x 16 B
  const unsigned col = (unsigned)(tid * 16);
  const unsigned slot_pitch = (unsigned)(BD * 16);
  unsigned char* tst = smem + (tile_s - sbase);
  const int s0 = blk * BD;
  const int s = s0 + tid;
  const bool act = s < p.S;
  const int c_begin = sg.cuts[seg] / kChunkL;
  const int r_end = sg.cuts[seg + 1];
  const int nchunks = (r_end + kChunkL - 1) / kChunkL;
  const unsigned tile_bytes = (unsigned)(kChunkL * BD) * ES;
  auto issue = [&](int c) {
    const int st = (c - c_begin) % kStagesL;
    const int nrec = min(kChunkL, r_end - c * kChunkL);
    const unsigned pb = (unsigned)(nrec * sizeof(Rec));
    if (DK == 0) {
      l_expect(&bars[st], 2 * pb);
      l_bulk(pst + st * kChunkL, p.prog + (long long)c * kChunkL, pb, &bars[st]);
      l_bulk(tst + (size_t)st * kChunkL * 16, dp->rows + (long long)c * kChunkL, pb, &bars[st]);
      return;
    }
    l_expect(&bars[st], pb + tile_bytes);
    l_bulk(pst + st * kChunkL, p.prog + (long long)c * kChunkL, pb, &bars[st]);
    l_tile(tst + (size_t)st * kChunkL * BD * ES, tmap, s0, c * kChunkL, &bars[st]);
  };
  if (tid == 0) {
    for (int i = 0; i < kStagesL; ++i) l_mbar_init(&bars[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int c = c_begin; c < min(c_begin + kStagesL, nchunks); ++c) issue(c);

  Sym<LN> Y;
#pragma unroll
  for (int l = 0; l <= NLANE; ++l)
#pragma unroll
    for (int c = 0; c < LN; ++c) Y.v[l][c] = (l == c) ? 0 : kNegSym;
  const unsigned row_pitch = DK == 0 ? 16u : (unsigned)BD * ES;
  Prog P;
  if (DK == 0) prog_load(dp, s, act, P);

  for (int c = c_begin; c < nchunks; ++c) {
    const int st = (c - c_begin) % kStagesL;
    l_wait(&bars[st], (unsigned)(((c - c_begin) / kStagesL) & 1));
    const unsigned rec0 = prog_s + (unsigned)(st * kChunkL * sizeof(Rec));
    const unsigned t0 = DK == 0 ? tile_s + (unsigned)(st * kChunkL) * 16u
                                : tile_s + (unsigned)(st * kChunkL) * row_pitch + (unsigned)tid * ES;
    const int nrec = min(kChunkL, r_end - c * kChunkL);
    // prefetched record and duration of the next record (the decode and the
    // shared-memory loads overlap this record's coefficient updates)
    int4 raw = l_lds128(rec0);
    long long dn = 0;
    auto load_d = [&](unsigned ta) {
      if (DK == 0) {
        const int4 rd = l_lds128(ta);
        dn = derived_dur(dp, ((long long)rd.y << 32) | (unsigned)rd.x, (unsigned)rd.z, rd.w, s,
                         p.S, act, P);
      } else if (DK == 1) {
        int x;
        asm volatile("ld.shared.s32 %0, [%1];" : "=r"(x) : "r"(ta));
        dn = x;
      } else {
        asm volatile("ld.shared.s64 %0, [%1];" : "=l"(dn) : "r"(ta));
      }
    };
    load_d(t0);
    auto record = [&](int j) {
      const int4 r = raw;
      const long long d = dn;
      if (j + 1 < nrec) {
        raw = l_lds128(rec0 + (unsigned)(j + 1) * 16u);
        load_d(t0 + (unsigned)(j + 1) * row_pitch);
      }
      const int gp = r.x;  // gap < 2^30 (host: every segment's gap sum is)
      const unsigned w = (unsigned)r.w;
      const unsigned h = w >> 24;
      const unsigned rare = (w >> 16) & 0xffu;
      if constexpr (CH) {
        if (rare & (R_CHAIN | R_NOP)) {
          if (rare & R_CHAIN)
            chain_sym<DK, LN>(p, *cpp, Y, (int)(short)(r.z & 0xffff), c * kChunkL + j, s, act,
                              slot_s, slot_pitch, col, dp, P);
          return;
        }
      }
      const int dv = (int)d;
      if (rare & R_PRE) {
        // slot predecessors (all in shared memory on this path) -> temp lane
        int x[4] = {kNegSym, kNegSym, kNegSym, kNegSym}, y[4];
        const int row = c * kChunkL + j;
        if (rare & R_S0) {
          sym_slot_ld(slot_s + (unsigned)((r.z << 16) >> 16) * slot_pitch + col, y);
#pragma unroll
          for (int q = 0; q < 4; ++q) x[q] = imax(x[q], y[q]);
        }
        if (rare & R_S1) {
          sym_slot_ld(slot_s + (unsigned)(r.z >> 16) * slot_pitch + col, y);
#pragma unroll
          for (int q = 0; q < 4; ++q) x[q] = imax(x[q], y[q]);
        }
        if ((rare & R_SIDE) && p.side_off)
          for (int k = p.side_off[row]; k < p.side_off[row + 1]; ++k) {
            sym_slot_ld(slot_s + (unsigned)p.side_slots[k] * slot_pitch + col, y);
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = imax(x[q], y[q]);
          }
#pragma unroll
        for (int q = 0; q < LN; ++q) Y.v[NLANE][q] = x[q];
      }
      DDSIM_SYM_DISPATCH(h)
      if (rare & R_OUT_SMEM) {
        int y[4];
        sym_get<LN>(Y, (int)(h & 3), y);
        sym_slot_st(slot_s + (unsigned)((w << 16) >> 16) * slot_pitch + col, y);
      } else if ((rare & R_OUT_GLOBAL) && act) {
        // a carry (read only in the chain segment): its coefficients
        int y[4];
        sym_get<LN>(Y, (int)(h & 3), y);
        int* o = sg.carry_coef + (long long)((int)(w << 16) >> 16) * LN * sg.s_pad + s;
#pragma unroll
        for (int q = 0; q < LN; ++q) o[(long long)q * sg.s_pad] = y[q];
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
#pragma unroll
  for (int j = 0; j < LN; ++j)
#pragma unroll
    for (int i = 0; i < LN; ++i) coef[j][i] = Y.v[j][i];
}

// Two scenarios per thread: the transfer pass is instruction-bound (record
// decode and dispatch dominate the L x L coefficient updates), so a thread
// decodes each record once for two adjacent scenarios.  Duration tiles hold
// both scenarios' durations (one 8/16-byte load); derived durations (DK 0)
// share the record's RowDur and derive twice.  Chains and carries as sym_pass,
// per scenario.  DDSIM_SYM_DISPATCH2(h) applies the handler to (Y, dv, gp)
// and (Y2, dv2, gp).
template <int DK, int LN, bool CH>
__device__ __forceinline__ void sym_pass2(const Tmap* tmap, const Params& p, const SegParams& sg,
                                          const ChainParams* cpp, int seg, int blk,
                                          int (&coef)[LN][LN], int (&coef2)[LN][LN],
                                          const DerivedParams* dp) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int BD = blockDim.x;
  const int W = 2 * BD;
  const int tid = threadIdx.x;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem);
  Rec* pst = reinterpret_cast<Rec*>(smem + 128);
  unsigned sbase = su32l(smem);
  asm volatile("" : "+r"(sbase));
  const unsigned prog_s = sbase + 128;
  const unsigned tile_s = prog_s + kStagesL * kChunkL * (unsigned)sizeof(Rec);
  constexpr unsigned ES = DK == 1 ? 4u : 8u;
  const unsigned tile_all = DK == 0 ? (unsigned)(kStagesL * kChunkL * 16)
                                    : (unsigned)(kStagesL * kChunkL * W) * ES;
  const unsigned slot_s = tile_s + tile_all;  // [ksm][BD] x 32 B (two scenarios)
  const unsigned col = (unsigned)(tid * 32);
  const unsigned slot_pitch = (unsigned)(BD * 32);
  unsigned char* tst = smem + (tile_s - sbase);
  const int s0 = blk * W;
  const long long s = s0 + 2 * tid, s2 = s + 1;
  const bool act = s < p.S, act2 = s2 < p.S;
  const int c_begin = sg.cuts[seg] / kChunkL;
  const int r_end = sg.cuts[seg + 1];
  const int nchunks = (r_end + kChunkL - 1) / kChunkL;
  const unsigned tile_bytes = (unsigned)(kChunkL * W) * ES;
  auto issue = [&](int c) {
    const int st = (c - c_begin) % kStagesL;
    const int nrec = min(kChunkL, r_end - c * kChunkL);
    const unsigned pb = (unsigned)(nrec * sizeof(Rec));
    if (DK == 0) {
      l_expect(&bars[st], 2 * pb);
      l_bulk(pst + st * kChunkL, p.prog + (long long)c * kChunkL, pb, &bars[st]);
      l_bulk(tst + (size_t)st * kChunkL * 16, dp->rows + (long long)c * kChunkL, pb, &bars[st]);
      return;
    }
    l_expect(&bars[st], pb + tile_bytes);
    l_bulk(pst + st * kChunkL, p.prog + (long long)c * kChunkL, pb, &bars[st]);
    l_tile(tst + (size_t)st * kChunkL * W * ES, tmap, s0, c * kChunkL, &bars[st]);
  };
  if (tid == 0) {
    for (int i = 0; i < kStagesL; ++i) l_mbar_init(&bars[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int c = c_begin; c < min(c_begin + kStagesL, nchunks); ++c) issue(c);

  Sym<LN> Y, Y2;
#pragma unroll
  for (int l = 0; l <= NLANE; ++l)
#pragma unroll
    for (int c = 0; c < LN; ++c) Y.v[l][c] = Y2.v[l][c] = (l == c) ? 0 : kNegSym;
  const unsigned row_pitch = DK == 0 ? 16u : (unsigned)W * ES;
  Prog P, P2;
  if (DK == 0) {
    prog_load(dp, s, act, P);
    prog_load(dp, s2, act2, P2);
  }

  for (int c = c_begin; c < nchunks; ++c) {
    const int st = (c - c_begin) % kStagesL;
    l_wait(&bars[st], (unsigned)(((c - c_begin) / kStagesL) & 1));
    const unsigned rec0 = prog_s + (unsigned)(st * kChunkL * sizeof(Rec));
    const unsigned t0 = DK == 0 ? tile_s + (unsigned)(st * kChunkL) * 16u
                                : tile_s + (unsigned)(st * kChunkL) * row_pitch + (unsigned)tid * ES * 2u;
    const int nrec = min(kChunkL, r_end - c * kChunkL);
    int4 raw = l_lds128(rec0);
    int dn = 0, dn2 = 0;
    auto load_d = [&](unsigned ta) {
      if (DK == 0) {
        const int4 rd = l_lds128(ta);
        const long long b = ((long long)rd.y << 32) | (unsigned)rd.x;
        dn = (int)derived_dur(dp, b, (unsigned)rd.z, rd.w, s, p.S, act, P);
        dn2 = (int)derived_dur(dp, b, (unsigned)rd.z, rd.w, s2, p.S, act2, P2);
      } else if (DK == 1) {
        const int2 v = l_lds64i(ta);
        dn = v.x;
        dn2 = v.y;
      } else {
        const longlong2 v = l_lds128ll(ta);
        dn = (int)v.x;
        dn2 = (int)v.y;
      }
    };
    load_d(t0);
    auto record = [&](int j) {
      const int4 r = raw;
      const int dv = dn, dv2 = dn2;
      if (j + 1 < nrec) {
        raw = l_lds128(rec0 + (unsigned)(j + 1) * 16u);
        load_d(t0 + (unsigned)(j + 1) * row_pitch);
      }
      const int gp = r.x;
      const unsigned w = (unsigned)r.w;
      const unsigned h = w >> 24;
      const unsigned rare = (w >> 16) & 0xffu;
      if constexpr (CH) {
        if (rare & (R_CHAIN | R_NOP)) {
          if (rare & R_CHAIN) {
            const int cid = (int)(short)(r.z & 0xffff), row = c * kChunkL + j;
            chain_sym<DK, LN>(p, *cpp, Y, cid, row, s, act, slot_s, slot_pitch, col, dp, P);
            chain_sym<DK, LN>(p, *cpp, Y2, cid, row, s2, act2, slot_s, slot_pitch, col + 16u, dp,
                              P2);
          }
          return;
        }
      }
      if (rare & R_PRE) {
        int x[4] = {kNegSym, kNegSym, kNegSym, kNegSym}, x2[4] = {kNegSym, kNegSym, kNegSym, kNegSym};
        int y[4], y2[4];
        const int row = c * kChunkL + j;
        auto take = [&](unsigned code) {
          const unsigned a = slot_s + code * slot_pitch + col;
          sym_slot_ld(a, y);
          sym_slot_ld(a + 16u, y2);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            x[q] = imax(x[q], y[q]);
            x2[q] = imax(x2[q], y2[q]);
          }
        };
        if (rare & R_S0) take((unsigned)((r.z << 16) >> 16));
        if (rare & R_S1) take((unsigned)(r.z >> 16));
        if ((rare & R_SIDE) && p.side_off)
          for (int k = p.side_off[row]; k < p.side_off[row + 1]; ++k) take((unsigned)p.side_slots[k]);
#pragma unroll
        for (int q = 0; q < LN; ++q) {
          Y.v[NLANE][q] = x[q];
          Y2.v[NLANE][q] = x2[q];
        }
      }
      DDSIM_SYM_DISPATCH2(h)
      if (rare & R_OUT_SMEM) {
        int y[4], y2[4];
        sym_get<LN>(Y, (int)(h & 3), y);
        sym_get<LN>(Y2, (int)(h & 3), y2);
        const unsigned a = slot_s + (unsigned)((w << 16) >> 16) * slot_pitch + col;
        sym_slot_st(a, y);
        sym_slot_st(a + 16u, y2);
      } else if (rare & R_OUT_GLOBAL) {
        // a carry (read only in the chain segment): its coefficients
        int y[4], y2[4];
        sym_get<LN>(Y, (int)(h & 3), y);
        sym_get<LN>(Y2, (int)(h & 3), y2);
        int* o = sg.carry_coef + (long long)((int)(w << 16) >> 16) * LN * sg.s_pad + s;
#pragma unroll
        for (int q = 0; q < LN; ++q) {
          if (act) o[(long long)q * sg.s_pad] = y[q];
          if (act2) o[(long long)q * sg.s_pad + 1] = y2[q];
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
#pragma unroll
  for (int j = 0; j < LN; ++j)
#pragma unroll
    for (int i = 0; i < LN; ++i) {
      coef[j][i] = Y.v[j][i];
      coef2[j][i] = Y2.v[j][i];
    }
}

template <int DK, int LN, bool CH>
__device__ __forceinline__ void sym_body2(const Tmap* tmap, const Params& p, const SegParams& sg,
                                          const ChainParams* cpp, const DerivedParams* dp) {
  if ((int)blockIdx.y == sg.kc) return;  // the chain segment is replayed numerically
  int coef[LN][LN], coef2[LN][LN];
  sym_pass2<DK, LN, CH>(tmap, p, sg, cpp, (int)blockIdx.y, (int)blockIdx.x, coef, coef2, dp);
  const long long s = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (s < p.S) {  // (an odd S leaves the last thread's second scenario out)
    int* out = sg.trans + (long long)blockIdx.y * LN * LN * sg.s_pad + s;
    const bool second = s + 1 < p.S;
#pragma unroll
    for (int j = 0; j < LN; ++j)
#pragma unroll
      for (int i = 0; i < LN; ++i) {
        out[(long long)(j * LN + i) * sg.s_pad] = coef[j][i];
        if (second) out[(long long)(j * LN + i) * sg.s_pad + 1] = coef2[j][i];
      }
  }
}

// Three-kernel path, pass 1: blockIdx.y = segment, coefficients to sg.trans.
template <int DK, int LN, bool CH>
__device__ __forceinline__ void sym_body(const Tmap* tmap, const Params& p, const SegParams& sg,
                                         const ChainParams* cpp, const DerivedParams* dp) {
  if ((int)blockIdx.y == sg.kc) return;  // the chain segment is replayed numerically
  int coef[LN][LN];
  sym_pass<DK, LN, CH>(tmap, p, sg, cpp, (int)blockIdx.y, (int)blockIdx.x, coef, dp);
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < p.S) {
    int* out = sg.trans + (long long)blockIdx.y * LN * LN * sg.s_pad + s;
#pragma unroll
    for (int j = 0; j < LN; ++j)
#pragma unroll
      for (int i = 0; i < LN; ++i) out[(long long)(j * LN + i) * sg.s_pad] = coef[j][i];
  }
}

// Three-kernel path, pass 3: replay of segment blockIdx.y from seg_scan's
// state; RV scenarios per thread (2: one record decode for both, S even).
template <int DK, int LN, bool CH, int RV = 1>
__device__ __forceinline__ void replay_body(const Tmap* tmap, const Params& p,
                                            const SegParams& sg, const ChainParams* cpp,
                                            const DerivedParams* dp) {
  const int k = sg.replay_only >= 0 ? sg.replay_only : (int)blockIdx.y;
  if (sg.replay_only < 0 && k == sg.kc) return;  // replayed before the second scan
  long long init[NLANE * RV];
#pragma unroll
  for (int q = 0; q < NLANE * RV; ++q) init[q] = 0;
  const long long s = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * RV;
  if (k > 0 && s < p.S)
#pragma unroll
    for (int l = 0; l < LN; ++l)
#pragma unroll
      for (int i = 0; i < RV; ++i)
        init[l * RV + i] = sg.state[((long long)k * LN + l) * sg.s_pad + s + i];
  lanes_body<DK, RV, CH, true>(tmap, p, cpp, &sg, k, (int)blockIdx.x, init, dp);
}
template <int DK, int LN, bool CH>
__device__ __forceinline__ void replay_body2(const Tmap* tmap, const Params& p,
                                             const SegParams& sg, const ChainParams* cpp,
                                             const DerivedParams* dp) {
  replay_body<DK, LN, CH, 2>(tmap, p, sg, cpp, dp);
}

// Fused single pass with decoupled look-back: CTAs take (segment, block) work
// items in ticket order (segment-major), compute their segment's transfer,
// wait until the previous segment of the same block published this segment's
// input lane heads, publish the next segment's, then replay.  A CTA only waits
// on an item with a smaller ticket (already running), so the chain always
// progresses; later items' transfers overlap earlier items' replays.
template <int DK, int LN, bool CH>
__device__ __forceinline__ void fused_body(const Tmap* tmap, const Params& p, const SegParams& sg,
                                           const ChainParams* cpp, const DerivedParams* dp) {
  __shared__ int tk;
  if (threadIdx.x == 0) tk = atomicAdd(sg.ticket, 1);
  __syncthreads();
  const int k = tk / sg.nb, b = tk % sg.nb;
  const long long s = (long long)b * blockDim.x + threadIdx.x;
  const bool act = s < p.S;
  const bool last = k + 1 >= sg.K;
  int coef[LN][LN];
  if (!last) sym_pass<DK, LN, CH>(tmap, p, sg, cpp, k, b, coef, dp);
  long long st[NLANE] = {0, 0, 0, 0};
  if (k > 0) {
    if (threadIdx.x == 0) {
      const int* f = sg.flags + (long long)k * sg.nb + b;
      int v = 0;
      while (true) {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v) break;
        __nanosleep(64);
      }
    }
    __syncthreads();
    if (act)
#pragma unroll
      for (int l = 0; l < LN; ++l)
        st[l] = __ldcg(sg.state + ((long long)k * LN + l) * sg.s_pad + s);
  }
  if (!last) {
    if (act) {
      long long* out = sg.state + (long long)(k + 1) * LN * sg.s_pad + s;
#pragma unroll
      for (int j = 0; j < LN; ++j) {
        long long m = 0;  // values >= 0: 0 is the identity of max
#pragma unroll
        for (int i = 0; i < LN; ++i)
          if (coef[j][i] >= 0) m = max(m, (long long)coef[j][i] + st[i]);
        __stcg(out + (long long)j * sg.s_pad, m);
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      int* f = sg.flags + (long long)(k + 1) * sg.nb + b;
      asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(f), "r"(1) : "memory");
    }
  }
  // the transfer pass's generic shared-memory accesses precede the replay's
  // TMA writes into the same bytes
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  lanes_body<DK, 1, CH, true>(tmap, p, cpp, &sg, k, b, st, dp);
}

}  // namespace ddsim_lanes
