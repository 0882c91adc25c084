/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Only tests/, __graft_entry__.
 * smoke() and bench.py's cpu_baseline / --impl reference legs may load this.
 * The product path (paper_2006_03318_b200) never links or calls it.
 *
 * A plain-C restatement of the reference algorithms on dense arrays:
 *
 *   ora_simulate      Alg. 1 frontier simulation, kernsim.sim.simulate
 *                     (pkg/src/kernsim/sim.py:89-142) with the policies
 *                     DefaultSchedule (sim.py:55-69), PrioritySchedule
 *                     (sim.py:72-86) and VdnnPrefetchPolicy
 *                     (pkg/src/kernsim/scenarios.py:593-630).  Frontier choice
 *                     is a linear scan exactly like the reference.
 *   ora_toposort      verify_acyclic (graph.py:129-148): Kahn, min-heap on id.
 *   ora_longest_path  longest_path_makespan (synthetic.py:35-48): DP over the
 *                     verify_acyclic order.
 *   ora_scale         round_half_up(d * num / den) (transform.py:174-183).
 *   ora_simulate_batch  ora_simulate over S scenarios of dense durations,
 *                     pthread-parallel (CPU baseline of bench.py).
 *
 * Task "id order" is given by rank[] (rank of the external id).  Edges are a
 * multiset exactly like DependencyGraph.edges (sim.py:95-98 counts every
 * (u, v, kind) triple).
 */
#include <limits.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define POL_DEFAULT 0
#define POL_PRIORITY 1
#define POL_VDNN 2
#define F_COMM 1
#define F_VDNN_MALLOC 2

typedef struct {
  int n, L;
  const int64_t *dur, *gap, *ready;
  const int32_t *lane, *rank, *prio, *vrank;
  const uint8_t* flags;
  int64_t E;
  const int32_t *src, *dst;
} ora_graph;

static void build_children(const ora_graph* g, int32_t** ptr_out, int32_t** adj_out,
                           int32_t** indeg_out) {
  int32_t* ptr = (int32_t*)calloc((size_t)g->n + 1, sizeof(int32_t));
  int32_t* adj = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->E > 0 ? g->E : 1));
  int32_t* indeg = (int32_t*)calloc((size_t)(g->n > 0 ? g->n : 1), sizeof(int32_t));
  for (int64_t k = 0; k < g->E; ++k) {
    ptr[g->src[k] + 1]++;
    indeg[g->dst[k]]++;
  }
  for (int i = 0; i < g->n; ++i) ptr[i + 1] += ptr[i];
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n > 0 ? g->n : 1));
  for (int i = 0; i < g->n; ++i) fill[i] = ptr[i];
  for (int64_t k = 0; k < g->E; ++k) adj[fill[g->src[k]]++] = g->dst[k];
  free(fill);
  *ptr_out = ptr;
  *adj_out = adj;
  *indeg_out = indeg;
}

/* Effective start (sim.py:26-28). */
static inline int64_t eff_start(const int64_t* lane_prog, const int64_t* ready_time,
                                const int32_t* lane, int t) {
  int64_t a = lane_prog[lane[t]], b = ready_time[t];
  return a > b ? a : b;
}

/* DefaultSchedule.choose over candidates (skip[] marks excluded entries). */
static int choose_default(const int32_t* front, int F, const char* skip, const int64_t* lp,
                          const int64_t* rt, const int32_t* lane, const int32_t* rank) {
  int best = -1;
  int64_t be = 0;
  for (int i = 0; i < F; ++i) {
    if (skip && skip[i]) continue;
    const int t = front[i];
    const int64_t e = eff_start(lp, rt, lane, t);
    if (best < 0 || e < be || (e == be && rank[t] < rank[front[best]])) {
      best = i;
      be = e;
    }
  }
  return best;
}

/*
 * Returns the number of dispatched tasks (n unless Deadlock).
 * dur_override: optional per-task durations for this scenario (NULL = g->dur).
 */
int ora_simulate_core(const ora_graph* g, const int32_t* cptr, const int32_t* cadj,
                      const int32_t* indeg, const int64_t* dur_override, int policy,
                      int64_t* start_out, int32_t* trace_out, int64_t* lane_busy_out,
                      int64_t* makespan_out, int32_t* scratch_i, int64_t* scratch_l) {
  const int n = g->n;
  const int64_t* dur = dur_override ? dur_override : g->dur;
  int32_t* remaining = scratch_i;          /* n */
  int32_t* front = scratch_i + n;          /* n */
  int64_t* rt = scratch_l;                 /* n */
  int64_t* lp = scratch_l + n;             /* L */
  int64_t* lb = lane_busy_out;             /* L */
  char* skip = NULL;
  for (int i = 0; i < g->L; ++i) {
    lp[i] = 0;
    lb[i] = 0;
  }
  int F = 0;
  for (int i = 0; i < n; ++i) {
    remaining[i] = indeg[i];
    rt[i] = g->ready ? g->ready[i] : 0;
    if (indeg[i] == 0) front[F++] = i;
  }
  if (policy == POL_VDNN) skip = (char*)malloc((size_t)(n > 0 ? n : 1));
  int* tied = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  int64_t makespan = 0;
  int done = 0;
  while (F > 0) {
    int pos;
    if (policy == POL_VDNN) {
      /* mallocs: only the one with max (rank(layer), -id) stays eligible */
      int elig = -1;
      for (int i = 0; i < F; ++i) {
        const int t = front[i];
        skip[i] = 0;
        if (!(g->flags[t] & F_VDNN_MALLOC)) continue;
        if (elig < 0) {
          elig = i;
          continue;
        }
        const int e = front[elig];
        const int kt = g->vrank ? g->vrank[t] : -1, ke = g->vrank ? g->vrank[e] : -1;
        if (kt > ke || (kt == ke && g->rank[t] < g->rank[e])) elig = i;
      }
      for (int i = 0; i < F; ++i)
        if ((g->flags[front[i]] & F_VDNN_MALLOC) && i != elig) skip[i] = 1;
      pos = choose_default(front, F, skip, lp, rt, g->lane, g->rank);
    } else {
      pos = choose_default(front, F, NULL, lp, rt, g->lane, g->rank);
      if (policy == POL_PRIORITY) {
        /* literal restatement of sim.py:80-86: tied tasks sorted by id; a
         * later one replaces the incumbent iff both are comm and its
         * priority is strictly greater */
        const int64_t low = eff_start(lp, rt, g->lane, front[pos]);
        int nt = 0;
        for (int i = 0; i < F; ++i)
          if (eff_start(lp, rt, g->lane, front[i]) == low) tied[nt++] = i;
        for (int a = 1; a < nt; ++a) { /* insertion sort by id rank */
          const int x = tied[a];
          int b = a - 1;
          while (b >= 0 && g->rank[front[tied[b]]] > g->rank[front[x]]) {
            tied[b + 1] = tied[b];
            --b;
          }
          tied[b + 1] = x;
        }
        int best = tied[0];
        for (int a = 1; a < nt; ++a) {
          const int t = front[tied[a]], b = front[best];
          if ((g->flags[t] & F_COMM) && (g->flags[b] & F_COMM) && g->prio[t] > g->prio[b])
            best = tied[a];
        }
        pos = best;
      }
    }
    const int t = front[pos];
    front[pos] = front[--F];
    const int64_t st = eff_start(lp, rt, g->lane, t);
    const int64_t fin = st + dur[t];
    const int64_t rel = fin + g->gap[t];
    start_out[t] = st;
    if (trace_out) trace_out[done] = t;
    ++done;
    lp[g->lane[t]] = rel;
    lb[g->lane[t]] += dur[t];
    if (fin > makespan) makespan = fin;
    for (int k = cptr[t]; k < cptr[t + 1]; ++k) {
      const int c = cadj[k];
      if (rel > rt[c]) rt[c] = rel;
      if (--remaining[c] == 0) front[F++] = c;
    }
  }
  if (skip) free(skip);
  free(tied);
  *makespan_out = makespan;
  return done;
}

int ora_simulate(const ora_graph* g, int policy, int64_t* start_out, int32_t* trace_out,
                 int64_t* lane_busy_out, int64_t* makespan_out) {
  int32_t *cptr, *cadj, *indeg;
  build_children(g, &cptr, &cadj, &indeg);
  int32_t* si = (int32_t*)malloc(sizeof(int32_t) * (2 * (size_t)g->n + 1));
  int64_t* sl = (int64_t*)malloc(sizeof(int64_t) * ((size_t)g->n + g->L + 1));
  const int done = ora_simulate_core(g, cptr, cadj, indeg, NULL, policy, start_out, trace_out,
                                     lane_busy_out, makespan_out, si, sl);
  free(si);
  free(sl);
  free(cptr);
  free(cadj);
  free(indeg);
  return done;
}

/* ---- verify_acyclic: Kahn with a binary min-heap on rank ---------------- */
static void heap_push(int32_t* h, int* hn, int v, const int32_t* rank) {
  int i = (*hn)++;
  h[i] = v;
  while (i > 0) {
    int p = (i - 1) / 2;
    if (rank[h[p]] <= rank[h[i]]) break;
    int tmp = h[p];
    h[p] = h[i];
    h[i] = tmp;
    i = p;
  }
}
static int heap_pop(int32_t* h, int* hn, const int32_t* rank) {
  int top = h[0];
  h[0] = h[--(*hn)];
  int i = 0;
  for (;;) {
    int l = 2 * i + 1, r = l + 1, m = i;
    if (l < *hn && rank[h[l]] < rank[h[m]]) m = l;
    if (r < *hn && rank[h[r]] < rank[h[m]]) m = r;
    if (m == i) break;
    int tmp = h[m];
    h[m] = h[i];
    h[i] = tmp;
    i = m;
  }
  return top;
}

int ora_toposort(const ora_graph* g, int32_t* order_out) {
  int32_t *cptr, *cadj, *indeg;
  build_children(g, &cptr, &cadj, &indeg);
  int32_t* heap = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n > 0 ? g->n : 1));
  int hn = 0, k = 0;
  for (int i = 0; i < g->n; ++i)
    if (indeg[i] == 0) heap_push(heap, &hn, i, g->rank);
  while (hn > 0) {
    const int u = heap_pop(heap, &hn, g->rank);
    order_out[k++] = u;
    for (int j = cptr[u]; j < cptr[u + 1]; ++j)
      if (--indeg[cadj[j]] == 0) heap_push(heap, &hn, cadj[j], g->rank);
  }
  free(heap);
  free(cptr);
  free(cadj);
  free(indeg);
  return k;
}

/* longest_path_makespan: start(v) = max(0, max_p start(p)+dur(p)+gap(p)). */
int ora_longest_path(const ora_graph* g, int64_t* start_out, int64_t* makespan_out) {
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n > 0 ? g->n : 1));
  const int k = ora_toposort(g, order);
  /* parents via reverse CSR */
  int32_t* pptr = (int32_t*)calloc((size_t)g->n + 1, sizeof(int32_t));
  int32_t* padj = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->E > 0 ? g->E : 1));
  for (int64_t e = 0; e < g->E; ++e) pptr[g->dst[e] + 1]++;
  for (int i = 0; i < g->n; ++i) pptr[i + 1] += pptr[i];
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n > 0 ? g->n : 1));
  for (int i = 0; i < g->n; ++i) fill[i] = pptr[i];
  for (int64_t e = 0; e < g->E; ++e) padj[fill[g->dst[e]]++] = g->src[e];
  int64_t ms = 0;
  for (int i = 0; i < k; ++i) {
    const int v = order[i];
    int64_t s = 0;
    for (int j = pptr[v]; j < pptr[v + 1]; ++j) {
      const int p = padj[j];
      const int64_t r = start_out[p] + g->dur[p] + g->gap[p];
      if (r > s) s = r;
    }
    start_out[v] = s;
    if (s + g->dur[v] > ms) ms = s + g->dur[v];
  }
  *makespan_out = ms;
  free(order);
  free(pptr);
  free(padj);
  free(fill);
  return k;
}

int64_t ora_scale(int64_t d, int64_t num, int64_t den) {
  const int neg = d < 0;
  const unsigned __int128 a = (unsigned __int128)(neg ? -(__int128)d : (__int128)d);
  const unsigned __int128 q = (a * (unsigned __int128)num * 2 + (unsigned __int128)den) /
                              ((unsigned __int128)den * 2);
  return neg ? -(int64_t)q : (int64_t)q;
}

/* ---- batch: S scenarios of dense per-task durations, pthreads ---------- */
typedef struct {
  const ora_graph* g;
  const int32_t *cptr, *cadj, *indeg;
  const int32_t* dense; /* [n][ld] int32, task-major */
  int64_t ld;
  int s_begin, s_end;
  int64_t* makespan; /* [S] */
  int64_t* start;    /* optional [n][ld] */
  int policy;
  int64_t updates;
} ora_job;

static void* ora_worker(void* arg) {
  ora_job* j = (ora_job*)arg;
  const ora_graph* g = j->g;
  int32_t* si = (int32_t*)malloc(sizeof(int32_t) * (2 * (size_t)g->n + 1));
  int64_t* sl = (int64_t*)malloc(sizeof(int64_t) * ((size_t)g->n + g->L + 1));
  int64_t* d = (int64_t*)malloc(sizeof(int64_t) * ((size_t)g->n + 1));
  int64_t* st = (int64_t*)malloc(sizeof(int64_t) * ((size_t)g->n + 1));
  int64_t* lb = (int64_t*)malloc(sizeof(int64_t) * ((size_t)g->L + 1));
  for (int s = j->s_begin; s < j->s_end; ++s) {
    for (int i = 0; i < g->n; ++i) d[i] = j->dense[(int64_t)i * j->ld + s];
    int64_t ms = 0;
    ora_simulate_core(g, j->cptr, j->cadj, j->indeg, d, j->policy, st, NULL, lb, &ms, si, sl);
    j->makespan[s] = ms;
    if (j->start)
      for (int i = 0; i < g->n; ++i) j->start[(int64_t)i * j->ld + s] = st[i];
    j->updates += g->n;
  }
  free(si);
  free(sl);
  free(d);
  free(st);
  free(lb);
  return NULL;
}

int64_t ora_simulate_batch(const ora_graph* g, const int32_t* dense, int64_t ld, int S,
                           int policy, int threads, int64_t* makespan_out, int64_t* start_out) {
  int32_t *cptr, *cadj, *indeg;
  build_children(g, &cptr, &cadj, &indeg);
  if (threads < 1) threads = 1;
  if (threads > S) threads = S;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  ora_job* jobs = (ora_job*)calloc(threads, sizeof(ora_job));
  for (int t = 0; t < threads; ++t) {
    jobs[t].g = g;
    jobs[t].cptr = cptr;
    jobs[t].cadj = cadj;
    jobs[t].indeg = indeg;
    jobs[t].dense = dense;
    jobs[t].ld = ld;
    jobs[t].s_begin = (int)((int64_t)S * t / threads);
    jobs[t].s_end = (int)((int64_t)S * (t + 1) / threads);
    jobs[t].makespan = makespan_out;
    jobs[t].start = start_out;
    jobs[t].policy = policy;
    pthread_create(&th[t], NULL, ora_worker, &jobs[t]);
  }
  int64_t total = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    total += jobs[t].updates;
  }
  free(th);
  free(jobs);
  free(cptr);
  free(cadj);
  free(indeg);
  return total;
}

/* ======================================================================
 * Ingest restatement (TEST INFRASTRUCTURE): build_graph rules 1-5 + gaps
 * (pkg/src/kernsim/graph.py:189-312) and map_tasks_to_layers
 * (layers.py:30-81), written the straightforward way (sorts + scans).
 * ==================================================================== */
typedef struct {
  int64_t n;
  const int64_t *id, *start, *dur, *corr;
  const uint8_t *kind, *is_dtoh;
  const int32_t *lane, *sync_target;
  int32_t n_lanes;
  const uint8_t* lane_class; /* 0 cpu 1 gpu 2 comm */
} ora_trace;

static int is_cpu_k(int k) { return k == 0 || k == 1 || k == 4 || k == 6; }
static int is_gpu_k(int k) { return k == 2 || k == 3; }

static const ora_trace* g_sort_tr;
static int cmp_lane_start_id(const void* a, const void* b) {
  const int i = *(const int*)a, j = *(const int*)b;
  const ora_trace* t = g_sort_tr;
  if (t->lane[i] != t->lane[j]) return t->lane[i] < t->lane[j] ? -1 : 1;
  if (t->start[i] != t->start[j]) return t->start[i] < t->start[j] ? -1 : 1;
  if (t->id[i] != t->id[j]) return t->id[i] < t->id[j] ? -1 : 1;
  return 0;
}

/* stream entries (lane, launch start, id) */
typedef struct {
  int32_t lane;
  int64_t ls, id;
  int32_t idx;
} ora_entry;
static int cmp_entry(const void* a, const void* b) {
  const ora_entry *x = (const ora_entry*)a, *y = (const ora_entry*)b;
  if (x->lane != y->lane) return x->lane < y->lane ? -1 : 1;
  if (x->ls != y->ls) return x->ls < y->ls ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return 0;
}
typedef struct {
  int64_t key;
  int32_t idx;
} ora_kv;
static int cmp_kv(const void* a, const void* b) {
  const ora_kv *x = (const ora_kv*)a, *y = (const ora_kv*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* Returns the number of edges written (src, dst, kind as event indices,
 * kinds 0 LaneSeqCpu 1 LaneSeqGpu 2 LaunchCorrelation 3 SyncBlock 4 CommOrder);
 * gap[n], launcher[n].  Edges may be written in any order. */
int64_t ora_build_graph(const ora_trace* t, int32_t* esrc, int32_t* edst, uint8_t* ekind,
                        int64_t* gap, int32_t* launcher) {
  const int64_t n = t->n;
  int64_t m = 0;
  int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
  g_sort_tr = t;
  qsort(perm, (size_t)n, sizeof(int32_t), cmp_lane_start_id);
  for (int64_t i = 0; i < n; ++i) gap[i] = 0;
  for (int64_t k = 0; k + 1 < n; ++k) {
    const int a = perm[k], b = perm[k + 1];
    if (t->lane[a] != t->lane[b]) continue;
    const int cls = t->lane_class[t->lane[a]];
    esrc[m] = a; edst[m] = b; ekind[m] = cls == 0 ? 0 : (cls == 1 ? 1 : 4); ++m;
    if (cls == 0) {
      const int64_t d = t->start[b] - (t->start[a] + t->dur[a]);
      gap[a] = d > 0 ? d : 0;
    }
  }
  /* rule 3: last CPU-kind event per correlation (document order) */
  ora_kv* cpu = (ora_kv*)malloc(sizeof(ora_kv) * (size_t)(n > 0 ? n : 1));
  ora_kv* gpu = (ora_kv*)malloc(sizeof(ora_kv) * (size_t)(n > 0 ? n : 1));
  int64_t nc = 0, ng = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (t->corr[i] < 0) continue;
    if (is_cpu_k(t->kind[i])) { cpu[nc].key = t->corr[i]; cpu[nc].idx = (int32_t)i; ++nc; }
    if (is_gpu_k(t->kind[i])) { gpu[ng].key = t->corr[i]; gpu[ng].idx = (int32_t)i; ++ng; }
  }
  qsort(cpu, (size_t)nc, sizeof(ora_kv), cmp_kv);
  qsort(gpu, (size_t)ng, sizeof(ora_kv), cmp_kv);
  for (int64_t i = 0; i < n; ++i) {
    launcher[i] = -1;
    if (!is_gpu_k(t->kind[i]) || t->corr[i] < 0) continue;
    int64_t lo = 0, hi = nc; /* upper_bound(corr) - 1 */
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (cpu[mid].key <= t->corr[i]) lo = mid + 1; else hi = mid; }
    if (lo > 0 && cpu[lo - 1].key == t->corr[i]) {
      launcher[i] = cpu[lo - 1].idx;
      esrc[m] = launcher[i]; edst[m] = (int32_t)i; ekind[m] = 2; ++m;
    }
  }
  /* rule 4 */
  ora_entry* ent = (ora_entry*)malloc(sizeof(ora_entry) * (size_t)(n > 0 ? n : 1));
  int64_t ne = 0;
  for (int64_t i = 0; i < n; ++i)
    if (is_gpu_k(t->kind[i]) && launcher[i] >= 0) {
      ent[ne].lane = t->lane[i]; ent[ne].ls = t->start[launcher[i]]; ent[ne].id = t->id[i];
      ent[ne].idx = (int32_t)i; ++ne;
    }
  qsort(ent, (size_t)ne, sizeof(ora_entry), cmp_entry);
  int64_t* seg_b = (int64_t*)calloc((size_t)t->n_lanes + 1, sizeof(int64_t));
  int64_t* seg_e = (int64_t*)calloc((size_t)t->n_lanes + 1, sizeof(int64_t));
  for (int64_t k = 0; k < ne; ++k) {
    if (k == 0 || ent[k - 1].lane != ent[k].lane) seg_b[ent[k].lane] = k;
    seg_e[ent[k].lane] = k + 1;
  }
  char* has_ev = (char*)calloc((size_t)t->n_lanes + 1, 1);
  for (int64_t i = 0; i < n; ++i) has_ev[t->lane[i]] = 1;
  for (int64_t e = 0; e < n; ++e) {
    const int k = t->kind[e];
    int targets[1024];
    int nt = 0;
    int64_t exclude = -1;
    if (k == 6) {
      if (t->sync_target[e] >= 0) targets[nt++] = t->sync_target[e];
      else
        for (int l = 0; l < t->n_lanes && nt < 1024; ++l)
          if (t->lane_class[l] == 1 && has_ev[l]) targets[nt++] = l;
    } else if (is_cpu_k(k) && t->is_dtoh[e] && t->corr[e] >= 0) {
      int64_t lo = 0, hi = ng; /* lower_bound: first GPU event with the correlation */
      while (lo < hi) { int64_t mid = (lo + hi) / 2; if (gpu[mid].key < t->corr[e]) lo = mid + 1; else hi = mid; }
      if (lo >= ng || gpu[lo].key != t->corr[e]) continue;
      targets[nt++] = t->lane[gpu[lo].idx];
      exclude = gpu[lo].idx;
    } else {
      continue;
    }
    for (int q = 0; q < nt; ++q) {
      const int l = targets[q];
      /* newest entry with launch start < e.start, skipping `exclude` (graph.py:269-276) */
      int32_t best = -1;
      for (int64_t p = seg_b[l]; p < seg_e[l]; ++p) {
        if (ent[p].ls >= t->start[e]) break;
        if (ent[p].idx != exclude) best = ent[p].idx;
      }
      if (best >= 0) { esrc[m] = best; edst[m] = (int32_t)e; ekind[m] = 3; ++m; }
    }
  }
  free(perm); free(cpu); free(gpu); free(ent); free(seg_b); free(seg_e); free(has_ev);
  return m;
}

/* map_tasks_to_layers: CPU-kind events by innermost containing marker on the
 * same lane ((length, tag, list order) minimum; ambiguity if the best two are
 * not nested), GPU-kind events inherit their launcher's tag.  Returns -1 or
 * the index of the first ambiguous event.  Markers are scanned per task from
 * a per-lane list (O(N * markers per lane) -- test sizes only). */
int64_t ora_map_layers(const ora_trace* t, const int32_t* launcher, int64_t M, const int32_t* mlane,
                       const int64_t* mstart, const int64_t* mend, const int32_t* mtag, int32_t* tag_out) {
  int64_t bad = -1;
  for (int64_t i = 0; i < t->n; ++i) {
    tag_out[i] = -1;
    if (!is_cpu_k(t->kind[i]) || t->lane[i] < 0) continue;
    const int64_t s = t->start[i], e = t->start[i] + t->dur[i];
    int64_t a = -1, b = -1;
    for (int64_t j = 0; j < M; ++j) {
      if (mlane[j] != t->lane[i] || mstart[j] > s || mend[j] < e) continue;
      const int64_t len = mend[j] - mstart[j];
      if (a < 0 || len < mend[a] - mstart[a] || (len == mend[a] - mstart[a] && (mtag[j] < mtag[a]))) {
        b = a; a = j;
      } else if (b < 0 || len < mend[b] - mstart[b] || (len == mend[b] - mstart[b] && mtag[j] < mtag[b])) {
        b = j;
      }
    }
    if (a < 0) continue;
    if (b >= 0 && !(mstart[b] <= mstart[a] && mend[a] <= mend[b]) && bad < 0) bad = i;
    tag_out[i] = mtag[a];
  }
  for (int64_t i = 0; i < t->n; ++i)
    if (is_gpu_k(t->kind[i]) && launcher[i] >= 0 && tag_out[launcher[i]] >= 0)
      tag_out[i] = tag_out[launcher[i]];
  return bad;
}
