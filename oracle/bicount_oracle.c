/*
 * bicount_oracle.c -- CPU restatement of the reference (p,q)-biclique
 * counting hot path.  TEST INFRASTRUCTURE ONLY: imported by tests/, by
 * __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
 * --impl reference legs.  The product path (paper_2403_07858_b200) never
 * links or calls this file.
 *
 * Every stage follows the reference Python package under
 * /root/reference/pkg/src/bicount (read-only, not shipped):
 *
 *   anchor choice          graph.py:246-269   (wedge mass, ties -> U, V swaps p/q)
 *   2-hop index            graph.py:192-215   (multiplicity >= k, w != u, sorted)
 *   vertex priority        graph.py:227-243   (ascending size, ties -> smaller id
 *                                              gets the higher rank; rank in [1,n])
 *   rank override          engine.py:128-134
 *   directed filter        graph.py:218-224   (keep rank[w] < rank[u])
 *   HTB build              htb.py:89-115      (idx = id>>5, val = OR 1<<(id&31))
 *   task emission          engine.py:147-173  (priority order, und-size filter,
 *                                              round-robin over workers)
 *   progress board         engine.py:176-242  (claim under a latch, DONE sentinel,
 *                                              own entry first, then steal)
 *   search                 engine.py:245-374  (level 1, hybrid batches, 1-hop then
 *                                              2-hop phase, prune_keep, leaves add
 *                                              C(|C_R|, q))
 *   intersection           htb.py:122-154     (walk shorter idx, bisect_left the
 *                                              longer, AND, drop zero words)
 *   capacity check         engine.py:377-393
 *
 * Counts are exact unsigned 128-bit (the reference uses Python ints; an
 * overflow past 2^128 sets the overflow flag).  Besides the count and the
 * CountReport fields the oracle also tallies, per the SURVEY section 8(d)
 * measurement definition, every htb_intersect call it performs: number of
 * calls, operand words sum(|a|+|b|) (-> B_enum = 8 B x words) and
 * sum(min(|a|,|b|)) (-> B_min = 16 B x words).
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef unsigned __int128 u128;

#define ORC_DONE 0xFFFFFFFFu

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ------------------------------------------------------------------ */
/* public structs (mirrored by oracle/oracle.py via ctypes)            */
/* ------------------------------------------------------------------ */
typedef struct {
  int32_t p, q;
  int32_t workers;        /* EngineConfig.worker_count */
  int32_t capacity;       /* EngineConfig.batch_buffer_capacity (words) */
  int32_t mode;           /* 0 = dfs, 1 = hybrid */
  int32_t anchor;         /* -1 auto, 0 U, 1 V */
  const int64_t *rank_override; /* NULL or one distinct value per anchor vertex */
  const uint8_t *root_mask;     /* NULL or n_anchor flags: roots= restriction */
  int64_t *task_words;    /* NULL or [emitted] operand words per task (priority order) */
  uint64_t *task_count;   /* NULL or [2*emitted] u128 count per task (lo,hi) */
  int64_t *task_l1;       /* NULL or [4*emitted]: |C_R1|, words(C_R1), |C_L1|, words(C_L1)
                             (-1 where the reference stops before computing it) */
} orc_config;

typedef struct {
  uint64_t count_lo, count_hi;
  int32_t overflow;
  int32_t anchor;         /* 0 = U, 1 = V */
  int32_t p_eff, q_eff;
  int64_t batches, stolen, roots_filtered, emitted, consumed;
  int64_t intersections, operand_words, min_words;
  double prep_time, wall_time, time_1hop, time_2hop;
} orc_report;

/* ------------------------------------------------------------------ */
/* prepared structures                                                 */
/* ------------------------------------------------------------------ */
typedef struct {
  int32_t anchor, p_eff, q_eff;
  int64_t n, m;                    /* anchor layer size, opposite layer size */
  int64_t *aoff; int32_t *aidx;    /* anchor-layer adjacency (work.u_adj) */
  int64_t *boff; int32_t *bidx;    /* opposite-layer adjacency (work.v_adj) */
  int64_t *und_off; int32_t *und_idx; int64_t *und_size;
  int64_t *rank, *order;
  int64_t *dir_off; int32_t *dir_idx;
  int64_t *hadj_off; uint32_t *hadj_idx, *hadj_val;
  int64_t *hdir_off; uint32_t *hdir_idx, *hdir_val;
  double prep_time;
} orc_struct;

static char g_err[512];
const char *orc_last_error(void) { return g_err; }

static void *xmalloc(size_t n) {
  void *p = malloc(n ? n : 1);
  if (!p) { fprintf(stderr, "oracle: out of memory (%zu bytes)\n", n); abort(); }
  return p;
}

static int64_t wedge_mass(const int64_t *off, int64_t n) {
  int64_t s = 0;
  for (int64_t i = 0; i < n; i++) { int64_t d = off[i + 1] - off[i]; s += d * (d - 1) / 2; }
  return s;
}

/* --- 2-hop index, graph.py:192-215; parallel over anchor vertices --- */
typedef struct {
  const orc_struct *s; int32_t k; int64_t lo, hi;
  int32_t **lists; int64_t *sizes;
  int64_t *next;  /* shared claim counter (vertices in blocks of 16: hubs balance) */
} twohop_job;

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

static void *twohop_worker(void *arg) {
  twohop_job *j = (twohop_job *)arg;
  const orc_struct *s = j->s;
  int32_t *cnt = (int32_t *)calloc((size_t)s->n, sizeof(int32_t));
  int32_t *touched = (int32_t *)xmalloc((size_t)(s->n ? s->n : 1) * sizeof(int32_t));
  for (;;) {
   int64_t u0 = __atomic_fetch_add(j->next, 16, __ATOMIC_RELAXED);
   if (u0 >= j->hi) break;
   for (int64_t u = u0; u < u0 + 16 && u < j->hi; u++) {
    int64_t nt = 0;
    for (int64_t e = s->aoff[u]; e < s->aoff[u + 1]; e++) {
      int32_t v = s->aidx[e];
      for (int64_t f = s->boff[v]; f < s->boff[v + 1]; f++) {
        int32_t w = s->bidx[f];
        if (cnt[w]++ == 0) touched[nt++] = w;
      }
    }
    int64_t keep = 0;
    for (int64_t t = 0; t < nt; t++) {
      int32_t w = touched[t];
      if (cnt[w] >= j->k && w != u) touched[keep++] = w;
      cnt[w] = 0;
    }
    /* reset counters of dropped ids too: the loop above zeroed all touched */
    qsort(touched, (size_t)keep, sizeof(int32_t), cmp_i32);
    int32_t *out = (int32_t *)xmalloc((size_t)(keep ? keep : 1) * sizeof(int32_t));
    memcpy(out, touched, (size_t)keep * sizeof(int32_t));
    j->lists[u] = out;
    j->sizes[u] = keep;
   }
  }
  free(cnt); free(touched);
  return NULL;
}

static int n_threads_default(void) {
  cpu_set_t cs;
  if (sched_getaffinity(0, sizeof(cs), &cs) == 0) return CPU_COUNT(&cs);
  return 1;
}

/* --- HTB encode of a CSR family, htb.py:89-115 --- */
static void htb_build_csr(int64_t n, const int64_t *off, const int32_t *idx,
                          int64_t **hoff, uint32_t **hidx, uint32_t **hval) {
  int64_t *o = (int64_t *)xmalloc((size_t)(n + 1) * sizeof(int64_t));
  o[0] = 0;
  for (int64_t i = 0; i < n; i++) {
    int64_t w = 0; int64_t last = -1;
    for (int64_t e = off[i]; e < off[i + 1]; e++) {
      int64_t word = idx[e] >> 5;
      if (word != last) { w++; last = word; }
    }
    o[i + 1] = o[i] + w;
  }
  uint32_t *ix = (uint32_t *)xmalloc((size_t)(o[n] ? o[n] : 1) * 4);
  uint32_t *vl = (uint32_t *)xmalloc((size_t)(o[n] ? o[n] : 1) * 4);
  for (int64_t i = 0; i < n; i++) {
    int64_t t = o[i] - 1; int64_t last = -1;
    for (int64_t e = off[i]; e < off[i + 1]; e++) {
      int64_t word = idx[e] >> 5;
      if (word != last) { t++; ix[t] = (uint32_t)word; vl[t] = 0; last = word; }
      vl[t] |= 1u << (idx[e] & 31);
    }
  }
  *hoff = o; *hidx = ix; *hval = vl;
}

static int64_t *g_sort_size;  /* for qsort of the priority order */
static int cmp_prio(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  if (g_sort_size[x] != g_sort_size[y]) return g_sort_size[x] < g_sort_size[y] ? -1 : 1;
  return (x > y) - (x < y);
}
static int64_t *g_sort_rank;
static int cmp_rank_desc(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  if (g_sort_rank[x] != g_sort_rank[y]) return g_sort_rank[x] > g_sort_rank[y] ? -1 : 1;
  return (x > y) - (x < y);
}

void orc_free(orc_struct *s);

/* prepare_structures, engine.py:115-144 */
orc_struct *orc_prepare(const int64_t *u_off, const int32_t *u_idx, int64_t n_u,
                        const int64_t *v_off, const int32_t *v_idx, int64_t n_v,
                        int32_t p, int32_t q, int32_t anchor,
                        const int64_t *rank_override, int32_t threads) {
  g_err[0] = 0;
  if (p < 1 || q < 1) { snprintf(g_err, sizeof g_err, "p and q must be >= 1"); return NULL; }
  double t0 = now_s();
  orc_struct *s = (orc_struct *)calloc(1, sizeof(orc_struct));
  int layer;
  if (anchor < 0) layer = wedge_mass(v_off, n_v) <= wedge_mass(u_off, n_u) ? 0 : 1;
  else layer = anchor;
  s->anchor = layer;
  s->p_eff = layer == 0 ? p : q;
  s->q_eff = layer == 0 ? q : p;
  /* work = g or transpose(g), engine.py:126 -- borrowed pointers */
  s->n = layer == 0 ? n_u : n_v;
  s->m = layer == 0 ? n_v : n_u;
  s->aoff = (int64_t *)(layer == 0 ? u_off : v_off);
  s->aidx = (int32_t *)(layer == 0 ? u_idx : v_idx);
  s->boff = (int64_t *)(layer == 0 ? v_off : u_off);
  s->bidx = (int32_t *)(layer == 0 ? v_idx : u_idx);
  int64_t n = s->n;

  /* undirected 2-hop index with k = q_eff */
  int32_t **lists = (int32_t **)xmalloc((size_t)(n ? n : 1) * sizeof(int32_t *));
  s->und_size = (int64_t *)xmalloc((size_t)(n ? n : 1) * sizeof(int64_t));
  if (threads < 1) threads = n_threads_default();
  if (threads > 256) threads = 256;
  pthread_t th[256]; twohop_job jobs[256];
  int64_t next = 0;
  int nt = 0;
  for (int t = 0; t < threads && t < (n + 15) / 16; t++) {
    jobs[t] = (twohop_job){s, s->q_eff, 0, n, lists, s->und_size, &next};
    pthread_create(&th[t], NULL, twohop_worker, &jobs[t]);
    nt++;
  }
  for (int t = 0; t < nt; t++) pthread_join(th[t], NULL);
  s->und_off = (int64_t *)xmalloc((size_t)(n + 1) * sizeof(int64_t));
  s->und_off[0] = 0;
  for (int64_t u = 0; u < n; u++) s->und_off[u + 1] = s->und_off[u] + s->und_size[u];
  s->und_idx = (int32_t *)xmalloc((size_t)(s->und_off[n] ? s->und_off[n] : 1) * 4);
  for (int64_t u = 0; u < n; u++) {
    memcpy(s->und_idx + s->und_off[u], lists[u], (size_t)s->und_size[u] * 4);
    free(lists[u]);
  }
  free(lists);

  /* priority (graph.py:227-243) or override (engine.py:130-134) */
  s->rank = (int64_t *)xmalloc((size_t)(n ? n : 1) * sizeof(int64_t));
  s->order = (int64_t *)xmalloc((size_t)(n ? n : 1) * sizeof(int64_t));
  for (int64_t u = 0; u < n; u++) s->order[u] = u;
  if (!rank_override) {
    g_sort_size = s->und_size;
    qsort(s->order, (size_t)n, sizeof(int64_t), cmp_prio);   /* lexsort((id, size)) */
    for (int64_t i = 0; i < n; i++) s->rank[s->order[i]] = n - i;
    /* PriorityOrder.order lists highest priority first: order = lexsort result */
  } else {
    memcpy(s->rank, rank_override, (size_t)n * sizeof(int64_t));
    int64_t *tmp = (int64_t *)xmalloc((size_t)(n ? n : 1) * sizeof(int64_t));
    memcpy(tmp, rank_override, (size_t)n * sizeof(int64_t));
    g_sort_size = tmp;
    int64_t *ids = (int64_t *)xmalloc((size_t)(n ? n : 1) * sizeof(int64_t));
    for (int64_t u = 0; u < n; u++) ids[u] = u;
    qsort(ids, (size_t)n, sizeof(int64_t), cmp_prio);
    for (int64_t i = 1; i < n; i++)
      if (tmp[ids[i]] == tmp[ids[i - 1]]) {
        snprintf(g_err, sizeof g_err,
                 "rank override must give one distinct value per anchor vertex");
        free(tmp); free(ids); orc_free(s); return NULL;
      }
    free(tmp); free(ids);
    /* argsort(-rank, kind="stable") */
    g_sort_rank = s->rank;
    qsort(s->order, (size_t)n, sizeof(int64_t), cmp_rank_desc);
  }
  /* NB: vertex_priority's `order` is lexsort ascending (size,id); the
   * reference iterates tasks over order.order which is that lexsort result,
   * i.e. rank n first. */

  /* directed filter, graph.py:218-224 */
  s->dir_off = (int64_t *)xmalloc((size_t)(n + 1) * sizeof(int64_t));
  s->dir_idx = (int32_t *)xmalloc((size_t)(s->und_off[n] ? s->und_off[n] : 1) * 4);
  s->dir_off[0] = 0;
  for (int64_t u = 0; u < n; u++) {
    int64_t c = s->dir_off[u];
    for (int64_t e = s->und_off[u]; e < s->und_off[u + 1]; e++) {
      int32_t w = s->und_idx[e];
      if (s->rank[w] < s->rank[u]) s->dir_idx[c++] = w;
    }
    s->dir_off[u + 1] = c;
  }
  htb_build_csr(n, s->aoff, s->aidx, &s->hadj_off, &s->hadj_idx, &s->hadj_val);
  htb_build_csr(n, s->dir_off, s->dir_idx, &s->hdir_off, &s->hdir_idx, &s->hdir_val);
  s->prep_time = now_s() - t0;
  return s;
}

void orc_free(orc_struct *s) {
  if (!s) return;
  free(s->und_off); free(s->und_idx); free(s->und_size);
  free(s->rank); free(s->order); free(s->dir_off); free(s->dir_idx);
  free(s->hadj_off); free(s->hadj_idx); free(s->hadj_val);
  free(s->hdir_off); free(s->hdir_idx); free(s->hdir_val);
  free(s);
}

/* structure export for parity tests */
enum { X_UND_SIZE, X_RANK, X_ORDER, X_UND_OFF, X_UND_IDX, X_DIR_OFF, X_DIR_IDX,
       X_HADJ_OFF, X_HADJ_IDX, X_HADJ_VAL, X_HDIR_OFF, X_HDIR_IDX, X_HDIR_VAL, X_META };

int64_t orc_export_len(const orc_struct *s, int what) {
  int64_t n = s->n;
  switch (what) {
    case X_UND_SIZE: case X_RANK: case X_ORDER: return n;
    case X_UND_OFF: case X_DIR_OFF: case X_HADJ_OFF: case X_HDIR_OFF: return n + 1;
    case X_UND_IDX: return s->und_off[n];
    case X_DIR_IDX: return s->dir_off[n];
    case X_HADJ_IDX: case X_HADJ_VAL: return s->hadj_off[n];
    case X_HDIR_IDX: case X_HDIR_VAL: return s->hdir_off[n];
    case X_META: return 4;
  }
  return -1;
}

void orc_export(const orc_struct *s, int what, void *dst) {
  int64_t n = s->n, len = orc_export_len(s, what);
  const void *src = NULL; size_t el = 8;
  switch (what) {
    case X_UND_SIZE: src = s->und_size; break;
    case X_RANK: src = s->rank; break;
    case X_ORDER: src = s->order; break;
    case X_UND_OFF: src = s->und_off; break;
    case X_UND_IDX: src = s->und_idx; el = 4; break;
    case X_DIR_OFF: src = s->dir_off; break;
    case X_DIR_IDX: src = s->dir_idx; el = 4; break;
    case X_HADJ_OFF: src = s->hadj_off; break;
    case X_HADJ_IDX: src = s->hadj_idx; el = 4; break;
    case X_HADJ_VAL: src = s->hadj_val; el = 4; break;
    case X_HDIR_OFF: src = s->hdir_off; break;
    case X_HDIR_IDX: src = s->hdir_idx; el = 4; break;
    case X_HDIR_VAL: src = s->hdir_val; el = 4; break;
    case X_META: {
      int64_t *d = (int64_t *)dst;
      d[0] = s->anchor; d[1] = s->p_eff; d[2] = s->q_eff; d[3] = n;
      return;
    }
  }
  memcpy(dst, src, (size_t)len * el);
}

/* ------------------------------------------------------------------ */
/* search                                                              */
/* ------------------------------------------------------------------ */
typedef struct {                  /* HtbSlice: window [lo,hi) over idx/val */
  const uint32_t *idx, *val; int64_t lo, hi;
} slice_t;

typedef struct {                  /* batch child record */
  int32_t u; int64_t rlo, rhi; int64_t card;
  int64_t llo, lhi; int64_t lcard;
} child_t;

typedef struct {
  const orc_struct *s;
  int32_t p_eff, q_eff, capacity, mode, levels;
  const u128 *comb_q; int64_t max_deg;
  /* per-level scratch (engine.py:250-255) */
  uint32_t **cr_idx, **cr_val, **cl_idx, **cl_val;
  int32_t **cands; child_t **kids;
  /* tallies */
  u128 count; int overflow; int64_t first_bad;
  int64_t batches, inter, op_words, min_words;
  double t1, t2;
  int timing;
  int64_t *l1;
} searcher_t;

/* htb_intersect, htb.py:122-154: walk shorter idx, bisect the longer. */
static inline int64_t intersect(searcher_t *S, slice_t a, slice_t b,
                                uint32_t *oi, uint32_t *ov, int64_t pos) {
  int64_t la = a.hi - a.lo, lb = b.hi - b.lo;
  S->inter++;
  S->op_words += la + lb;
  S->min_words += la < lb ? la : lb;
  if (la > lb) { slice_t t = a; a = b; b = t; }
  int64_t t = a.lo, blo = b.lo, bhi = b.hi;
  while (t < a.hi) {
    uint32_t w = a.idx[t];
    /* bisect_left(b.idx, w, blo, bhi) */
    int64_t lo = blo, hi = bhi;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (b.idx[mid] < w) lo = mid + 1; else hi = mid;
    }
    int64_t j = lo;
    if (j == bhi) break;
    if (b.idx[j] == w) {
      uint32_t x = a.val[t] & b.val[j];
      if (x) { oi[pos] = w; ov[pos] = x; pos++; }
      blo = j + 1;
    } else {
      blo = j;
    }
    t++;
  }
  return pos;
}

static inline int64_t card_of(const uint32_t *val, int64_t lo, int64_t hi) {
  int64_t c = 0;
  for (int64_t t = lo; t < hi; t++) c += __builtin_popcount(val[t]);
  return c;
}

static inline void add_count(searcher_t *S, int64_t card) {
  if (card >= S->first_bad) { S->overflow = 1; return; }
  u128 x = S->comb_q[card];
  u128 before = S->count;
  S->count += x;
  if (S->count < before) S->overflow = 1;
}

static inline slice_t adj_slice(const orc_struct *s, int64_t u) {
  return (slice_t){s->hadj_idx, s->hadj_val, s->hadj_off[u], s->hadj_off[u + 1]};
}
static inline slice_t dir_slice(const orc_struct *s, int64_t u) {
  return (slice_t){s->hdir_idx, s->hdir_val, s->hdir_off[u], s->hdir_off[u + 1]};
}

/* batch_size, engine.py:306-313 */
static inline int64_t batch_size(const searcher_t *S, int64_t clw, int64_t crw, int leaf) {
  if (S->mode == 0) return 1;
  int64_t cap = S->capacity;
  int64_t b = cap / (crw > 1 ? crw : 1);
  if (!leaf) { int64_t b2 = cap / (clw > 1 ? clw : 1); if (b2 < b) b = b2; }
  return b > 1 ? b : 1;
}

/* prune_keep, engine.py:110-112 */
static inline int prune_keep(int64_t cr, int64_t cl, int level, int p_eff, int q_eff) {
  return cr >= q_eff && cl >= p_eff - level - 1;
}

/* Searcher._descend, engine.py:315-374 */
static void descend(searcher_t *S, int level, slice_t cl, slice_t cr) {
  const orc_struct *s = S->s;
  int32_t *cands = S->cands[level];
  int64_t nc = 0;
  for (int64_t t = cl.lo; t < cl.hi; t++) {   /* HtbSlice.decode, htb.py:42-52 */
    uint32_t w = cl.val[t]; int64_t base = (int64_t)cl.idx[t] * 32;
    while (w) { cands[nc++] = (int32_t)(base + __builtin_ctz(w)); w &= w - 1; }
  }
  int child_level = level + 1;
  int leaf = child_level == S->p_eff - 1;
  int64_t batch = batch_size(S, cl.hi - cl.lo, cr.hi - cr.lo, leaf);
  uint32_t *ci = S->cr_idx[child_level], *cv = S->cr_val[child_level];
  uint32_t *li = S->cl_idx[child_level], *lv = S->cl_val[child_level];
  child_t *kids = S->kids[child_level];
  for (int64_t lo = 0; lo < nc; lo += batch) {
    int64_t hi = lo + batch < nc ? lo + batch : nc;
    S->batches++;
    double t0 = S->timing ? now_s() : 0;
    int64_t pos = 0;
    for (int64_t k = lo; k < hi; k++) {
      int32_t u = cands[k];
      int64_t end = intersect(S, cr, adj_slice(s, u), ci, cv, pos);
      child_t *c = &kids[k - lo];
      c->u = u; c->rlo = pos; c->rhi = end; c->card = card_of(cv, pos, end);
      pos = end;
    }
    if (S->timing) S->t1 += now_s() - t0;
    if (leaf) {
      for (int64_t k = 0; k < hi - lo; k++)
        if (kids[k].card >= S->q_eff) add_count(S, kids[k].card);
    } else {
      double t1 = S->timing ? now_s() : 0;
      pos = 0;
      for (int64_t k = 0; k < hi - lo; k++) {
        child_t *c = &kids[k];
        if (c->card < S->q_eff) { c->lcard = -1; continue; }
        int64_t end = intersect(S, cl, dir_slice(s, c->u), li, lv, pos);
        c->llo = pos; c->lhi = end; c->lcard = card_of(lv, pos, end);
        pos = end;
      }
      if (S->timing) S->t2 += now_s() - t1;
      for (int64_t k = 0; k < hi - lo; k++) {
        child_t *c = &kids[k];
        if (c->lcard < 0) continue;
        if (prune_keep(c->card, c->lcard, child_level, S->p_eff, S->q_eff)) {
          slice_t ncl = {li, lv, c->llo, c->lhi};
          slice_t ncr = {ci, cv, c->rlo, c->rhi};
          descend(S, child_level, ncl, ncr);
        }
      }
    }
  }
}

/* Searcher.run_task, engine.py:265-299 */
static void run_task(searcher_t *S, int64_t root, int64_t second) {
  const orc_struct *s = S->s;
  if (S->p_eff == 1) {
    int64_t card = s->aoff[root + 1] - s->aoff[root];
    if (card >= S->q_eff) add_count(S, card);
    return;
  }
  double t0 = S->timing ? now_s() : 0;
  int64_t end = intersect(S, adj_slice(s, root), adj_slice(s, second),
                          S->cr_idx[1], S->cr_val[1], 0);
  int64_t cr_card = card_of(S->cr_val[1], 0, end);
  if (S->timing) S->t1 += now_s() - t0;
  S->batches++;
  if (S->l1) { S->l1[0] = cr_card; S->l1[1] = end; }
  if (cr_card < S->q_eff) return;
  if (S->p_eff == 2) { add_count(S, cr_card); return; }
  double t1 = S->timing ? now_s() : 0;
  int64_t lend = intersect(S, dir_slice(s, root), dir_slice(s, second),
                           S->cl_idx[1], S->cl_val[1], 0);
  int64_t cl_card = card_of(S->cl_val[1], 0, lend);
  if (S->timing) S->t2 += now_s() - t1;
  if (S->l1) { S->l1[2] = cl_card; S->l1[3] = lend; }
  if (!prune_keep(cr_card, cl_card, 1, S->p_eff, S->q_eff)) return;
  slice_t cl = {S->cl_idx[1], S->cl_val[1], 0, lend};
  slice_t cr = {S->cr_idx[1], S->cr_val[1], 0, end};
  descend(S, 1, cl, cr);
}

static void searcher_init(searcher_t *S, const orc_struct *s, const orc_config *cfg,
                          const u128 *comb_q, int64_t max_deg) {
  memset(S, 0, sizeof *S);
  S->s = s; S->p_eff = s->p_eff; S->q_eff = s->q_eff;
  S->capacity = cfg->capacity; S->mode = cfg->mode;
  S->comb_q = comb_q; S->max_deg = max_deg;
  S->levels = s->p_eff > 2 ? s->p_eff : 2;
  int L = S->levels + 1;
  size_t cap = (size_t)cfg->capacity;
  S->cr_idx = calloc(L, sizeof(void *)); S->cr_val = calloc(L, sizeof(void *));
  S->cl_idx = calloc(L, sizeof(void *)); S->cl_val = calloc(L, sizeof(void *));
  S->cands = calloc(L, sizeof(void *)); S->kids = calloc(L, sizeof(void *));
  for (int l = 0; l < L; l++) {
    S->cr_idx[l] = xmalloc(cap * 4); S->cr_val[l] = xmalloc(cap * 4);
    S->cl_idx[l] = xmalloc(cap * 4); S->cl_val[l] = xmalloc(cap * 4);
    S->cands[l] = xmalloc(cap * 32 * 4);
    S->kids[l] = xmalloc(cap * sizeof(child_t));
  }
}

static void searcher_free(searcher_t *S) {
  for (int l = 0; l <= S->levels; l++) {
    free(S->cr_idx[l]); free(S->cr_val[l]); free(S->cl_idx[l]); free(S->cl_val[l]);
    free(S->cands[l]); free(S->kids[l]);
  }
  free(S->cr_idx); free(S->cr_val); free(S->cl_idx); free(S->cl_val);
  free(S->cands); free(S->kids);
}

/* progress board, engine.py:176-242 */
typedef struct {
  int W; int64_t *sizes; uint32_t *counters; pthread_mutex_t *latches;
} board_t;

static int64_t board_claim(board_t *b, int e) {
  pthread_mutex_lock(&b->latches[e]);
  uint32_t c = b->counters[e];
  int64_t r;
  if (c == ORC_DONE) r = -1;
  else if ((int64_t)c >= b->sizes[e]) { b->counters[e] = ORC_DONE; r = -1; }
  else { b->counters[e] = c + 1; r = c; }
  pthread_mutex_unlock(&b->latches[e]);
  return r;
}

typedef struct {
  searcher_t S; board_t *board; int me;
  int64_t **lists; /* per-worker list of task ids (index into task arrays) */
  const int64_t *troot, *tsecond;
  int64_t consumed, stolen;
  int64_t *task_words; uint64_t *task_count; int64_t *task_l1;
} worker_t;

static void do_task(worker_t *w, int64_t tid) {
  searcher_t *S = &w->S;
  int64_t ow = S->op_words; u128 c0 = S->count;
  S->l1 = w->task_l1 ? w->task_l1 + 4 * tid : NULL;
  if (S->l1) S->l1[0] = S->l1[1] = S->l1[2] = S->l1[3] = -1;
  run_task(S, w->troot[tid], w->tsecond[tid]);
  if (w->task_words) w->task_words[tid] = S->op_words - ow;
  if (w->task_count) {
    u128 d = S->count - c0;
    w->task_count[2 * tid] = (uint64_t)d; w->task_count[2 * tid + 1] = (uint64_t)(d >> 64);
  }
}

static void *worker_main(void *arg) {
  worker_t *w = (worker_t *)arg;
  board_t *b = w->board;
  int n = b->W;
  for (;;) {
    int alive = 0, got = 0;
    for (int k = 0; k < n; k++) {
      int e = (w->me + k) % n;
      if (__atomic_load_n(&b->counters[e], __ATOMIC_RELAXED) == ORC_DONE) continue;
      alive = 1;
      int64_t i = board_claim(b, e);
      if (i < 0) continue;
      do_task(w, w->lists[e][i]);
      w->consumed++;
      if (e != w->me) w->stolen++;
      got = 1;
      break;
    }
    if (!alive) break;
    (void)got;
  }
  return NULL;
}

/* count_bicliques, engine.py:419-500 */
int orc_count(const orc_struct *s, const orc_config *cfg, orc_report *out) {
  g_err[0] = 0;
  memset(out, 0, sizeof *out);
  if (cfg->workers < 1) { snprintf(g_err, sizeof g_err, "worker_count must be >= 1"); return -1; }
  if (cfg->capacity < 1) { snprintf(g_err, sizeof g_err, "batch_buffer_capacity must be >= 1"); return -1; }
  if (cfg->mode != 0 && cfg->mode != 1) { snprintf(g_err, sizeof g_err, "mode must be one of ('dfs', 'hybrid')"); return -1; }
  int64_t n = s->n;
  /* _build_shared, engine.py:377-406 */
  int64_t max_words = 0, max_deg = 0;
  for (int64_t u = 0; u < n; u++) {
    int64_t a = s->hadj_off[u + 1] - s->hadj_off[u];
    int64_t d = s->hdir_off[u + 1] - s->hdir_off[u];
    if (a > max_words) max_words = a;
    if (d > max_words) max_words = d;
    int64_t dg = s->aoff[u + 1] - s->aoff[u];
    if (dg > max_deg) max_deg = dg;
  }
  if (cfg->capacity < max_words) {
    snprintf(g_err, sizeof g_err,
             "batch_buffer_capacity %d words is below the largest candidate slice "
             "(%lld words); raise --batch-words", cfg->capacity, (long long)max_words);
    return -1;
  }
  u128 *comb_q = (u128 *)xmalloc((size_t)(max_deg + 1) * sizeof(u128));
  int64_t first_bad = max_deg + 1;   /* C(c,q) >= 2^128 from here on */
  {
    /* C(c, q) by the multiplicative recurrence C(c,q) = C(c-1,q) * c / (c-q) */
    int64_t q = s->q_eff;
    for (int64_t c = 0; c <= max_deg; c++) {
      if (c < q) comb_q[c] = 0;
      else if (c == q) comb_q[c] = 1;
      else {
        u128 prev = comb_q[c - 1];
        /* prev * c / (c - q): exact; guard overflow of prev * c */
        u128 g = prev / (u128)(c - q), r = prev % (u128)(c - q);
        /* prev*c/(c-q) = g*c + r*c/(c-q); r*c divisible-part exact */
        u128 hi = g * (u128)c;
        u128 v = hi + (r * (u128)c) / (u128)(c - q);
        if ((c && hi / (u128)c != g) || v < hi) { first_bad = c; break; }
        comb_q[c] = v;
      }
    }
  }
  double t_start = now_s();
  /* pre_runtime_tasks, engine.py:147-173 */
  int W = cfg->workers;
  int64_t emitted = 0, filtered = 0, need = s->p_eff - 1;
  for (int64_t i = 0; i < n; i++) {
    int64_t r = s->order[i];
    if (cfg->root_mask && !cfg->root_mask[r]) continue;
    if (s->und_size[r] < need) { filtered++; continue; }
    emitted += s->p_eff == 1 ? 1 : (s->dir_off[r + 1] - s->dir_off[r]);
  }
  int64_t *troot = xmalloc((size_t)(emitted ? emitted : 1) * 8);
  int64_t *tsec = xmalloc((size_t)(emitted ? emitted : 1) * 8);
  int64_t **lists = calloc(W, sizeof(int64_t *));
  int64_t *sizes = calloc(W, sizeof(int64_t));
  for (int w = 0; w < W; w++) lists[w] = xmalloc((size_t)(emitted / W + 2) * 8);
  int64_t e = 0;
  for (int64_t i = 0; i < n; i++) {
    int64_t r = s->order[i];
    if (cfg->root_mask && !cfg->root_mask[r]) continue;
    if (s->und_size[r] < need) continue;
    if (s->p_eff == 1) {
      troot[e] = r; tsec[e] = -1; lists[e % W][sizes[e % W]++] = e; e++;
    } else {
      for (int64_t f = s->dir_off[r]; f < s->dir_off[r + 1]; f++) {
        troot[e] = r; tsec[e] = s->dir_idx[f]; lists[e % W][sizes[e % W]++] = e; e++;
      }
    }
  }
  board_t board = {W, sizes, calloc(W, sizeof(uint32_t)), calloc(W, sizeof(pthread_mutex_t))};
  for (int w = 0; w < W; w++) pthread_mutex_init(&board.latches[w], NULL);
  worker_t *ws = calloc(W, sizeof(worker_t));
  pthread_t *th = calloc(W, sizeof(pthread_t));
  for (int w = 0; w < W; w++) {
    searcher_init(&ws[w].S, s, cfg, comb_q, max_deg);
    ws[w].S.first_bad = first_bad;
    ws[w].S.timing = (W == 1);
    ws[w].board = &board; ws[w].me = w; ws[w].lists = lists;
    ws[w].troot = troot; ws[w].tsecond = tsec;
    ws[w].task_words = cfg->task_words; ws[w].task_count = cfg->task_count;
    ws[w].task_l1 = cfg->task_l1;
  }
  if (W == 1) {
    /* engine.py:437-447: straight loop, nothing stolen */
    for (int64_t i = 0; i < sizes[0]; i++) do_task(&ws[0], lists[0][i]);
    ws[0].consumed = sizes[0];
  } else {
    for (int w = 0; w < W; w++) pthread_create(&th[w], NULL, worker_main, &ws[w]);
    for (int w = 0; w < W; w++) pthread_join(th[w], NULL);
  }
  u128 total = 0; int over = 0;
  for (int w = 0; w < W; w++) {
    u128 before = total;
    total += ws[w].S.count;
    if (total < before || ws[w].S.overflow) over = 1;
    out->batches += ws[w].S.batches;
    out->intersections += ws[w].S.inter;
    out->operand_words += ws[w].S.op_words;
    out->min_words += ws[w].S.min_words;
    out->time_1hop += ws[w].S.t1; out->time_2hop += ws[w].S.t2;
    out->consumed += ws[w].consumed;
    out->stolen += ws[w].stolen;
    searcher_free(&ws[w].S);
  }
  out->wall_time = now_s() - t_start;
  out->prep_time = s->prep_time;
  out->count_lo = (uint64_t)total; out->count_hi = (uint64_t)(total >> 64);
  out->overflow = over;
  out->anchor = s->anchor; out->p_eff = s->p_eff; out->q_eff = s->q_eff;
  out->roots_filtered = filtered; out->emitted = emitted;
  for (int w = 0; w < W; w++) { free(lists[w]); pthread_mutex_destroy(&board.latches[w]); }
  free(lists); free(sizes); free(board.counters); free(board.latches);
  free(ws); free(th); free(troot); free(tsec); free(comb_q);
  return 0;
}
