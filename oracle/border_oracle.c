/* border_oracle.c -- CPU restatement of the reference's Border column reordering.
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the device Border pass
 * (paper_2403_07858_b200/csrc/border.cu).  Only tests/, __graft_entry__.smoke() and
 * bench/timing scripts' CPU legs may call it; the product path never does.
 *
 * Follows pkg/src/bicount/reorder.py step by step, deliberately the literal way
 * (the device pass uses an algebraic decomposition of the swap profit, so the two
 * are independent restatements):
 *   build_block_matrix  reorder.py:44-64   (row, block) -> mask, pos / colv identity
 *   count_one_blocks    reorder.py:67-68
 *   per-vertex 1-blocks reorder.py:71-79   (owner of the single bit via colv)
 *   swap_profit         reorder.py:82-110  (rows in the symmetric difference only)
 *   apply_swap          reorder.py:113-134 (zero masks are deleted: here kept as 0,
 *                                           which every count treats the same)
 *   border_reorder      reorder.py:146-179 (argmax -> min-overlap partners ->
 *                                           first strictly best profit; stop at none)
 *   _row_overlap        reorder.py:182-188
 * Parity pinned by tests/golden/border.json (reference runs, make_border_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t *key;  /* r * nblocks + b, UINT64_MAX = empty */
  uint32_t *val;
  uint64_t cap, used;
} bmap;

static uint64_t hmix(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  return k;
}

static int bmap_init(bmap *m, uint64_t want) {
  uint64_t cap = 16;
  while (cap < 2 * want + 16) cap <<= 1;
  m->key = (uint64_t *)malloc(cap * sizeof(uint64_t));
  m->val = (uint32_t *)calloc(cap, sizeof(uint32_t));
  if (!m->key || !m->val) return -1;
  memset(m->key, 0xff, cap * sizeof(uint64_t));
  m->cap = cap;
  m->used = 0;
  return 0;
}

static uint32_t *bmap_slot(bmap *m, uint64_t k, int insert);

static int bmap_grow(bmap *m) {
  bmap n;
  if (bmap_init(&n, m->cap) != 0) return -1;
  for (uint64_t i = 0; i < m->cap; i++)
    if (m->key[i] != UINT64_MAX) *bmap_slot(&n, m->key[i], 1) = m->val[i];
  free(m->key);
  free(m->val);
  *m = n;
  return 0;
}

/* value slot of key k; NULL when absent and !insert */
static uint32_t *bmap_slot(bmap *m, uint64_t k, int insert) {
  uint64_t i = hmix(k) & (m->cap - 1);
  for (;;) {
    if (m->key[i] == k) return &m->val[i];
    if (m->key[i] == UINT64_MAX) {
      if (!insert) return NULL;
      if (2 * (m->used + 1) > m->cap) {
        if (bmap_grow(m) != 0) return NULL;
        return bmap_slot(m, k, 1);
      }
      m->key[i] = k;
      m->val[i] = 0;
      m->used++;
      return &m->val[i];
    }
    i = (i + 1) & (m->cap - 1);
  }
}

static uint32_t bget(bmap *m, uint64_t k) {
  const uint32_t *s = bmap_slot(m, k, 0);
  return s ? *s : 0u;
}

static int one(uint32_t w) { return __builtin_popcount(w) == 1; }

typedef struct {
  const int64_t *coff;
  const int32_t *cidx; /* rows_of[c], sorted */
  const int64_t *roff;
  const int32_t *ridx; /* row_cols[r] (column vertex ids) */
  int64_t ncols, nrows, nblocks;
  int64_t *pos, *colv;
  bmap blocks;
} bstate;

/* reorder.py:82-110 */
static int64_t swap_profit(bstate *s, int64_t vm, int64_t vn) {
  if (vm == vn) return 0;
  const int64_t bm = s->pos[vm] >> 5, jm = s->pos[vm] & 31;
  const int64_t bn = s->pos[vn] >> 5, jn = s->pos[vn] & 31;
  if (bm == bn) return 0;
  const uint32_t bit_m = 1u << jm, bit_n = 1u << jn;
  int64_t a = s->coff[vm], ae = s->coff[vm + 1], b = s->coff[vn], be = s->coff[vn + 1];
  int64_t profit = 0;
  while (a < ae || b < be) {
    int64_t r;
    int in_m;
    if (b >= be || (a < ae && s->cidx[a] < s->cidx[b])) {
      r = s->cidx[a++];
      in_m = 1;
    } else if (a >= ae || s->cidx[b] < s->cidx[a]) {
      r = s->cidx[b++];
      in_m = 0;
    } else { /* in both: not in the symmetric difference */
      a++;
      b++;
      continue;
    }
    const uint32_t wm = bget(&s->blocks, (uint64_t)r * s->nblocks + bm);
    const uint32_t wn = bget(&s->blocks, (uint64_t)r * s->nblocks + bn);
    uint32_t wm2, wn2;
    if (in_m) {
      wm2 = wm & ~bit_m;
      wn2 = wn | bit_n;
    } else {
      wm2 = wm | bit_m;
      wn2 = wn & ~bit_n;
    }
    profit += one(wm) + one(wn) - one(wm2) - one(wn2);
  }
  return profit;
}

/* reorder.py:113-134 */
static int apply_swap(bstate *s, int64_t vm, int64_t vn) {
  const int64_t pm = s->pos[vm], pn = s->pos[vn];
  const int64_t bm = pm >> 5, bn = pn >> 5;
  const uint32_t bit_m = 1u << (pm & 31), bit_n = 1u << (pn & 31);
  int64_t a = s->coff[vm], ae = s->coff[vm + 1], b = s->coff[vn], be = s->coff[vn + 1];
  while (a < ae || b < be) {
    int64_t r, sb_blk, db_blk;
    uint32_t sbit, dbit;
    if (b >= be || (a < ae && s->cidx[a] < s->cidx[b])) {
      r = s->cidx[a++];
      sb_blk = bm, sbit = bit_m, db_blk = bn, dbit = bit_n;
    } else if (a >= ae || s->cidx[b] < s->cidx[a]) {
      r = s->cidx[b++];
      sb_blk = bn, sbit = bit_n, db_blk = bm, dbit = bit_m;
    } else {
      a++;
      b++;
      continue;
    }
    uint32_t *src = bmap_slot(&s->blocks, (uint64_t)r * s->nblocks + sb_blk, 0);
    if (src) *src &= ~sbit;
    uint32_t *dst = bmap_slot(&s->blocks, (uint64_t)r * s->nblocks + db_blk, 1);
    if (!dst) return -1;
    *dst |= dbit;
  }
  s->pos[vm] = pn;
  s->pos[vn] = pm;
  s->colv[pm] = vn;
  s->colv[pn] = vm;
  return 0;
}

/* border_reorder (reorder.py:146-179).  Columns: the layer reordered (coff/cidx:
 * column -> rows); rows: the other layer (roff/ridx: row -> columns).  Writes the
 * permutation (old id -> new position) and the 1-block history (<= iters + 1
 * entries); returns the history length, or -1 on allocation failure. */
int64_t orc_border(const int64_t *coff, const int32_t *cidx, int64_t ncols, const int64_t *roff,
                   const int32_t *ridx, int64_t nrows, int64_t iters, int64_t *perm_out,
                   int64_t *hist_out) {
  bstate s;
  memset(&s, 0, sizeof s);
  s.coff = coff;
  s.cidx = cidx;
  s.roff = roff;
  s.ridx = ridx;
  s.ncols = ncols;
  s.nrows = nrows;
  s.nblocks = (ncols + 31) / 32;
  const int64_t E = ncols ? coff[ncols] : 0;
  s.pos = (int64_t *)malloc((ncols + 1) * sizeof(int64_t));
  s.colv = (int64_t *)malloc((ncols + 1) * sizeof(int64_t));
  int64_t *per = (int64_t *)malloc((ncols + 1) * sizeof(int64_t));
  int64_t *ov = (int64_t *)malloc((ncols + 1) * sizeof(int64_t));
  if (!s.pos || !s.colv || !per || !ov || bmap_init(&s.blocks, (uint64_t)E) != 0) return -1;
  for (int64_t c = 0; c < ncols; c++) {
    s.pos[c] = s.colv[c] = c;
    for (int64_t e = coff[c]; e < coff[c + 1]; e++) {
      uint32_t *w = bmap_slot(&s.blocks, (uint64_t)cidx[e] * s.nblocks + (c >> 5), 1);
      if (!w) return -1;
      *w |= 1u << (c & 31);
    }
  }
  int64_t total = 0;
  for (uint64_t i = 0; i < s.blocks.cap; i++)
    if (s.blocks.key[i] != UINT64_MAX && one(s.blocks.val[i])) total++;
  int64_t nh = 0;
  hist_out[nh++] = total;
  if (ncols >= 2) {
    for (int64_t it = 0; it < iters; it++) {
      memset(per, 0, ncols * sizeof(int64_t));
      for (uint64_t i = 0; i < s.blocks.cap; i++) {
        const uint32_t w = s.blocks.val[i];
        if (s.blocks.key[i] == UINT64_MAX || !one(w)) continue;
        const int64_t b = (int64_t)(s.blocks.key[i] % (uint64_t)s.nblocks);
        per[s.colv[b * 32 + (31 - __builtin_clz(w))]]++;
      }
      int64_t vm = 0;
      for (int64_t c = 1; c < ncols; c++)
        if (per[c] > per[vm]) vm = c;
      memset(ov, 0, ncols * sizeof(int64_t));
      for (int64_t e = coff[vm]; e < coff[vm + 1]; e++) {
        const int64_t r = cidx[e];
        for (int64_t f = roff[r]; f < roff[r + 1]; f++) ov[ridx[f]]++;
      }
      ov[vm] = INT64_MAX;
      int64_t floor = INT64_MAX;
      for (int64_t c = 0; c < ncols; c++)
        if (ov[c] < floor) floor = ov[c];
      int64_t best = -1, best_profit = 0;
      for (int64_t c = 0; c < ncols; c++) {
        if (ov[c] != floor) continue;
        const int64_t pr = swap_profit(&s, vm, c);
        if (pr > best_profit) {
          best_profit = pr;
          best = c;
        }
      }
      if (best < 0) break;
      if (apply_swap(&s, vm, best) != 0) return -1;
      total -= best_profit;
      hist_out[nh++] = total;
    }
  }
  memcpy(perm_out, s.pos, ncols * sizeof(int64_t));
  free(s.pos);
  free(s.colv);
  free(per);
  free(ov);
  free(s.blocks.key);
  free(s.blocks.val);
  return nh;
}
