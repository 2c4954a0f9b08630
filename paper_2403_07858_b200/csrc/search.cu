// search.cu -- level-1 pass and hybrid DFS-BFS enumeration on sm_100a.
//
// Restates Searcher.run_task / Searcher._descend (reference engine.py:245-374)
// and the leaf rule C(|C_R|, q) (engine.py:285, 346-347), for all tasks of
// this shard, with exact 128-bit counts.
//
// Level 1 (level1_kernel, warp per task): C_R1 = adj[r] & adj[s] and, when
// p_eff >= 3 and |C_R1| >= q, C_L1 = dir2[r] & dir2[s] -- the same two HTB
// intersections the reference performs first (engine.py:277-292).  The warp
// walks the shorter Idx run 32 words at a time; each lane finds its word in
// the longer run by lower_bound (the reference's bisect, htb.py:122-154) or,
// when the longer row is a hub with a dense bitmap, by one direct load; the
// matched Val words are ANDed and reduced with __popc / __reduce_add_sync.
// p_eff = 2 finishes here.  Deeper searches record |C_R1|, |C_L1| and their
// HTB word counts, drop tasks failing prune_keep (engine.py:110-112) and emit
// the cost key |C_L1|*|C_R1| for the pre-runtime LPT order.
//
// Enumeration (enum_kernel): persistent warps pull tasks, heaviest first,
// from one global atomic cursor (runtime stealing).  Every deeper C_R is a
// subset of C_R1 and every deeper C_L a subset of C_L1 (engine.py:296-297,
// 365-366), so the warp re-materialises C_R1 / C_L1 as HTB words and
// re-indexes them as a task-local universe:
//   rowR[x] = N(x) & C_R1,   rowL[x] = dir2(x) & C_L1   for x in C_L1,
// dense bitsets over the local indices (the reference's level 1->2
// intersections, engine.py:338, 360).  Every deeper intersection is then an
// aligned AND of ceil(|C_R1|/32) resp. ceil(|C_L1|/32) words + popcount.
// A node's candidates are expanded as one BFS batch across the 32 lanes and
// the search descends depth-first into survivors (hybrid DFS-BFS, Alg. 1).
//
// Heavy tasks (the head of the LPT queue, p_eff >= 5) are split: their frame
// goes to a global arena and the nodes of the split level are pushed to a
// sub-task array that sub_kernel drains with every warp (composite balancing:
// pre-runtime LPT order + runtime stealing + intra-task splitting).
//
// The reference's batch accounting (engine.py:306-331) is reproduced exactly:
// a node's C_R / C_L word counts in the original id space are the number of
// C_R1 / C_L1 HTB words its local bitset touches.
#include <cub/cub.cuh>

#include <algorithm>
#include <ctime>
#include <cstdlib>
#include <vector>

#include "engine.h"

namespace bc {

// Per-phase SM-cycle tallies (lane 0 of every warp) in -DBC_PHASE_PROF builds:
// 0 claim, 1 level-1 re-materialisation, 2 decode + slot map, 3 rows,
// 4 expansions, 5 leaf-parents, 6 finish.
#ifdef BC_PHASE_PROF
__device__ unsigned long long g_phase[16];
__device__ __forceinline__ long long clk() {
  long long c = 0;
#ifdef __CUDA_ARCH__
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
#endif
  return c;
}
struct PhaseClock {
  unsigned long long t[8];
  long long last;
  __device__ __forceinline__ PhaseClock() : last(clk()) {
    for (int i = 0; i < 8; i++) t[i] = 0;
  }
  __device__ __forceinline__ void mark(int i) {
    const long long n = clk();
    t[i] += (unsigned long long)(n - last);
    last = n;
  }
  __device__ __forceinline__ void flush() {
    if ((threadIdx.x & 31) == 0)
      for (int i = 0; i < 8; i++) atomicAdd(&g_phase[i], t[i]);
  }
};
#else
struct PhaseClock {
  __device__ __forceinline__ void mark(int) {}
  __device__ __forceinline__ void flush() {}
};
#endif
#define PH_DECL PhaseClock ph_;
#define PH_MARK(i) ph_.mark(i)
#define PH_FLUSH() ph_.flush()

int64_t debug_phase_cycles(uint64_t *out, int n) {
#ifdef BC_PHASE_PROF
  unsigned long long h[16];
  BC_CUDA(cudaMemcpyFromSymbol(h, g_phase, sizeof h));
  for (int i = 0; i < n && i < 16; i++) out[i] = h[i];
  const unsigned long long z[16] = {0};
  BC_CUDA(cudaMemcpyToSymbol(g_phase, z, sizeof z));
  return 16;
#else
  for (int i = 0; i < n; i++) out[i] = 0;
  return 0;
#endif
}

namespace {

struct Graph2 {  // HTB arenas (htb.py:64-86) + dense hub rows
  const int64_t *__restrict__ aoff;
  const uint32_t *__restrict__ aidx;
  const uint32_t *__restrict__ aval;
  const int64_t *__restrict__ doff;
  const uint32_t *__restrict__ didx;
  const uint32_t *__restrict__ dval;
  const int32_t *__restrict__ dense_id;
  const uint32_t *__restrict__ dense;
  int64_t mw;
  const int64_t *__restrict__ boff;  // opposite layer -> anchor CSR (graph.py:15-49 v_adj
  const int32_t *__restrict__ bidx;  // of the work graph): the wedge-scatter rows
};

struct Params {
  Graph2 g;
  const int2 *__restrict__ tasks;
  int64_t n_tasks;
  int shard, nshards;
  int p_eff, q_eff;
  int cap;       // batch_buffer_capacity
  int mode_dfs;  // EngineConfig.mode == "dfs"
  const ulonglong2 *__restrict__ comb;  // C(c, q_eff), c <= max anchor degree
  int64_t first_bad;                    // C(c, q) >= 2^128 for c >= first_bad
  unsigned long long *acc;              // [2] shard count (lo, hi)
  int *overflow;
  unsigned long long *ctr;              // counters, see CTR_*
  unsigned long long *task_counts;      // optional [2 * n_tasks]
  int map_words;                        // anchor-word slot map entries (0 = no map)
  const int64_t *__restrict__ roff;     // wedge-scatter level 1: C_R1 of local task j is
  const int32_t *__restrict__ lists;    //   lists[roff[j], roff[j+1]) (ascending ids), or null
  int rowR_mode;                        // 0 = per-task choice, 1 = scatter, 2 = probe
};

enum { CTR_ALIVE = 0, CTR_BATCHES, CTR_STOLEN, CTR_INTER, CTR_OPW, CTR_MINW, CTR_MAXRO,
       CTR_MAXSCR, CTR_SPILL, CTR_NEXT, CTR_SUB_USED, CTR_SUB_N, CTR_SUB_NEXT, CTR_SPLIT,
       CTR_HEAVY, CTR_MAXRO_T, CTR_MAXSCR_T, CTR_COUNT };

struct Info {  // level-1 facts of one task
  int32_t cr, wr, cl, wl;
};

struct Dims {
  int nR, nL, wR, wL, WR, WL;
  bool r_single, l_single;  // every C_R1 / C_L1 HTB word holds exactly one id
};

__device__ __forceinline__ Dims dims_of(const Info &in) {
  Dims d;
  d.nR = in.cr;
  d.nL = in.cl;
  d.wR = in.wr;
  d.wL = in.wl;
  d.WR = (in.cr + 31) >> 5;
  d.WL = (in.cl + 31) >> 5;
  d.r_single = in.wr == in.cr;
  d.l_single = in.wl == in.cl;
  return d;
}

__device__ __forceinline__ void add_comb(const Params &P, Acc128 &a, int c) {
  if (c >= P.first_bad) {
    atomicExch(P.overflow, 1);
    return;
  }
  const ulonglong2 v = __ldg(P.comb + c);
  a.add(v.x, v.y);
}

// Warp-cooperative HTB intersection of slices [a0,a1) and [b0,b1) of one arena
// (htb.py:122-154).  Walks the shorter slice 32 words at a time.  Matches in
// the longer slice come from `dense_b` (its dense bitmap row) when given, else
// from a per-lane lower_bound with a moving lower bound.  Returns |A & B| in
// card and the number of nonzero words; with OUT, writes the nonzero words
// (ascending) and exclusive prefix popcounts (o_pre[words] = card).
template <bool OUT>
__device__ __forceinline__ int warp_isect(const uint32_t *__restrict__ idx,
                                          const uint32_t *__restrict__ val, int64_t a0,
                                          int64_t a1, int64_t b0, int64_t b1,
                                          const uint32_t *__restrict__ dense_b, int &card,
                                          uint32_t *o_idx, uint32_t *o_val, int *o_pre) {
  const int lane = lane_id();
  int pos = 0, run = 0;
  int64_t lo = b0;
  for (int64_t base = a0; base < a1; base += 32) {
    const int64_t i = base + lane;
    int64_t j = b1;
    uint32_t x = 0, key = 0;
    if (i < a1) {
      key = __ldg(idx + i);
      if (dense_b) {
        x = __ldg(val + i) & __ldg(dense_b + key);
        j = b0;
      } else {
        j = lower_bound_u32(idx, lo, b1, key);
        if (j < b1 && __ldg(idx + j) == key) x = __ldg(val + i) & __ldg(val + j);
      }
    }
    const unsigned nz = __ballot_sync(FULL, x != 0);
    const int c = __popc(x);
    if (OUT) {
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += t;
      }
      if (x) {
        const int k = pos + __popc(nz & lanemask_lt());
        o_idx[k] = key;
        o_val[k] = x;
        o_pre[k] = run + incl - c;
      }
      run += __shfl_sync(FULL, incl, 31);
    } else {
      run += __reduce_add_sync(FULL, c);
    }
    pos += __popc(nz);
    if (!dense_b) {
      const int64_t jl = __shfl_sync(FULL, j, 31);
      if (jl >= b1) break;
      lo = jl;
    }
  }
  if (OUT) {
    if (lane == 0) o_pre[pos] = run;
    __syncwarp();
  }
  card = run;
  return pos;
}

// adj[r] & adj[s] with the shorter side walked and the longer side probed.
template <bool OUT>
__device__ __forceinline__ int isect_adj(const Graph2 &g, int r, int s, int &card,
                                         uint32_t *o_idx, uint32_t *o_val, int *o_pre) {
  int64_t a0 = g.aoff[r], a1 = g.aoff[r + 1], b0 = g.aoff[s], b1 = g.aoff[s + 1];
  int lng = s;
  if (a1 - a0 > b1 - b0) {
    int64_t t0 = a0, t1 = a1;
    a0 = b0; a1 = b1; b0 = t0; b1 = t1;
    lng = r;
  }
  const int sl = g.dense_id[lng];
  const uint32_t *db = sl >= 0 ? g.dense + (int64_t)sl * g.mw : nullptr;
  return warp_isect<OUT>(g.aidx, g.aval, a0, a1, b0, b1, db, card, o_idx, o_val, o_pre);
}

template <bool OUT>
__device__ __forceinline__ int isect_dir(const Graph2 &g, int r, int s, int &card,
                                         uint32_t *o_idx, uint32_t *o_val, int *o_pre) {
  int64_t a0 = g.doff[r], a1 = g.doff[r + 1], b0 = g.doff[s], b1 = g.doff[s + 1];
  if (a1 - a0 > b1 - b0) {
    int64_t t0 = a0, t1 = a1;
    a0 = b0; a1 = b1; b0 = t0; b1 = t1;
  }
  return warp_isect<OUT>(g.didx, g.dval, a0, a1, b0, b1, nullptr, card, o_idx, o_val, o_pre);
}

// Frame: the task-local universe.  The read-only part (built once) and the
// per-warp DFS scratch are carved separately so split tasks can share the
// former from global memory.  rowL rows exist only for the level-1
// R-survivors (x with |rowR[x]| >= q): every candidate whose rowL is ever read
// has passed |R & rowR[x]| >= q at some node, and R is a subset of C_R1, so it
// passed at level 1 too; lslot[x] is its rowL row (-1: none).
struct Frame {
  uint32_t *r_idx, *r_val;
  int *r_pre;
  uint32_t *l_idx, *l_val;
  int *l_pre;
  int *lids, *lslot;
  uint32_t *rowR, *rowL;
  int *adjw, *dirw;
  int *cand;
  uint32_t *setR, *setL;
  int *surv;
  int *ns, *cur;
  int surv_cap;
};

// rowL is materialised for p_eff >= 5 (reused at every depth) and for p_eff = 4
// without a slot map; p_eff = 4 with a map walks dir2(u) lazily instead.
__host__ __device__ __forceinline__ bool has_rowL(int p_eff, int map_words) {
  return p_eff >= 5 || (p_eff == 4 && map_words == 0);
}

// rowL rows allocated: level-1 R-survivors, bounded by nL (or by the triage cap).
__host__ __device__ __forceinline__ int64_t rowl_rows(int nL, bool rowL, int cap) {
  return rowL ? (cap > 0 && cap < nL ? cap : nL) : 0;
}

__host__ __device__ __forceinline__ int64_t ro_words(int nR, int nL, int wR, int wL, bool rowL,
                                                     bool instr, int cap = 0) {
  const int64_t WR = (nR + 31) / 32, WL = (nL + 31) / 32;
  int64_t w = 3 * (int64_t)wR + 1 + 3 * (int64_t)wL + 1;  // C_R1 / C_L1 HTB words + prefixes
  w += 2 * (int64_t)nL;                                    // lids, lslot
  w += (int64_t)nL * WR;                                   // rowR
  w += rowl_rows(nL, rowL, cap) * WL;                      // rowL
  if (instr) w += 2 * (int64_t)nL;                         // adj / dir2 slice words
  return (w + 3) & ~int64_t(3);
}

// DFS stack: nodes at levels 1 .. p_eff-3 are expanded warp-cooperatively
// (leaf-parents at p_eff-2 are finished lane-parallel without a frame).
__host__ __device__ __forceinline__ int stack_levels(int p_eff) {
  return p_eff - 3 > 1 ? p_eff - 3 : 1;
}

// survivors listed per level: level-1 R-survivors, bounded by nL (or the triage cap)
__host__ __device__ __forceinline__ int surv_cap_of(int nL, int cap) {
  return cap > 0 && cap < nL ? cap : nL;
}

__host__ __device__ __forceinline__ int64_t scratch_words(int nR, int nL, int p_eff, int cap = 0) {
  const int64_t WR = (nR + 31) / 32, WL = (nL + 31) / 32;
  const int64_t levels = stack_levels(p_eff);
  return ((int64_t)nL + levels * (WR + WL + surv_cap_of(nL, cap) + 2) + 3) & ~int64_t(3);
}

__device__ __forceinline__ void carve_ro(Frame &f, uint32_t *p, const Dims &d, bool rowL,
                                         bool instr, int cap = 0) {
  f.r_idx = p; p += d.wR;
  f.r_val = p; p += d.wR;
  f.r_pre = (int *)p; p += d.wR + 1;
  f.l_idx = p; p += d.wL;
  f.l_val = p; p += d.wL;
  f.l_pre = (int *)p; p += d.wL + 1;
  f.lids = (int *)p; p += d.nL;
  f.lslot = (int *)p; p += d.nL;
  f.rowR = p; p += (int64_t)d.nL * d.WR;
  f.rowL = p; p += rowl_rows(d.nL, rowL, cap) * d.WL;
  f.adjw = (int *)p; if (instr) p += d.nL;
  f.dirw = (int *)p;
}

__device__ __forceinline__ void carve_scratch(Frame &f, uint32_t *p, const Dims &d, int p_eff,
                                              int cap = 0) {
  const int levels = stack_levels(p_eff);
  f.surv_cap = surv_cap_of(d.nL, cap);
  f.cand = (int *)p; p += d.nL;
  f.setR = p; p += (int64_t)levels * d.WR;
  f.setL = p; p += (int64_t)levels * d.WL;
  f.surv = (int *)p; p += (int64_t)levels * f.surv_cap;
  f.ns = (int *)p; p += levels;
  f.cur = (int *)p;
}

__device__ __forceinline__ const uint32_t *rowL_of(const Frame &f, const Dims &d, int u) {
  return f.rowL + (int64_t)f.lslot[u] * d.WL;
}

// Writes a local-universe row whose set positions arrive in ascending order:
// each 32-bit word is stored once, from a register, with no read-modify-write.
struct RowWriter {
  uint32_t *row;
  int W, cur;
  uint32_t bits;
  __device__ __forceinline__ RowWriter(uint32_t *r, int w) : row(r), W(w), cur(0), bits(0) {}
  __device__ __forceinline__ void flush_to(int w) {
    row[cur] = bits;
    for (int x = cur + 1; x < w; x++) row[x] = 0;
    cur = w;
    bits = 0;
  }
  __device__ __forceinline__ void set(int pos) {
    const int w = pos >> 5;
    if (w != cur) flush_to(w);
    bits |= 1u << (pos & 31);
  }
  __device__ __forceinline__ void set_run(int pos, int len) {  // len <= 32
    const int w = pos >> 5, sh = pos & 31;
    if (w != cur) flush_to(w);
    const unsigned long long x = (len == 32 ? 0xffffffffull : ((1ull << len) - 1ull)) << sh;
    bits |= (uint32_t)x;
    if (x >> 32) {
      flush_to(w + 1);
      bits = (uint32_t)(x >> 32);
    }
  }
  // bits m (a subset of HTB word v whose first local index is pre)
  __device__ __forceinline__ void add(int pre, uint32_t v, uint32_t m) {
    if (m == v) {
      set_run(pre, __popc(v));
      return;
    }
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      set(pre + __popc(v & ((1u << b) - 1u)));
    }
  }
  __device__ __forceinline__ void finish() {
    if (W) flush_to(W);
  }
};

// row = (local word list S) & (global HTB slice [g0,g1)), mapped to local bits.
// Dense hub rows answer each S word with one load; short rows walk the shorter
// side and bisect the longer (htb.py:122-154).
__device__ __forceinline__ void local_row(const uint32_t *s_idx, const uint32_t *s_val,
                                          const int *s_pre, int ns, const uint32_t *__restrict__ gidx,
                                          const uint32_t *__restrict__ gval, int64_t g0, int64_t g1,
                                          const uint32_t *__restrict__ dense_row, uint32_t *row,
                                          int W) {
  RowWriter rw(row, W);
  if (dense_row) {
    int k = 0;
    for (; k + 4 <= ns; k += 4) {  // four independent probes in flight
      uint32_t d[4];
#pragma unroll
      for (int t = 0; t < 4; t++) d[t] = __ldg(dense_row + s_idx[k + t]);
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const uint32_t m = s_val[k + t] & d[t];
        if (m) rw.add(s_pre[k + t], s_val[k + t], m);
      }
    }
    for (; k < ns; k++) {
      const uint32_t m = s_val[k] & __ldg(dense_row + s_idx[k]);
      if (m) rw.add(s_pre[k], s_val[k], m);
    }
  } else if (ns <= g1 - g0) {
    int64_t lo = g0;
    for (int k = 0; k < ns; k++) {
      const uint32_t key = s_idx[k];
      const int64_t j = lower_bound_u32(gidx, lo, g1, key);
      if (j == g1) break;
      if (__ldg(gidx + j) == key) {
        const uint32_t m = s_val[k] & __ldg(gval + j);
        if (m) rw.add(s_pre[k], s_val[k], m);
        lo = j + 1;
      } else {
        lo = j;
      }
    }
  } else {
    int lo = 0;
    for (int64_t j = g0; j < g1; j++) {
      const uint32_t key = __ldg(gidx + j);
      int a = lo, b = ns;
      while (a < b) {
        const int mid = (a + b) >> 1;
        if (s_idx[mid] < key) a = mid + 1;
        else b = mid;
      }
      if (a == ns) break;
      if (s_idx[a] == key) {
        const uint32_t m = s_val[a] & __ldg(gval + j);
        if (m) rw.add(s_pre[a], s_val[a], m);
        lo = a + 1;
      } else {
        lo = a;
      }
    }
  }
  rw.finish();
}

// rowL via the anchor-word slot map: walk dir2(x)'s HTB words, one map lookup each.
__device__ __forceinline__ void local_row_map(const uint16_t *map, const uint32_t *l_val,
                                              const int *l_pre, const uint32_t *__restrict__ gidx,
                                              const uint32_t *__restrict__ gval, int64_t g0,
                                              int64_t g1, uint32_t *row, int W) {
  RowWriter rw(row, W);
  for (int64_t j = g0; j < g1; j++) {
    const int k = map[__ldg(gidx + j)];
    if (k != 0xffff) {
      const uint32_t m = l_val[k] & __ldg(gval + j);
      if (m) rw.add(l_pre[k], l_val[k], m);
    }
  }
  rw.finish();
}

// Number of original HTB words (ranges [pre[k], pre[k+1])) a local bitset touches.
__device__ __forceinline__ int words_touched(const uint32_t *set, const int *pre, int nwords,
                                             int W, bool single) {
  int c = 0;
  if (single) {
    for (int w = lane_id(); w < W; w += 32) c += __popc(set[w]);
  } else {
    for (int k = lane_id(); k < nwords; k += 32) {
      const int a = pre[k], b = pre[k + 1];
      const int w0 = a >> 5, w1 = (b - 1) >> 5;
      unsigned long long x = set[w0];
      if (w1 > w0) x |= (unsigned long long)set[w1] << 32;
      x >>= (a & 31);
      const int len = b - a;
      const unsigned long long mask = len >= 64 ? ~0ull : ((1ull << len) - 1ull);
      c += (x & mask) != 0;
    }
  }
  return __reduce_add_sync(FULL, c);
}

// Same count for R & ru, by one lane.
__device__ __forceinline__ int lane_words(const uint32_t *R, const uint32_t *ru, const int *pre,
                                          int nwords, int W, bool single) {
  int c = 0;
  if (single) {
    for (int w = 0; w < W; w++) c += __popc(R[w] & ru[w]);
    return c;
  }
  for (int k = 0; k < nwords; k++) {
    const int a = pre[k], b = pre[k + 1];
    const int w0 = a >> 5, w1 = (b - 1) >> 5;
    unsigned long long x = R[w0] & ru[w0];
    if (w1 > w0) x |= (unsigned long long)(R[w1] & ru[w1]) << 32;
    x >>= (a & 31);
    const int len = b - a;
    const unsigned long long mask = len >= 64 ? ~0ull : ((1ull << len) - 1ull);
    c += (x & mask) != 0;
  }
  return c;
}

// order-preserving compaction of the set bits of a W-word set into cand[]
__device__ __forceinline__ int compact_bits(const uint32_t *set, int W, int *cand) {
  const int lane = lane_id();
  int n = 0;
  for (int w0 = 0; w0 < W; w0 += 32) {
    const uint32_t mine = w0 + lane < W ? set[w0 + lane] : 0u;
    unsigned nz = __ballot_sync(FULL, mine != 0);
    while (nz) {
      const int x = __ffs(nz) - 1;
      nz &= nz - 1;
      const uint32_t bits = __shfl_sync(FULL, mine, x);
      if ((bits >> lane) & 1u) cand[n + __popc(bits & lanemask_lt())] = (w0 + x) * 32 + lane;
      n += __popc(bits);
    }
  }
  __syncwarp();
  return n;
}

struct Tally {
  unsigned long long batches = 0, inter = 0, opw = 0, minw = 0;
};

// reference batch count for one node expansion (engine.py:306-313, 329-331)
__device__ __forceinline__ unsigned node_batches(const Params &P, unsigned ncand, int wr, int wl,
                                                 bool leaf) {
  if (!ncand) return 0;
  if (P.mode_dfs) return ncand;
  const unsigned cap = (unsigned)P.cap;
  const unsigned w = (unsigned)(wr > 1 ? wr : 1), w2 = leaf ? 1u : (unsigned)(wl > 1 ? wl : 1);
  const unsigned wm = w > w2 ? w : w2;  // b = cap / max(wr, wl)
  if ((unsigned long long)ncand * wm <= cap) return 1;  // one batch: no division
  unsigned b = cap / wm;
  if (b < 1) b = 1;
  return (ncand + b - 1) / b;
}

// Per-warp shared-memory staging of (leaf-parent slot, leaf) pairs.
constexpr int LEAF_BUF = 256;
struct LeafBuf {
  uint32_t *pairs;  // [LEAF_BUF]: slot << 27 | local leaf index
  int *wr;          // [32]: C_R word count of each slot's leaf-parent
  int *ncand;       // [32]: leaves of each slot's leaf-parent (batch accounting)
};

// Evaluate buffered leaves: add C(|R & rowR[u] & rowR[w]|, q) (engine.py:342-347).
template <bool INSTR>
__device__ __forceinline__ void flush_leaves(const Params &P, const Frame &f, const Dims &d,
                                             const uint32_t *R, const int *slot_u,
                                             const LeafBuf &lb, int fill, Acc128 &acc,
                                             Tally &tl) {
  __syncwarp();
  const int WR = d.WR, q = P.q_eff;
  for (int p0 = 0; p0 < fill; p0 += 32) {
    const int i = p0 + lane_id();
    if (i < fill) {
      const uint32_t pr = lb.pairs[i];
      const int slot = pr >> 27, w = pr & 0x7ffffff;
      const int u = slot_u[slot];
      const uint32_t *ru = f.rowR + (int64_t)u * WR, *rw = f.rowR + (int64_t)w * WR;
      int c = 0;
      for (int x = 0; x < WR; x++) c += __popc(R[x] & ru[x] & rw[x]);
      if (INSTR) {
        const int wr = lb.wr[slot];
        tl.inter++;
        tl.opw += wr + f.adjw[w];
        tl.minw += wr < f.adjw[w] ? wr : f.adjw[w];
      }
      if (c >= q) add_comb(P, acc, c);
    }
  }
  __syncwarp();
}

// Stage the leaves of one round: lane holds HTB-style word (v, pre) with
// present bits m for leaf-parent `slot`; leaves are compacted into the pair
// buffer (flushed 32 at a time when full).
template <bool INSTR>
__device__ __forceinline__ void stage_leaves(const Params &P, const Frame &f, const Dims &d,
                                             const uint32_t *R, const int *slot_u,
                                             const LeafBuf &lb, int &fill, int slot, uint32_t v,
                                             int pre, uint32_t m, int wr, Acc128 &acc,
                                             Tally &tl) {
  const int lane = lane_id();
  const int cnt = __popc(m);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += t;
  }
  const int total = __shfl_sync(FULL, incl, 31);
  if (fill + total > LEAF_BUF) {
    flush_leaves<INSTR>(P, f, d, R, slot_u, lb, fill, acc, tl);
    fill = 0;
  }
  if (total > LEAF_BUF) {  // a round too wide to stage: evaluate in place
    const int WR = d.WR;
    const uint32_t *ru = f.rowR + (int64_t)slot_u[slot] * WR;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int w = pre + __popc(v & ((1u << b) - 1u));
      const uint32_t *rw = f.rowR + (int64_t)w * WR;
      int c = 0;
      for (int x = 0; x < WR; x++) c += __popc(R[x] & ru[x] & rw[x]);
      if (INSTR) {
        tl.inter++;
        tl.opw += wr + f.adjw[w];
        tl.minw += wr < f.adjw[w] ? wr : f.adjw[w];
      }
      if (c >= P.q_eff) add_comb(P, acc, c);
    }
    return;
  }
  int o = fill + incl - cnt;
  while (m) {
    const int b = __ffs(m) - 1;
    m &= m - 1;
    lb.pairs[o++] = ((uint32_t)slot << 27) | (uint32_t)(pre + __popc(v & ((1u << b) - 1u)));
  }
  fill += total;
}

// Leaf-parent nodes, 32 at a time (one slot per lane): node u (a survivor
// of the node at `level`) has R' = R & rowR[u] and L' = L & rowL[u] -- or,
// with LAZY (p_eff = 4, level 1), L' = dir2(u) & C_L1 read through the slot
// map -- and its children are leaves (engine.py:342-347).  The L' words of
// the 32 leaf-parents are walked as one flattened stream (LAZY: every lane
// loads a different dir2 word each round, so the gathers overlap), and the
// leaves are compacted and evaluated 32 at a time.
template <bool INSTR, bool LAZY>
__device__ __forceinline__ void leaf_parents(const Params &P, const Frame &f, const Dims &d,
                                             int level, const int *list, int n,
                                             const uint16_t *map, const LeafBuf &lb, Acc128 &acc,
                                             Tally &tl) {
  const int lane = lane_id();
  const int WR = d.WR, WL = d.WL;
  const uint32_t *R = f.setR + (level - 1) * WR;
  const uint32_t *Ls = f.setL + (level - 1) * WL;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const bool act = i < n;
    const int u = act ? list[i] : 0;
    const int wr = act ? lane_words(R, f.rowR + (int64_t)u * WR, f.r_pre, d.wR, WR, d.r_single) : 0;
    lb.wr[lane] = wr;
    lb.ncand[lane] = 0;
    __syncwarp();
    int fill = 0;
    if (LAZY) {
      int64_t start = 0;
      int len = 0;
      if (act) {
        const int id = f.lids[u];
        start = P.g.doff[id];
        len = (int)(P.g.doff[id + 1] - start);
      }
      int incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += t;
      }
      const int excl = incl - len;
      const int T = __shfl_sync(FULL, incl, 31);
      for (int r0 = 0; r0 < T; r0 += 32) {
        const int pos = r0 + lane;
        // owning slot: the last lane whose exclusive offset is <= pos
        int sl = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const int c = sl + step;
          const int e = __shfl_sync(FULL, excl, c < 32 ? c : 31);
          if (c < 32 && e <= pos) sl = c;
        }
        const int64_t st = __shfl_sync(FULL, start, sl);
        const int ex = __shfl_sync(FULL, excl, sl);
        uint32_t m = 0, v = 0xffffffffu;
        int pre = 0;
        if (pos < T) {
          const int64_t j = st + (pos - ex);
          const uint32_t key = __ldg(P.g.didx + j), dv = __ldg(P.g.dval + j);
          const int k = map[key];
          if (k != 0xffff) {
            v = f.l_val[k];
            m = v & dv;
            pre = f.l_pre[k];
            if (m) atomicAdd(&lb.ncand[sl], __popc(m));
          }
        }
        stage_leaves<INSTR>(P, f, d, R, list + base, lb, fill, sl, v, pre, m, lb.wr[sl], acc, tl);
      }
    } else {
      int ncand = 0;
      const uint32_t *rl = act ? rowL_of(f, d, u) : f.rowL;
      for (int x = 0; __any_sync(FULL, act && x < WL); x++) {
        uint32_t m = 0;
        if (act && x < WL) m = Ls[x] & rl[x];
        ncand += __popc(m);
        stage_leaves<INSTR>(P, f, d, R, list + base, lb, fill, lane, 0xffffffffu, x * 32, m, wr,
                            acc, tl);
      }
      lb.ncand[lane] = ncand;
    }
    flush_leaves<INSTR>(P, f, d, R, list + base, lb, fill, acc, tl);
    if (act) tl.batches += node_batches(P, (unsigned)lb.ncand[lane], wr, 0, true);
    __syncwarp();
  }
}

// Expand node at `level` (1-based): children at level+1 (engine.py:315-374).
// Children that are leaves are counted here; children that are leaf-parents
// are finished lane-parallel (leaf_parents); deeper survivors are listed in
// surv[level-1] for the depth-first descent.
template <bool INSTR, bool LAZY>
__device__ __forceinline__ void expand(const Params &P, const Frame &f, const Dims &d, int level,
                                       const uint16_t *map, const LeafBuf &lb, Acc128 &acc,
                                       Tally &tl, PhaseClock &ph_) {
  const int lane = lane_id();
  const int WR = d.WR, WL = d.WL, nL = d.nL;
  const int li = level - 1;
  const uint32_t *R = f.setR + li * WR;
  const uint32_t *Ls = f.setL + li * WL;
  const bool leaf = level + 1 == P.p_eff - 1;
  const bool lp = level + 1 == P.p_eff - 2;  // children are leaf-parents
  const int ncand = compact_bits(Ls, WL, f.cand);
  const int wr = level == 1 ? d.wR : words_touched(R, f.r_pre, d.wR, WR, d.r_single);
  const int wl = leaf ? 0 : (level == 1 ? d.wL : words_touched(Ls, f.l_pre, d.wL, WL, d.l_single));
  if (lane == 0) tl.batches += node_batches(P, (unsigned)ncand, wr, wl, leaf);
  int ns = 0;
  const int need_l = P.p_eff - level - 2;  // prune_keep(cr, cl, level+1): cl >= p - (level+1) - 1
  int *out = f.surv + li * f.surv_cap;
  for (int c0 = 0; c0 < ncand; c0 += 32) {
    const int i = c0 + lane;
    bool keep = false;
    int u = 0;
    if (i < ncand) {
      u = f.cand[i];
      const uint32_t *row = f.rowR + (int64_t)u * WR;
      int cr = 0;
      for (int w = 0; w < WR; w++) cr += __popc(R[w] & row[w]);
      if (INSTR) {
        tl.inter++;
        tl.opw += wr + f.adjw[u];
        tl.minw += wr < f.adjw[u] ? wr : f.adjw[u];
      }
      if (cr >= P.q_eff) {
        if (leaf) {
          add_comb(P, acc, cr);
        } else {
          if (INSTR) {
            tl.inter++;
            tl.opw += wl + f.dirw[u];
            tl.minw += wl < f.dirw[u] ? wl : f.dirw[u];
          }
          if (LAZY) {
            keep = true;  // |L'| >= 1 is checked when the leaf-parent is walked
          } else {
            const uint32_t *rl = rowL_of(f, d, u);
            int cl = 0;
            for (int w = 0; w < WL; w++) cl += __popc(Ls[w] & rl[w]);
            keep = cl >= need_l;
          }
        }
      }
    }
    if (!leaf) {
      const unsigned m = __ballot_sync(FULL, keep);
      if (keep) out[ns + __popc(m & lanemask_lt())] = u;
      ns += __popc(m);
    }
  }
  __syncwarp();
  if (lp && ns) {
    PH_MARK(4);
    leaf_parents<INSTR, LAZY>(P, f, d, level, out, ns, map, lb, acc, tl);
    PH_MARK(5);
    ns = 0;
  }
  if (lane == 0) {
    f.ns[li] = ns;
    f.cur[li] = 0;
  }
  __syncwarp();
}

// Where split nodes go (heavy tasks only).
struct SplitSink {
  uint32_t *arena;          // sub-task records
  int64_t arena_words;
  unsigned long long *index; // record offsets
  int64_t index_cap;
  int level;                // emit nodes of this level instead of descending
  int64_t frame_off;        // this task's read-only frame in the frame arena
  int task_j;               // local task index
};

// Push node (level lv, sets R, L) as a sub-task; false if the arena is full.
__device__ __forceinline__ bool emit_node(const Params &P, const SplitSink &S, const Dims &d,
                                          int lv, const uint32_t *R, const uint32_t *rr,
                                          const uint32_t *Ls, const uint32_t *rl) {
  const int lane = lane_id();
  const int64_t words = 4 + d.WR + d.WL;
  long long off = -1;
  if (lane == 0) {
    const unsigned long long o = atomicAdd(P.ctr + CTR_SUB_USED, (unsigned long long)words);
    if ((int64_t)(o + words) <= S.arena_words) {
      const unsigned long long k = atomicAdd(P.ctr + CTR_SUB_N, 1ull);
      if ((int64_t)k < S.index_cap) {
        off = (long long)o;
        S.index[k] = o;
      }
    }
  }
  off = __shfl_sync(FULL, off, 0);
  if (off < 0) return false;
  uint32_t *rec = S.arena + off;
  if (lane == 0) {
    rec[0] = (uint32_t)S.task_j;
    rec[1] = (uint32_t)lv;
    rec[2] = (uint32_t)(S.frame_off & 0xffffffffll);
    rec[3] = (uint32_t)(S.frame_off >> 32);
  }
  for (int w = lane; w < d.WR; w += 32) rec[4 + w] = R[w] & rr[w];
  for (int w = lane; w < d.WL; w += 32) rec[4 + d.WR + w] = Ls[w] & rl[w];
  __syncwarp();
  return true;
}

// DFS from a node at `start` whose sets sit in setR/setL[start-1].
template <bool INSTR, bool LAZY>
__device__ __forceinline__ void dfs(const Params &P, const Frame &f, const Dims &d, int start,
                                    const uint16_t *map, const LeafBuf &lb, Acc128 &acc, Tally &tl,
                                    const SplitSink *sink, PhaseClock &ph_) {
  const int lane = lane_id();
  const int WR = d.WR, WL = d.WL, nL = d.nL, p_eff = P.p_eff;
  expand<INSTR, LAZY>(P, f, d, start, map, lb, acc, tl, ph_);
  int level = start;
  while (level >= start) {
    const int li = level - 1;
    if (level + 1 < p_eff - 2 && f.cur[li] < f.ns[li]) {
      const int u = f.surv[li * f.surv_cap + f.cur[li]];
      __syncwarp();
      if (lane == 0) f.cur[li]++;
      const uint32_t *rr = f.rowR + (int64_t)u * WR;
      const uint32_t *rl = rowL_of(f, d, u);
      if (sink && level + 1 == sink->level &&
          emit_node(P, *sink, d, level + 1, f.setR + li * WR, rr, f.setL + li * WL, rl))
        continue;
      for (int w = lane; w < WR; w += 32) f.setR[(li + 1) * WR + w] = f.setR[li * WR + w] & rr[w];
      for (int w = lane; w < WL; w += 32) f.setL[(li + 1) * WL + w] = f.setL[li * WL + w] & rl[w];
      __syncwarp();
      level++;
      expand<INSTR, LAZY>(P, f, d, level, map, lb, acc, tl, ph_);
    } else {
      level--;
    }
  }
}

// Sorted id list -> HTB words (htb.py:89-115) with exclusive prefix
// popcounts (o_pre[words] = n); returns the word count.
__device__ __forceinline__ int list_to_htb(const int32_t *__restrict__ ids, int n,
                                           uint32_t *o_idx, uint32_t *o_val, int *o_pre) {
  const int lane = lane_id();
  int pos = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    uint32_t word = 0;
    bool start = false;
    if (i < n) {
      word = (uint32_t)__ldg(ids + i) >> 5;
      start = i == 0 || ((uint32_t)__ldg(ids + i - 1) >> 5) != word;
    }
    const unsigned m = __ballot_sync(FULL, start);
    if (start) {
      uint32_t v = 0;
      for (int k = i; k < n; k++) {
        const uint32_t id = (uint32_t)__ldg(ids + k);
        if ((id >> 5) != word) break;
        v |= 1u << (id & 31);
      }
      const int o = pos + __popc(m & lanemask_lt());
      o_idx[o] = word;
      o_val[o] = v;
      o_pre[o] = i;
    }
    pos += __popc(m);
  }
  if (lane == 0) o_pre[pos] = n;
  __syncwarp();
  return pos;
}

// rowR by wedge scatter: for every C_R1 member v (local index i, ascending id
// order) and every anchor x in N(v) that lies in C_L1 (slot map), set bit i of
// rowR[x].  Work is sum_{v in C_R1} deg(v) over contiguous opposite-layer rows
// instead of |C_L1| probes of (possibly hub-sized) adjacency rows.
__device__ __forceinline__ void scatter_rowR(const Params &P, const Frame &f, const Dims &d,
                                             const uint16_t *map) {
  const int lane = lane_id();
  const int64_t total = (int64_t)d.nL * d.WR;
  for (int64_t w = lane; w < total; w += 32) f.rowR[w] = 0;
  __syncwarp();
  for (int k = lane; k < d.wR; k += 32) {
    uint32_t bits = f.r_val[k];
    const int64_t vb = (int64_t)f.r_idx[k] * 32;
    int i = f.r_pre[k];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int64_t v = vb + b;
      const uint32_t ibit = 1u << (i & 31);
      const int iw = i >> 5;
      for (int64_t e = __ldg(P.g.boff + v), e1 = __ldg(P.g.boff + v + 1); e < e1; e++) {
        const int x = __ldg(P.g.bidx + e);
        const int kk = map[x >> 5];
        if (kk == 0xffff) continue;
        const uint32_t lv = f.l_val[kk];
        const int xb = x & 31;
        if (!((lv >> xb) & 1u)) continue;
        const int lx = f.l_pre[kk] + __popc(lv & ((1u << xb) - 1u));
        atomicOr(f.rowR + (int64_t)lx * d.WR + iw, ibit);
      }
      i++;
    }
  }
  __syncwarp();
}

// Frame part 1 for task (r, s) (local index j): C_R1 / C_L1 (engine.py:277-292)
// -- C_R1 from the wedge-scatter level-1 lists when present -- the decoded C_L1
// ids + slot map, and rowR[x] = N(x) & C_R1 for x in C_L1 (engine.py:338).
// Returns the number of level-1 R-survivors (|rowR[x]| >= q).
template <bool INSTR>
__device__ __forceinline__ int build_frame_R(const Params &P, const Frame &f, const Dims &d,
                                             int r, int s, int64_t j, uint16_t *map,
                                             PhaseClock &ph_) {
  const int lane = lane_id();
  int card;
  if (P.lists) list_to_htb(P.lists + P.roff[j], d.nR, f.r_idx, f.r_val, f.r_pre);
  else isect_adj<true>(P.g, r, s, card, f.r_idx, f.r_val, f.r_pre);
  isect_dir<true>(P.g, r, s, card, f.l_idx, f.l_val, f.l_pre);
  PH_MARK(1);
  // decode C_L1 ids (ascending, htb.py:42-52); fill the slot map
  for (int k = lane; k < d.wL; k += 32) {
    uint32_t v = f.l_val[k];
    const int base_id = (int)f.l_idx[k] * 32;
    int pos = f.l_pre[k];
    if (map) map[f.l_idx[k]] = (uint16_t)k;
    while (v) {
      f.lids[pos++] = base_id + __ffs(v) - 1;
      v &= v - 1;
    }
  }
  __syncwarp();
  PH_MARK(2);
  bool scatter = false;
  if (map && P.rowR_mode != 2) {
    if (P.rowR_mode == 1) {
      scatter = true;
    } else {
      // sum of C_R1 members' degrees vs ~2 probes per (x, C_R1 word)
      long long sdeg = 0;
      for (int k = lane; k < d.wR; k += 32) {
        uint32_t bits = f.r_val[k];
        const int64_t vb = (int64_t)f.r_idx[k] * 32;
        while (bits) {
          const int64_t v = vb + __ffs(bits) - 1;
          bits &= bits - 1;
          sdeg += __ldg(P.g.boff + v + 1) - __ldg(P.g.boff + v);
        }
      }
      sdeg = warp_sum(sdeg);
      scatter = sdeg < 2ll * d.nL * d.wR;
    }
  }
  if (scatter) {
    scatter_rowR(P, f, d, map);
  } else {
    for (int x = lane; x < d.nL; x += 32) {
      const int id = f.lids[x];
      const int sl = P.g.dense_id[id];
      local_row(f.r_idx, f.r_val, f.r_pre, d.wR, P.g.aidx, P.g.aval, P.g.aoff[id],
                P.g.aoff[id + 1], sl >= 0 ? P.g.dense + (int64_t)sl * P.g.mw : nullptr,
                f.rowR + (int64_t)x * d.WR, d.WR);
    }
    __syncwarp();
  }
  int ns1 = 0;
  for (int x = lane; x < d.nL; x += 32) {
    const uint32_t *row = f.rowR + (int64_t)x * d.WR;
    int c = 0;
    for (int w = 0; w < d.WR; w++) c += __popc(row[w]);
    ns1 += c >= P.q_eff;
  }
  return __reduce_add_sync(FULL, ns1);
}

// Frame part 2: rowL[x] = dir2(x) & C_L1 (engine.py:360) for the level-1
// R-survivors only (lslot), and the slice lengths the instrumented tallies use.
template <bool INSTR, bool LAZY>
__device__ __forceinline__ void build_frame_L(const Params &P, const Frame &f, const Dims &d,
                                              const uint16_t *map, bool rowL, PhaseClock &ph_) {
  const int lane = lane_id();
  const bool build = rowL && P.p_eff >= 4 && !LAZY;
  int base = 0;
  for (int x0 = 0; x0 < d.nL; x0 += 32) {
    const int x = x0 + lane;
    bool sv = false;
    if (x < d.nL) {
      const uint32_t *row = f.rowR + (int64_t)x * d.WR;
      int c = 0;
      for (int w = 0; w < d.WR; w++) c += __popc(row[w]);
      sv = c >= P.q_eff;
    }
    const unsigned m = __ballot_sync(FULL, sv);
    if (x < d.nL) {
      const int slot = sv ? base + __popc(m & lanemask_lt()) : -1;
      f.lslot[x] = slot;
      const int id = f.lids[x];
      if (build && sv) {
        const int64_t d0 = P.g.doff[id], d1 = P.g.doff[id + 1];
        uint32_t *out = f.rowL + (int64_t)slot * d.WL;
        if (map)
          local_row_map(map, f.l_val, f.l_pre, P.g.didx, P.g.dval, d0, d1, out, d.WL);
        else
          local_row(f.l_idx, f.l_val, f.l_pre, d.wL, P.g.didx, P.g.dval, d0, d1, nullptr, out,
                    d.WL);
      }
      if (INSTR) {
        f.adjw[x] = (int)(P.g.aoff[id + 1] - P.g.aoff[id]);
        f.dirw[x] = (int)(P.g.doff[id + 1] - P.g.doff[id]);
      }
    }
    base += __popc(m);
  }
  __syncwarp();
  PH_MARK(3);
}

__device__ __forceinline__ void clear_map(uint16_t *map, const Frame &f, const Dims &d) {
  if (!map) return;
  for (int k = lane_id(); k < d.wL; k += 32) map[f.l_idx[k]] = 0xffff;
  __syncwarp();
}

__device__ __forceinline__ void init_root_sets(const Frame &f, const Dims &d) {
  const int lane = lane_id();
  for (int w = lane; w < d.WR; w += 32) {
    const int rem = d.nR - w * 32;
    f.setR[w] = rem >= 32 ? FULL : ((1u << rem) - 1u);
  }
  for (int w = lane; w < d.WL; w += 32) {
    const int rem = d.nL - w * 32;
    f.setL[w] = rem >= 32 ? FULL : ((1u << rem) - 1u);
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// p_eff = 1: C(deg(root), q) per task (engine.py:267-275)
// ---------------------------------------------------------------------------
__global__ void p1_kernel(Params P, const int64_t *__restrict__ deg_off) {
  Acc128 a{0, 0};
  const int64_t nloc = P.n_tasks > P.shard ? (P.n_tasks - P.shard + P.nshards - 1) / P.nshards : 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nloc;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = P.shard + j * P.nshards;
    const int r = P.tasks[t].x;
    const int d = (int)(deg_off[r + 1] - deg_off[r]);
    Acc128 one{0, 0};
    if (d >= P.q_eff) add_comb(P, one, d);
    if (P.task_counts) {
      P.task_counts[2 * t] = one.lo;
      P.task_counts[2 * t + 1] = one.hi;
    }
    a.add(one.lo, one.hi);
  }
  a = warp_sum128(a);
  if (lane_id() == 0) atomic_add128(P.acc, P.overflow, a.lo, a.hi);
}

// ---------------------------------------------------------------------------
// level 1 (engine.py:265-299 up to the descent)
// ---------------------------------------------------------------------------
template <bool INSTR>
__global__ void __launch_bounds__(256) level1_kernel(Params P, Info *__restrict__ info,
                                                     uint32_t *__restrict__ cost) {
  const int lane = lane_id();
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nloc = P.n_tasks > P.shard ? (P.n_tasks - P.shard + P.nshards - 1) / P.nshards : 0;
  Acc128 a{0, 0};
  unsigned long long alive = 0, inter = 0, opw = 0, minw = 0, maxro = 0, maxscr = 0;
  for (int64_t j = gw; j < nloc; j += nw) {
    const int64_t t = P.shard + j * P.nshards;
    const int2 tk = P.tasks[t];
    int cr, wr;
    if (P.lists) {  // C_R1 from the wedge-scatter pass: |C_R1| and its HTB word count
      const int64_t l0 = P.roff[j];
      cr = (int)(P.roff[j + 1] - l0);
      wr = 0;
      for (int b = 0; b < cr; b += 32) {
        const int i = b + lane;
        bool start = false;
        if (i < cr) {
          const uint32_t w = (uint32_t)__ldg(P.lists + l0 + i) >> 5;
          start = i == 0 || ((uint32_t)__ldg(P.lists + l0 + i - 1) >> 5) != w;
        }
        wr += __popc(__ballot_sync(FULL, start));
      }
    } else {
      wr = isect_adj<false>(P.g, tk.x, tk.y, cr, nullptr, nullptr, nullptr);
    }
    if (INSTR) {
      const int64_t la = P.g.aoff[tk.x + 1] - P.g.aoff[tk.x], lb = P.g.aoff[tk.y + 1] - P.g.aoff[tk.y];
      inter++;
      opw += la + lb;
      minw += la < lb ? la : lb;
    }
    Info in{cr, wr, -1, -1};
    uint32_t key = 0;
    Acc128 one{0, 0};
    if (cr >= P.q_eff) {
      if (P.p_eff == 2) {
        add_comb(P, one, cr);
      } else {
        int cl;
        const int wl = isect_dir<false>(P.g, tk.x, tk.y, cl, nullptr, nullptr, nullptr);
        if (INSTR) {
          const int64_t la = P.g.doff[tk.x + 1] - P.g.doff[tk.x], lb = P.g.doff[tk.y + 1] - P.g.doff[tk.y];
          inter++;
          opw += la + lb;
          minw += la < lb ? la : lb;
        }
        in.cl = cl;
        in.wl = wl;
        if (cl >= P.p_eff - 2) {  // prune_keep(cr, cl, 1, p, q)
          const unsigned long long c = (unsigned long long)cl * (unsigned long long)cr;
          key = c > 0xfffffffeull ? 0xffffffffu : (uint32_t)(c ? c : 1);
          alive++;
          const unsigned long long ro =
              ro_words(cr, cl, wr, wl, has_rowL(P.p_eff, P.map_words), INSTR);
          const unsigned long long sc = scratch_words(cr, cl, P.p_eff);
          maxro = ro > maxro ? ro : maxro;
          maxscr = sc > maxscr ? sc : maxscr;
        }
      }
    }
    if (lane == 0) {
      info[j] = in;
      cost[j] = key;
      if (P.task_counts && P.p_eff == 2) {
        P.task_counts[2 * t] = one.lo;
        P.task_counts[2 * t + 1] = one.hi;
      }
    }
    a.add(one.lo, one.hi);  // lane-uniform: only lane 0 contributes below
  }
  if (lane == 0) {
    atomic_add128(P.acc, P.overflow, a.lo, a.hi);
    if (alive) atomicAdd(P.ctr + CTR_ALIVE, alive);
    if (INSTR) {
      atomicAdd(P.ctr + CTR_INTER, inter);
      atomicAdd(P.ctr + CTR_OPW, opw);
      atomicAdd(P.ctr + CTR_MINW, minw);
    }
    if (maxro) atomicMax(P.ctr + CTR_MAXRO, maxro);
    if (maxscr) atomicMax(P.ctr + CTR_MAXSCR, maxscr);
  }
}

// ---------------------------------------------------------------------------
// Level 1 by wedge scatter (root-grouped).  For root r, C_R1(r, s) =
// N(r) & N(s) for every task (r, s) at once: walk the wedges r - v - s with
// v in N(r) and s in N(v) & dir2(r) and append v to the list of task (r, s).
// The work is the root's 2-hop pool, sum_{v in N(r)} deg(v), read as short
// contiguous opposite-layer rows, instead of |dir2(r)| HTB intersections
// against (possibly hub-sized) adjacency rows (htb.py:122-154).  The lists
// are exactly the reference's C_R1 sets in ascending id order.
//
// Units are (root, chunk of L1_CH consecutive neighbours), one warp each,
// drawn from an atomic queue.  dir2(r) membership and slot (= position in
// dir2(r) = task offset from troot[r]) come from a per-warp shared-memory
// bitmap over anchor ids plus a u16 prefix per word (n <= 65536), else from a
// binary search of dir2(r).  Pass 1 counts hits per (unit, slot); a column
// scan turns them into per-task list offsets and per-unit cursors; pass 2
// appends, 32 neighbours per round, ranking same-slot hits by lane with a
// per-warp hit mask so every list comes out sorted.
// ---------------------------------------------------------------------------
constexpr int L1_CH = 1024;
constexpr int L1_THREADS = 128;

struct L1Args {
  const int64_t *__restrict__ aoff;  // anchor -> opposite
  const int32_t *__restrict__ aidx;
  const int64_t *__restrict__ boff;  // opposite -> anchor
  const int32_t *__restrict__ bidx;
  const int64_t *__restrict__ doff;  // dir2 lists (sorted ascending)
  const int32_t *__restrict__ didx;
  const int64_t *__restrict__ troot;
  const int32_t *__restrict__ unit_root;
  const int64_t *__restrict__ ubase;  // per root: aux offset of chunk 0 (stride |dir2(r)|)
  const int32_t *__restrict__ unit_first;  // per root: first unit id
  int64_t n_units;
  unsigned long long *aux;  // pass 1: counts; pass 2: cursors
  int map_words;            // bitmap words per warp (0 = binary search)
  int shard, nshards;
  int32_t *lists;           // pass 2
  uint32_t *masks;          // pass 2: per-warp hit masks [mask_stride]
  int64_t mask_stride;
  unsigned long long *next;
};

struct RootMap {
  uint32_t *bits;
  uint16_t *pre;
  const int32_t *__restrict__ d;
  int D;
  __device__ __forceinline__ int slot(int x) const {
    if (bits) {
      const uint32_t b = bits[x >> 5];
      const int xb = x & 31;
      if (!((b >> xb) & 1u)) return -1;
      return pre[x >> 5] + __popc(b & ((1u << xb) - 1u));
    }
    int lo = 0, hi = D;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(d + mid) < x) lo = mid + 1;
      else hi = mid;
    }
    return lo < D && __ldg(d + lo) == x ? lo : -1;
  }
};

__device__ __forceinline__ void rootmap_set(RootMap &m, bool on) {
  if (!m.bits) return;
  const int lane = lane_id();
  for (int i = lane; i < m.D; i += 32) {
    const int x = __ldg(m.d + i);
    if (on) {
      atomicOr(m.bits + (x >> 5), 1u << (x & 31));
      if (i == 0 || (__ldg(m.d + i - 1) >> 5) != (x >> 5)) m.pre[x >> 5] = (uint16_t)i;
    } else {
      m.bits[x >> 5] = 0;
    }
  }
  __syncwarp();
}

template <bool FILL>
__global__ void __launch_bounds__(L1_THREADS) l1_scatter(L1Args A) {
  extern __shared__ uint32_t sm[];
  const int lane = lane_id();
  const int wib = threadIdx.x >> 5;
  const int64_t gwarp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int mw = A.map_words;
  uint32_t *bits = mw ? sm + (int64_t)wib * (mw + (mw + 1) / 2) : nullptr;
  uint16_t *pre = mw ? (uint16_t *)(bits + mw) : nullptr;
  if (bits)
    for (int i = lane; i < mw; i += 32) bits[i] = 0;
  __syncwarp();
  uint32_t *mask = FILL ? A.masks + gwarp * A.mask_stride : nullptr;
  for (;;) {
    long long u = 0;
    if (lane == 0) u = (long long)atomicAdd(A.next, 1ull);
    u = __shfl_sync(FULL, u, 0);
    if (u >= A.n_units) break;
    const int r = A.unit_root[u];
    const int c = (int)(u - A.unit_first[r]);
    const int64_t d0 = A.doff[r];
    RootMap m{bits, pre, A.didx + d0, (int)(A.doff[r + 1] - d0)};
    rootmap_set(m, true);
    const int64_t T0 = A.troot[r];
    unsigned long long *col = A.aux + A.ubase[r] + (int64_t)c * m.D;
    const int64_t e0 = A.aoff[r] + (int64_t)c * L1_CH;
    const int64_t e1 = min(A.aoff[r + 1], e0 + L1_CH);
    for (int64_t base = e0; base < e1; base += 32) {
      const int64_t e = base + lane;
      int32_t v = 0;
      int64_t f0 = 0, f1 = 0;
      if (e < e1) {
        v = __ldg(A.aidx + e);
        f0 = __ldg(A.boff + v);
        f1 = __ldg(A.boff + v + 1);
      }
      if (!FILL) {
        for (int64_t f = f0; f < f1; f++) {
          const int k = m.slot(__ldg(A.bidx + f));
          if (k >= 0 && (T0 + k) % A.nshards == A.shard) atomicAdd(col + k, 1ull);
        }
      } else {
        // (a) hit masks, (b) ranked writes, (c) the lowest hitter advances the cursor
        for (int64_t f = f0; f < f1; f++) {
          const int k = m.slot(__ldg(A.bidx + f));
          if (k >= 0 && (T0 + k) % A.nshards == A.shard) atomicOr(mask + k, 1u << lane);
        }
        __syncwarp();
        for (int64_t f = f0; f < f1; f++) {
          const int k = m.slot(__ldg(A.bidx + f));
          if (k >= 0 && (T0 + k) % A.nshards == A.shard) {
            const uint32_t mk = *(volatile uint32_t *)(mask + k);
            A.lists[col[k] + __popc(mk & lanemask_lt())] = v;
          }
        }
        __syncwarp();
        for (int64_t f = f0; f < f1; f++) {
          const int k = m.slot(__ldg(A.bidx + f));
          if (k >= 0 && (T0 + k) % A.nshards == A.shard) {
            const uint32_t mk = *(volatile uint32_t *)(mask + k);
            if (mk && __ffs(mk) - 1 == lane) {
              col[k] += __popc(mk);
              mask[k] = 0;
            }
          }
        }
        __syncwarp();
      }
    }
    __syncwarp();  // lanes still probing the map must finish before it is cleared
    rootmap_set(m, false);
  }
}

// development check: |N(r) & N(s)| by merge, thread per local task
__global__ void l1_naive(const int2 *__restrict__ tasks, int64_t nloc, int shard, int nshards,
                         const int64_t *__restrict__ aoff, const int32_t *__restrict__ aidx,
                         const int64_t *__restrict__ cnt, unsigned long long *bad) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nloc) return;
  const int2 tk = tasks[shard + j * nshards];
  int64_t a = aoff[tk.x], a1 = aoff[tk.x + 1], b = aoff[tk.y], b1 = aoff[tk.y + 1], c = 0;
  while (a < a1 && b < b1) {
    const int x = aidx[a], y = aidx[b];
    c += x == y;
    a += x <= y;
    b += y <= x;
  }
  if (c != cnt[j]) {
    const unsigned long long k = atomicAdd(bad, 1ull);
    if (k < 5) printf("l1 check: task %lld (%d,%d) naive %lld pass1 %lld\n", (long long)j, tk.x, tk.y,
                      (long long)c, (long long)cnt[j]);
  }
}

// per local task: |C_R1| = sum over its root's chunks (pass-1 columns)
__global__ void l1_task_totals(const int2 *__restrict__ tasks, int64_t nloc, int shard, int nshards,
                               const int64_t *__restrict__ troot, const int64_t *__restrict__ ubase,
                               const int32_t *__restrict__ unit_first, const int64_t *__restrict__ doff,
                               const unsigned long long *__restrict__ aux, int64_t *__restrict__ cnt) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nloc) return;
  const int64_t t = shard + j * nshards;
  const int r = tasks[t].x;
  const int64_t k = t - troot[r], D = doff[r + 1] - doff[r];
  const int nch = unit_first[r + 1] - unit_first[r];
  unsigned long long c = 0;
  for (int ch = 0; ch < nch; ch++) c += aux[ubase[r] + ch * D + k];
  cnt[j] = (int64_t)c;
}

// per local task: pass-1 counts -> per-chunk write cursors (list offset + earlier chunks)
__global__ void l1_cursors(const int2 *__restrict__ tasks, int64_t nloc, int shard, int nshards,
                           const int64_t *__restrict__ troot, const int64_t *__restrict__ ubase,
                           const int32_t *__restrict__ unit_first, const int64_t *__restrict__ doff,
                           const int64_t *__restrict__ roff, unsigned long long *__restrict__ aux) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nloc) return;
  const int64_t t = shard + j * nshards;
  const int r = tasks[t].x;
  const int64_t k = t - troot[r], D = doff[r + 1] - doff[r];
  const int nch = unit_first[r + 1] - unit_first[r];
  unsigned long long run = (unsigned long long)roff[j];
  for (int ch = 0; ch < nch; ch++) {
    unsigned long long *p = aux + ubase[r] + ch * D + k;
    const unsigned long long x = *p;
    *p = run;
    run += x;
  }
}

// per root: chunks (units) and aux block size (0 for roots without tasks)
__global__ void l1_root_sizes(const int64_t *__restrict__ aoff, const int64_t *__restrict__ doff,
                              const int64_t *__restrict__ troot, int64_t n, int32_t *__restrict__ nunits,
                              int64_t *__restrict__ auxw) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  int32_t nu = 0;
  int64_t w = 0;
  const int64_t D = doff[r + 1] - doff[r];
  if (troot[r] >= 0 && D > 0) {
    const int64_t deg = aoff[r + 1] - aoff[r];
    nu = (int32_t)((deg + L1_CH - 1) / L1_CH);
    w = (int64_t)nu * D;
  }
  nunits[r] = nu;
  auxw[r] = w;
}

__global__ void l1_unit_roots(const int32_t *__restrict__ unit_first, int64_t n,
                              int32_t *__restrict__ unit_root) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int32_t u = unit_first[r]; u < unit_first[r + 1]; u++) unit_root[u] = (int32_t)r;
}

__global__ void max_dir_len(const int64_t *__restrict__ doff, int64_t n, unsigned long long *out) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long v = r < n ? (unsigned long long)(doff[r + 1] - doff[r]) : 0ull;
  v = __reduce_max_sync(FULL, (unsigned)v);
  if ((threadIdx.x & 31) == 0 && v) atomicMax(out, v);
}

// probe-cost estimate of level 1 (sum over local tasks of the shorter adjacency
// slice) vs the wedge pool of the roots: decides the level-1 mode
__global__ void l1_probe_cost(const int2 *__restrict__ tasks, int64_t nloc, int shard, int nshards,
                             const int64_t *__restrict__ hoff, unsigned long long *out) {
  unsigned long long c = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nloc;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int2 tk = tasks[shard + j * nshards];
    const int64_t a = hoff[tk.x + 1] - hoff[tk.x], b = hoff[tk.y + 1] - hoff[tk.y];
    c += (unsigned long long)(a < b ? a : b);
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void l1_pool(const int64_t *__restrict__ aoff, const int32_t *__restrict__ aidx,
                        const int64_t *__restrict__ boff, const int64_t *__restrict__ troot,
                        int64_t n, unsigned long long *out) {
  // warp per root with tasks: sum of its neighbours' degrees
  const int lane = lane_id();
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long c = 0;
  for (int64_t r = gw; r < n; r += nw) {
    if (troot[r] < 0) continue;
    for (int64_t e = aoff[r] + lane; e < aoff[r + 1]; e += 32) {
      const int v = aidx[e];
      c += (unsigned long long)(boff[v + 1] - boff[v]);
    }
  }
  c = warp_sum(c);
  if (lane == 0 && c) atomicAdd(out, c);
}

// ---------------------------------------------------------------------------
// enumeration (engine.py:315-374) over the task-local universe
// ---------------------------------------------------------------------------
struct EnumArgs {
  const Info *__restrict__ info;
  const int32_t *__restrict__ queue;  // local task ids, LPT order
  int64_t q0, q1;                     // this launch drains queue[q0, q1)
  int budget_words;                   // shared memory per warp for frames
  uint32_t *gscratch;                 // per-warp global fallback
  int64_t gscratch_words;
  uint32_t *frames;                   // SPLIT: read-only frames of queue[q0, q1)
  const int64_t *frame_off;           // SPLIT: [q1 - q0]
  SplitSink sink;
  const unsigned long long *sub_order;  // sub_kernel: record offsets, LPT order
  int triage;                           // > 0: defer tasks with more level-1 R-survivors
  int32_t *heavy;                       //   (or a frame over the scratch) to heavy[]
};

__device__ __forceinline__ void finish_task(const Params &P, Acc128 acc, int64_t t, bool atomic,
                                            Acc128 &total) {
  acc = warp_sum128(acc);
  if (lane_id() == 0) {
    total.add(acc.lo, acc.hi);
    if (P.task_counts) {
      if (atomic) atomic_add128(P.task_counts + 2 * t, P.overflow, acc.lo, acc.hi);
      else {
        P.task_counts[2 * t] = acc.lo;
        P.task_counts[2 * t + 1] = acc.hi;
      }
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void flush_tallies(const Params &P, const Acc128 &total, const Tally &tl,
                                              unsigned long long claims, unsigned long long spills,
                                              bool instr) {
  const int lane = lane_id();
  const unsigned long long batches = warp_sum(tl.batches);  // leaf_parents tally per lane
  if (lane == 0) {
    atomic_add128(P.acc, P.overflow, total.lo, total.hi);
    atomicAdd(P.ctr + CTR_BATCHES, batches);
    if (claims > 1) atomicAdd(P.ctr + CTR_STOLEN, claims - 1);
    if (spills) atomicAdd(P.ctr + CTR_SPILL, spills);
  }
  if (instr) {
    const unsigned long long a = warp_sum(tl.inter), b = warp_sum(tl.opw), c = warp_sum(tl.minw);
    if (lane == 0) {
      atomicAdd(P.ctr + CTR_INTER, a);
      atomicAdd(P.ctr + CTR_OPW, b);
      atomicAdd(P.ctr + CTR_MINW, c);
    }
  }
}

constexpr int ENUM_THREADS = 256;
#ifndef ENUM_MIN_BLOCKS
#define ENUM_MIN_BLOCKS 3
#endif
constexpr int LEAF_WORDS = LEAF_BUF + 64;  // per-warp leaf staging in shared memory

// Whole tasks (SPLIT = false) or the top levels of every task with its frame
// written to the global frame arena and split-level nodes pushed as sub-tasks
// (SPLIT = true, p_eff >= 5).
template <bool INSTR, bool LAZY, bool SPLIT>
__global__ void __launch_bounds__(ENUM_THREADS, ENUM_MIN_BLOCKS) enum_kernel(Params P, EnumArgs A) {
  extern __shared__ uint32_t smem[];
  const int lane = lane_id();
  const int wib = threadIdx.x >> 5;
  const int64_t gwarp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int map_w = (P.map_words + 1) / 2;  // u16 entries packed in words
  uint32_t *my = smem + (int64_t)wib * (map_w + LEAF_WORDS + A.budget_words);
  uint16_t *map = P.map_words ? (uint16_t *)my : nullptr;
  const LeafBuf lb{my + map_w, (int *)(my + map_w + LEAF_BUF), (int *)(my + map_w + LEAF_BUF + 32)};
  uint32_t *my_smem = my + map_w + LEAF_WORDS;
  uint32_t *my_global = A.gscratch ? A.gscratch + gwarp * A.gscratch_words : nullptr;
  if (map)
    for (int i = lane; i < map_w; i += 32) my[i] = 0xffffffffu;
  __syncwarp();
  Acc128 total{0, 0};
  Tally tl;
  unsigned long long claims = 0, spills = 0;
  const int p_eff = P.p_eff;
  PH_DECL
  for (;;) {
    long long qi = 0;
    if (lane == 0) qi = (long long)atomicAdd(P.ctr + CTR_NEXT, 1ull);
    qi = __shfl_sync(FULL, qi, 0) + A.q0;
    PH_MARK(0);
    if (qi >= A.q1) break;
    claims++;
    const int j = A.queue[qi];
    const int64_t t = P.shard + (int64_t)j * P.nshards;
    const int2 tk = P.tasks[t];
    const Dims d = dims_of(A.info[j]);
    const bool rowL = SPLIT || has_rowL(p_eff, P.map_words);
    const int cap = SPLIT ? 0 : A.triage;
    const int64_t ro = ro_words(d.nR, d.nL, d.wR, d.wL, rowL, INSTR, cap);
    const int64_t sc = scratch_words(d.nR, d.nL, p_eff, cap);
    uint32_t *ro_base, *sc_base;
    if (SPLIT) {
      ro_base = A.frames + A.frame_off[qi - A.q0];
      if (sc <= A.budget_words) sc_base = my_smem;
      else { sc_base = my_global; spills++; }
    } else if (ro + sc <= A.budget_words) {
      ro_base = my_smem;
      sc_base = my_smem + ro;
    } else {
      ro_base = my_global;
      sc_base = my_global + ro;
      spills++;
    }
    if (!sc_base || (sc_base == my_global && (SPLIT ? sc : ro + sc) > A.gscratch_words)) {
      if (A.triage > 0 && !SPLIT) {  // frame too large for the scratch: the split path takes it
        if (lane == 0) A.heavy[atomicAdd(P.ctr + CTR_HEAVY, 1ull)] = j;
        __syncwarp();
      } else if (lane == 0) {
        atomicExch(P.overflow, 2);  // cannot happen: sized from level-1 maxima
      }
      continue;
    }
    Frame f;
    carve_ro(f, ro_base, d, rowL, INSTR, cap);
    carve_scratch(f, sc_base, d, p_eff, cap);
    const int ns1 = build_frame_R<INSTR>(P, f, d, tk.x, tk.y, j, map, ph_);
    if (!SPLIT && A.triage > 0 && ns1 > A.triage) {  // heavy: defer to the split path
      if (lane == 0) A.heavy[atomicAdd(P.ctr + CTR_HEAVY, 1ull)] = j;
      clear_map(map, f, d);
      continue;
    }
    build_frame_L<INSTR, LAZY>(P, f, d, map, rowL, ph_);
    init_root_sets(f, d);
    Acc128 acc{0, 0};
    if (SPLIT) {
      SplitSink sink = A.sink;
      sink.frame_off = A.frame_off[qi - A.q0];
      sink.task_j = j;
      dfs<INSTR, false>(P, f, d, 1, map, lb, acc, tl, &sink, ph_);
    } else {
      dfs<INSTR, LAZY>(P, f, d, 1, map, lb, acc, tl, nullptr, ph_);
    }
    PH_MARK(4);
    clear_map(map, f, d);
    finish_task(P, acc, t, SPLIT, total);
    PH_MARK(6);
  }
  PH_FLUSH();
  flush_tallies(P, total, tl, claims, spills, INSTR);
}

// Split nodes: warp per sub-task record, records in LPT order.
template <bool INSTR>
__global__ void __launch_bounds__(ENUM_THREADS, ENUM_MIN_BLOCKS) sub_kernel(Params P, EnumArgs A, int64_t n_sub) {
  extern __shared__ uint32_t smem[];
  const int lane = lane_id();
  const int wib = threadIdx.x >> 5;
  const int64_t gwarp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  uint32_t *my = smem + (int64_t)wib * (LEAF_WORDS + A.budget_words);
  const LeafBuf lb{my, (int *)(my + LEAF_BUF), (int *)(my + LEAF_BUF + 32)};
  uint32_t *my_smem = my + LEAF_WORDS;
  uint32_t *my_global = A.gscratch ? A.gscratch + gwarp * A.gscratch_words : nullptr;
  Acc128 total{0, 0};
  Tally tl;
  unsigned long long spills = 0;
  const int p_eff = P.p_eff;
  PH_DECL
  for (;;) {
    long long k = 0;
    if (lane == 0) k = (long long)atomicAdd(P.ctr + CTR_SUB_NEXT, 1ull);
    k = __shfl_sync(FULL, k, 0);
    if (k >= n_sub) break;
    const uint32_t *rec = A.sink.arena + A.sub_order[k];
    const int j = (int)rec[0];
    const int lv = (int)rec[1];
    const int64_t foff = (int64_t)rec[2] | ((int64_t)rec[3] << 32);
    const int64_t t = P.shard + (int64_t)j * P.nshards;
    const Dims d = dims_of(A.info[j]);
    const int64_t sc = scratch_words(d.nR, d.nL, p_eff);
    uint32_t *sc_base = sc <= A.budget_words ? my_smem : my_global;
    if (sc_base == my_global) spills++;
    if (!sc_base || (sc_base == my_global && sc > A.gscratch_words)) {
      if (lane == 0) atomicExch(P.overflow, 2);
      continue;
    }
    Frame f;
    carve_ro(f, A.frames + foff, d, true, INSTR);
    carve_scratch(f, sc_base, d, p_eff);
    for (int w = lane; w < d.WR; w += 32) f.setR[(lv - 1) * d.WR + w] = rec[4 + w];
    for (int w = lane; w < d.WL; w += 32) f.setL[(lv - 1) * d.WL + w] = rec[4 + d.WR + w];
    __syncwarp();
    Acc128 acc{0, 0};
    PH_MARK(0);
    dfs<INSTR, false>(P, f, d, lv, nullptr, lb, acc, tl, nullptr, ph_);
    PH_MARK(4);
    finish_task(P, acc, t, true, total);
    PH_MARK(6);
  }
  PH_FLUSH();
  flush_tallies(P, total, tl, 0, spills, INSTR);
}

__global__ void gather_keys(const int32_t *ids, int64_t n, const uint32_t *cost, uint32_t *out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = cost[ids[i]];
}

__global__ void iota32(int32_t *a, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int32_t)i;
}

// frame / sub-task arena sizes for queue[q0, q1)
__global__ void split_sizes(const Info *info, const int32_t *queue, int64_t q0, int64_t q1,
                            bool instr, int split_level, int64_t *ro, int64_t *sub) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= q1 - q0) return;
  const Info in = info[queue[q0 + i]];
  ro[i] = ro_words(in.cr, in.cl, in.wr, in.wl, true, instr);
  const int64_t WR = (in.cr + 31) / 32, WL = (in.cl + 31) / 32;
  const int64_t nodes = split_level == 2 ? in.cl : (int64_t)in.cl * (in.cl - 1) / 2;
  sub[i] = nodes * (4 + WR + WL);
}

// sub-task LPT key: candidates left below the node, |L| * |R| (saturating)
__global__ void sub_keys(const uint32_t *arena, const unsigned long long *index, int64_t n,
                         const Info *info, uint32_t *key, unsigned long long *val) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t *rec = arena + index[i];
  const Info in = info[rec[0]];
  const int WR = (in.cr + 31) >> 5, WL = (in.cl + 31) >> 5;
  unsigned cr = 0, cl = 0;
  for (int w = 0; w < WR; w++) cr += __popc(rec[4 + w]);
  for (int w = 0; w < WL; w++) cl += __popc(rec[4 + WR + w]);
  const unsigned long long k = (unsigned long long)cl * cl * (cr ? cr : 1);
  key[i] = k > 0xffffffffull ? 0xffffffffu : (uint32_t)k;
  val[i] = index[i];
}

// C(c, q) for c <= max_deg as exact u128; returns first c whose value needs > 128 bits.
int64_t binomials(int q, int max_deg, std::vector<ulonglong2> &out) {
  out.assign((size_t)max_deg + 1, make_ulonglong2(0, 0));
  int64_t first_bad = (int64_t)max_deg + 1;
  u128 prev = 0;
  for (int64_t c = 0; c <= max_deg; c++) {
    u128 v;
    if (c < q) v = 0;
    else if (c == q) v = 1;
    else {
      // C(c,q) = C(c-1,q) * c / (c-q), exact via the split prev = g*(c-q) + r
      const u128 d = (u128)(c - q);
      const u128 g = prev / d, r = prev % d;
      const u128 hi = g * (u128)c;
      if (hi / (u128)c != g) { first_bad = c; break; }
      v = hi + (r * (u128)c) / d;
      if (v < hi) { first_bad = c; break; }
    }
    out[c] = make_ulonglong2((unsigned long long)v, (unsigned long long)(v >> 64));
    prev = v;
  }
  return first_bad;
}

template <typename T>
T sum_device(const T *p, int64_t n, cudaStream_t st) {
  DBuf<T> out;
  out.alloc(1, st);
  size_t tmp = 0;
  BC_CUDA(cub::DeviceReduce::Sum(nullptr, tmp, p, out.p, n, st));
  DBuf<char> t;
  t.alloc(tmp, st);
  BC_CUDA(cub::DeviceReduce::Sum(t.p, tmp, p, out.p, n, st));
  T h;
  copy_d2h(&h, out.p, sizeof(T), st);
  BC_CUDA(cudaStreamSynchronize(st));
  return h;
}

// BC_DEBUG=1: synchronising stage timer on stderr (development only)
struct DbgTimer {
  bool on;
  cudaStream_t st;
  double t0;
  explicit DbgTimer(cudaStream_t s) : on(getenv("BC_DEBUG") != nullptr), st(s), t0(now()) {}
  static double now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
  }
  void mark(const char *what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const double t = now();
    fprintf(stderr, "[bc search] %-14s %9.3f ms\n", what, 1e3 * (t - t0));
    t0 = t;
  }
};

int env_int(const char *name, int dflt) {  // development knobs
  const char *v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

template <typename K, typename V>
void sort_pairs_desc(const K *kin, K *kout, const V *vin, V *vout, int64_t n, cudaStream_t st) {
  size_t tmp = 0;
  BC_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, kin, kout, vin, vout, n, 0,
                                                    (int)sizeof(K) * 8, st));
  DBuf<char> t;
  t.alloc(tmp, st);
  BC_CUDA(cub::DeviceRadixSort::SortPairsDescending(t.p, tmp, kin, kout, vin, vout, n, 0,
                                                    (int)sizeof(K) * 8, st));
}

template <typename T>
void scan_excl(const T *in, T *out, int64_t n, cudaStream_t st) {
  size_t tmp = 0;
  BC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, st));
  DBuf<char> t;
  t.alloc(tmp, st);
  BC_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, n, st));
}

template <typename KERN>
int blocks_per_sm(KERN kern, size_t smem) {
  BC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  BC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, ENUM_THREADS, smem));
  return per_sm < 1 ? 1 : per_sm;
}

}  // namespace

void search(const DevStructs &s, const bc_config &cfg, bc_report &out) {
  cudaStream_t st = s.stream;
  int device = 0;
  BC_CUDA(cudaGetDevice(&device));
  const int sms = num_sms(device);
  const bool instr = (cfg.flags & BC_FLAG_INSTRUMENT) != 0;
  const bool allow_split = (cfg.flags & BC_FLAG_NO_SPLIT) == 0;
  const int nshards = cfg.shard_count > 0 ? cfg.shard_count : 1;
  const int shard = cfg.shard_index;
  if (shard < 0 || shard >= nshards) throw Error(BC_EINVAL, "shard_index out of range");
  const int64_t n_tasks = s.emitted;
  const int64_t nloc = n_tasks > shard ? (n_tasks - shard + nshards - 1) / nshards : 0;
  int64_t launches = 0;

  std::vector<ulonglong2> comb;
  const int64_t first_bad = binomials(s.q_eff, s.max_deg_anchor, comb);
  DBuf<ulonglong2> dcomb;
  dcomb.alloc(comb.size(), st);
  copy_h2d(dcomb.p, comb.data(), comb.size() * sizeof(ulonglong2), st);
  DBuf<unsigned long long> acc, ctr;
  DBuf<int> ovf;
  acc.alloc(2, st);
  acc.zero();
  ctr.alloc(CTR_COUNT, st);
  ctr.zero();
  ovf.alloc(1, st);
  ovf.zero();
  DBuf<unsigned long long> tcounts;
  const bool want_tc = (cfg.flags & BC_FLAG_TASK_COUNTS) && cfg.task_counts;
  if (want_tc) {
    if (cfg.task_counts_cap < n_tasks) throw Error(BC_EINVAL, "task_counts buffer too small");
    tcounts.alloc(2 * (size_t)(n_tasks ? n_tasks : 1), st);
    tcounts.zero();
  }
  Params P;
  P.g = Graph2{s.hadj_off.p, s.hadj_idx.p, s.hadj_val.p, s.hdir_off.p, s.hdir_idx.p, s.hdir_val.p,
               s.dense_id.p, s.dense.p, s.dense_mw, s.boff, s.bidx};
  P.tasks = s.tasks.p;
  P.n_tasks = n_tasks;
  P.shard = shard;
  P.nshards = nshards;
  P.p_eff = s.p_eff;
  P.q_eff = s.q_eff;
  P.cap = cfg.batch_words;
  P.mode_dfs = cfg.mode == 0;
  P.comb = dcomb.p;
  P.first_bad = first_bad;
  P.acc = acc.p;
  P.overflow = ovf.p;
  P.ctr = ctr.p;
  P.task_counts = want_tc ? tcounts.p : nullptr;
  P.roff = nullptr;
  P.lists = nullptr;
  P.rowR_mode = (cfg.flags & BC_FLAG_ROWR_SCATTER) ? 1 : (cfg.flags & BC_FLAG_ROWR_PROBE) ? 2 : 0;
  // slot map over anchor words for rowL (u16 per word) when it is small
  const int64_t anchor_words = (s.n + 31) / 32;
  P.map_words = (s.p_eff >= 4 && anchor_words <= 4096) ? (int)((anchor_words + 1) & ~1) : 0;
  const int map_w = (P.map_words + 1) / 2;
  const int wpb = ENUM_THREADS / 32;

  cudaEvent_t e0, e1, e2;
  BC_CUDA(cudaEventCreate(&e0));
  BC_CUDA(cudaEventCreate(&e1));
  BC_CUDA(cudaEventCreate(&e2));
  BC_CUDA(cudaEventRecord(e0, st));
  int64_t n_alive = 0, n_split = 0, n_sub_total = 0;
  if (nloc > 0 && s.p_eff == 1) {
    p1_kernel<<<sms * 8, 256, 0, st>>>(P, s.aoff);
    BC_CHECK_LAUNCH();
    launches++;
    BC_CUDA(cudaEventRecord(e1, st));
  } else if (nloc > 0) {
    DBuf<Info> info;
    DBuf<uint32_t> cost;
    info.alloc(nloc, st);
    cost.alloc(nloc, st);
    // ---- level-1 mode: wedge scatter (root-grouped C_R1 lists) when the roots'
    // 2-hop pools cost less than the per-task probes of the shorter adjacency slice
    DBuf<int64_t> l1_roff;
    DBuf<int32_t> l1_lists;
    int l1_mode = (cfg.flags & BC_FLAG_L1_SCATTER) ? 1 : (cfg.flags & BC_FLAG_L1_PROBE) ? 2 : 0;
    if (l1_mode == 0) {
      DBuf<unsigned long long> c2;
      c2.alloc(2, st);
      c2.zero();
      l1_probe_cost<<<sms * 8, 256, 0, st>>>(s.tasks.p, nloc, shard, nshards, s.hadj_off.p, c2.p);
      l1_pool<<<sms * 8, 256, 0, st>>>(s.aoff, s.aidx, s.boff, s.troot.p, s.n, c2.p + 1);
      BC_CHECK_LAUNCH();
      unsigned long long hc[2];
      copy_d2h(hc, c2.p, sizeof hc, st);
      BC_CUDA(cudaStreamSynchronize(st));
      launches += 2;
      // a probe is a bisect step chain (~4x a streamed id); the scatter walks each
      // pool ~4 times (count, mask, write, cursor)
      l1_mode = 4.0 * (double)hc[1] < 4.0 * (double)hc[0] ? 1 : 2;
      if (getenv("BC_DEBUG"))
        fprintf(stderr, "[bc level1] probe words %llu  pool %llu  -> %s\n", hc[0], hc[1],
                l1_mode == 1 ? "scatter" : "probe");
    }
    DbgTimer dt(st);
    if (l1_mode == 1) {
      const int64_t n = s.n;
      DBuf<int32_t> nunits, unit_first, unit_root;
      DBuf<int64_t> auxw, ubase;
      nunits.alloc(n + 1, st);
      auxw.alloc(n + 1, st);
      nunits.zero();
      auxw.zero();
      l1_root_sizes<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s.aoff, s.dir_off.p, s.troot.p, n,
                                                                 nunits.p, auxw.p);
      unit_first.alloc(n + 1, st);
      ubase.alloc(n + 1, st);
      scan_excl(nunits.p, unit_first.p, n + 1, st);
      scan_excl(auxw.p, ubase.p, n + 1, st);
      DBuf<unsigned long long> mx;
      mx.alloc(1, st);
      mx.zero();
      max_dir_len<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s.dir_off.p, n, mx.p);
      int32_t n_units = 0;
      int64_t aux_total = 0;
      unsigned long long maxD = 0;
      copy_d2h(&n_units, unit_first.p + n, sizeof n_units, st);
      copy_d2h(&aux_total, ubase.p + n, sizeof aux_total, st);
      copy_d2h(&maxD, mx.p, sizeof maxD, st);
      BC_CUDA(cudaStreamSynchronize(st));
      unit_root.alloc(n_units, st);
      l1_unit_roots<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(unit_first.p, n, unit_root.p);
      DBuf<unsigned long long> aux, nxt;
      aux.alloc(aux_total, st);
      aux.zero();
      nxt.alloc(2, st);
      nxt.zero();
      L1Args A1{};
      A1.aoff = s.aoff;
      A1.aidx = s.aidx;
      A1.boff = s.boff;
      A1.bidx = s.bidx;
      A1.doff = s.dir_off.p;
      A1.didx = s.dir_idx.p;
      A1.troot = s.troot.p;
      A1.unit_root = unit_root.p;
      A1.ubase = ubase.p;
      A1.unit_first = unit_first.p;
      A1.n_units = n_units;
      A1.aux = aux.p;
      A1.map_words = n <= 65536 ? (int)((n + 31) / 32) : 0;
      A1.shard = shard;
      A1.nshards = nshards;
      A1.next = nxt.p;
      const int l1w = L1_THREADS / 32;
      const size_t l1smem = (size_t)l1w * (A1.map_words + (A1.map_words + 1) / 2) * 4;
      int per_sm = 0;
      BC_CUDA(cudaFuncSetAttribute(l1_scatter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)l1smem));
      BC_CUDA(cudaFuncSetAttribute(l1_scatter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)l1smem));
      BC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, l1_scatter<true>, L1_THREADS,
                                                            l1smem));
      const int64_t l1blocks = (int64_t)sms * std::max(per_sm, 1);
      dt.mark("l1 setup");
      l1_scatter<false><<<(unsigned)l1blocks, L1_THREADS, l1smem, st>>>(A1);
      BC_CHECK_LAUNCH();
      dt.mark("l1 count");
      DBuf<int64_t> cnt;
      cnt.alloc(nloc + 1, st);
      cnt.zero();
      l1_task_totals<<<(unsigned)((nloc + 255) / 256), 256, 0, st>>>(
          s.tasks.p, nloc, shard, nshards, s.troot.p, ubase.p, unit_first.p, s.dir_off.p, aux.p,
          cnt.p);
      if (getenv("BC_CHECK_L1")) {
        DBuf<unsigned long long> bad;
        bad.alloc(1, st);
        bad.zero();
        l1_naive<<<(unsigned)((nloc + 255) / 256), 256, 0, st>>>(s.tasks.p, nloc, shard, nshards,
                                                                 s.aoff, s.aidx, cnt.p, bad.p);
        unsigned long long hb = 0;
        copy_d2h(&hb, bad.p, 8, st);
        BC_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "[bc level1] check: %llu of %lld task counts differ\n", hb, (long long)nloc);
      }
      l1_roff.alloc(nloc + 1, st);
      scan_excl(cnt.p, l1_roff.p, nloc + 1, st);
      int64_t n_entries = 0;
      copy_d2h(&n_entries, l1_roff.p + nloc, sizeof n_entries, st);
      BC_CUDA(cudaStreamSynchronize(st));
      l1_lists.alloc(n_entries, st);
      l1_cursors<<<(unsigned)((nloc + 255) / 256), 256, 0, st>>>(
          s.tasks.p, nloc, shard, nshards, s.troot.p, ubase.p, unit_first.p, s.dir_off.p,
          l1_roff.p, aux.p);
      DBuf<uint32_t> masks;
      A1.mask_stride = (int64_t)std::max<unsigned long long>(maxD, 1);
      masks.alloc((size_t)l1blocks * l1w * A1.mask_stride, st);
      masks.zero();
      A1.masks = masks.p;
      A1.lists = l1_lists.p;
      A1.next = nxt.p + 1;
      dt.mark("l1 offsets");
      l1_scatter<true><<<(unsigned)l1blocks, L1_THREADS, l1smem, st>>>(A1);
      BC_CHECK_LAUNCH();
      dt.mark("l1 fill");
      launches += 12;
      P.roff = l1_roff.p;
      P.lists = l1_lists.p;
      if (getenv("BC_DEBUG")) {
        BC_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "[bc level1] scatter: %d units, %lld aux, %lld C_R1 entries\n", n_units,
                (long long)aux_total, (long long)n_entries);
      }
    }
    {
      int64_t blocks = (nloc * 32 + 255) / 256;
      blocks = std::min<int64_t>(blocks, (int64_t)sms * 32);
      if (instr) level1_kernel<true><<<(unsigned)blocks, 256, 0, st>>>(P, info.p, cost.p);
      else level1_kernel<false><<<(unsigned)blocks, 256, 0, st>>>(P, info.p, cost.p);
      BC_CHECK_LAUNCH();
      dt.mark("level1_kernel");
      launches++;
    }
    BC_CUDA(cudaEventRecord(e1, st));
    if (s.p_eff >= 3) {
      unsigned long long h[CTR_COUNT];
      copy_d2h(h, ctr.p, sizeof h, st);
      BC_CUDA(cudaStreamSynchronize(st));
      n_alive = (int64_t)h[CTR_ALIVE];
      const int64_t max_ro = (int64_t)h[CTR_MAXRO], max_scr = (int64_t)h[CTR_MAXSCR];
      if (const char *dump = getenv("BC_DUMP_L1")) {  // development: Info + C_R1 lists
        std::vector<Info> hi(nloc);
        copy_d2h(hi.data(), info.p, nloc * sizeof(Info), st);
        std::vector<int64_t> ro;
        std::vector<int32_t> li;
        if (P.lists) {
          ro.resize(nloc + 1);
          copy_d2h(ro.data(), P.roff, (nloc + 1) * 8, st);
          BC_CUDA(cudaStreamSynchronize(st));
          li.resize(ro[nloc]);
          copy_d2h(li.data(), P.lists, ro[nloc] * 4, st);
        }
        BC_CUDA(cudaStreamSynchronize(st));
        if (FILE *fh = fopen(dump, "wb")) {
          int64_t n = nloc, nl = (int64_t)li.size();
          fwrite(&n, 8, 1, fh);
          fwrite(hi.data(), sizeof(Info), nloc, fh);
          fwrite(&nl, 8, 1, fh);
          if (nl) {
            fwrite(ro.data(), 8, nloc + 1, fh);
            fwrite(li.data(), 4, nl, fh);
          }
          fclose(fh);
        }
      }
      if (getenv("BC_LEVEL1_STATS")) {  // development: level-1 shape of the workload
        std::vector<Info> hi(nloc);
        copy_d2h(hi.data(), info.p, nloc * sizeof(Info), st);
        BC_CUDA(cudaStreamSynchronize(st));
        std::vector<int> crs, cls;
        double sum_lr = 0, sum_rowR = 0;
        for (const Info &x : hi)
          if (x.cl >= s.p_eff - 2 && x.cr >= s.q_eff) {
            crs.push_back(x.cr);
            cls.push_back(x.cl);
            sum_lr += (double)x.cl * x.cr;
            sum_rowR += (double)x.cl * ((x.cr + 31) / 32);
          }
        std::sort(crs.begin(), crs.end());
        std::sort(cls.begin(), cls.end());
        auto pct = [](const std::vector<int> &v, double f) {
          return v.empty() ? 0 : v[std::min(v.size() - 1, (size_t)(f * v.size()))];
        };
        float l1ms = 0;
        BC_CUDA(cudaEventRecord(e1, st));
        BC_CUDA(cudaEventSynchronize(e1));
        BC_CUDA(cudaEventElapsedTime(&l1ms, e0, e1));
        fprintf(stderr,
                "[bc level1] tasks %lld alive %lld  level1 %.3f ms  max_ro %lld max_scr %lld words\n"
                "  |C_R1| p50 %d p90 %d p99 %d max %d   |C_L1| p50 %d p90 %d p99 %d max %d\n"
                "  sum |C_L1||C_R1| %.4g  sum rowR words %.4g\n",
                (long long)nloc, (long long)n_alive, l1ms, (long long)max_ro, (long long)max_scr,
                pct(crs, .5), pct(crs, .9), pct(crs, .99), crs.empty() ? 0 : crs.back(),
                pct(cls, .5), pct(cls, .9), pct(cls, .99), cls.empty() ? 0 : cls.back(), sum_lr,
                sum_rowR);
        if (getenv("BC_LEVEL1_ONLY")) n_alive = 0;
      }
      if (n_alive > 0) {
        // pre-runtime LPT order: alive tasks by |C_L1|*|C_R1| descending
        DBuf<int32_t> ids, queue;
        DBuf<uint32_t> skeys;
        ids.alloc(nloc, st);
        queue.alloc(nloc, st);
        skeys.alloc(nloc, st);
        iota32<<<(unsigned)((nloc + 255) / 256), 256, 0, st>>>(ids.p, nloc);
        sort_pairs_desc(cost.p, skeys.p, ids.p, queue.p, nloc, st);
        launches += 2;
        EnumArgs A{};
        A.info = info.p;
        A.queue = queue.p;
        const bool split = allow_split && s.p_eff >= 5;
        if (!split) {
          // whole tasks per warp; frames in shared memory
          const bool lazy = s.p_eff == 4 && !has_rowL(s.p_eff, P.map_words);
          const int budget = env_int("BC_ENUM_BUDGET", 1200);
          const size_t smem = (size_t)wpb * (budget + map_w + LEAF_WORDS) * 4;
          auto kern = instr ? (lazy ? enum_kernel<true, true, false> : enum_kernel<true, false, false>)
                            : (lazy ? enum_kernel<false, true, false> : enum_kernel<false, false, false>);
          const int64_t blocks = (int64_t)sms * blocks_per_sm(kern, smem);
          A.q0 = 0;
          A.q1 = n_alive;
          A.budget_words = budget;
          DBuf<uint32_t> gs;
          if (max_ro + max_scr > budget) {
            A.gscratch_words = (max_ro + max_scr + 31) & ~int64_t(31);
            gs.alloc((size_t)blocks * wpb * A.gscratch_words, st);
            A.gscratch = gs.p;
          }
          kern<<<(unsigned)blocks, ENUM_THREADS, smem, st>>>(P, A);
          BC_CHECK_LAUNCH();
          launches++;
        } else {
          // triage (p_eff >= 5): every task is started whole by one warp; a task with
          // at most T level-1 R-survivors (whose frame fits the scratch) finishes in
          // place, the rest are deferred, heaviest first, to the split path below.
          int64_t n_heavy = n_alive;
          const int32_t *hq_p = queue.p;
          DBuf<int32_t> heavy, hq;
          const int T = env_int("BC_TRIAGE", 32);
          if (T > 0) {
            const int budget = env_int("BC_TRIAGE_BUDGET", 1536);
            const size_t smem = (size_t)wpb * (budget + map_w + LEAF_WORDS) * 4;
            auto kern = instr ? enum_kernel<true, false, false> : enum_kernel<false, false, false>;
            const int64_t blocks = (int64_t)sms * blocks_per_sm(kern, smem);
            heavy.alloc(n_alive, st);
            EnumArgs B = A;
            B.q0 = 0;
            B.q1 = n_alive;
            B.budget_words = budget;
            B.triage = T;
            B.heavy = heavy.p;
            DBuf<uint32_t> gs;
            if (max_ro + max_scr > budget) {
              // per-warp frame scratch, capped at 4 GiB in total (larger frames defer)
              int64_t w = (max_ro + max_scr + 31) & ~int64_t(31);
              const int64_t cap_w = ((int64_t(1) << 30) / (blocks * wpb)) & ~int64_t(31);
              B.gscratch_words = std::min(w, cap_w);
              gs.alloc((size_t)blocks * wpb * B.gscratch_words, st);
              B.gscratch = gs.p;
            }
            BC_CUDA(cudaMemsetAsync(ctr.p + CTR_NEXT, 0, 8, st));
            dt.mark("pre-triage");
            kern<<<(unsigned)blocks, ENUM_THREADS, smem, st>>>(P, B);
            BC_CHECK_LAUNCH();
            dt.mark("triage");
            launches++;
            unsigned long long hn = 0;
            copy_d2h(&hn, ctr.p + CTR_HEAVY, sizeof hn, st);
            BC_CUDA(cudaStreamSynchronize(st));
            n_heavy = (int64_t)hn;
            if (n_heavy > 0) {  // deferred tasks in LPT order again (deterministic)
              DBuf<uint32_t> hk, hk2;
              hk.alloc(n_heavy, st);
              hk2.alloc(n_heavy, st);
              hq.alloc(n_heavy, st);
              gather_keys<<<(unsigned)((n_heavy + 255) / 256), 256, 0, st>>>(heavy.p, n_heavy,
                                                                              cost.p, hk.p);
              sort_pairs_desc(hk.p, hk2.p, heavy.p, hq.p, n_heavy, st);
              launches += 2;
            }
            hq_p = hq.p;
          }
          A.queue = hq_p;
          if (n_heavy > 0) {
          // split mode (p_eff >= 5): chunks of the LPT queue; per chunk, enum_kernel
            // writes every frame to the frame arena and pushes the split-level nodes,
            // then sub_kernel drains them heaviest first with every warp.
            const int split_level = s.p_eff <= 6 ? 2 : 3;
            const int budget = env_int("BC_SPLIT_BUDGET", 1024);
            const size_t smem = (size_t)wpb * (budget + map_w + LEAF_WORDS) * 4;
            auto kern = instr ? enum_kernel<true, false, true> : enum_kernel<false, false, true>;
            auto sk = instr ? sub_kernel<true> : sub_kernel<false>;
            const size_t ssmem = (size_t)wpb * (budget + LEAF_WORDS) * 4;
            const int64_t blocks = (int64_t)sms * blocks_per_sm(kern, smem);
            const int64_t sblocks = std::min<int64_t>((int64_t)sms * blocks_per_sm(sk, ssmem), blocks);
            A.budget_words = budget;
            DBuf<uint32_t> gs;
            if (max_scr > budget) {
              A.gscratch_words = (max_scr + 31) & ~int64_t(31);
              gs.alloc((size_t)blocks * wpb * A.gscratch_words, st);
              A.gscratch = gs.p;
            }
            const int64_t arena_limit = int64_t(1) << 28;  // words per arena (1 GiB)
            DBuf<int64_t> ro, sub, foff, soff;
            ro.alloc(n_heavy + 1, st);
            sub.alloc(n_heavy + 1, st);
            foff.alloc(n_heavy + 1, st);
            soff.alloc(n_heavy + 1, st);
            ro.zero();
            sub.zero();
            split_sizes<<<(unsigned)((n_heavy + 255) / 256), 256, 0, st>>>(
                info.p, hq_p, 0, n_heavy, instr, split_level, ro.p, sub.p);
            scan_excl(ro.p, foff.p, n_heavy + 1, st);
            scan_excl(sub.p, soff.p, n_heavy + 1, st);
            std::vector<int64_t> hf(n_heavy + 1), hs(n_heavy + 1);
            copy_d2h(hf.data(), foff.p, (n_heavy + 1) * 8, st);
            copy_d2h(hs.data(), soff.p, (n_heavy + 1) * 8, st);
            BC_CUDA(cudaStreamSynchronize(st));
            launches += 3;
            int64_t q0 = 0;
            while (q0 < n_heavy) {
              // grow the chunk while both arenas stay under the limit
              int64_t q1 = q0 + 1;
              {
                int64_t lo = q0 + 1, hi = n_heavy;
                while (lo < hi) {
                  const int64_t mid = (lo + hi + 1) / 2;
                  if (hf[mid] - hf[q0] <= arena_limit && hs[mid] - hs[q0] <= arena_limit) lo = mid;
                  else hi = mid - 1;
                }
                q1 = lo;
              }
              const int64_t fw = hf[q1] - hf[q0];
              const int64_t sw = std::max<int64_t>(hs[q1] - hs[q0], 8);
              DBuf<uint32_t> frames, arena;
              DBuf<unsigned long long> index;
              DBuf<int64_t> local_off;
              frames.alloc(fw, st);
              arena.alloc(sw, st);
              const int64_t cap = sw / 6 + 1;
              index.alloc(cap, st);
              local_off.alloc(q1 - q0, st);
              // frame offsets relative to the chunk
              {
                std::vector<int64_t> lo_off(q1 - q0);
                for (int64_t i = q0; i < q1; i++) lo_off[i - q0] = hf[i] - hf[q0];
                copy_h2d(local_off.p, lo_off.data(), (q1 - q0) * 8, st);
              }
              BC_CUDA(cudaMemsetAsync(ctr.p + CTR_NEXT, 0, 8, st));
              BC_CUDA(cudaMemsetAsync(ctr.p + CTR_SUB_USED, 0, 8, st));
              BC_CUDA(cudaMemsetAsync(ctr.p + CTR_SUB_N, 0, 8, st));
              BC_CUDA(cudaMemsetAsync(ctr.p + CTR_SUB_NEXT, 0, 8, st));
              A.q0 = q0;
              A.q1 = q1;
              A.frames = frames.p;
              A.frame_off = local_off.p;
              A.sink.arena = arena.p;
              A.sink.arena_words = sw;
              A.sink.index = index.p;
              A.sink.index_cap = cap;
              A.sink.level = split_level;
              kern<<<(unsigned)blocks, ENUM_THREADS, smem, st>>>(P, A);
              BC_CHECK_LAUNCH();
              unsigned long long hn = 0;
              copy_d2h(&hn, ctr.p + CTR_SUB_N, sizeof hn, st);
              BC_CUDA(cudaStreamSynchronize(st));
              const int64_t n_sub = std::min<int64_t>((int64_t)hn, cap);
              launches += 1;
              if (n_sub > 0) {
                DBuf<uint32_t> k0, k1;
                DBuf<unsigned long long> v1;
                k0.alloc(n_sub, st);
                k1.alloc(n_sub, st);
                DBuf<unsigned long long> v0;
                v0.alloc(n_sub, st);
                v1.alloc(n_sub, st);
                sub_keys<<<(unsigned)((n_sub + 255) / 256), 256, 0, st>>>(arena.p, index.p, n_sub,
                                                                        info.p, k0.p, v0.p);
                sort_pairs_desc(k0.p, k1.p, v0.p, v1.p, n_sub, st);
                A.sub_order = v1.p;
                sk<<<(unsigned)sblocks, ENUM_THREADS, ssmem, st>>>(P, A, n_sub);
                BC_CHECK_LAUNCH();
                launches += 3;
              }
              n_sub_total += n_sub;
              q0 = q1;
            }
          }
          dt.mark("split");
          if (dt.on) fprintf(stderr, "[bc search] alive %lld heavy %lld\n", (long long)n_alive,
                             (long long)n_heavy);
          n_split = n_heavy;
        }
      }
    }
  } else {
    BC_CUDA(cudaEventRecord(e1, st));
  }
  BC_CUDA(cudaEventRecord(e2, st));
  unsigned long long h_acc[2], h_ctr[CTR_COUNT];
  int h_ovf = 0;
  copy_d2h(h_acc, acc.p, sizeof h_acc, st);
  copy_d2h(h_ctr, ctr.p, sizeof h_ctr, st);
  copy_d2h(&h_ovf, ovf.p, sizeof h_ovf, st);
  if (want_tc) copy_d2h(cfg.task_counts, tcounts.p, 2 * n_tasks * sizeof(uint64_t), st);
  BC_CUDA(cudaStreamSynchronize(st));
  float t1 = 0, t2 = 0;
  BC_CUDA(cudaEventElapsedTime(&t1, e0, e1));
  BC_CUDA(cudaEventElapsedTime(&t2, e1, e2));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  if (h_ovf == 2) throw Error(BC_ECUDA, "enumeration frame exceeded its scratch sizing");
  out.count_lo = h_acc[0];
  out.count_hi = h_acc[1];
  out.overflow = h_ovf ? 1 : 0;
  out.tasks_consumed = nloc;
  out.tasks_alive = n_alive;
  out.tasks_split = n_split;
  out.tasks_stolen = (int64_t)h_ctr[CTR_STOLEN];
  out.batches_executed = (s.p_eff >= 2 ? nloc : 0) + (int64_t)h_ctr[CTR_BATCHES];
  out.intersections = (int64_t)h_ctr[CTR_INTER];
  out.operand_words = (int64_t)h_ctr[CTR_OPW];
  out.min_words = (int64_t)h_ctr[CTR_MINW];
  out.time_level1 = t1 * 1e-3;
  out.time_enum = t2 * 1e-3;
  out.kernel_launches += launches;
  (void)n_sub_total;
}

}  // namespace bc
