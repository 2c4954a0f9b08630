// search_dev.cuh -- device side of the enumeration, shared by search.cu (level 1,
// orchestration) and the two instantiation units enum_plain.cu / enum_compact.cu
// (candidate rows probed for every x, or wedge-scattered for the level-1
// survivors only: COMPACT).  Types live in bc::sk so launchers can be declared
// across units; each kernel instantiation is compiled in exactly one unit.
#pragma once
#include <climits>

// Loops over task-local words and lists run a handful of iterations (C_R1 / C_L1 are a
// few words): compiler unrolling only multiplies the code of kernels whose hot set
// already exceeds the instruction cache (ncu: no_instruction was 65% of C5 sub_kernel's
// stall samples), so loops are kept rolled unless marked otherwise.
#ifndef BC_UNROLL_DEFAULT
#define BC_LOOP _Pragma("unroll 1")
#else
#define BC_LOOP
#endif

#include "engine.h"

namespace bc {
namespace sk {

// Per-phase SM-cycle tallies (lane 0 of every warp) in -DBC_PHASE_PROF builds:
// 0 claim, 1 level-1 re-materialisation, 2 decode + slot map, 3 rows,
// 4 expansions, 5 leaf-parents, 6 finish.
#ifdef BC_PHASE_PROF
static __device__ unsigned long long g_phase[16];  // one copy per unit
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
    BC_LOOP
    for (int i = 0; i < 8; i++) t[i] = 0;
  }
  __device__ __forceinline__ void mark(int i) {
    const long long n = clk();
    t[i] += (unsigned long long)(n - last);
    last = n;
  }
  __device__ __forceinline__ void flush() {
    if ((threadIdx.x & 31) == 0)
      BC_LOOP
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
  int64_t n_local;  // tasks of this shard
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
  const int64_t *__restrict__ ltask;    // root sharding: global id of local task j (or null:
                                        //   task interleave t = shard + j * nshards)
  unsigned *claims;                     // optional [n_tasks]: claims per task (track_tasks)
  // root-restricted rows (wedge-scatter level 1; roffE null: not built, lists hold ids and
  // the wedge walks read the whole rows N(v)).  With them, C_R1 list entry i of task (r, s)
  // is the rank-local index e of the edge (r, v): v = csr_aidx[csr_aoff[r] - rebase[r] + e]
  // and R(r, v) = N(v) & dir2(r) is rrows[roffE[e], roffE[e + 1])
  const int64_t *__restrict__ roffE;
  const int64_t *__restrict__ rebase;   // per root: its first edge index
  const int64_t *__restrict__ csr_aoff; // anchor -> opposite CSR (work graph)
  const int32_t *__restrict__ csr_aidx;
  const int32_t *__restrict__ rrows;   // R(r, v) entries: rank-order positions in dir2(r)
  const int32_t *__restrict__ rdir;    // dir2(r) in rank order at dir_off[r] (position -> id)
  const int32_t *__restrict__ rpos;    // dir2 entry (id order) -> its rank-order position
  const int64_t *__restrict__ dir_off; // plain dir2 list offsets
  const int64_t *__restrict__ troot;   // first task of each root
};

// global task id of this shard's local task j
__host__ __device__ __forceinline__ int64_t task_id(const int64_t *ltask, int shard, int nshards,
                                                    int64_t j) {
  return ltask ? ltask[j] : shard + j * (int64_t)nshards;
}

enum { CTR_ALIVE = 0, CTR_BATCHES, CTR_STOLEN, CTR_INTER, CTR_OPW, CTR_MINW, CTR_MAXRO,
       CTR_MAXSCR, CTR_SPILL, CTR_NEXT, CTR_SUB_USED, CTR_SUB_N, CTR_SUB_NEXT, CTR_SPLIT,
       CTR_HEAVY, CTR_OPW_L1, CTR_CONSUMED, CTR_NEST_BAD, CTR_NEST_CHECKED, CTR_COUNT };

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
  BC_LOOP
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
// former from global memory.
//
// Candidate rows exist for the level-1 R-survivors (x with |N(x) & C_R1| >= q)
// only: every candidate whose rowL (or, in compact mode, rowR) is read has
// passed |R & N(x)| >= q at some node, and R is a subset of C_R1, so it passed
// at level 1 too; lslot[x] is its row (-1: none, which reads as |R & N(x)| = 0
// < q).  In full mode (probe-built rows) rowR has a row for every x.
struct FrameSpec {
  bool rowL;     // rowL rows for the survivors
  bool compact;  // rowR rows for the survivors only (scatter-built)
  bool instr;    // adj / dir2 slice lengths for the B_enum tallies
  int cap;       // > 0: at most cap survivors (triage), else nL
  __host__ __device__ __forceinline__ int64_t rows(int nL) const {
    return cap > 0 && cap < nL ? cap : nL;
  }
  __host__ __device__ __forceinline__ bool lslot() const { return rowL || compact; }
};

struct Frame {
  // two bases and 32-bit word offsets (frames are far below 2^31 words): row and set
  // addresses are one 32-bit multiply-add and one wide add, not 64-bit pointer math
  uint32_t *ro;  // read-only part (built once; split tasks share it from the arena)
  uint32_t *sc;  // per-warp DFS scratch
  int o_r_idx, o_r_val, o_r_pre, o_l_idx, o_l_val, o_l_pre, o_r_last, o_l_last, o_s1, o_s1h, o_lids, o_lslot, o_rids, o_rowR, o_rowL, o_adjw, o_dirw;
  int o_cand, o_setR, o_setL, o_surv, o_ns, o_cur;
  int surv_cap;
  bool compact;
  // every node of this task fits one reference batch (|C_L1| * max(words) <= capacity, or
  // dfs mode): node_batches then needs no HTB word counts, so they are not computed
  bool skip_words;
  __device__ __forceinline__ uint32_t *r_idx() const { return (uint32_t *)(ro + o_r_idx); }
  __device__ __forceinline__ uint32_t *r_val() const { return (uint32_t *)(ro + o_r_val); }
  __device__ __forceinline__ int *r_pre() const { return (int *)(ro + o_r_pre); }
  __device__ __forceinline__ uint32_t *l_idx() const { return (uint32_t *)(ro + o_l_idx); }
  __device__ __forceinline__ uint32_t *l_val() const { return (uint32_t *)(ro + o_l_val); }
  __device__ __forceinline__ int *l_pre() const { return (int *)(ro + o_l_pre); }
  __device__ __forceinline__ uint32_t *r_last() const { return (uint32_t *)(ro + o_r_last); }
  __device__ __forceinline__ uint32_t *l_last() const { return (uint32_t *)(ro + o_l_last); }
  __device__ __forceinline__ uint32_t *s1() const { return (uint32_t *)(ro + o_s1); }
  __device__ __forceinline__ uint32_t *s1h() const { return (uint32_t *)(ro + o_s1h); }
  __device__ __forceinline__ int *lids() const { return (int *)(ro + o_lids); }
  __device__ __forceinline__ int *lslot() const { return (int *)(ro + o_lslot); }
  __device__ __forceinline__ int *rids() const { return (int *)(ro + o_rids); }
  __device__ __forceinline__ uint32_t *rowR() const { return (uint32_t *)(ro + o_rowR); }
  __device__ __forceinline__ uint32_t *rowL() const { return (uint32_t *)(ro + o_rowL); }
  __device__ __forceinline__ int *adjw() const { return (int *)(ro + o_adjw); }
  __device__ __forceinline__ int *dirw() const { return (int *)(ro + o_dirw); }
  __device__ __forceinline__ int *cand() const { return (int *)(sc + o_cand); }
  __device__ __forceinline__ uint32_t *setR() const { return (uint32_t *)(sc + o_setR); }
  __device__ __forceinline__ uint32_t *setL() const { return (uint32_t *)(sc + o_setL); }
  __device__ __forceinline__ int *surv() const { return (int *)(sc + o_surv); }
  __device__ __forceinline__ int *ns() const { return (int *)(sc + o_ns); }
  __device__ __forceinline__ int *cur() const { return (int *)(sc + o_cur); }
};

// rowL is materialised for p_eff >= 5 (reused at every depth) and for p_eff = 4
// without a slot map; p_eff = 4 with a map walks dir2(u) lazily instead.
__host__ __device__ __forceinline__ bool has_rowL(int p_eff, int map_words) {
  return p_eff >= 5 || (p_eff == 4 && map_words == 0);
}

__host__ __device__ __forceinline__ int64_t ro_words(int nR, int nL, int wR, int wL,
                                                     const FrameSpec &sp) {
  const int64_t WR = (nR + 31) / 32, WL = (nL + 31) / 32;
  int64_t w = 3 * (int64_t)wR + 1 + 3 * (int64_t)wL + 1;  // C_R1 / C_L1 HTB words + prefixes
  w += WR + WL;                                            // r_last, l_last
  if (sp.compact) w += WL + wL;                            // s1, s1h
  if (!sp.compact) w += nL;                                // lids (compact: lid_of)
  if (sp.lslot()) w += nL;                                 // lslot
  if (sp.compact) w += nR;                                 // rids (C_R1 members)
  w += (sp.compact ? sp.rows(nL) : nL) * WR;               // rowR
  if (sp.rowL) w += sp.rows(nL) * WL;                      // rowL
  if (sp.instr) w += 2 * (int64_t)nL;                      // adj / dir2 slice words
  return (w + 3) & ~int64_t(3);
}

// frame words whichever row mode the launch uses (sizing before the choice)
__host__ __device__ __forceinline__ int64_t ro_words_any(int nR, int nL, int wR, int wL,
                                                         FrameSpec sp) {
  sp.compact = false;
  const int64_t a = ro_words(nR, nL, wR, wL, sp);
  sp.compact = true;
  const int64_t b = ro_words(nR, nL, wR, wL, sp);
  return a > b ? a : b;
}

// DFS stack: nodes at levels 1 .. p_eff-3 are expanded warp-cooperatively
// (leaf-parents at p_eff-2 are finished lane-parallel without a frame).
__host__ __device__ __forceinline__ int stack_levels(int p_eff) {
  return p_eff - 3 > 1 ? p_eff - 3 : 1;
}

// survivors listed per level are level-1 R-survivors: bounded by nL or the cap
__host__ __device__ __forceinline__ int64_t scratch_words(int nR, int nL, int p_eff,
                                                          const FrameSpec &sp) {
  const int64_t WR = (nR + 31) / 32, WL = (nL + 31) / 32;
  const int64_t levels = stack_levels(p_eff);
  return ((int64_t)nL + levels * (WR + WL + sp.rows(nL) + 2) + 3) & ~int64_t(3);
}

__device__ __forceinline__ void carve_ro(Frame &f, uint32_t *p, const Dims &d,
                                         const FrameSpec &sp) {
  int o = 0;
  f.ro = p;
  f.o_r_idx = o; o += d.wR;
  f.o_r_val = o; o += d.wR;
  f.o_r_pre = o; o += d.wR + 1;
  f.o_l_idx = o; o += d.wL;
  f.o_l_val = o; o += d.wL;
  f.o_l_pre = o; o += d.wL + 1;
  f.o_r_last = o; o += d.WR;
  f.o_l_last = o; o += d.WL;
  f.o_s1 = o; if (sp.compact) o += d.WL;
  f.o_s1h = o; if (sp.compact) o += d.wL;
  f.o_lids = o; if (!sp.compact) o += d.nL;
  f.o_lslot = o; if (sp.lslot()) o += d.nL;
  f.o_rids = o; if (sp.compact) o += d.nR;
  f.o_rowR = o; o += (int)(sp.compact ? sp.rows(d.nL) : d.nL) * d.WR;
  f.o_rowL = o; if (sp.rowL) o += (int)sp.rows(d.nL) * d.WL;
  f.o_adjw = o; if (sp.instr) o += d.nL;
  f.o_dirw = o;
  f.compact = sp.compact;
  f.skip_words = false;
}

// set once per task (frame or sub-task) in non-instrumented launches: a node's candidates
// are a subset of C_L1 and its word counts at most C_R1's / C_L1's, so node_batches is
// (ncand > 0) whenever |C_L1| * max(words(C_R1), words(C_L1), 1) fits the capacity
__device__ __forceinline__ void set_skip_words(Frame &f, const Params &P, const Dims &d, bool instr) {
  const int64_t wm = d.wR > d.wL ? (d.wR > 1 ? d.wR : 1) : (d.wL > 1 ? d.wL : 1);
  f.skip_words = !instr && (P.mode_dfs || (int64_t)d.nL * wm <= (int64_t)P.cap);
}

__device__ __forceinline__ void carve_scratch(Frame &f, uint32_t *p, const Dims &d, int p_eff,
                                              const FrameSpec &sp) {
  const int levels = stack_levels(p_eff);
  f.surv_cap = (int)sp.rows(d.nL);
  int o = 0;
  f.sc = p;
  f.o_cand = o; o += d.nL;
  f.o_setR = o; o += levels * d.WR;
  f.o_setL = o; o += levels * d.WL;
  f.o_surv = o; o += levels * f.surv_cap;
  f.o_ns = o; o += levels;
  f.o_cur = o;
}

__device__ __forceinline__ const uint32_t *rowL_of(const Frame &f, const Dims &d, int u) {
  return f.ro + (f.o_rowL + f.lslot()[u] * d.WL);
}

// anchor id of C_L1 local index x: decoded list (full mode) or, in compact mode,
// the word holding x (bisect on the prefix counts) and its bit of that rank
__device__ __forceinline__ int lid_of(const Frame &f, const Dims &d, int x) {
  if (!f.compact) return f.lids()[x];
  int lo = 0, hi = d.wL - 1;
  BC_LOOP
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (f.l_pre()[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return (int)f.l_idx()[lo] * 32 + (int)__fns(f.l_val()[lo], 0, x - f.l_pre()[lo] + 1);
}

// rowR of candidate u, or null when u has no row (not a level-1 R-survivor)
__device__ __forceinline__ const uint32_t *rowR_of(const Frame &f, const Dims &d, int u) {
  if (!f.compact) return f.ro + (f.o_rowR + u * d.WR);
  const int sl = f.lslot()[u];
  return sl >= 0 ? f.ro + (f.o_rowR + sl * d.WR) : nullptr;
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
    BC_LOOP
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
    BC_LOOP
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
    BC_LOOP
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
    BC_LOOP
    for (; k < ns; k++) {
      const uint32_t m = s_val[k] & __ldg(dense_row + s_idx[k]);
      if (m) rw.add(s_pre[k], s_val[k], m);
    }
  } else if (ns <= g1 - g0) {
    int64_t lo = g0;
    BC_LOOP
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
    BC_LOOP
    for (int64_t j = g0; j < g1; j++) {
      const uint32_t key = __ldg(gidx + j);
      int a = lo, b = ns;
      BC_LOOP
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
  BC_LOOP
  for (int64_t j = g0; j < g1; j++) {
    const int k = map[__ldg(gidx + j)];
    if (k != 0xffff) {
      const uint32_t m = l_val[k] & __ldg(gval + j);
      if (m) rw.add(l_pre[k], l_val[k], m);
    }
  }
  rw.finish();
}

// Number of original HTB words a local bitset touches (the reference's word count
// of the node's set, engine.py:306-313), warp-parallel over the W local words with
// the field trick of lane_words below.  A field (one HTB word's local indices) has
// at most 32 bits, so it spans at most two words and a word's carry-out depends on
// that word alone: each lane forms its carry-out, the next lane takes it as carry-in.
__device__ __forceinline__ int words_touched(const uint32_t *set, const uint32_t *last, int W) {
  const int lane = lane_id();
  int c = 0;
  unsigned long long cin_chunk = 0;
  BC_LOOP
  for (int w0 = 0; w0 < W; w0 += 32) {
    const int w = w0 + lane;
    const uint32_t x = w < W ? set[w] : 0u, L = w < W ? last[w] : FULL;
    const unsigned long long base = (unsigned long long)(x & ~L) + (unsigned long long)(~L);
    const unsigned long long cout = base >> 32;
    unsigned long long cin = __shfl_up_sync(FULL, cout, 1);
    if (lane == 0) cin = cin_chunk;
    c += __popc(((uint32_t)(base + cin) | x) & L);
    cin_chunk = __shfl_sync(FULL, cout, 31);
  }
  return __reduce_add_sync(FULL, c);
}

// Same count for X = R & ru, by one lane, in O(W) words: the local indices of
// one HTB word form a field ending at a `last` bit; (X & ~last) + ~last, added
// across words with carry, sets a field's last bit iff its low bits are non-zero
// and never carries out of a field, so the touched fields are
// popc(((X & ~last) + ~last | X) & last).
__device__ __forceinline__ int lane_words(const uint32_t *R, const uint32_t *ru,
                                          const uint32_t *last, int W,
                                          const uint32_t *ru2 = nullptr) {
  int c = 0;
  unsigned long long carry = 0;
  BC_LOOP
  for (int w = 0; w < W; w++) {
    const uint32_t x = R[w] & ru[w] & (ru2 ? ru2[w] : FULL), L = last[w];
    const unsigned long long sum = (unsigned long long)(x & ~L) + (unsigned long long)(~L) + carry;
    carry = sum >> 32;
    c += __popc(((uint32_t)sum | x) & L);
  }
  return c;
}

// order-preserving compaction of the set bits of a W-word set into cand[]
__device__ __forceinline__ int compact_bits(const uint32_t *set, int W, int *cand) {
  const int lane = lane_id();
  int n = 0;
  BC_LOOP
  for (int w0 = 0; w0 < W; w0 += 32) {
    const uint32_t mine = w0 + lane < W ? set[w0 + lane] : 0u;
    unsigned nz = __ballot_sync(FULL, mine != 0);
    BC_LOOP
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

// compact_bits of set & filter
__device__ __forceinline__ int compact_bits_and(const uint32_t *set, const uint32_t *filter, int W,
                                                int *cand) {
  const int lane = lane_id();
  int n = 0;
  BC_LOOP
  for (int w0 = 0; w0 < W; w0 += 32) {
    const uint32_t mine = w0 + lane < W ? set[w0 + lane] & filter[w0 + lane] : 0u;
    unsigned nz = __ballot_sync(FULL, mine != 0);
    BC_LOOP
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

// several batches: the divisions stay out of line (one copy, off the hot path)
static __device__ __noinline__ unsigned node_batches_div(unsigned ncand, unsigned wm, unsigned cap) {
  unsigned b = cap / wm;
  if (b < 1) b = 1;
  return (ncand + b - 1) / b;
}

// reference batch count for one node expansion (engine.py:306-313, 329-331)
__device__ __forceinline__ unsigned node_batches(const Params &P, unsigned ncand, int wr, int wl,
                                                 bool leaf) {
  if (!ncand) return 0;
  if (P.mode_dfs) return ncand;
  const unsigned cap = (unsigned)P.cap;
  const unsigned w = (unsigned)(wr > 1 ? wr : 1), w2 = leaf ? 1u : (unsigned)(wl > 1 ? wl : 1);
  const unsigned wm = w > w2 ? w : w2;  // b = cap / max(wr, wl)
  if ((unsigned long long)ncand * wm <= cap) return 1;  // one batch: no division
  return node_batches_div(ncand, wm, cap);
}

// Per-warp shared-memory staging of (leaf-parent slot, leaf) pairs.
constexpr int RP_WORDS = 2;  // leaf-parent R' words kept in registers

struct LeafBuf {
  int *wr;     // [32]: C_R word count of each slot's leaf-parent
  int *ncand;  // [32]: leaves of each slot's leaf-parent (batch accounting)
  int *pu, *pw;  // [64] each: (child, grandchild) leaf-parent pairs awaiting evaluation
};
constexpr int LEAF_WORDS = 64 + 128;  // per-warp leaf-parent bookkeeping in shared memory

// Evaluate one round of leaves (engine.py:342-347): lane i offers the present bits m
// of an HTB-style word (v, pre) for leaf-parent `slot`; all offered leaves, as one
// flattened list, are spread over the 32 lanes (owner lane by a shuffle bisection
// over the exclusive popcount prefix, leaf = that lane's k-th set bit), and each
// adds C(|R & rowR[u] & rowR[w]|, q).
template <bool INSTR>
__device__ __forceinline__ void eval_leaves(const Params &P, const Frame &f, const Dims &d,
                                            const uint32_t *R, const int *slot_u, int slot,
                                            uint32_t v, int pre, uint32_t m, int wr,
                                            const uint32_t (&rp)[RP_WORDS], Acc128 &acc,
                                            Tally &tl) {
  const int lane = lane_id();
  const int cnt = __popc(m);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += t;
  }
  const int excl = incl - cnt;
  const int total = __shfl_sync(FULL, incl, 31);
  const int WR = d.WR;
  BC_LOOP
  for (int r0 = 0; r0 < total; r0 += 32) {
    const int k = r0 + lane;
    int o = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
      const int c = o + step;
      const int e = __shfl_sync(FULL, excl, c < 32 ? c : 31);
      if (c < 32 && e <= k) o = c;
    }
    const int so = __shfl_sync(FULL, slot, o);
    const uint32_t vo = __shfl_sync(FULL, v, o), mo = __shfl_sync(FULL, m, o);
    const int po = __shfl_sync(FULL, pre, o), eo = __shfl_sync(FULL, excl, o);
    const int wro = INSTR ? __shfl_sync(FULL, wr, o) : 0;
    // R & rowR[u] of the leaf-parent, held in its lane's registers when it is short
    uint32_t pr[RP_WORDS];
#pragma unroll
    for (int x = 0; x < RP_WORDS; x++) pr[x] = x < WR ? __shfl_sync(FULL, rp[x], so) : 0u;
    if (k < total) {
      const int b = (int)__fns(mo, 0, k - eo + 1);
      const int w = po + __popc(vo & ((1u << b) - 1u));
      const uint32_t *rw = rowR_of(f, d, w);
      int c = 0;
      if (rw) {
        if (WR <= RP_WORDS) {
#pragma unroll
          for (int x = 0; x < RP_WORDS; x++)
            if (x < WR) c += __popc(pr[x] & rw[x]);
        } else {
          const uint32_t *ru = rowR_of(f, d, slot_u[so]);
          BC_LOOP
          for (int x = 0; x < WR; x++) c += __popc(R[x] & ru[x] & rw[x]);
        }
      }
      if (INSTR) {
        tl.inter++;
        tl.opw += wro + f.adjw()[w];
        tl.minw += wro < f.adjw()[w] ? wro : f.adjw()[w];
      }
      if (c >= P.q_eff) add_comb(P, acc, c);
    }
  }
}

// Leaf-parent nodes, 32 at a time (one slot per lane): node u (a survivor
// of the node at `level`) has R' = R & rowR[u] and L' = L & rowL[u] -- or,
// with LAZY (p_eff = 4, level 1), L' = dir2(u) & C_L1 read through the slot
// map -- and its children are leaves (engine.py:342-347).  The L' words of
// the 32 leaf-parents are walked as one flattened stream (LAZY: every lane
// loads a different dir2 word each round, so the gathers overlap), and each
// round's leaves are spread over the lanes (eval_leaves).
template <bool INSTR, bool LAZY>
__device__ __forceinline__ void leaf_parents(const Params &P, const Frame &f, const Dims &d,
                                             int level, const int *list, int n,
                                             const uint16_t *map, const LeafBuf &lb, Acc128 &acc,
                                             Tally &tl, const int *list2 = nullptr) {
  const int lane = lane_id();
  const int WR = d.WR, WL = d.WL;
  const uint32_t *R = f.setR() + (level - 1) * WR;
  const uint32_t *Ls = f.setL() + (level - 1) * WL;
  BC_LOOP
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const bool act = i < n;
    const int u = act ? list[i] : 0;
    const uint32_t *ru_mine = act ? rowR_of(f, d, u) : nullptr;
    const uint32_t *ru2 = act && list2 ? rowR_of(f, d, list2[i]) : nullptr;
    const int wr = act ? (f.skip_words ? 1 : lane_words(R, ru_mine, f.r_last(), WR, ru2)) : 0;
    uint32_t rp[RP_WORDS];
#pragma unroll
    for (int x = 0; x < RP_WORDS; x++)
      rp[x] = act && x < WR ? R[x] & ru_mine[x] & (ru2 ? ru2[x] : FULL) : 0u;
    lb.wr[lane] = wr;
    lb.ncand[lane] = 0;
    __syncwarp();
    if (LAZY) {
      int64_t start = 0;
      int len = 0;
      if (act) {
        const int id = lid_of(f, d, u);
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
      BC_LOOP
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
            v = f.l_val()[k];
            m = v & dv;
            pre = f.l_pre()[k];
            if (m) atomicAdd(&lb.ncand[sl], __popc(m));
            if (!INSTR && f.compact) m &= f.s1h()[k];  // non-survivor leaves add 0
          }
        }
        eval_leaves<INSTR>(P, f, d, R, list + base, sl, v, pre, m, lb.wr[sl], rp, acc, tl);
      }
    } else {
      int ncand = 0;
      const uint32_t *rl = act ? rowL_of(f, d, u) : f.rowL();
      const uint32_t *rl2 = act && list2 ? rowL_of(f, d, list2[i]) : nullptr;
      BC_LOOP
      for (int x = 0; __any_sync(FULL, act && x < WL); x++) {
        uint32_t m = 0;
        if (act && x < WL) m = Ls[x] & rl[x] & (rl2 ? rl2[x] : FULL);
        ncand += __popc(m);
        if (!INSTR && f.compact) m &= f.s1()[x];
        if (__any_sync(FULL, m != 0u))  // a word with no leaf anywhere in the warp: skip
          eval_leaves<INSTR>(P, f, d, R, list + base, lane, 0xffffffffu, x * 32, m, wr, rp, acc,
                             tl);
      }
      lb.ncand[lane] = ncand;
    }
    if (act) tl.batches += node_batches(P, (unsigned)lb.ncand[lane], wr, 0, true);
    __syncwarp();
  }
}

// Expand all children of the node at `level` at once when its grandchildren are
// leaf-parents (engine.py:315-374 applied to each child): a child u has
// R_u = R & rowR[u] (<= RP_WORDS words, in its lane's registers) and
// L_u = L & rowL[u]; the candidates w of 32 children are one flattened list over
// the lanes (owner bisection as in eval_leaves), each tested for
// |R_u & rowR[w]| >= q and |L_u & rowL[w]| >= p - level - 3, and the surviving
// (u, w) leaf-parents are finished 32 at a time (leaf_parents with pairs).
// Per-node batch accounting and intersection tallies are those of expand.
template <bool INSTR>
__device__ __forceinline__ int expand_children(const Params &P, const Frame &f, const Dims &d,
                                               int level, const LeafBuf &lb, Acc128 &acc,
                                               Tally &tl) {
  const int lane = lane_id();
  const int WR = d.WR, WL = d.WL;
  const int li = level - 1;
  const uint32_t *R = f.setR() + li * WR;
  const uint32_t *Ls = f.setL() + li * WL;
  const int n = f.ns()[li];
  const int *kids = f.surv() + li * f.surv_cap;
  const int need_g = P.p_eff - level - 3;  // prune_keep at level + 2
  int work = 0, fill = 0;
  BC_LOOP
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const bool act = i < n;
    const int u = act ? kids[i] : 0;
    const uint32_t *ru = act ? rowR_of(f, d, u) : nullptr;
    const uint32_t *rl = act ? rowL_of(f, d, u) : f.rowL();
    uint32_t rp[RP_WORDS];
#pragma unroll
    for (int x = 0; x < RP_WORDS; x++) rp[x] = act && x < WR ? R[x] & ru[x] : 0u;
    const int wr_u = act ? (f.skip_words ? 1 : lane_words(R, ru, f.r_last(), WR)) : 0;
    const int wl_u = act ? (f.skip_words ? 1 : lane_words(Ls, rl, f.l_last(), WL)) : 0;
    int ncand_u = 0;
    BC_LOOP
    for (int x = 0; __any_sync(FULL, act && x < WL); x++) {
      const uint32_t mall = act && x < WL ? Ls[x] & rl[x] : 0u;
      ncand_u += __popc(mall);
      const uint32_t m = INSTR || !f.compact ? mall : mall & f.s1()[x];
      if (!__any_sync(FULL, m != 0u)) continue;  // no candidate in this word anywhere
      const int cnt = __popc(m);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += t;
      }
      const int excl = incl - cnt;
      const int total = __shfl_sync(FULL, incl, 31);
      BC_LOOP
      for (int r0 = 0; r0 < total; r0 += 32) {
        const int k = r0 + lane;
        int o = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const int c = o + step;
          const int e = __shfl_sync(FULL, excl, c < 32 ? c : 31);
          if (c < 32 && e <= k) o = c;
        }
        const uint32_t mo = __shfl_sync(FULL, m, o);
        const int eo = __shfl_sync(FULL, excl, o);
        const int uo = __shfl_sync(FULL, u, o);
        const int wro = INSTR ? __shfl_sync(FULL, wr_u, o) : 0;
        const int wlo = INSTR ? __shfl_sync(FULL, wl_u, o) : 0;
        uint32_t pr[RP_WORDS];
#pragma unroll
        for (int x2 = 0; x2 < RP_WORDS; x2++) pr[x2] = x2 < WR ? __shfl_sync(FULL, rp[x2], o) : 0u;
        bool keep = false;
        int w = 0;
        if (k < total) {
          w = x * 32 + (int)__fns(mo, 0, k - eo + 1);
          const uint32_t *rw = rowR_of(f, d, w);
          int cr = 0;
          if (rw) {
#pragma unroll
            for (int x2 = 0; x2 < RP_WORDS; x2++)
              if (x2 < WR) cr += __popc(pr[x2] & rw[x2]);
          }
          if (INSTR) {
            tl.inter++;
            tl.opw += wro + f.adjw()[w];
            tl.minw += wro < f.adjw()[w] ? wro : f.adjw()[w];
          }
          if (cr >= P.q_eff) {
            if (INSTR) {
              tl.inter++;
              tl.opw += wlo + f.dirw()[w];
              tl.minw += wlo < f.dirw()[w] ? wlo : f.dirw()[w];
            }
            const uint32_t *rlo = rowL_of(f, d, uo), *rlw = rowL_of(f, d, w);
            int cl = 0;  // only |L'| >= need_g matters: stop once it is reached
            BC_LOOP
            for (int x2 = 0; x2 < WL && cl < need_g; x2++) cl += __popc(Ls[x2] & rlo[x2] & rlw[x2]);
            keep = cl >= need_g;
          }
        }
        const unsigned km = __ballot_sync(FULL, keep);
        if (keep) {
          const int at = fill + __popc(km & lanemask_lt());
          lb.pu[at] = uo;
          lb.pw[at] = w;
        }
        fill += __popc(km);
        __syncwarp();
        if (fill >= 32) {  // finish 32 leaf-parents, keep the rest
          leaf_parents<INSTR, false>(P, f, d, level, lb.pu, 32, nullptr, lb, acc, tl, lb.pw);
          work += 32 * (WL + 8);
          const int rest = fill - 32;
          int a = 0, b = 0;
          if (lane < rest) {
            a = lb.pu[32 + lane];
            b = lb.pw[32 + lane];
          }
          __syncwarp();
          if (lane < rest) {
            lb.pu[lane] = a;
            lb.pw[lane] = b;
          }
          fill = rest;
          __syncwarp();
        }
      }
    }
    if (act) tl.batches += node_batches(P, (unsigned)ncand_u, wr_u, wl_u, false);
    work += __reduce_add_sync(FULL, ncand_u);
  }
  if (fill) {
    leaf_parents<INSTR, false>(P, f, d, level, lb.pu, fill, nullptr, lb, acc, tl, lb.pw);
    work += fill * (WL + 8);
  }
  return work;
}

// Expand node at `level` (1-based): children at level+1 (engine.py:315-374).
// Children that are leaves are counted here; children that are leaf-parents
// are finished lane-parallel (leaf_parents); deeper survivors are listed in
// surv[level-1] for the depth-first descent.
template <bool INSTR, bool LAZY>
__device__ __forceinline__ int expand(const Params &P, const Frame &f, const Dims &d, int level,
                                       const uint16_t *map, const LeafBuf &lb, Acc128 &acc,
                                       Tally &tl, PhaseClock &ph_) {
  const int lane = lane_id();
  const int WR = d.WR, WL = d.WL, nL = d.nL;
  const int li = level - 1;
  const uint32_t *R = f.setR() + li * WR;
  const uint32_t *Ls = f.setL() + li * WL;
  const bool leaf = level + 1 == P.p_eff - 1;
  const bool lp = level + 1 == P.p_eff - 2;  // children are leaf-parents
  int ncand, ncand_eval;
  if (INSTR || !f.compact) {
    ncand = ncand_eval = compact_bits(Ls, WL, f.cand());
  } else {  // batches count every candidate; only survivors are evaluated
    int c = 0;
    BC_LOOP
    for (int w = lane; w < WL; w += 32) c += __popc(Ls[w]);
    ncand = __reduce_add_sync(FULL, c);
    ncand_eval = compact_bits_and(Ls, f.s1(), WL, f.cand());
  }
  const int wr = level == 1 ? d.wR : f.skip_words ? 1 : words_touched(R, f.r_last(), WR);
  const int wl = leaf ? 0 : (level == 1 ? d.wL : f.skip_words ? 1 : words_touched(Ls, f.l_last(), WL));
  if (lane == 0) tl.batches += node_batches(P, (unsigned)ncand, wr, wl, leaf);
  int ns = 0;
  const int need_l = P.p_eff - level - 2;  // prune_keep(cr, cl, level+1): cl >= p - (level+1) - 1
  int *out = f.surv() + li * f.surv_cap;
  BC_LOOP
  for (int c0 = 0; c0 < ncand_eval; c0 += 32) {
    const int i = c0 + lane;
    bool keep = false;
    int u = 0;
    if (i < ncand_eval) {
      u = f.cand()[i];
      const uint32_t *row = rowR_of(f, d, u);
      int cr = 0;
      if (row)
        BC_LOOP
        for (int w = 0; w < WR; w++) cr += __popc(R[w] & row[w]);
      if (INSTR) {
        tl.inter++;
        tl.opw += wr + f.adjw()[u];
        tl.minw += wr < f.adjw()[u] ? wr : f.adjw()[u];
      }
      if (cr >= P.q_eff) {
        if (leaf) {
          add_comb(P, acc, cr);
        } else {
          if (INSTR) {
            tl.inter++;
            tl.opw += wl + f.dirw()[u];
            tl.minw += wl < f.dirw()[u] ? wl : f.dirw()[u];
          }
          if (LAZY) {
            keep = true;  // |L'| >= 1 is checked when the leaf-parent is walked
          } else {
            const uint32_t *rl = rowL_of(f, d, u);
            int cl = 0;  // prune_keep only needs |L'| >= need_l: stop once it is reached
            BC_LOOP
            for (int w = 0; w < WL && cl < need_l; w++) cl += __popc(Ls[w] & rl[w]);
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
  int work = ncand_eval;
  if (lp && ns) {
    PH_MARK(4);
    leaf_parents<INSTR, LAZY>(P, f, d, level, out, ns, map, lb, acc, tl);
    PH_MARK(5);
    work += ns * (WL + 8);
    ns = 0;
  }
  if (lane == 0) {
    f.ns()[li] = ns;
    f.cur()[li] = 0;
  }
  __syncwarp();
  return work;
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
  int cap;                  // frame layout: FrameSpec::cap of the task
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
    rec[1] = (uint32_t)lv | ((uint32_t)S.cap << 8);
    rec[2] = (uint32_t)(S.frame_off & 0xffffffffll);
    rec[3] = (uint32_t)(S.frame_off >> 32);
  }
  BC_LOOP
  for (int w = lane; w < d.WR; w += 32) rec[4 + w] = R[w] & rr[w];
  BC_LOOP
  for (int w = lane; w < d.WL; w += 32) rec[4 + d.WR + w] = Ls[w] & rl[w];
  __syncwarp();
  return true;
}

// DFS from a node at `start` whose sets sit in setR/setL[start-1].  Returns
// false once the expansion work passes `limit` (triage: the caller discards
// the partial task and defers it to the split path).
template <bool INSTR, bool LAZY, bool FLAT = true>
__device__ __forceinline__ bool dfs(const Params &P, const Frame &f, const Dims &d, int start,
                                    const uint16_t *map, const LeafBuf &lb, Acc128 &acc, Tally &tl,
                                    const SplitSink *sink, PhaseClock &ph_,
                                    long long limit = LLONG_MAX) {
  const int lane = lane_id();
  const int WR = d.WR, WL = d.WL, p_eff = P.p_eff;
  long long work = 0;
  int level = start;
  bool fresh = true;  // one expand call site: the kernel stays small (I-cache)
  BC_LOOP
  for (;;) {
    if (fresh) {
      work += expand<INSTR, LAZY>(P, f, d, level, map, lb, acc, tl, ph_);
      if (work > limit) return false;
      fresh = false;
      const int li0 = level - 1;
      if (FLAT && !LAZY && level + 2 == p_eff - 2 && WR <= RP_WORDS && f.ns()[li0] > 0 &&
          !(sink && level + 1 == sink->level)) {
        // the children's children are leaf-parents: expand every child at once
        work += expand_children<INSTR>(P, f, d, level, lb, acc, tl);
        if (work > limit) return false;
        __syncwarp();  // every lane's read of ns[li0] above precedes lane 0's write
        if (lane == 0) f.ns()[li0] = 0;
        __syncwarp();
      }
    }
    const int li = level - 1;
    if (level + 1 < p_eff - 2 && f.cur()[li] < f.ns()[li]) {
      const int u = f.surv()[li * f.surv_cap + f.cur()[li]];
      __syncwarp();
      if (lane == 0) f.cur()[li]++;
      const uint32_t *rr = rowR_of(f, d, u);
      const uint32_t *rl = rowL_of(f, d, u);
      if (sink && level + 1 == sink->level &&
          emit_node(P, *sink, d, level + 1, f.setR() + li * WR, rr, f.setL() + li * WL, rl))
        continue;
      BC_LOOP
      for (int w = lane; w < WR; w += 32) f.setR()[(li + 1) * WR + w] = f.setR()[li * WR + w] & rr[w];
      BC_LOOP
      for (int w = lane; w < WL; w += 32) f.setL()[(li + 1) * WL + w] = f.setL()[li * WL + w] & rl[w];
      __syncwarp();
      level++;
      fresh = true;
    } else {
      if (level == start) break;
      level--;
    }
  }
  return true;
}

// Sorted id list -> HTB words (htb.py:89-115) with exclusive prefix
// popcounts (o_pre[words] = n); returns the word count.
__device__ __forceinline__ int list_to_htb(const int32_t *ids, int n,
                                           uint32_t *o_idx, uint32_t *o_val, int *o_pre) {
  const int lane = lane_id();
  int pos = 0;
  BC_LOOP
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    uint32_t word = 0;
    bool start = false;
    if (i < n) {
      word = (uint32_t)ids[i] >> 5;
      start = i == 0 || ((uint32_t)ids[i - 1] >> 5) != word;
    }
    const unsigned m = __ballot_sync(FULL, start);
    if (start) {
      uint32_t v = 0;
      BC_LOOP
      for (int k = i; k < n; k++) {
        const uint32_t id = (uint32_t)ids[k];
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

// Flattened wedge walk over the opposite-layer rows of the C_R1 members
// (members[i], ascending ids): calls fn(i, lx) for every anchor x in N(members[i])
// that lies in C_L1 (slot map), lx = its local index.  The 32 lanes share the
// concatenated rows, so every lane issues a load per step however short the
// rows are.  Work is sum_{v in C_R1} deg(v), read as contiguous rows, instead
// of |C_L1| probes of (possibly hub-sized) adjacency rows.
//
// With root-restricted rows (P.roffE), member i's row is R(r, v) = N(v) & dir2(r)
// (list entry lbase + i): every x of C_L1 = dir2(r) & dir2(s) in N(v) is in it, so the
// hits are the same and the walk is shorter.
template <typename F>
__device__ __forceinline__ void for_member_hits(const Params &P, const Frame &f, const Dims &d,
                                                const int *members, const uint16_t *map,
                                                int64_t lbase, int64_t rbase, F fn) {
  const int lane = lane_id();
  const int32_t *__restrict__ src = P.roffE ? P.rrows : P.g.bidx;
  BC_LOOP
  for (int b0 = 0; b0 < d.nR; b0 += 32) {
    const int i = b0 + lane;
    int64_t start = 0;
    int len = 0;
    if (i < d.nR) {
      if (P.roffE) {
        const int64_t e = __ldg(P.lists + lbase + i);
        start = __ldg(P.roffE + e);
        len = (int)(__ldg(P.roffE + e + 1) - start);
      } else {
        const int v = members[i];
        start = __ldg(P.g.boff + v);
        len = (int)(__ldg(P.g.boff + v + 1) - start);
      }
    }
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    const int excl = incl - len;
    const int T = __shfl_sync(FULL, incl, 31);
    constexpr int U = 4;  // gathers in flight per lane
    BC_LOOP
    for (int r0 = 0; r0 < T; r0 += 32 * U) {
      int xs[U], own[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int pos = r0 + 32 * u + lane;
        int sl = 0;  // owning member: the last lane whose exclusive offset is <= pos
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const int c = sl + step;
          const int e = __shfl_sync(FULL, excl, c < 32 ? c : 31);
          if (c < 32 && e <= pos) sl = c;
        }
        const int64_t st = __shfl_sync(FULL, start, sl);
        const int ex = __shfl_sync(FULL, excl, sl);
        own[u] = sl;
        xs[u] = pos < T ? __ldg(src + st + (pos - ex)) : -1;
        if (P.roffE && xs[u] >= 0) xs[u] = __ldg(P.rdir + rbase + xs[u]);  // position -> id
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int x = xs[u];
        if (x < 0) continue;
        const int k = map[x >> 5];
        if (k != 0xffff) {
          const uint32_t lv = f.l_val()[k];
          const int xb = x & 31;
          if ((lv >> xb) & 1u) fn(b0 + own[u], f.l_pre()[k] + __popc(lv & ((1u << xb) - 1u)));
        }
      }
    }
  }
  __syncwarp();
}

// Frame part 1 for task (r, s) (local index j): C_R1 / C_L1 (engine.py:277-292)
// -- C_R1 from the wedge-scatter level-1 lists when present -- the decoded C_L1
// ids + slot map, the level-1 R-survivors x (|N(x) & C_R1| >= q, engine.py:338)
// with their lslot rows, and rowR.  Compact (scatter) mode counts |N(x) & C_R1|
// for every x by the wedge walk, then sets bits for the survivors only (when
// they fit the cap); full mode probes a row for every x (local_row).
// Returns the number of survivors (-1 in full mode without lslot: not counted).
template <bool INSTR, bool ROWS = true>
__device__ __forceinline__ int build_frame_R(const Params &P, const Frame &f, const Dims &d,
                                             const FrameSpec &sp, int r, int s, int64_t j,
                                             uint16_t *map, PhaseClock &ph_) {
  const int lane = lane_id();
  int card;
  if (P.lists && P.roffE && sp.compact) {
    // edge-indexed list: members into rids (ascending: edges of r follow its sorted row),
    // then their HTB words
    const int64_t l0 = P.roff[j], abase = P.csr_aoff[r] - P.rebase[r];
    BC_LOOP
    for (int i = lane; i < d.nR; i += 32) f.rids()[i] = __ldg(P.csr_aidx + abase + __ldg(P.lists + l0 + i));
    __syncwarp();
    list_to_htb(f.rids(), d.nR, f.r_idx(), f.r_val(), f.r_pre());
  } else if (P.lists && !P.roffE) {
    list_to_htb(P.lists + P.roff[j], d.nR, f.r_idx(), f.r_val(), f.r_pre());
  } else {
    isect_adj<true>(P.g, r, s, card, f.r_idx(), f.r_val(), f.r_pre());
  }
  isect_dir<true>(P.g, r, s, card, f.l_idx(), f.l_val(), f.l_pre());
  PH_MARK(1);
  // decode C_L1 ids (ascending, htb.py:42-52); fill the slot map
  BC_LOOP
  for (int k = lane; k < d.wL; k += 32) {
    uint32_t v = f.l_val()[k];
    const int base_id = (int)f.l_idx()[k] * 32;
    int pos = f.l_pre()[k];
    if (map) map[f.l_idx()[k]] = (uint16_t)k;
    if (!sp.compact)
      BC_LOOP
      while (v) {
        f.lids()[pos++] = base_id + __ffs(v) - 1;
        v &= v - 1;
      }
  }
  if (sp.compact && !(P.lists && P.roffE)) {  // C_R1 members, ascending
    BC_LOOP
    for (int k = lane; k < d.wR; k += 32) {
      uint32_t v = f.r_val()[k];
      const int base_id = (int)f.r_idx()[k] * 32;
      int pos = f.r_pre()[k];
      BC_LOOP
      while (v) {
        f.rids()[pos++] = base_id + __ffs(v) - 1;
        v &= v - 1;
      }
    }
  }
  __syncwarp();
  PH_MARK(2);
  int ns1 = 0;
  if (sp.compact) {
    BC_LOOP
    for (int x = lane; x < d.nL; x += 32) f.lslot()[x] = 0;
    __syncwarp();
    // two walks with one inlined copy of the walk (instruction cache): pass 0 counts
    // |N(x) & C_R1| per x into lslot, pass 1 sets the survivors' rowR bits
    int *lslot = f.lslot();
    uint32_t *rowR = f.rowR();
    const int WR = d.WR;
    const int64_t lbase = P.roffE ? P.roff[j] : 0;
    const int64_t rbase = P.roffE ? P.dir_off[r] : 0;
    BC_LOOP
    for (int pass = 0; pass < 2; pass++) {
      for_member_hits(P, f, d, f.rids(), map, lbase, rbase, [&](int i, int lx) {
        if (pass == 0) {
          atomicAdd(lslot + lx, 1);
        } else {
          const int sl = lslot[lx];
          if (sl >= 0) atomicOr(rowR + (sl * WR + (i >> 5)), 1u << (i & 31));
        }
      });
      if (pass == 1) break;
      int base = 0;
      BC_LOOP
      for (int x0 = 0; x0 < d.nL; x0 += 32) {
        const int x = x0 + lane;
        const bool sv = x < d.nL && lslot[x] >= P.q_eff;
        const unsigned m = __ballot_sync(FULL, sv);
        if (x < d.nL) lslot[x] = sv ? base + __popc(m & lanemask_lt()) : -1;
        base += __popc(m);
      }
      ns1 = base;
      __syncwarp();
      if (!(ROWS && ns1 > 0 && ns1 <= sp.rows(d.nL))) break;
      const int total = ns1 * WR;
      BC_LOOP
      for (int w = lane; w < total; w += 32) rowR[w] = 0;
      __syncwarp();
    }
  } else {
    BC_LOOP
    for (int x = lane; x < d.nL; x += 32) {
      const int id = f.lids()[x];
      const int sl = P.g.dense_id[id];
      local_row(f.r_idx(), f.r_val(), f.r_pre(), d.wR, P.g.aidx, P.g.aval, P.g.aoff[id],
                P.g.aoff[id + 1], sl >= 0 ? P.g.dense + (int64_t)sl * P.g.mw : nullptr,
                f.rowR() + x * d.WR, d.WR);
    }
    __syncwarp();
    if (!sp.lslot()) return -1;  // survivors not needed (no rowL rows, no triage)
    int base = 0;
    BC_LOOP
    for (int x0 = 0; x0 < d.nL; x0 += 32) {
      const int x = x0 + lane;
      bool sv = false;
      if (x < d.nL) {
        const uint32_t *row = f.rowR() + x * d.WR;
        int c = 0;
        BC_LOOP
        for (int w = 0; w < d.WR; w++) c += __popc(row[w]);
        sv = c >= P.q_eff;
      }
      const unsigned m = __ballot_sync(FULL, sv);
      if (x < d.nL) f.lslot()[x] = sv ? base + __popc(m & lanemask_lt()) : -1;
      base += __popc(m);
    }
    ns1 = base;
    __syncwarp();
  }
  return ns1;
}

// Frame part 2: rowL[lslot[x]] = dir2(x) & C_L1 (engine.py:360) for the
// level-1 R-survivors, and the slice lengths the instrumented tallies use.
template <bool INSTR, bool LAZY>
__device__ __forceinline__ void build_frame_L(const Params &P, const Frame &f, const Dims &d,
                                              const FrameSpec &sp, const uint16_t *map,
                                              PhaseClock &ph_) {
  const int lane = lane_id();
  // word-boundary masks of the local universes for the batch accounting below level 1
  // (C_R: leaf-parents and deeper nodes; C_L: nodes at level >= 2, p_eff >= 5)
  const bool need_l = P.p_eff >= 5;
  BC_LOOP
  for (int w = lane; w < d.WR; w += 32) f.r_last()[w] = 0;
  if (need_l)
    BC_LOOP
    for (int w = lane; w < d.WL; w += 32) f.l_last()[w] = 0;
  __syncwarp();
  BC_LOOP
  for (int k = lane; k < d.wR; k += 32) {
    const int e = f.r_pre()[k + 1] - 1;
    atomicOr(f.r_last() + (e >> 5), 1u << (e & 31));
  }
  if (need_l)
    BC_LOOP
    for (int k = lane; k < d.wL; k += 32) {
      const int e = f.l_pre()[k + 1] - 1;
      atomicOr(f.l_last() + (e >> 5), 1u << (e & 31));
    }
  __syncwarp();
  // level-1 R-survivor masks: candidates outside them cannot pass |R & N(x)| >= q.
  // Used in compact mode (few survivors among many candidates, e.g. hub pairs);
  // where most candidates survive the extra masks do not pay.
  BC_LOOP
  for (int x0 = 0; sp.compact && x0 < d.nL; x0 += 32) {
    const int x = x0 + lane;
    bool sv = false;
    if (x < d.nL) {
      if (sp.compact || sp.lslot()) {
        sv = f.lslot()[x] >= 0;
      } else {
        const uint32_t *row = f.rowR() + x * d.WR;
        int c = 0;
        BC_LOOP
        for (int w = 0; w < d.WR; w++) c += __popc(row[w]);
        sv = c >= P.q_eff;
      }
    }
    const unsigned m = __ballot_sync(FULL, sv);
    if (lane == 0) f.s1()[x0 >> 5] = m;
  }
  __syncwarp();
  BC_LOOP
  for (int k = lane; sp.compact && k < d.wL; k += 32) {
    uint32_t v = f.l_val()[k], h = 0;
    int pos = f.l_pre()[k];
    BC_LOOP
    while (v) {
      const int b = __ffs(v) - 1;
      v &= v - 1;
      if ((f.s1()[pos >> 5] >> (pos & 31)) & 1u) h |= 1u << b;
      pos++;
    }
    f.s1h()[k] = h;
  }
  __syncwarp();
  const bool build = sp.rowL && P.p_eff >= 4 && !LAZY;
  if (!build && !INSTR) {
    PH_MARK(3);
    return;
  }
  BC_LOOP
  for (int x = lane; x < d.nL; x += 32) {
    if (sp.compact && !INSTR && f.lslot()[x] < 0) continue;
    const int id = lid_of(f, d, x);
    if (build) {
      const int slot = f.lslot()[x];
      if (slot >= 0) {
        const int64_t d0 = P.g.doff[id], d1 = P.g.doff[id + 1];
        uint32_t *out = f.rowL() + slot * d.WL;
        if (map)
          local_row_map(map, f.l_val(), f.l_pre(), P.g.didx, P.g.dval, d0, d1, out, d.WL);
        else
          local_row(f.l_idx(), f.l_val(), f.l_pre(), d.wL, P.g.didx, P.g.dval, d0, d1, nullptr, out,
                    d.WL);
      }
    }
    if (INSTR) {
      f.adjw()[x] = (int)(P.g.aoff[id + 1] - P.g.aoff[id]);
      f.dirw()[x] = (int)(P.g.doff[id + 1] - P.g.doff[id]);
    }
  }
  __syncwarp();
  PH_MARK(3);
}

__device__ __forceinline__ void clear_map(uint16_t *map, const Frame &f, const Dims &d) {
  if (!map) return;
  BC_LOOP
  for (int k = lane_id(); k < d.wL; k += 32) map[f.l_idx()[k]] = 0xffff;
  __syncwarp();
}

__device__ __forceinline__ void init_root_sets(const Frame &f, const Dims &d) {
  const int lane = lane_id();
  BC_LOOP
  for (int w = lane; w < d.WR; w += 32) {
    const int rem = d.nR - w * 32;
    f.setR()[w] = rem >= 32 ? FULL : ((1u << rem) - 1u);
  }
  BC_LOOP
  for (int w = lane; w < d.WL; w += 32) {
    const int rem = d.nL - w * 32;
    f.setL()[w] = rem >= 32 ? FULL : ((1u << rem) - 1u);
  }
  __syncwarp();
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
  int triage;                           // > 0: defer tasks with more level-1 R-survivors,
  long long triage_work;                //   more expansion work, or a frame over
  int32_t *heavy;                       //   the scratch to heavy[] (the split path),
  int32_t *heavy_ns1;                   //   with their level-1 survivor counts (0: unknown)
  const int32_t *caps;                  // SPLIT: survivor cap per queue entry (0: |C_L1|)
};

__device__ __forceinline__ void push_heavy(const Params &P, const EnumArgs &A, int j, int ns1) {
  const unsigned long long k = atomicAdd(P.ctr + CTR_HEAVY, 1ull);
  A.heavy[k] = j;
  A.heavy_ns1[k] = ns1;
}

__device__ __forceinline__ void finish_task(const Params &P, Acc128 acc, int64_t t, bool atomic,
                                            Acc128 &total) {
  acc = warp_sum128(acc);
  if (lane_id() == 0) {
    total.add(acc);
    if (P.task_counts) {
      if (atomic) atomic_add128(P.task_counts + 2 * t, P.overflow, acc);
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
    atomic_add128(P.acc, P.overflow, total);
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

// Whole tasks (SPLIT = false) or the top levels of every task with its frame
// written to the global frame arena and split-level nodes pushed as sub-tasks
// (SPLIT = true, p_eff >= 5).
template <bool INSTR, bool LAZY, bool SPLIT, bool TRIAGE, bool COMPACT>
__global__ void __launch_bounds__(ENUM_THREADS, ENUM_MIN_BLOCKS) enum_kernel(Params P, EnumArgs A) {
  extern __shared__ uint32_t smem[];
  const int lane = lane_id();
  const int wib = threadIdx.x >> 5;
  const int64_t gwarp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int map_w = (P.map_words + 1) / 2;  // u16 entries packed in words
  uint32_t *my = smem + (int64_t)wib * (map_w + LEAF_WORDS + A.budget_words);
  uint16_t *map = P.map_words ? (uint16_t *)my : nullptr;
  const LeafBuf lb{(int *)(my + map_w), (int *)(my + map_w + 32), (int *)(my + map_w + 64),
                   (int *)(my + map_w + 128)};
  uint32_t *my_smem = my + map_w + LEAF_WORDS;
  uint32_t *my_global = A.gscratch ? A.gscratch + gwarp * A.gscratch_words : nullptr;
  if (map)
    BC_LOOP
    for (int i = lane; i < map_w; i += 32) my[i] = 0xffffffffu;
  __syncwarp();
  Acc128 total{0, 0};
  Tally tl;
  unsigned long long claims = 0, spills = 0;
  const int p_eff = P.p_eff;
  PH_DECL
  BC_LOOP
  for (;;) {
    long long qi = 0;
    if (lane == 0) qi = (long long)atomicAdd(P.ctr + CTR_NEXT, 1ull);
    qi = __shfl_sync(FULL, qi, 0) + A.q0;
    PH_MARK(0);
    if (qi >= A.q1) break;
    claims++;
    const int j = A.queue[qi];
    const int64_t t = task_id(P.ltask, P.shard, P.nshards, j);
    const int2 tk = P.tasks[t];
    const Dims d = dims_of(A.info[j]);
    const FrameSpec sp{SPLIT || has_rowL(p_eff, P.map_words), COMPACT, INSTR,
                       TRIAGE ? A.triage : (SPLIT && A.caps ? A.caps[qi] : 0)};
    const int64_t ro = ro_words(d.nR, d.nL, d.wR, d.wL, sp);
    const int64_t sc = scratch_words(d.nR, d.nL, p_eff, sp);
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
      if (TRIAGE) {  // frame too large for the scratch: the split path takes it
        if (lane == 0) push_heavy(P, A, j, 0);
        __syncwarp();
      } else if (lane == 0) {
        atomicExch(P.overflow, 2);  // cannot happen: sized from level-1 maxima
      }
      continue;
    }
    Frame f;
    carve_ro(f, ro_base, d, sp);
    carve_scratch(f, sc_base, d, p_eff, sp);
    set_skip_words(f, P, d, INSTR);
    const int ns1 = build_frame_R<INSTR>(P, f, d, sp, tk.x, tk.y, j, map, ph_);
    if (TRIAGE && ns1 > A.triage) {  // too many survivor rows: split path
      if (lane == 0) push_heavy(P, A, j, ns1);
      clear_map(map, f, d);
      continue;
    }
    if (!INSTR && !SPLIT && ns1 == 0) {
      // no candidate survives level 1: count 0, the level-1 expansion is the only batch
      // work (engine.py:306-331); skip the frame's second half and the search
      if (lane == 0) tl.batches += node_batches(P, (unsigned)d.nL, d.wR, d.wL, p_eff == 3);
      clear_map(map, f, d);
      finish_task(P, Acc128{0, 0}, t, false, total);
      continue;
    }
    build_frame_L<INSTR, LAZY>(P, f, d, sp, map, ph_);
    init_root_sets(f, d);
    Acc128 acc{0, 0};
    if (SPLIT) {
      SplitSink sink = A.sink;
      sink.frame_off = A.frame_off[qi - A.q0];
      sink.task_j = j;
      sink.cap = sp.cap;
      dfs<INSTR, false>(P, f, d, 1, map, lb, acc, tl, &sink, ph_);
    } else if (TRIAGE) {
      const Tally tl0 = tl;
      if (!dfs<INSTR, LAZY, false>(P, f, d, 1, map, lb, acc, tl, nullptr, ph_,
                                   A.triage_work)) {
        // over the work budget: discard the partial task, the split path takes it
        tl = tl0;
        if (lane == 0) push_heavy(P, A, j, ns1);
        clear_map(map, f, d);
        continue;
      }
    } else if (LAZY) {  // p_eff = 4: level 1's children are the leaf-parents, no descent
      expand<INSTR, true>(P, f, d, 1, map, lb, acc, tl, ph_);
    } else {
      dfs<INSTR, false>(P, f, d, 1, map, lb, acc, tl, nullptr, ph_);
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
template <bool INSTR, bool COMPACT>
__global__ void __launch_bounds__(ENUM_THREADS, ENUM_MIN_BLOCKS) sub_kernel(Params P, EnumArgs A, int64_t n_sub) {
  extern __shared__ uint32_t smem[];
  const int lane = lane_id();
  const int wib = threadIdx.x >> 5;
  const int64_t gwarp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  uint32_t *my = smem + (int64_t)wib * (LEAF_WORDS + A.budget_words);
  const LeafBuf lb{(int *)my, (int *)(my + 32), (int *)(my + 64), (int *)(my + 128)};
  uint32_t *my_smem = my + LEAF_WORDS;
  uint32_t *my_global = A.gscratch ? A.gscratch + gwarp * A.gscratch_words : nullptr;
  Acc128 total{0, 0};
  Tally tl;
  unsigned long long spills = 0;
  const int p_eff = P.p_eff;
  PH_DECL
  BC_LOOP
  for (;;) {
    long long k = 0;
    if (lane == 0) k = (long long)atomicAdd(P.ctr + CTR_SUB_NEXT, 1ull);
    k = __shfl_sync(FULL, k, 0);
    if (k >= n_sub) break;
    const uint32_t *rec = A.sink.arena + A.sub_order[k];
    const int j = (int)rec[0];
    const int lv = (int)(rec[1] & 0xff);
    const FrameSpec sp{true, COMPACT, INSTR, (int)(rec[1] >> 8)};
    const int64_t foff = (int64_t)rec[2] | ((int64_t)rec[3] << 32);
    const int64_t t = task_id(P.ltask, P.shard, P.nshards, j);
    const Dims d = dims_of(A.info[j]);
    const int64_t sc = scratch_words(d.nR, d.nL, p_eff, sp);
    uint32_t *sc_base = sc <= A.budget_words ? my_smem : my_global;
    if (sc_base == my_global) spills++;
    if (!sc_base || (sc_base == my_global && sc > A.gscratch_words)) {
      if (lane == 0) atomicExch(P.overflow, 2);
      continue;
    }
    Frame f;
    carve_ro(f, A.frames + foff, d, sp);
    carve_scratch(f, sc_base, d, p_eff, sp);
    set_skip_words(f, P, d, INSTR);
    BC_LOOP
    for (int w = lane; w < d.WR; w += 32) f.setR()[(lv - 1) * d.WR + w] = rec[4 + w];
    BC_LOOP
    for (int w = lane; w < d.WL; w += 32) f.setL()[(lv - 1) * d.WL + w] = rec[4 + d.WR + w];
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

// Triage filter (p_eff >= 5, millions of tasks): only the first half of each task's
// frame -- C_R1, C_L1 and the level-1 R-survivor count.  A task without survivors
// is finished here (its level-1 expansion is its only batch work, engine.py:306-331);
// the others go to `heavy` (the medium list) for the triage kernel.  Kept separate
// so this kernel, which sees every task, stays small in instruction cache.
#ifndef FILTER_MIN_BLOCKS
#define FILTER_MIN_BLOCKS 4
#endif
template <bool COMPACT>
__global__ void __launch_bounds__(ENUM_THREADS, FILTER_MIN_BLOCKS) filter_kernel(Params P, EnumArgs A) {
  extern __shared__ uint32_t smem[];
  const int lane = lane_id();
  const int wib = threadIdx.x >> 5;
  const int64_t gwarp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int map_w = (P.map_words + 1) / 2;
  uint32_t *my = smem + (int64_t)wib * (map_w + A.budget_words);
  uint16_t *map = P.map_words ? (uint16_t *)my : nullptr;
  uint32_t *my_smem = my + map_w;
  uint32_t *my_global = A.gscratch ? A.gscratch + gwarp * A.gscratch_words : nullptr;
  if (map)
    BC_LOOP
    for (int i = lane; i < map_w; i += 32) my[i] = 0xffffffffu;
  __syncwarp();
  Tally tl;
  Acc128 total{0, 0};
  unsigned long long claims = 0;
  const int p_eff = P.p_eff;
  PH_DECL
  BC_LOOP
  for (;;) {
    long long qi = 0;
    if (lane == 0) qi = (long long)atomicAdd(P.ctr + CTR_NEXT, 1ull);
    qi = __shfl_sync(FULL, qi, 0) + A.q0;
    if (qi >= A.q1) break;
    claims++;
    const int j = A.queue[qi];
    const int64_t t = task_id(P.ltask, P.shard, P.nshards, j);
    const int2 tk = P.tasks[t];
    const Dims d = dims_of(A.info[j]);
    // only C_R1 / C_L1 and the survivor count: no candidate rows
    const FrameSpec sp{false, COMPACT, false, 1};
    const int64_t ro = ro_words(d.nR, d.nL, d.wR, d.wL, sp);
    uint32_t *ro_base = ro <= A.budget_words ? my_smem : my_global;
    if (!ro_base || (ro_base == my_global && ro > A.gscratch_words)) {
      if (lane == 0) push_heavy(P, A, j, 0);  // frame over the scratch: the next passes
      __syncwarp();
      continue;
    }
    Frame f;
    carve_ro(f, ro_base, d, sp);
    const int ns1 = build_frame_R<false, false>(P, f, d, sp, tk.x, tk.y, j, map, ph_);
    clear_map(map, f, d);
    if (ns1 == 0) {
      if (lane == 0) tl.batches += node_batches(P, (unsigned)d.nL, d.wR, d.wL, p_eff == 3);
      finish_task(P, Acc128{0, 0}, t, false, total);
    } else if (lane == 0) {
      push_heavy(P, A, j, 0);
    }
    __syncwarp();
  }
  flush_tallies(P, total, tl, claims, 0, false);
}

// ---- launchers (defined once per COMPACT value in enum_plain.cu / enum_compact.cu)
struct EnumVariant {
  bool instr, lazy, split, triage;
};
int enum_blocks_per_sm_c0(const EnumVariant &v, size_t smem);
int enum_blocks_per_sm_c1(const EnumVariant &v, size_t smem);
void enum_launch_c0(const EnumVariant &v, unsigned blocks, size_t smem, cudaStream_t st,
                    const Params &P, const EnumArgs &A);
void enum_launch_c1(const EnumVariant &v, unsigned blocks, size_t smem, cudaStream_t st,
                    const Params &P, const EnumArgs &A);
int sub_blocks_per_sm_c0(bool instr, size_t smem);
int sub_blocks_per_sm_c1(bool instr, size_t smem);
void sub_launch_c0(bool instr, unsigned blocks, size_t smem, cudaStream_t st, const Params &P,
                   const EnumArgs &A, int64_t n_sub);
void sub_launch_c1(bool instr, unsigned blocks, size_t smem, cudaStream_t st, const Params &P,
                   const EnumArgs &A, int64_t n_sub);
void phase_cycles_c0(unsigned long long *h, bool reset);
int filter_blocks_per_sm_c0(size_t smem);
int filter_blocks_per_sm_c1(size_t smem);
void filter_launch_c0(unsigned blocks, size_t smem, cudaStream_t st, const Params &P,
                      const EnumArgs &A);
void filter_launch_c1(unsigned blocks, size_t smem, cudaStream_t st, const Params &P,
                      const EnumArgs &A);
void phase_cycles_c1(unsigned long long *h, bool reset);

}  // namespace sk
}  // namespace bc
