// search.cu -- level-1 pass and hybrid DFS-BFS enumeration on sm_100a.
//
// Restates Searcher.run_task / Searcher._descend (reference engine.py:245-374)
// and the leaf rule C(|C_R|, q) (engine.py:285, 346-347), for all tasks of
// this shard, with exact 128-bit counts.
//
// Level 1 (kernel level1_kernel, warp per task): C_R1 = adj[r] & adj[s] and,
// when p_eff >= 3 and |C_R1| >= q, C_L1 = dir2[r] & dir2[s] -- the same two
// HTB intersections the reference performs first (engine.py:277-292), as a
// warp-cooperative walk of the shorter Idx run with per-lane lower_bound in the
// longer one (the reference's bisect, htb.py:122-154, 32 words at a time),
// AND of the matched Val words and __popc / __reduce_add_sync reductions.
// p_eff = 2 finishes here.  For deeper searches it records |C_R1|, |C_L1|
// and their HTB word counts, drops tasks failing prune_keep (engine.py:110-112)
// and emits a cost key |C_L1|*|C_R1| for the pre-runtime LPT order.
//
// Enumeration (kernel enum_kernel): persistent warps pull tasks, heaviest
// first, from one global atomic cursor (runtime stealing).  Every deeper
// C_R is a subset of C_R1 and every deeper C_L a subset of C_L1
// (engine.py:296-297, 365-366), so the warp re-materialises C_R1 / C_L1 as
// HTB words in shared memory and re-indexes them as a task-local universe:
//   rowR[x] = N(x) & C_R1,   rowL[x] = dir2(x) & C_L1   for x in C_L1,
// dense bitsets over the local indices (the reference's level 1->2
// intersections, engine.py:338, 360).  Every deeper intersection is then an
// aligned AND of ceil(|C_R1|/32) resp. ceil(|C_L1|/32) words + popcount.
// A node's candidates are expanded as one BFS batch across the 32 lanes and
// the search descends depth-first into survivors (hybrid DFS-BFS, Alg. 1).
// The reference's batch accounting (engine.py:306-331) is reproduced exactly:
// a node's C_R / C_L word counts in the original id space are the number of
// C_R1 / C_L1 HTB words its local bitset touches.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "engine.h"

namespace bc {

namespace {

struct Graph2 {  // HTB arenas (htb.py:64-86)
  const int64_t *__restrict__ aoff;
  const uint32_t *__restrict__ aidx;
  const uint32_t *__restrict__ aval;
  const int64_t *__restrict__ doff;
  const uint32_t *__restrict__ didx;
  const uint32_t *__restrict__ dval;
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
};

enum { CTR_ALIVE = 0, CTR_BATCHES, CTR_STOLEN, CTR_INTER, CTR_OPW, CTR_MINW, CTR_MAXNEED,
       CTR_SPILL, CTR_NEXT, CTR_COUNT };

struct Info {  // level-1 facts of one task
  int32_t cr, wr, cl, wl;
};

__device__ __forceinline__ void add_comb(const Params &P, Acc128 &a, int c) {
  if (c >= P.first_bad) {
    atomicExch(P.overflow, 1);
    return;
  }
  const ulonglong2 v = __ldg(P.comb + c);
  a.add(v.x, v.y);
}

// Warp-cooperative HTB intersection (htb.py:122-154) returning |A&B| and the
// number of nonzero result words.  Slices [a0,a1), [b0,b1) of one arena.
__device__ __forceinline__ void warp_isect_count(const uint32_t *__restrict__ idx,
                                                 const uint32_t *__restrict__ val, int64_t a0,
                                                 int64_t a1, int64_t b0, int64_t b1, int &card,
                                                 int &words) {
  const int lane = lane_id();
  if (a1 - a0 > b1 - b0) {
    int64_t t0 = a0, t1 = a1;
    a0 = b0; a1 = b1; b0 = t0; b1 = t1;
  }
  int c = 0, w = 0;
  int64_t lo = b0;
  for (int64_t base = a0; base < a1; base += 32) {
    const int64_t i = base + lane;
    int64_t j = b1;
    uint32_t x = 0;
    if (i < a1) {
      const uint32_t key = __ldg(idx + i);
      j = lower_bound_u32(idx, lo, b1, key);
      if (j < b1 && __ldg(idx + j) == key) x = __ldg(val + i) & __ldg(val + j);
    }
    c += __popc(x);
    w += x != 0;
    const int64_t jl = __shfl_sync(FULL, j, 31);
    if (jl >= b1) break;
    lo = jl;
  }
  card = __reduce_add_sync(FULL, c);
  words = __reduce_add_sync(FULL, w);
}

// Same walk, writing the nonzero result words (ascending) and the exclusive
// prefix popcounts pre[k] (pre[words] = card) to o_idx/o_val/o_pre.
__device__ __forceinline__ int warp_isect_out(const uint32_t *__restrict__ idx,
                                              const uint32_t *__restrict__ val, int64_t a0,
                                              int64_t a1, int64_t b0, int64_t b1,
                                              uint32_t *o_idx, uint32_t *o_val, int *o_pre) {
  const int lane = lane_id();
  if (a1 - a0 > b1 - b0) {
    int64_t t0 = a0, t1 = a1;
    a0 = b0; a1 = b1; b0 = t0; b1 = t1;
  }
  int pos = 0, run = 0;
  int64_t lo = b0;
  for (int64_t base = a0; base < a1; base += 32) {
    const int64_t i = base + lane;
    int64_t j = b1;
    uint32_t x = 0, key = 0;
    if (i < a1) {
      key = __ldg(idx + i);
      j = lower_bound_u32(idx, lo, b1, key);
      if (j < b1 && __ldg(idx + j) == key) x = __ldg(val + i) & __ldg(val + j);
    }
    const unsigned nz = __ballot_sync(FULL, x != 0);
    int c = __popc(x), incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    if (x) {
      const int k = pos + __popc(nz & lanemask_lt());
      o_idx[k] = key;
      o_val[k] = x;
      o_pre[k] = run + incl - c;
    }
    pos += __popc(nz);
    run += __shfl_sync(FULL, incl, 31);
    const int64_t jl = __shfl_sync(FULL, j, 31);
    if (jl >= b1) break;
    lo = jl;
  }
  if (lane == 0) o_pre[pos] = run;
  __syncwarp();
  return pos;
}

// Frame size in 32-bit words for a task-local universe.
__host__ __device__ __forceinline__ int64_t frame_words(int nR, int nL, int wR, int wL, int p_eff,
                                                        bool instr) {
  const int64_t WR = (nR + 31) / 32, WL = (nL + 31) / 32;
  const int64_t levels = p_eff - 2;
  int64_t w = 3 * (int64_t)wR + 1 + 3 * (int64_t)wL + 1;  // C_R1 / C_L1 HTB words + prefixes
  w += nL;                                                 // lids
  w += (int64_t)nL * WR;                                   // rowR
  if (p_eff >= 4) w += (int64_t)nL * WL;                   // rowL
  if (instr) w += 2 * (int64_t)nL;                         // adj / dir2 slice words
  w += nL;                                                 // candidate compaction
  w += levels * (WR + WL + nL + 2);                        // per-level R, L, survivors, ns/cur
  return w;
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
  unsigned long long alive = 0, inter = 0, opw = 0, minw = 0, maxneed = 0;
  for (int64_t j = gw; j < nloc; j += nw) {
    const int64_t t = P.shard + j * P.nshards;
    const int2 tk = P.tasks[t];
    const int64_t ra0 = P.g.aoff[tk.x], ra1 = P.g.aoff[tk.x + 1];
    const int64_t sa0 = P.g.aoff[tk.y], sa1 = P.g.aoff[tk.y + 1];
    int cr, wr;
    warp_isect_count(P.g.aidx, P.g.aval, ra0, ra1, sa0, sa1, cr, wr);
    if (INSTR) {
      const int64_t la = ra1 - ra0, lb = sa1 - sa0;
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
        const int64_t rd0 = P.g.doff[tk.x], rd1 = P.g.doff[tk.x + 1];
        const int64_t sd0 = P.g.doff[tk.y], sd1 = P.g.doff[tk.y + 1];
        int cl, wl;
        warp_isect_count(P.g.didx, P.g.dval, rd0, rd1, sd0, sd1, cl, wl);
        if (INSTR) {
          const int64_t la = rd1 - rd0, lb = sd1 - sd0;
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
          const int64_t need = frame_words(cr, cl, wr, wl, P.p_eff, INSTR);
          if ((unsigned long long)need > maxneed) maxneed = need;
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
    if (maxneed) atomicMax(P.ctr + CTR_MAXNEED, maxneed);
  }
}

// ---------------------------------------------------------------------------
// enumeration (engine.py:315-374) over the task-local universe
// ---------------------------------------------------------------------------
struct Frame {
  uint32_t *r_idx, *r_val;
  int *r_pre;
  uint32_t *l_idx, *l_val;
  int *l_pre;
  int *lids;
  uint32_t *rowR, *rowL;
  int *adjw, *dirw;
  int *cand;
  uint32_t *setR, *setL;
  int *surv;
  int *ns, *cur;
};

__device__ __forceinline__ Frame carve(uint32_t *base, int nR, int nL, int wR, int wL, int p_eff,
                                       bool instr) {
  const int WR = (nR + 31) >> 5, WL = (nL + 31) >> 5, levels = p_eff - 2;
  Frame f;
  uint32_t *p = base;
  f.r_idx = p; p += wR;
  f.r_val = p; p += wR;
  f.r_pre = (int *)p; p += wR + 1;
  f.l_idx = p; p += wL;
  f.l_val = p; p += wL;
  f.l_pre = (int *)p; p += wL + 1;
  f.lids = (int *)p; p += nL;
  f.rowR = p; p += (int64_t)nL * WR;
  f.rowL = p; if (p_eff >= 4) p += (int64_t)nL * WL;
  f.adjw = (int *)p; if (instr) p += nL;
  f.dirw = (int *)p; if (instr) p += nL;
  f.cand = (int *)p; p += nL;
  f.setR = p; p += (int64_t)levels * WR;
  f.setL = p; p += (int64_t)levels * WL;
  f.surv = (int *)p; p += (int64_t)levels * nL;
  f.ns = (int *)p; p += levels;
  f.cur = (int *)p; p += levels;
  return f;
}

// OR the bits m (a subset of v) of HTB word (v, local start pre) into row.
__device__ __forceinline__ void scatter_local(uint32_t *row, int pre, uint32_t v, uint32_t m) {
  while (m) {
    const int b = __ffs(m) - 1;
    m &= m - 1;
    const int pos = pre + __popc(v & ((1u << b) - 1u));
    row[pos >> 5] |= 1u << (pos & 31);
  }
}

// row = (local word list S) & (global HTB slice [g0,g1)), mapped to local bits.
// Walks the shorter side and bisects the longer (htb.py:122-154).
__device__ __forceinline__ void local_row(const uint32_t *s_idx, const uint32_t *s_val,
                                          const int *s_pre, int ns, const uint32_t *__restrict__ gidx,
                                          const uint32_t *__restrict__ gval, int64_t g0, int64_t g1,
                                          uint32_t *row, int W) {
  for (int w = 0; w < W; w++) row[w] = 0;
  if (ns <= g1 - g0) {
    int64_t lo = g0;
    for (int k = 0; k < ns; k++) {
      const uint32_t key = s_idx[k];
      const int64_t j = lower_bound_u32(gidx, lo, g1, key);
      if (j == g1) break;
      if (__ldg(gidx + j) == key) {
        const uint32_t m = s_val[k] & __ldg(gval + j);
        if (m) scatter_local(row, s_pre[k], s_val[k], m);
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
        if (m) scatter_local(row, s_pre[a], s_val[a], m);
        lo = a + 1;
      } else {
        lo = a;
      }
    }
  }
}

// Number of original HTB words (ranges [pre[k], pre[k+1])) a local bitset touches.
__device__ __forceinline__ int words_touched(const uint32_t *set, const int *pre, int nwords) {
  int c = 0;
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
  return __reduce_add_sync(FULL, c);
}

// popcount of a W-word set held in frame memory (warp-cooperative)
__device__ __forceinline__ int set_card(const uint32_t *set, int W) {
  int c = 0;
  for (int w = lane_id(); w < W; w += 32) c += __popc(set[w]);
  return __reduce_add_sync(FULL, c);
}

// order-preserving compaction of the set bits of a W-word set into cand[]
__device__ __forceinline__ int compact_bits(const uint32_t *set, int W, int *cand) {
  const int lane = lane_id();
  int n = 0;
  for (int w = 0; w < W; w++) {
    const uint32_t bits = set[w];
    if (!bits) continue;
    if ((bits >> lane) & 1u) cand[n + __popc(bits & lanemask_lt())] = w * 32 + lane;
    n += __popc(bits);
  }
  __syncwarp();
  return n;
}

template <bool INSTR>
struct Tally {
  unsigned long long batches = 0, inter = 0, opw = 0, minw = 0;
};

// Expand node at `level` (1-based): children at level+1 (engine.py:315-374).
template <bool INSTR>
__device__ __forceinline__ void expand(const Params &P, const Frame &f, int level, int nR, int nL,
                                       int wR1, int wL1, Acc128 &acc, Tally<INSTR> &tl) {
  const int lane = lane_id();
  const int WR = (nR + 31) >> 5, WL = (nL + 31) >> 5;
  const int li = level - 1;
  const uint32_t *R = f.setR + li * WR;
  const uint32_t *Ls = f.setL + li * WL;
  const bool leaf = level + 1 == P.p_eff - 1;
  const int ncand = compact_bits(Ls, WL, f.cand);
  // reference batch accounting (engine.py:306-313, 329-331)
  const int wr = level == 1 ? wR1 : words_touched(R, f.r_pre, wR1);
  const int wl = leaf ? 0 : (level == 1 ? wL1 : words_touched(Ls, f.l_pre, wL1));
  if (lane == 0 && ncand) {
    long long b = 1;
    if (!P.mode_dfs) {
      b = P.cap / (wr > 1 ? wr : 1);
      if (!leaf) {
        long long b2 = P.cap / (wl > 1 ? wl : 1);
        if (b2 < b) b = b2;
      }
      if (b < 1) b = 1;
    }
    tl.batches += (ncand + b - 1) / b;
  }
  int ns = 0;
  const int need_l = P.p_eff - level - 2;  // prune_keep(cr, cl, level+1): cl >= p - (level+1) - 1
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
          const uint32_t *rl = f.rowL + (int64_t)u * WL;
          int cl = 0;
          for (int w = 0; w < WL; w++) cl += __popc(Ls[w] & rl[w]);
          if (INSTR) {
            tl.inter++;
            tl.opw += wl + f.dirw[u];
            tl.minw += wl < f.dirw[u] ? wl : f.dirw[u];
          }
          keep = cl >= need_l;
        }
      }
    }
    if (!leaf) {
      const unsigned m = __ballot_sync(FULL, keep);
      if (keep) f.surv[li * nL + ns + __popc(m & lanemask_lt())] = u;
      ns += __popc(m);
    }
  }
  if (lane == 0) {
    f.ns[li] = ns;
    f.cur[li] = 0;
  }
  __syncwarp();
}

template <bool INSTR>
__global__ void __launch_bounds__(256) enum_kernel(Params P, const Info *__restrict__ info,
                                                   const int32_t *__restrict__ queue,
                                                   int64_t n_alive, int budget_words,
                                                   uint32_t *__restrict__ gscratch,
                                                   int64_t gscratch_words) {
  extern __shared__ uint32_t smem[];
  const int lane = lane_id();
  const int wib = threadIdx.x >> 5;
  const int64_t gwarp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  uint32_t *my_smem = smem + (int64_t)wib * budget_words;
  uint32_t *my_global = gscratch ? gscratch + gwarp * gscratch_words : nullptr;
  Acc128 total{0, 0};
  Tally<INSTR> tl;
  unsigned long long claims = 0, spills = 0;
  const int p_eff = P.p_eff;
  for (;;) {
    long long qi = 0;
    if (lane == 0) qi = (long long)atomicAdd(P.ctr + CTR_NEXT, 1ull);
    qi = __shfl_sync(FULL, qi, 0);
    if (qi >= n_alive) break;
    claims++;
    const int j = queue[qi];
    const int64_t t = P.shard + (int64_t)j * P.nshards;
    const int2 tk = P.tasks[t];
    const Info in = info[j];
    const int nR = in.cr, nL = in.cl, wR1 = in.wr, wL1 = in.wl;
    const int WR = (nR + 31) >> 5, WL = (nL + 31) >> 5;
    const int64_t need = frame_words(nR, nL, wR1, wL1, p_eff, INSTR);
    uint32_t *base;
    if (need <= budget_words) {
      base = my_smem;
    } else {
      base = my_global;
      spills++;
      if (!base || need > gscratch_words) {  // cannot happen: sized from level-1 maxima
        atomicExch(P.overflow, 2);
        continue;
      }
    }
    const Frame f = carve(base, nR, nL, wR1, wL1, p_eff, INSTR);
    // re-materialise C_R1, C_L1 (engine.py:277-292)
    warp_isect_out(P.g.aidx, P.g.aval, P.g.aoff[tk.x], P.g.aoff[tk.x + 1], P.g.aoff[tk.y],
                   P.g.aoff[tk.y + 1], f.r_idx, f.r_val, f.r_pre);
    warp_isect_out(P.g.didx, P.g.dval, P.g.doff[tk.x], P.g.doff[tk.x + 1], P.g.doff[tk.y],
                   P.g.doff[tk.y + 1], f.l_idx, f.l_val, f.l_pre);
    // decode C_L1 ids (ascending, htb.py:42-52)
    for (int k = lane; k < wL1; k += 32) {
      uint32_t v = f.l_val[k];
      const int base_id = (int)f.l_idx[k] * 32;
      int pos = f.l_pre[k];
      while (v) {
        f.lids[pos++] = base_id + __ffs(v) - 1;
        v &= v - 1;
      }
    }
    __syncwarp();
    // task-local rows
    for (int x = lane; x < nL; x += 32) {
      const int id = f.lids[x];
      const int64_t a0 = P.g.aoff[id], a1 = P.g.aoff[id + 1];
      local_row(f.r_idx, f.r_val, f.r_pre, wR1, P.g.aidx, P.g.aval, a0, a1,
                f.rowR + (int64_t)x * WR, WR);
      const int64_t d0 = P.g.doff[id], d1 = P.g.doff[id + 1];
      if (p_eff >= 4)
        local_row(f.l_idx, f.l_val, f.l_pre, wL1, P.g.didx, P.g.dval, d0, d1,
                  f.rowL + (int64_t)x * WL, WL);
      if (INSTR) {
        f.adjw[x] = (int)(a1 - a0);
        f.dirw[x] = (int)(d1 - d0);
      }
    }
    // level-1 node: C_R1, C_L1 = all local ids
    for (int w = lane; w < WR; w += 32) {
      const int rem = nR - w * 32;
      f.setR[w] = rem >= 32 ? FULL : ((1u << rem) - 1u);
    }
    for (int w = lane; w < WL; w += 32) {
      const int rem = nL - w * 32;
      f.setL[w] = rem >= 32 ? FULL : ((1u << rem) - 1u);
    }
    __syncwarp();
    Acc128 acc{0, 0};
    expand<INSTR>(P, f, 1, nR, nL, wR1, wL1, acc, tl);
    int level = 1;
    while (level >= 1) {
      const int li = level - 1;
      if (level + 1 < p_eff - 1 && f.cur[li] < f.ns[li]) {
        const int u = f.surv[li * nL + f.cur[li]];
        __syncwarp();
        if (lane == 0) f.cur[li]++;
        const uint32_t *rr = f.rowR + (int64_t)u * WR;
        const uint32_t *rl = f.rowL + (int64_t)u * WL;
        for (int w = lane; w < WR; w += 32) f.setR[(li + 1) * WR + w] = f.setR[li * WR + w] & rr[w];
        for (int w = lane; w < WL; w += 32) f.setL[(li + 1) * WL + w] = f.setL[li * WL + w] & rl[w];
        __syncwarp();
        level++;
        expand<INSTR>(P, f, level, nR, nL, wR1, wL1, acc, tl);
      } else {
        level--;
      }
    }
    acc = warp_sum128(acc);
    if (lane == 0) {
      total.add(acc.lo, acc.hi);
      if (P.task_counts) {
        P.task_counts[2 * t] = acc.lo;
        P.task_counts[2 * t + 1] = acc.hi;
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    atomic_add128(P.acc, P.overflow, total.lo, total.hi);
    atomicAdd(P.ctr + CTR_BATCHES, tl.batches);
    if (claims > 1) atomicAdd(P.ctr + CTR_STOLEN, claims - 1);
    if (spills) atomicAdd(P.ctr + CTR_SPILL, spills);
  }
  if (INSTR) {
    unsigned long long a = warp_sum(tl.inter), b = warp_sum(tl.opw), c = warp_sum(tl.minw);
    if (lane == 0) {
      atomicAdd(P.ctr + CTR_INTER, a);
      atomicAdd(P.ctr + CTR_OPW, b);
      atomicAdd(P.ctr + CTR_MINW, c);
    }
  }
}

__global__ void iota32(int32_t *a, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int32_t)i;
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

}  // namespace

void search(const DevStructs &s, const bc_config &cfg, bc_report &out) {
  cudaStream_t st = s.stream;
  int device = 0;
  BC_CUDA(cudaGetDevice(&device));
  const int sms = num_sms(device);
  const bool instr = (cfg.flags & BC_FLAG_INSTRUMENT) != 0;
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
  P.g = Graph2{s.hadj_off.p, s.hadj_idx.p, s.hadj_val.p, s.hdir_off.p, s.hdir_idx.p, s.hdir_val.p};
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

  cudaEvent_t e0, e1, e2;
  BC_CUDA(cudaEventCreate(&e0));
  BC_CUDA(cudaEventCreate(&e1));
  BC_CUDA(cudaEventCreate(&e2));
  BC_CUDA(cudaEventRecord(e0, st));
  int64_t n_alive = 0, spills = 0;
  if (nloc > 0) {
    if (s.p_eff == 1) {
      p1_kernel<<<sms * 8, 256, 0, st>>>(P, s.aoff);
      BC_CHECK_LAUNCH();
      launches++;
      BC_CUDA(cudaEventRecord(e1, st));
    } else {
      DBuf<Info> info;
      DBuf<uint32_t> cost;
      info.alloc(nloc, st);
      cost.alloc(nloc, st);
      {
        int64_t blocks = (nloc * 32 + 255) / 256;
        blocks = std::min<int64_t>(blocks, (int64_t)sms * 32);
        if (instr) level1_kernel<true><<<(unsigned)blocks, 256, 0, st>>>(P, info.p, cost.p);
        else level1_kernel<false><<<(unsigned)blocks, 256, 0, st>>>(P, info.p, cost.p);
        BC_CHECK_LAUNCH();
        launches++;
      }
      BC_CUDA(cudaEventRecord(e1, st));
      if (s.p_eff >= 3) {
        unsigned long long h[CTR_COUNT];
        copy_d2h(h, ctr.p, sizeof h, st);
        BC_CUDA(cudaStreamSynchronize(st));
        n_alive = (int64_t)h[CTR_ALIVE];
        const int64_t max_need = (int64_t)h[CTR_MAXNEED];
        if (n_alive > 0) {
          // pre-runtime LPT order: alive tasks by |C_L1|*|C_R1| descending
          DBuf<int32_t> ids, queue;
          DBuf<uint32_t> skeys;
          ids.alloc(nloc, st);
          queue.alloc(nloc, st);
          skeys.alloc(nloc, st);
          iota32<<<(unsigned)((nloc + 255) / 256), 256, 0, st>>>(ids.p, nloc);
          size_t tmp = 0;
          BC_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, cost.p, skeys.p, ids.p,
                                                            queue.p, nloc, 0, 32, st));
          DBuf<char> t;
          t.alloc(tmp, st);
          BC_CUDA(cub::DeviceRadixSort::SortPairsDescending(t.p, tmp, cost.p, skeys.p, ids.p,
                                                            queue.p, nloc, 0, 32, st));
          launches += 2;
          const int threads = 256, wpb = threads / 32;
          const int budget = 2048;  // words of shared memory per warp
          const size_t smem = (size_t)wpb * budget * 4;
          auto kern = instr ? enum_kernel<true> : enum_kernel<false>;
          BC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
          int per_sm = 0;
          BC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
          if (per_sm < 1) per_sm = 1;
          const int64_t blocks = (int64_t)sms * per_sm;
          DBuf<uint32_t> gs;
          int64_t gs_words = 0;
          if (max_need > budget) {
            gs_words = (max_need + 31) & ~int64_t(31);
            gs.alloc((size_t)blocks * wpb * gs_words, st);
          }
          kern<<<(unsigned)blocks, threads, smem, st>>>(P, info.p, queue.p, n_alive, budget,
                                                       gs_words ? gs.p : nullptr, gs_words);
          BC_CHECK_LAUNCH();
          launches++;
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
  if (want_tc)
    copy_d2h(cfg.task_counts, tcounts.p, 2 * n_tasks * sizeof(uint64_t), st);
  BC_CUDA(cudaStreamSynchronize(st));
  float t1 = 0, t2 = 0;
  BC_CUDA(cudaEventElapsedTime(&t1, e0, e1));
  BC_CUDA(cudaEventElapsedTime(&t2, e1, e2));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  if (h_ovf == 2) throw Error(BC_ECUDA, "enumeration frame exceeded its scratch sizing");
  spills = (int64_t)h_ctr[CTR_SPILL];
  (void)spills;
  out.count_lo = h_acc[0];
  out.count_hi = h_acc[1];
  out.overflow = h_ovf ? 1 : 0;
  out.tasks_consumed = nloc;
  out.tasks_alive = n_alive;
  out.tasks_stolen = (int64_t)h_ctr[CTR_STOLEN];
  out.batches_executed = (s.p_eff >= 2 ? nloc : 0) + (int64_t)h_ctr[CTR_BATCHES];
  out.intersections = (int64_t)h_ctr[CTR_INTER];
  out.operand_words = (int64_t)h_ctr[CTR_OPW];
  out.min_words = (int64_t)h_ctr[CTR_MINW];
  out.time_level1 = t1 * 1e-3;
  out.time_enum = t2 * 1e-3;
  out.kernel_launches += launches;
}

}  // namespace bc
