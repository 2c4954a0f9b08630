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
#include <climits>
#include <ctime>
#include <cstdlib>
#include <vector>

#include "search_dev.cuh"

namespace bc {

int64_t debug_phase_cycles(uint64_t *out, int n) {
#ifdef BC_PHASE_PROF
  unsigned long long a[16], b[16];
  sk::phase_cycles_c0(a, true);
  sk::phase_cycles_c1(b, true);
  for (int i = 0; i < n && i < 16; i++) out[i] = a[i] + b[i];
  return 16;
#else
  for (int i = 0; i < n; i++) out[i] = 0;
  return 0;
#endif
}

namespace {
using namespace sk;

// ---------------------------------------------------------------------------
// p_eff = 1: C(deg(root), q) per task (engine.py:267-275)
// ---------------------------------------------------------------------------
__global__ void p1_kernel(Params P, const int64_t *__restrict__ deg_off) {
  Acc128 a{0, 0};
  unsigned long long mine = 0;
  const int64_t nloc = P.n_local;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nloc;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = task_id(P.ltask, P.shard, P.nshards, j);
    const int r = P.tasks[t].x;
    const int d = (int)(deg_off[r + 1] - deg_off[r]);
    mine++;
    if (P.claims) atomicAdd(P.claims + t, 1u);
    Acc128 one{0, 0};
    if (d >= P.q_eff) add_comb(P, one, d);
    if (P.task_counts) {
      P.task_counts[2 * t] = one.lo;
      P.task_counts[2 * t + 1] = one.hi;
    }
    a.add(one);
  }
  a = warp_sum128(a);
  const unsigned long long consumed = warp_sum(mine);
  if (lane_id() == 0) {
    atomic_add128(P.acc, P.overflow, a);
    if (consumed) atomicAdd(P.ctr + CTR_CONSUMED, consumed);
  }
}

// ---------------------------------------------------------------------------
// level 1 (engine.py:265-299 up to the descent)
// ---------------------------------------------------------------------------
template <bool INSTR, int RUN>
__global__ void __launch_bounds__(256) level1_kernel(Params P, Info *__restrict__ info,
                                                     uint32_t *__restrict__ cost) {
  const int lane = lane_id();
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nloc = P.n_local;
  Acc128 a{0, 0};
  unsigned long long alive = 0, inter = 0, opw = 0, minw = 0, maxro = 0, maxscr = 0, claimed = 0;
  // runs of 32 consecutive local tasks per warp: lane k resolves task k's loads (task,
  // list offsets, member-id base) for the run at once, then the warp takes them in turn
  int64_t b_t = 0, b_l0 = 0, b_l1 = 0, b_ab = 0;
  int2 b_tk{0, 0};
  // (RUN = 32 only when there are many tasks per warp: C5's 18.9 M, not C2's 0.7 M)
  for (int64_t j0 = gw * RUN; j0 < nloc; j0 += nw * RUN) {
    const int nrun = (int)min((int64_t)RUN, nloc - j0);
    if (RUN == 1 || lane < nrun) {
      const int64_t jl = RUN == 1 ? j0 : j0 + lane;  // RUN = 1: every lane loads task j0
      b_t = task_id(P.ltask, P.shard, P.nshards, jl);
      b_tk = P.tasks[b_t];
      if (P.lists) {
        b_l0 = P.roff[jl];
        b_l1 = P.roff[jl + 1];
        if (P.roffE) b_ab = P.csr_aoff[b_tk.x] - P.rebase[b_tk.x];
      }
    }
  for (int kk = 0; kk < nrun; kk++) {
    const int64_t j = j0 + kk;
    const int64_t t = RUN == 1 ? b_t : __shfl_sync(FULL, b_t, kk);
    const int2 tk = RUN == 1 ? b_tk : int2{__shfl_sync(FULL, b_tk.x, kk), __shfl_sync(FULL, b_tk.y, kk)};
    claimed++;
    if (P.claims && lane == 0) atomicAdd(P.claims + t, 1u);
    int cr, wr;
    if (P.lists) {  // C_R1 from the wedge-scatter pass: |C_R1| and its HTB word count
      const int64_t l0 = RUN == 1 ? b_l0 : __shfl_sync(FULL, b_l0, kk);
      cr = (int)((RUN == 1 ? b_l1 : __shfl_sync(FULL, b_l1, kk)) - l0);
      const int64_t ab = RUN == 1 ? b_ab : __shfl_sync(FULL, b_ab, kk);
      wr = 0;
      uint32_t last = 0xffffffffu;  // word of the previous batch's last member
      for (int b = 0; b < cr; b += 32) {
        const int i = b + lane;
        uint32_t w = 0xffffffffu;
        if (i < cr) {
          // edge-indexed list: member ids through the anchor CSR
          w = P.roffE ? (uint32_t)__ldg(P.csr_aidx + ab + __ldg(P.lists + l0 + i)) >> 5
                      : (uint32_t)__ldg(P.lists + l0 + i) >> 5;
        }
        uint32_t wp = __shfl_up_sync(FULL, w, 1);
        if (lane == 0) wp = last;
        wr += __popc(__ballot_sync(FULL, i < cr && (i == 0 || wp != w)));
        last = __shfl_sync(FULL, w, 31);
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
          const FrameSpec sp{has_rowL(P.p_eff, P.map_words), true, INSTR, 0};  // upper bound
          const unsigned long long ro = ro_words_any(cr, cl, wr, wl, sp);
          const unsigned long long sc = scratch_words(cr, cl, P.p_eff, sp);
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
    a.add(one);  // lane-uniform: only lane 0 contributes below
  }
  }
  if (lane == 0) {
    atomic_add128(P.acc, P.overflow, a);
    if (alive) atomicAdd(P.ctr + CTR_ALIVE, alive);
    if (claimed) atomicAdd(P.ctr + CTR_CONSUMED, claimed);
    if (INSTR) {
      atomicAdd(P.ctr + CTR_INTER, inter);
      atomicAdd(P.ctr + CTR_OPW, opw);
      atomicAdd(P.ctr + CTR_OPW_L1, opw);
      atomicAdd(P.ctr + CTR_MINW, minw);
    }
    if (maxro) atomicMax(P.ctr + CTR_MAXRO, maxro);
    if (maxscr) atomicMax(P.ctr + CTR_MAXSCR, maxscr);
  }
}

// ---------------------------------------------------------------------------
// check_nesting (engine.py:296-297, 365-366): the reference asserts, for every
// child it expands below level 1, that C_L' = C_L & dir2(u) is a subset of
// dir2(root).  Every deeper C_L is an AND-subset of a level-2 set, so this
// kernel recomputes every level-2 set of every task that descends -- C_L1 =
// dir2(r) & dir2(s) and C_L1 & dir2(x) for each x in C_L1, from the HTB arenas
// with the same warp intersection the search uses -- and checks each id against
// the root's directed 2-hop list by binary search in the CSR (an independent
// path).  Violations and checked ids are tallied; the host raises BC_EASSERT.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) nesting_check(Params P, const Info *__restrict__ info,
                                                     const int64_t *__restrict__ dir_off,
                                                     const int32_t *__restrict__ dir_idx,
                                                     uint32_t *__restrict__ scratch, int64_t maxw) {
  const int lane = lane_id();
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t *c_idx = scratch + gw * 3 * (maxw + 1);
  uint32_t *c_val = c_idx + maxw + 1;
  int *c_pre = (int *)(c_val + maxw + 1);
  unsigned long long bad = 0, checked = 0;
  for (int64_t j = gw; j < P.n_local; j += nw) {
    const Info in = info[j];
    if (in.cr < P.q_eff || in.cl < P.p_eff - 2) continue;  // no descent (prune_keep)
    const int64_t t = task_id(P.ltask, P.shard, P.nshards, j);
    const int2 tk = P.tasks[t];
    int cl = 0;
    const int wl = isect_dir<true>(P.g, tk.x, tk.y, cl, c_idx, c_val, c_pre);
    const int64_t r0 = dir_off[tk.x], r1 = dir_off[tk.x + 1];
    for (int k = 0; k < wl; k++) {
      uint32_t v = c_val[k];
      while (v) {
        const int x = (int)(c_idx[k] * 32u) + __ffs(v) - 1;
        v &= v - 1;
        const int64_t x0 = P.g.doff[x], x1 = P.g.doff[x + 1];
        for (int b = lane; b < wl; b += 32) {
          const uint32_t key = c_idx[b];
          const int64_t i = lower_bound_u32(P.g.didx, x0, x1, key);
          uint32_t w = i < x1 && __ldg(P.g.didx + i) == key ? c_val[b] & __ldg(P.g.dval + i) : 0u;
          while (w) {
            const int id = (int)(key * 32u) + __ffs(w) - 1;
            w &= w - 1;
            int64_t lo = r0, hi = r1;
            while (lo < hi) {
              const int64_t mid = (lo + hi) >> 1;
              if (__ldg(dir_idx + mid) < id) lo = mid + 1;
              else hi = mid;
            }
            checked++;
            if (!(lo < r1 && __ldg(dir_idx + lo) == id)) bad++;
          }
        }
      }
    }
    __syncwarp();
  }
  bad = warp_sum(bad);
  checked = warp_sum(checked);
  if (lane == 0) {
    if (bad) atomicAdd(P.ctr + CTR_NEST_BAD, bad);
    if (checked) atomicAdd(P.ctr + CTR_NEST_CHECKED, checked);
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
// binary search of dir2(r).  The rows of 32 neighbours are walked as one
// flattened list over the lanes (four gathers in flight per lane).  Pass 1
// counts hits per (unit, slot); a column scan turns them into per-task list
// offsets and per-unit cursors; pass 2 appends, ranking the same-slot hits of a
// round by lane (__match_any_sync) so every list comes out sorted.
//
// The same walk also yields the root-restricted rows R(r, v) = N(v) & dir2(r): every
// later wedge walk of a task (r, s) (the survivor counts and candidate rows of
// build_frame_R) only looks for x in C_L1 = dir2(r) & dir2(s), so it can walk R(r, v)
// instead of the whole row N(v) (C5: 4.0e9 instead of 1.7e10 wedges).  Per-edge
// cursors live in shared memory (one per lane's edge of the current 32-edge round);
// a row's order is free, so hits take their places by shared-memory atomics.
// ---------------------------------------------------------------------------
// Rank-order positions inside each root's directed list (for the restricted rows): the
// j-th entry of root r's segment after the sort is the j-th lowest-ranked member of dir2(r).
// pos[ids[i]] = i: a vertex's position in ascending rank order
__global__ void scatter_pos(const int32_t *__restrict__ ids, int64_t n, int64_t *__restrict__ pos) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) pos[ids[i]] = i;
}

// Keys (root << rb) | rank position of every dir2 entry (warp per root): one radix sort by these
// orders each root's list by rank -- cheaper than a segmented sort of 44 K short segments
__global__ void dir_rank_keys64(const int64_t *__restrict__ doff, const int32_t *__restrict__ didx,
                                const int64_t *__restrict__ rpos_of, int64_t n, int rb,
                                unsigned long long *__restrict__ keys, int32_t *__restrict__ vals) {
  const int lane = lane_id();
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw; r < n; r += nw)
    for (int64_t i = doff[r] + lane; i < doff[r + 1]; i += 32) {
      keys[i] = ((unsigned long long)r << rb) | (unsigned long long)rpos_of[didx[i]];
      vals[i] = (int32_t)i;
    }
}

// warp per root: rpos[i] = rank-order position of dir2 entry i inside its root's list,
// rdir[doff[r] + j] = the j-th lowest-ranked member of dir2(r)
__global__ void dir_rank_pos(const int64_t *__restrict__ doff, const int64_t *__restrict__ dend,
                             const int32_t *__restrict__ didx, int64_t n,
                             const int32_t *__restrict__ sorted_vals,
                             int32_t *__restrict__ rpos, int32_t *__restrict__ rdir) {
  const int lane = lane_id();
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw; r < n; r += nw) {
    const int64_t d0 = doff[r], d1 = dend[r];  // roots this rank does not walk: empty
    for (int64_t pidx = d0 + lane; pidx < d1; pidx += 32) {
      const int32_t i = sorted_vals[pidx];
      rpos[i] = (int32_t)(pidx - d0);
      rdir[pidx] = didx[i];
    }
  }
}

struct U32ToI64 {
  __host__ __device__ __forceinline__ int64_t operator()(uint32_t x) const { return (int64_t)x; }
};

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
  unsigned long long *next;
  // root-restricted rows R(r, v) = N(v) & dir2(r) for every edge e = (r, v) of a unit
  // (null: not built).  Pass 1 counts |R(r, v)| into rcnt[e]; pass 2 writes the rows at
  // roffE[e] and, as the C_R1 list entry of task (r, s), the edge index e instead of v
  uint32_t *rcnt;
  const int64_t *__restrict__ roffE;
  int32_t *rrows;  // entries are rank-order positions in dir2(r) (rpos), not anchor ids
  const int32_t *__restrict__ rpos;  // rank-order position of each dir2 entry
  int cur_words;  // pass 2: shared-memory list cursors per warp (0: global cursors)
  const int64_t *__restrict__ rebase;  // per root: first index of its edges in rcnt / roffE
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
  uint32_t *wsm = sm + (int64_t)wib * (mw + (mw + 1) / 2 + 32 + (FILL ? A.cur_words : 0));
  uint32_t *bits = mw ? wsm : nullptr;
  uint16_t *pre = mw ? (uint16_t *)(bits + mw) : nullptr;
  uint32_t *runs = wsm + mw + (mw + 1) / 2;  // R(r, v) cursor of the round's edge base + lane
  uint32_t *ccur = runs + 32;  // pass 2: the unit's list cursors (u32) when they fit
  const bool rr = A.rcnt != nullptr;
  if (bits)
    for (int i = lane; i < mw; i += 32) bits[i] = 0;
  __syncwarp();
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
    const int t0mod = A.nshards > 1 ? (int)(T0 % A.nshards) : 0;  // 32-bit shard test per hit
    unsigned long long *col = A.aux + A.ubase[r] + (int64_t)c * m.D;
    // the unit's cursors in shared memory: the per-hit cursor read is then an LDS, not a
    // dependent global load (list offsets fit u32 when cur_words > 0)
    const bool scur = FILL && m.D <= A.cur_words;
    if (scur) {
      BC_LOOP
      for (int i = lane; i < m.D; i += 32) ccur[i] = (uint32_t)col[i];
      __syncwarp();
    }
    const int64_t e0 = A.aoff[r] + (int64_t)c * L1_CH;
    const int64_t e1 = min(A.aoff[r + 1], e0 + L1_CH);
    // the rows of 32 neighbours at a time as one flattened list over the lanes; rounds of
    // 32 consecutive positions keep the owners (hence v) ascending across the lanes
    for (int64_t base = e0; base < e1; base += 32) {
      const int64_t e = base + lane;
      const int64_t el = rr ? A.rebase[r] + (e - A.aoff[r]) : 0;  // this rank's edge index
      int32_t v = 0;
      int64_t st = 0;
      int len = 0;
      uint32_t rs = 0;  // this lane's edge: R(r, v) start (pass 2)
      if (e < e1) {
        v = __ldg(A.aidx + e);
        st = __ldg(A.boff + v);
        len = (int)(__ldg(A.boff + v + 1) - st);
        if (rr && FILL) rs = (uint32_t)A.roffE[el];
      }
      if (rr) runs[lane] = rs;
      __syncwarp();
      int incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += t;
      }
      const int excl = incl - len;
      const int T = __shfl_sync(FULL, incl, 31);
      constexpr int U = 4;  // gathers in flight per lane
      for (int r0 = 0; r0 < T; r0 += 32 * U) {
        int ks[U], os[U];
        int32_t vs[U];
        int32_t els[U];
#pragma unroll
        for (int uu = 0; uu < U; uu++) {
          const int pos = r0 + 32 * uu + lane;
          int sl = 0;
#pragma unroll
          for (int step = 16; step >= 1; step >>= 1) {
            const int cc = sl + step;
            const int ee = __shfl_sync(FULL, excl, cc < 32 ? cc : 31);
            if (cc < 32 && ee <= pos) sl = cc;
          }
          const int64_t so = __shfl_sync(FULL, st, sl);
          const int eo = __shfl_sync(FULL, excl, sl);
          vs[uu] = __shfl_sync(FULL, v, sl);
          os[uu] = sl;
          if (FILL && rr) els[uu] = __shfl_sync(FULL, (int32_t)el, sl);
          ks[uu] = pos < T ? __ldg(A.bidx + so + (pos - eo)) : -1;
        }
#pragma unroll
        for (int uu = 0; uu < U; uu++) {
          const int kd = ks[uu] >= 0 ? m.slot(ks[uu]) : -1;  // s in dir2(r)
          int k = kd;
          if (k >= 0 && A.nshards > 1 && (t0mod + k) % A.nshards != A.shard) k = -1;
          // R(r, v) of every local edge holds all of dir2(r), whatever the shard; its order
          // is free (the walks only count), so a shared-memory atomic places each hit
          if (rr && kd >= 0) {
            const uint32_t at = atomicAdd(runs + os[uu], 1u);
            if (FILL) A.rrows[at] = __ldg(A.rpos + d0 + kd);
          }
          if (!FILL) {
            if (k >= 0) atomicAdd(col + k, 1ull);
          } else {
            // same-slot hits of this round, ranked by lane (= by ascending v)
            const unsigned grp = __match_any_sync(FULL, k >= 0 ? k : -1 - lane);
            const unsigned long long c0 = k < 0 ? 0ull : scur ? (unsigned long long)ccur[k] : col[k];
            __syncwarp();
            if (k >= 0) {
              const unsigned long long at = c0 + __popc(grp & lanemask_lt());
              // with restricted rows the entry is the edge (r, v): its member id and its row
              // R(r, v) both follow from it, one 4-byte scattered write per entry
              A.lists[at] = rr ? els[uu] : vs[uu];
              if (((grp >> lane) >> 1) == 0) {
                if (scur) ccur[k] = (uint32_t)(c0 + __popc(grp));
                else col[k] = c0 + __popc(grp);
              }
            }
            __syncwarp();
          }
        }
      }
      __syncwarp();
      if (rr && !FILL && e < e1) A.rcnt[el] = runs[lane];
      __syncwarp();
    }
    __syncwarp();  // lanes still probing the map must finish before it is cleared
    rootmap_set(m, false);
  }
}

// per local task: |C_R1| = sum over its root's chunks (pass-1 columns)
__global__ void l1_task_totals(const int2 *__restrict__ tasks, const int64_t *ltask, int64_t nloc,
                               int shard, int nshards,
                               const int64_t *__restrict__ troot, const int64_t *__restrict__ ubase,
                               const int32_t *__restrict__ unit_first, const int64_t *__restrict__ doff,
                               const unsigned long long *__restrict__ aux, int64_t *__restrict__ cnt) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nloc) return;
  const int64_t t = task_id(ltask, shard, nshards, j);
  const int r = tasks[t].x;
  const int64_t k = t - troot[r], D = doff[r + 1] - doff[r];
  const int nch = unit_first[r + 1] - unit_first[r];
  unsigned long long c = 0;
  const unsigned long long *col = aux + ubase[r] + k;
#pragma unroll 8
  for (int ch = 0; ch < nch; ch++) c += col[ch * D];  // independent loads in flight
  cnt[j] = (int64_t)c;
}

// per local task: pass-1 counts -> per-chunk write cursors (list offset + earlier chunks)
__global__ void l1_cursors(const int2 *__restrict__ tasks, const int64_t *ltask, int64_t nloc,
                               int shard, int nshards,
                           const int64_t *__restrict__ troot, const int64_t *__restrict__ ubase,
                           const int32_t *__restrict__ unit_first, const int64_t *__restrict__ doff,
                           const int64_t *__restrict__ roff, unsigned long long *__restrict__ aux) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nloc) return;
  const int64_t t = task_id(ltask, shard, nshards, j);
  const int r = tasks[t].x;
  const int64_t k = t - troot[r], D = doff[r + 1] - doff[r];
  const int nch = unit_first[r + 1] - unit_first[r];
  unsigned long long run = (unsigned long long)roff[j];
  unsigned long long *col = aux + ubase[r] + k;
  int ch = 0;
  for (; ch + 8 <= nch; ch += 8) {  // eight independent loads in flight, then the prefix
    unsigned long long x[8];
#pragma unroll
    for (int u = 0; u < 8; u++) x[u] = col[(ch + u) * D];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      col[(ch + u) * D] = run;
      run += x[u];
    }
  }
  for (; ch < nch; ch++) {
    const unsigned long long x = col[ch * D];
    col[ch * D] = run;
    run += x;
  }
}

// per root: chunks (units) and aux block size (0 for roots without tasks)
__global__ void l1_root_sizes(const int64_t *__restrict__ aoff, const int64_t *__restrict__ doff,
                              const int64_t *__restrict__ troot, int64_t n, int32_t *__restrict__ nunits,
                              int64_t *__restrict__ auxw, int64_t *__restrict__ redges,
                              const int32_t *__restrict__ owner, int shard) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  int32_t nu = 0;
  int64_t w = 0, de = 0;
  const int64_t D = doff[r + 1] - doff[r];
  if (troot[r] >= 0 && D > 0 && (!owner || owner[r] == shard)) {
    const int64_t deg = aoff[r + 1] - aoff[r];
    nu = (int32_t)((deg + L1_CH - 1) / L1_CH);
    w = (int64_t)nu * D;
    de = deg;
  }
  nunits[r] = nu;
  auxw[r] = w;
  redges[r] = de;  // edges this rank walks: restricted rows are indexed by them only
}

// dir2 segments of the roots this rank walks (others empty): the rank-position sort
// covers only those
__global__ void l1_owned_segments(const int64_t *__restrict__ doff, const int32_t *__restrict__ nunits,
                                  int64_t n, int64_t *__restrict__ seg_end) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  seg_end[r] = nunits[r] > 0 ? doff[r + 1] : doff[r];
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
__global__ void l1_probe_cost(const int2 *__restrict__ tasks, const int64_t *ltask, int64_t nloc,
                              int shard, int nshards,
                             const int64_t *__restrict__ hoff, unsigned long long *out) {
  unsigned long long c = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nloc;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int2 tk = tasks[task_id(ltask, shard, nshards, j)];
    const int64_t a = hoff[tk.x + 1] - hoff[tk.x], b = hoff[tk.y + 1] - hoff[tk.y];
    c += (unsigned long long)(a < b ? a : b);
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void l1_pool_sum(const int32_t *__restrict__ pool, const int64_t *__restrict__ troot,
                            int64_t n, unsigned long long *out, const int32_t *__restrict__ owner,
                            int shard) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long c = 0;
  if (r < n && troot[r] >= 0 && (!owner || owner[r] == shard)) c = (unsigned long long)pool[r];
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void l1_pool(const int64_t *__restrict__ aoff, const int32_t *__restrict__ aidx,
                        const int64_t *__restrict__ boff, const int64_t *__restrict__ troot,
                        int64_t n, unsigned long long *out, const int32_t *__restrict__ owner,
                        int shard) {
  // warp per root with tasks: sum of its neighbours' degrees
  const int lane = lane_id();
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long c = 0;
  for (int64_t r = gw; r < n; r += nw) {
    if (troot[r] < 0 || (owner && owner[r] != shard)) continue;
    for (int64_t e = aoff[r] + lane; e < aoff[r + 1]; e += 32) {
      const int v = aidx[e];
      c += (unsigned long long)(boff[v + 1] - boff[v]);
    }
  }
  c = warp_sum(c);
  if (lane == 0 && c) atomicAdd(out, c);
}

// sampled cost of the two candidate-row builds: sum over alive tasks of the C_R1
// members' degrees (wedge scatter) vs 2 * |C_L1| * words(C_R1) (probes)
__global__ void rows_cost(const Info *__restrict__ info, int64_t nloc, int stride,
                          const int64_t *__restrict__ roff, const int32_t *__restrict__ lists,
                          const int64_t *__restrict__ boff, const int64_t *__restrict__ roffE,
                          int p_eff, int q, unsigned long long *out) {
  const int lane = lane_id();
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long sc = 0, pr = 0;
  for (int64_t j = gw * stride; j < nloc; j += nw * stride) {
    const Info in = info[j];
    if (in.cr < q || in.cl < p_eff - 2) continue;
    for (int64_t i = roff[j] + lane; i < roff[j + 1]; i += 32) {
      if (roffE) {  // the walk reads the root-restricted row R(r, v)
        const int64_t e = lists[i];
        sc += (unsigned long long)(roffE[e + 1] - roffE[e]);
      } else {
        const int v = lists[i];
        sc += (unsigned long long)(boff[v + 1] - boff[v]);
      }
    }
    if (lane == 0) pr += 2ull * (unsigned long long)in.cl * (unsigned long long)in.wr;
  }
  sc = warp_sum(sc);
  if (lane == 0) {
    atomicAdd(out, sc);
    atomicAdd(out + 1, pr);
  }
}

// root sharding: keys |tasks| x (degree + 1) (0 for roots without tasks), snake owners
__global__ void root_keys(const int64_t *__restrict__ aoff, const int64_t *__restrict__ doff,
                          const int64_t *__restrict__ troot, int64_t n,
                          unsigned long long *__restrict__ keys, int32_t *__restrict__ ids) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const unsigned long long d = (unsigned long long)(doff[r + 1] - doff[r]);
  keys[r] = troot[r] >= 0 ? d * (unsigned long long)(aoff[r + 1] - aoff[r] + 1) : 0ull;
  ids[r] = (int32_t)r;
}

__global__ void snake_owner(const int32_t *__restrict__ sorted, int64_t n, int nshards,
                            int32_t *__restrict__ owner) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t round = i / nshards, pos = i % nshards;
  owner[sorted[i]] = (int32_t)(round & 1 ? nshards - 1 - pos : pos);
}

__global__ void local_task_flags(const int2 *__restrict__ tasks, int64_t n_tasks,
                                 const int32_t *__restrict__ owner, int shard,
                                 int64_t *__restrict__ tids, uint8_t *__restrict__ flags) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_tasks) return;
  tids[t] = t;
  flags[t] = owner[tasks[t].x] == shard;
}

__global__ void alive_flags(const uint32_t *cost, int64_t n, uint8_t *flags) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) flags[i] = cost[i] != 0;
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
// frame and sub-task arena words of queue[q0, q1): rows and split-level nodes are
// bounded by the level-1 survivor count when triage measured it (caps), else |C_L1|
__global__ void split_sizes(const Info *info, const int32_t *queue, const int32_t *caps,
                            int64_t q0, int64_t q1, bool instr, bool compact, int split_level,
                            int64_t *ro, int64_t *sub) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= q1 - q0) return;
  const Info in = info[queue[q0 + i]];
  const int cap = caps ? caps[q0 + i] : 0;
  const FrameSpec sp{true, compact, instr, cap};
  ro[i] = ro_words(in.cr, in.cl, in.wr, in.wl, sp);
  const int64_t WR = (in.cr + 31) / 32, WL = (in.cl + 31) / 32, ns = sp.rows(in.cl);
  const int64_t nodes = split_level == 2 ? ns : ns * (ns - 1) / 2;
  sub[i] = nodes * (4 + WR + WL);
}

__global__ void gather2(const int32_t *perm, int64_t n, const int32_t *a, const int32_t *b,
                        int32_t *oa, int32_t *ob) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    oa[i] = a[perm[i]];
    ob[i] = b[perm[i]];
  }
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
  // candidates below the node ~ |L|^2 |R|, each an AND over the task's WR + WL words
  const unsigned long long k =
      (unsigned long long)cl * cl * (cr ? cr : 1) * (unsigned long long)(WR + WL) / 4 + 1;
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

// ---------------------------------------------------------------------------
// Level-1 survivor filter on the restricted rows (p_eff >= 5, wedge-scatter level 1).
// A task (r, s) has a level-1 R-survivor x iff x is in C_L1 = dir2(r) & dir2(s) and
// |N(x) & C_R1| >= q (engine.py:331-338).  dir2(s) = {x : |N(x) & N(s)| >= q,
// rank(x) < rank(s)} (graph.py:192-224, k = q_eff, engine.py:127-135) and C_R1 is a
// subset of N(s), so for x in dir2(r): x survives iff rank(x) < rank(s) and
// |N(x) & C_R1| >= q.  The rows R(r, v) hold rank-order positions in dir2(r), so the
// test is `position < position of s` and the counters are indexed by position: no
// C_L1 intersection, no slot map, no HTB words.  Counters are u16 pairs in shared
// memory (a carry into the neighbour only adds false survivors, which the triage
// kernel re-checks exactly; a count is flagged the moment it reaches q < 2^16).
// Tasks without a survivor finish here (their level-1 batch is their only work);
// the others go to the medium list as before.
// ---------------------------------------------------------------------------
constexpr int RF_THREADS = 256;
constexpr int RF_RUN = 32;  // tasks claimed per warp at a time

__global__ void __launch_bounds__(RF_THREADS, 4) rfilter_kernel(Params P, EnumArgs A,
                                                               int budget_words) {
  extern __shared__ uint32_t smem[];
  const int lane = lane_id();
  uint32_t *cnt = smem + (int64_t)(threadIdx.x >> 5) * budget_words;
  Tally tl;
  Acc128 total{0, 0, 0};
  unsigned long long claims = 0;
  const int q = P.q_eff;
  // tasks are claimed RF_RUN at a time and lane k resolves task k's chain of dependent
  // loads (queue -> task -> root offsets -> rank position, list offset, level-1 facts)
  // for the whole run at once; the warp then takes the run's tasks one by one
  int nb = 0, k = 0;
  int b_j = 0, b_rps = 0;
  int64_t b_t = 0, b_l0 = 0;
  int b_nR = 0, b_nL = 0, b_wR = 0, b_wL = 0;
  BC_LOOP
  for (;;) {
    if (k >= nb) {
      long long q0 = 0;
      if (lane == 0) q0 = (long long)atomicAdd(P.ctr + CTR_NEXT, (unsigned long long)RF_RUN);
      q0 = __shfl_sync(FULL, q0, 0) + A.q0;
      if (q0 >= A.q1) break;
      nb = (int)min((long long)RF_RUN, A.q1 - q0);
      k = 0;
      if (lane < nb) {
        b_j = A.queue[q0 + lane];
        b_t = task_id(P.ltask, P.shard, P.nshards, b_j);
        const int br = P.tasks[b_t].x;
        b_rps = P.rpos[P.dir_off[br] + (b_t - P.troot[br])];
        b_l0 = P.roff[b_j];
        const Info in = A.info[b_j];
        b_nR = in.cr;
        b_nL = in.cl;
        b_wR = in.wr;
        b_wL = in.wl;
      }
    }
    claims++;
    const int j = __shfl_sync(FULL, b_j, k);
    const int64_t t = __shfl_sync(FULL, b_t, k);
    const int rps = __shfl_sync(FULL, b_rps, k);  // candidates: positions [0, rps)
    const int64_t lbase = __shfl_sync(FULL, b_l0, k);
    const Dims d = dims_of(Info{__shfl_sync(FULL, b_nR, k), __shfl_sync(FULL, b_wR, k),
                                __shfl_sync(FULL, b_nL, k), __shfl_sync(FULL, b_wL, k)});
    k++;
    bool surv = false;
    if (rps > 2 * budget_words) {
      surv = true;  // counters do not fit: the triage kernel decides
    } else if (rps > 0) {
      BC_LOOP
      for (int w = lane; w < (rps + 1) / 2; w += 32) cnt[w] = 0;
      __syncwarp();
      BC_LOOP
      for (int b0 = 0; b0 < d.nR && !surv; b0 += 32) {
        const int i = b0 + lane;
        int64_t start = 0;
        int len = 0;
        if (i < d.nR) {
          const int64_t e = __ldg(P.lists + lbase + i);
          start = __ldg(P.roffE + e);
          len = (int)(__ldg(P.roffE + e + 1) - start);
        }
        int incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int tt = __shfl_up_sync(FULL, incl, o);
          if (lane >= o) incl += tt;
        }
        const int excl = incl - len;
        const int T = __shfl_sync(FULL, incl, 31);
        constexpr int U = 4;  // gathers in flight per lane
        BC_LOOP
        for (int r0 = 0; r0 < T; r0 += 32 * U) {
          int xs[U];
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
            xs[u] = pos < T ? __ldg(P.rrows + st + (pos - ex)) : INT_MAX;
          }
          bool hit = false;
#pragma unroll
          for (int u = 0; u < U; u++) {
            const int x = xs[u];
            if (x < rps) {
              const int sh = (x & 1) * 16;
              const uint32_t old = atomicAdd(cnt + (x >> 1), 1u << sh);
              hit |= ((old >> sh) & 0xffffu) + 1 >= (uint32_t)q;
            }
          }
          if (__any_sync(FULL, hit)) {
            surv = true;
            break;
          }
        }
      }
      __syncwarp();
    }
    if (!surv) {
      if (lane == 0) tl.batches += node_batches(P, (unsigned)d.nL, d.wR, d.wL, P.p_eff == 3);
      finish_task(P, Acc128{0, 0, 0}, t, false, total);
    } else if (lane == 0) {
      push_heavy(P, A, j, 0);
    }
    __syncwarp();
  }
  flush_tallies(P, total, tl, claims, 0, false);
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
  int64_t nloc = n_tasks > shard ? (n_tasks - shard + nshards - 1) / nshards : 0;
  int64_t launches = 0;
  // Multi-GPU sharding: by root, degree-balanced -- roots ordered by
  // |tasks| x (degree + 1) and dealt in snake order, each shard keeps whole roots, so the
  // level-1 wedge walk of a root runs on one GPU only -- or, with BC_FLAG_TASK_SHARD,
  // task-interleaved (t % shards).  Either way the shard counts sum to the total.
  DBuf<int32_t> owner;
  DBuf<int64_t> ltask;
  if (nshards > 1 && !(cfg.flags & BC_FLAG_TASK_SHARD) && s.n > 0 && n_tasks > 0) {
    const int64_t n = s.n;
    DBuf<unsigned long long> keys, skeys;
    DBuf<int32_t> ids, sids;
    keys.alloc(n, st);
    skeys.alloc(n, st);
    ids.alloc(n, st);
    sids.alloc(n, st);
    owner.alloc(n, st);
    root_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s.aoff, s.dir_off.p, s.troot.p, n,
                                                           keys.p, ids.p);
    sort_pairs_desc(keys.p, skeys.p, ids.p, sids.p, n, st);
    snake_owner<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(sids.p, n, nshards, owner.p);
    DBuf<int64_t> tids;
    DBuf<uint8_t> flags;
    DBuf<int64_t> nsel;
    tids.alloc(n_tasks, st);
    flags.alloc(n_tasks, st);
    ltask.alloc(n_tasks, st);
    nsel.alloc(1, st);
    local_task_flags<<<(unsigned)((n_tasks + 255) / 256), 256, 0, st>>>(s.tasks.p, n_tasks,
                                                                         owner.p, shard, tids.p,
                                                                         flags.p);
    size_t tmp = 0;
    BC_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, tids.p, flags.p, ltask.p, nsel.p, n_tasks, st));
    DBuf<char> tb;
    tb.alloc(tmp, st);
    BC_CUDA(cub::DeviceSelect::Flagged(tb.p, tmp, tids.p, flags.p, ltask.p, nsel.p, n_tasks, st));
    copy_d2h(&nloc, nsel.p, sizeof nloc, st);
    BC_CUDA(cudaStreamSynchronize(st));
    launches += 6;
  }

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
  DBuf<uint32_t> claims;
  const bool want_claims = (cfg.flags & BC_FLAG_TRACK_TASKS) && cfg.task_claims;
  if (want_claims) {
    if (cfg.task_claims_cap < n_tasks) throw Error(BC_EINVAL, "task_claims buffer too small");
    claims.alloc((size_t)(n_tasks ? n_tasks : 1), st);
    claims.zero();
  }
  Params P;
  P.g = Graph2{s.hadj_off.p, s.hadj_idx.p, s.hadj_val.p, s.hdir_off.p, s.hdir_idx.p, s.hdir_val.p,
               s.dense_id.p, s.dense.p, s.dense_mw, s.boff, s.bidx};
  P.tasks = s.tasks.p;
  P.n_tasks = n_tasks;
  P.n_local = nloc;
  P.ltask = ltask.p;
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
  P.claims = want_claims ? claims.p : nullptr;
  P.roff = nullptr;
  P.lists = nullptr;
  P.roffE = nullptr;
  P.rebase = nullptr;
  P.csr_aoff = nullptr;
  P.csr_aidx = nullptr;
  P.rrows = nullptr;
  P.rdir = nullptr;
  P.rpos = nullptr;
  P.dir_off = nullptr;
  P.troot = nullptr;
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
  int64_t n_alive = 0, n_split = 0, n_sub_total = 0, l1_entries = 0;
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
    DBuf<uint32_t> rr_cnt;  // root-restricted rows (l1_scatter)
    DBuf<int64_t> rr_ebase;
    DBuf<int64_t> rr_off;
    DBuf<int32_t> rr_rows;
    DBuf<int32_t> rr_rpos, rr_rdir;  // rank-order positions / dir2 lists in rank order
    int l1_mode = (cfg.flags & BC_FLAG_L1_SCATTER) ? 1 : (cfg.flags & BC_FLAG_L1_PROBE) ? 2 : 0;
    if (l1_mode == 0) {
      DBuf<unsigned long long> c2;
      c2.alloc(2, st);
      c2.zero();
      l1_probe_cost<<<sms * 8, 256, 0, st>>>(s.tasks.p, ltask.p, nloc, shard, nshards,
                                             s.hadj_off.p, c2.p);
      if (s.pool.p) {  // the pools the 2-hop construction measured
        l1_pool_sum<<<(unsigned)((s.n + 255) / 256), 256, 0, st>>>(s.pool.p, s.troot.p, s.n,
                                                                  c2.p + 1, owner.p, shard);
      } else {
        l1_pool<<<sms * 8, 256, 0, st>>>(s.aoff, s.aidx, s.boff, s.troot.p, s.n, c2.p + 1,
                                         owner.p, shard);
      }
      BC_CHECK_LAUNCH();
      unsigned long long hc[2];
      copy_d2h(hc, c2.p, sizeof hc, st);
      BC_CUDA(cudaStreamSynchronize(st));
      launches += 2;
      // the scatter walks each pool ~4 times (count, mask, write, cursor) with an
      // atomic per hit; a probe word is a short bisect in L2.  Measured break-even
      // is near pool ~ probe / 8 (C2 probes, C5 scatters)
      l1_mode = 8.0 * (double)hc[1] < (double)hc[0] ? 1 : 2;
      if (getenv("BC_DEBUG"))
        fprintf(stderr, "[bc level1] probe words %llu  pool %llu  -> %s\n", hc[0], hc[1],
                l1_mode == 1 ? "scatter" : "probe");
    }
    DbgTimer dt(st);
    if (l1_mode == 1) {
      const int64_t n = s.n;
      DBuf<int32_t> nunits, unit_first, unit_root;
      DBuf<int64_t> auxw, ubase, redges;
      nunits.alloc(n + 1, st);
      auxw.alloc(n + 1, st);
      redges.alloc(n + 1, st);
      nunits.zero();
      auxw.zero();
      redges.zero();
      l1_root_sizes<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
          s.aoff, s.dir_off.p, s.troot.p, n, nunits.p, auxw.p, redges.p, owner.p, shard);
      unit_first.alloc(n + 1, st);
      ubase.alloc(n + 1, st);
      rr_ebase.alloc(n + 1, st);
      scan_excl(nunits.p, unit_first.p, n + 1, st);
      scan_excl(auxw.p, ubase.p, n + 1, st);
      scan_excl(redges.p, rr_ebase.p, n + 1, st);
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
      A1.shard = owner.p ? 0 : shard;  // root sharding: every slot of an owned root is local
      A1.nshards = owner.p ? 1 : nshards;
      A1.next = nxt.p;
      // root-restricted rows for the compact frames' wedge walks (slot map needed, p_eff >= 4)
      const bool want_rr = s.p_eff >= 4 && (s.n + 31) / 32 <= 4096 &&
                           !(cfg.flags & BC_FLAG_FULL_ROWS);
      int64_t n_anchor_edges = 0;  // edges of the roots this rank walks
      if (want_rr) {
        copy_d2h(&n_anchor_edges, rr_ebase.p + n, sizeof n_anchor_edges, st);
        BC_CUDA(cudaStreamSynchronize(st));
        A1.rebase = rr_ebase.p;
        rr_cnt.alloc(n_anchor_edges, st);
        rr_cnt.zero();
        A1.rcnt = rr_cnt.p;
        // rank-order positions: restricted rows hold them, so a task (r, s) finds the
        // candidates x with rank(x) < rank(s) by comparing positions (rfilter_kernel)
        const int64_t D = s.dir2_pairs;
        rr_rpos.alloc(D, st);
        rr_rdir.alloc(D, st);
        {
          DBuf<unsigned long long> k0, k1;
          DBuf<int32_t> v0, v1;
          k0.alloc(D, st);
          k1.alloc(D, st);
          v0.alloc(D, st);
          v1.alloc(D, st);
          // dense rank positions 0..n-1 of the anchors (rank overrides, e.g. a partitioned
          // count's global ranks, can be any distinct int64s): one small sort of the ranks
          DBuf<int64_t> dpos, rk2;
          DBuf<int32_t> vid, vid2;
          dpos.alloc(n, st);
          rk2.alloc(n, st);
          vid.alloc(n, st);
          vid2.alloc(n, st);
          iota32<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(vid.p, n);
          {
            size_t t0 = 0;
            BC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t0, s.rank.p, rk2.p, vid.p, vid2.p, n,
                                                    0, 64, st));
            DBuf<char> tb0;
            tb0.alloc(t0, st);
            BC_CUDA(cub::DeviceRadixSort::SortPairs(tb0.p, t0, s.rank.p, rk2.p, vid.p, vid2.p, n,
                                                    0, 64, st));
          }
          scatter_pos<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(vid2.p, n, dpos.p);
          int rb = 1;  // bits of a rank position (< n)
          while ((int64_t(1) << rb) < n) rb++;
          int nb = 1;  // bits of a root id
          while ((int64_t(1) << nb) < n) nb++;
          dir_rank_keys64<<<sms * 8, 256, 0, st>>>(s.dir_off.p, s.dir_idx.p, dpos.p, n, rb, k0.p,
                                                   v0.p);
          DBuf<int64_t> seg_end;
          seg_end.alloc(n, st);
          l1_owned_segments<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s.dir_off.p, nunits.p, n,
                                                                        seg_end.p);
          size_t tmp = 0;
          BC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0.p, k1.p, v0.p, v1.p, D, 0,
                                                  rb + nb, st));
          DBuf<char> tb;
          tb.alloc(tmp, st);
          BC_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, tmp, k0.p, k1.p, v0.p, v1.p, D, 0, rb + nb,
                                                  st));
          dir_rank_pos<<<sms * 8, 256, 0, st>>>(s.dir_off.p, seg_end.p, s.dir_idx.p, n, v1.p,
                                                rr_rpos.p, rr_rdir.p);
          BC_CHECK_LAUNCH();
          launches += 3;
        }
        A1.rpos = rr_rpos.p;
      }
      const int l1w = L1_THREADS / 32;
      const size_t l1smem = (size_t)l1w * (A1.map_words + (A1.map_words + 1) / 2 + 32) * 4;
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
          s.tasks.p, ltask.p, nloc, shard, nshards, s.troot.p, ubase.p, unit_first.p,
          s.dir_off.p, aux.p, cnt.p);
      l1_roff.alloc(nloc + 1, st);
      scan_excl(cnt.p, l1_roff.p, nloc + 1, st);
      int64_t n_entries = 0;
      copy_d2h(&n_entries, l1_roff.p + nloc, sizeof n_entries, st);
      BC_CUDA(cudaStreamSynchronize(st));
      l1_lists.alloc(n_entries, st);
      l1_entries = n_entries;
      if (A1.rcnt) {
        // restricted-row offsets; the per-entry row starts are u32 (else: whole rows)
        const int64_t E = n_anchor_edges;
        rr_off.alloc(E + 1, st);
        U32ToI64 cv;
        cub::TransformInputIterator<int64_t, U32ToI64, const uint32_t *> it(rr_cnt.p, cv);
        size_t tmp = 0;
        BC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, it, rr_off.p + 1, E, st));
        DBuf<char> tb;
        tb.alloc(tmp, st);
        BC_CUDA(cub::DeviceScan::InclusiveSum(tb.p, tmp, it, rr_off.p + 1, E, st));
        BC_CUDA(cudaMemsetAsync(rr_off.p, 0, sizeof(int64_t), st));
        int64_t rr_total = 0;
        copy_d2h(&rr_total, rr_off.p + E, sizeof rr_total, st);
        BC_CUDA(cudaStreamSynchronize(st));
        launches += 2;
        if (rr_total < (int64_t(1) << 32) && E < (int64_t(1) << 31)) {
          rr_rows.alloc(rr_total, st);
          A1.roffE = rr_off.p;
          A1.rrows = rr_rows.p;
          if (getenv("BC_DEBUG"))
            fprintf(stderr, "[bc level1] restricted rows: %lld entries\n", (long long)rr_total);
        } else {
          A1.rcnt = nullptr;
        }
      }
      l1_cursors<<<(unsigned)((nloc + 255) / 256), 256, 0, st>>>(
          s.tasks.p, ltask.p, nloc, shard, nshards, s.troot.p, ubase.p, unit_first.p,
          s.dir_off.p, l1_roff.p, aux.p);
      A1.lists = l1_lists.p;
      A1.next = nxt.p + 1;
#ifndef L1_CUR_WORDS
#define L1_CUR_WORDS 512
#endif
      A1.cur_words = n_entries < (int64_t(1) << 32) ? (int)std::min<unsigned long long>(maxD, L1_CUR_WORDS) : 0;
      const size_t l1smem2 = l1smem + (size_t)l1w * A1.cur_words * 4;
      BC_CUDA(cudaFuncSetAttribute(l1_scatter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)l1smem2));
      int per_sm2 = 0;
      BC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, l1_scatter<true>, L1_THREADS,
                                                            l1smem2));
      const int64_t l1blocks2 = (int64_t)sms * std::max(per_sm2, 1);
      dt.mark("l1 offsets");
      l1_scatter<true><<<(unsigned)l1blocks2, L1_THREADS, l1smem2, st>>>(A1);
      BC_CHECK_LAUNCH();
      dt.mark("l1 fill");
      launches += 12;
      P.roff = l1_roff.p;
      P.lists = l1_lists.p;
      if (A1.rcnt) {
        P.roffE = rr_off.p;
        P.rebase = rr_ebase.p;
        P.csr_aoff = s.aoff;
        P.csr_aidx = s.aidx;
        P.rrows = rr_rows.p;
        P.rdir = rr_rdir.p;
        P.rpos = rr_rpos.p;
        P.dir_off = s.dir_off.p;
        P.troot = s.troot.p;
      }
      if (getenv("BC_DEBUG")) {
        BC_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "[bc level1] scatter: %d units, %lld aux, %lld C_R1 entries\n", n_units,
                (long long)aux_total, (long long)n_entries);
      }
    }
    {
      int64_t blocks = (nloc * 32 + 255) / 256;
      blocks = std::min<int64_t>(blocks, (int64_t)sms * 32);
      const bool runs = nloc >= blocks * 8 * 128;  // many tasks per warp: batched loads
      if (instr && runs) level1_kernel<true, 32><<<(unsigned)blocks, 256, 0, st>>>(P, info.p, cost.p);
      else if (instr) level1_kernel<true, 1><<<(unsigned)blocks, 256, 0, st>>>(P, info.p, cost.p);
      else if (runs) level1_kernel<false, 32><<<(unsigned)blocks, 256, 0, st>>>(P, info.p, cost.p);
      else level1_kernel<false, 1><<<(unsigned)blocks, 256, 0, st>>>(P, info.p, cost.p);
      BC_CHECK_LAUNCH();
      dt.mark("level1_kernel");
      launches++;
    }
    BC_CUDA(cudaEventRecord(e1, st));
    if ((cfg.flags & BC_FLAG_CHECK_NESTING) && s.p_eff >= 4) {
      const int64_t maxw = std::max<int64_t>(s.max_dir_slice, 1);
      const int nb = sms * 2;
      DBuf<uint32_t> scr;
      scr.alloc((size_t)nb * 8 * 3 * (maxw + 1), st);
      nesting_check<<<nb, 256, 0, st>>>(P, info.p, s.dir_off.p, s.dir_idx.p, scr.p, maxw);
      BC_CHECK_LAUNCH();
      launches++;
    }
    if (s.p_eff >= 3) {
      unsigned long long h[CTR_COUNT];
      copy_d2h(h, ctr.p, sizeof h, st);
      BC_CUDA(cudaStreamSynchronize(st));
      n_alive = (int64_t)h[CTR_ALIVE];
      const int64_t max_ro = (int64_t)h[CTR_MAXRO], max_scr = (int64_t)h[CTR_MAXSCR];
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
        // candidate rows: wedge-scattered for the level-1 survivors (compact) when the
        // sampled sum of C_R1 members' degrees beats ~2 probes per (candidate, C_R1 word)
        bool compact = false;
        if (P.map_words > 0) {
          if (P.rowR_mode == 1) {
            compact = true;
          } else if (P.rowR_mode == 0 && P.lists) {
            DBuf<unsigned long long> rc;
            rc.alloc(2, st);
            rc.zero();
            const int stride = nloc > (int64_t(1) << 20) ? 16 : 1;
            rows_cost<<<(unsigned)std::min<int64_t>((nloc / stride * 32 + 255) / 256 + 1, sms * 16), 256,
                        0, st>>>(info.p, nloc, stride, P.roff, P.lists, s.boff, P.roffE, s.p_eff,
                                 s.q_eff, rc.p);
            unsigned long long hc[2];
            copy_d2h(hc, rc.p, sizeof hc, st);
            BC_CUDA(cudaStreamSynchronize(st));
            launches++;
            compact = hc[0] < hc[1];
            if (dt.on)
              fprintf(stderr, "[bc search] rows: scatter %llu vs probe %llu -> %s\n", hc[0], hc[1],
                      compact ? "compact" : "full");
          }
        }
        auto eblocks = [&](const EnumVariant &v, size_t sm) {
          return compact ? enum_blocks_per_sm_c1(v, sm) : enum_blocks_per_sm_c0(v, sm);
        };
        auto elaunch = [&](const EnumVariant &v, unsigned b, size_t sm, const Params &p,
                           const EnumArgs &a) {
          if (compact) enum_launch_c1(v, b, sm, st, p, a);
          else enum_launch_c0(v, b, sm, st, p, a);
        };
        if (!split) {
          // whole tasks per warp; frames in shared memory
          const bool lazy = s.p_eff == 4 && !has_rowL(s.p_eff, P.map_words);
          const int budget = 1200;  // frame words per warp (measured optimum on C2, p_eff = 4)
          const size_t smem = (size_t)wpb * (budget + map_w + LEAF_WORDS) * 4;
          const EnumVariant ev{instr, lazy, false, false};
          const int64_t blocks = (int64_t)sms * eblocks(ev, smem);
          A.q0 = 0;
          A.q1 = n_alive;
          A.budget_words = budget;
          DBuf<uint32_t> gs;
          if (max_ro + max_scr > budget) {
            A.gscratch_words = (max_ro + max_scr + 31) & ~int64_t(31);
            gs.alloc((size_t)blocks * wpb * A.gscratch_words, st);
            A.gscratch = gs.p;
          }
          elaunch(ev, (unsigned)blocks, smem, P, A);
          launches++;
        } else {
          // triage (p_eff >= 5): every task is started whole by one warp; a task with
          // at most T level-1 R-survivors (whose frame fits the scratch) finishes in
          // place, the rest are deferred, heaviest first, to the split path below.
          int64_t n_heavy = n_alive;
          const int32_t *hq_p = queue.p, *hcap_p = nullptr;
          DBuf<int32_t> heavy, heavy_ns1, hq, hcap;
          // triage only when splitting everything would not fit one frame arena
          // (millions of mostly light tasks, e.g. C5); C3/C4-sized queues split all
          // level-1 survivors a triaged task may have before it goes to the split path:
          // 10 measured best (C5 enumeration 118.6 ms at 16 -> 109.5 ms; C5H 9.14 -> 7.92 s)
          int T = 10;
          if (!(cfg.flags & BC_FLAG_FORCE_TRIAGE)) {
            DBuf<int64_t> ro_all, sub_all, sum;
            ro_all.alloc(n_alive, st);
            sub_all.alloc(n_alive, st);
            sum.alloc(1, st);
            split_sizes<<<(unsigned)((n_alive + 255) / 256), 256, 0, st>>>(
                info.p, queue.p, nullptr, 0, n_alive, instr, compact, s.p_eff <= 6 ? 2 : 3,
                ro_all.p, sub_all.p);
            size_t tmp = 0;
            BC_CUDA(cub::DeviceReduce::Sum(nullptr, tmp, ro_all.p, sum.p, n_alive, st));
            DBuf<char> tb;
            tb.alloc(tmp, st);
            BC_CUDA(cub::DeviceReduce::Sum(tb.p, tmp, ro_all.p, sum.p, n_alive, st));
            int64_t frames_total = 0;
            copy_d2h(&frames_total, sum.p, 8, st);
            BC_CUDA(cudaStreamSynchronize(st));
            launches += 2;
            // (or when the queue is long: a shard of C5 is 2.4 M mostly light tasks)
            if (frames_total <= (int64_t(1) << 28) && n_alive <= (int64_t(1) << 18)) T = 0;
          }
          if (T > 0) {
            const int budget = 1024;
            const size_t smem = (size_t)wpb * (budget + map_w + LEAF_WORDS) * 4;
            const EnumVariant ev{instr, false, false, true};
            const int64_t blocks = (int64_t)sms * eblocks(ev, smem);
            heavy.alloc(n_alive, st);
            heavy_ns1.alloc(n_alive, st);
            EnumArgs B = A;
            B.q0 = 0;
            B.q1 = n_alive;
            // triage drains the alive tasks in emission order: the tasks of one root are
            // adjacent, so their C_R1 members' rows (all in N(root)) are re-read from L2
            DBuf<int32_t> tq;
            {
              DBuf<int32_t> ids;
              DBuf<uint8_t> flags;
              DBuf<int64_t> nsel;
              ids.alloc(nloc, st);
              flags.alloc(nloc, st);
              tq.alloc(nloc, st);
              nsel.alloc(1, st);
              iota32<<<(unsigned)((nloc + 255) / 256), 256, 0, st>>>(ids.p, nloc);
              alive_flags<<<(unsigned)((nloc + 255) / 256), 256, 0, st>>>(cost.p, nloc, flags.p);
              size_t tmp = 0;
              BC_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, ids.p, flags.p, tq.p, nsel.p, nloc,
                                                 st));
              DBuf<char> tb;
              tb.alloc(tmp, st);
              BC_CUDA(cub::DeviceSelect::Flagged(tb.p, tmp, ids.p, flags.p, tq.p, nsel.p, nloc,
                                                 st));
              B.queue = tq.p;
              launches += 3;
            }
            B.budget_words = budget;
            B.triage = T;
            B.triage_work = 1 << 16;  // expansion budget before a task is deferred
            B.heavy = heavy.p;
            B.heavy_ns1 = heavy_ns1.p;
            DBuf<uint32_t> gs;
            if (max_ro + max_scr > budget) {
              // per-warp frame scratch, capped at 4 GiB in total (larger frames defer)
              int64_t w = (max_ro + max_scr + 31) & ~int64_t(31);
              const int64_t cap_w = ((int64_t(1) << 30) / (blocks * wpb)) & ~int64_t(31);
              B.gscratch_words = std::min(w, cap_w);
              gs.alloc((size_t)blocks * wpb * B.gscratch_words, st);
              B.gscratch = gs.p;
            }
            DBuf<int32_t> medium, medium_ns1;
            if (!instr) {
              // filter: tasks without level-1 survivors finish in a small kernel; the
              // rest (the medium list) go through the triage kernel
              const size_t fsmem = (size_t)wpb * (budget + map_w) * 4;
              const int64_t fblocks =
                  (int64_t)sms * (compact ? filter_blocks_per_sm_c1(fsmem) : filter_blocks_per_sm_c0(fsmem));
              medium.alloc(n_alive, st);
              medium_ns1.alloc(n_alive, st);
              EnumArgs F = B;
              F.heavy = medium.p;
              F.heavy_ns1 = medium_ns1.p;
              // the filter's frames are the first half only (C_R1, C_L1, ids, counters);
              // its own per-warp scratch when it runs more warps than the triage kernel
              DBuf<uint32_t> fgs;
              if (B.gscratch && fblocks > blocks) {
                const int64_t w = (max_ro + 31) & ~int64_t(31);
                const int64_t cap_w = ((int64_t(1) << 30) / (fblocks * wpb)) & ~int64_t(31);
                F.gscratch_words = std::min(w, cap_w);
                fgs.alloc((size_t)fblocks * wpb * F.gscratch_words, st);
                F.gscratch = fgs.p;
              }
              BC_CUDA(cudaMemsetAsync(ctr.p + CTR_NEXT, 0, 8, st));
              BC_CUDA(cudaMemsetAsync(ctr.p + CTR_HEAVY, 0, 8, st));
              dt.mark("pre-filter");
              if (P.roffE && s.q_eff < 65536) {
                // restricted rows: the rank-position filter (no frames, no slot map)
                const int rbudget = 1024;  // words per warp: 2048 u16 counters
                const size_t rsmem = (size_t)(RF_THREADS / 32) * rbudget * 4;
                BC_CUDA(cudaFuncSetAttribute(rfilter_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)rsmem));
                int per_sm = 0;
                BC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rfilter_kernel,
                                                                      RF_THREADS, rsmem));
                rfilter_kernel<<<(unsigned)(sms * std::max(per_sm, 1)), RF_THREADS, rsmem, st>>>(
                    P, F, rbudget);
                BC_CHECK_LAUNCH();
              } else if (compact) {
                filter_launch_c1((unsigned)fblocks, fsmem, st, P, F);
              } else {
                filter_launch_c0((unsigned)fblocks, fsmem, st, P, F);
              }
              dt.mark("filter");
              unsigned long long hm = 0;
              copy_d2h(&hm, ctr.p + CTR_HEAVY, sizeof hm, st);
              BC_CUDA(cudaStreamSynchronize(st));
              // back to emission order (the filter pushes in completion order): a root's
              // tasks stay adjacent, so the triage kernel re-reads their rows from L2
              DBuf<int32_t> msorted;
              msorted.alloc(hm, st);
              {
                size_t tmp = 0;
                BC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, medium.p, msorted.p,
                                                       (int64_t)hm, 0, 32, st));
                DBuf<char> tb;
                tb.alloc(tmp, st);
                BC_CUDA(cub::DeviceRadixSort::SortKeys(tb.p, tmp, medium.p, msorted.p,
                                                       (int64_t)hm, 0, 32, st));
              }
              medium = std::move(msorted);
              B.queue = medium.p;
              B.q1 = (int64_t)hm;
              launches += 2;
              if (dt.on) fprintf(stderr, "[bc search] medium %llu\n", hm);
            }
            BC_CUDA(cudaMemsetAsync(ctr.p + CTR_NEXT, 0, 8, st));
            BC_CUDA(cudaMemsetAsync(ctr.p + CTR_HEAVY, 0, 8, st));
            dt.mark("pre-triage");
            elaunch(ev, (unsigned)blocks, smem, P, B);
            dt.mark("triage");
            launches++;
            unsigned long long hn = 0;
            copy_d2h(&hn, ctr.p + CTR_HEAVY, sizeof hn, st);
            BC_CUDA(cudaStreamSynchronize(st));
            n_heavy = (int64_t)hn;
            if (n_heavy > 0) {  // deferred tasks in LPT order again, with their survivor caps
              DBuf<uint32_t> hk, hk2;
              DBuf<int32_t> slot, perm;
              hk.alloc(n_heavy, st);
              hk2.alloc(n_heavy, st);
              slot.alloc(n_heavy, st);
              perm.alloc(n_heavy, st);
              hq.alloc(n_heavy, st);
              hcap.alloc(n_heavy, st);
              gather_keys<<<(unsigned)((n_heavy + 255) / 256), 256, 0, st>>>(heavy.p, n_heavy,
                                                                              cost.p, hk.p);
              iota32<<<(unsigned)((n_heavy + 255) / 256), 256, 0, st>>>(slot.p, n_heavy);
              sort_pairs_desc(hk.p, hk2.p, slot.p, perm.p, n_heavy, st);
              gather2<<<(unsigned)((n_heavy + 255) / 256), 256, 0, st>>>(
                  perm.p, n_heavy, heavy.p, heavy_ns1.p, hq.p, hcap.p);
              launches += 4;
            }
            hq_p = hq.p;
            hcap_p = hcap.p;
          }
          A.queue = hq_p;
          A.caps = hcap_p;
          if (n_heavy > 0) {
          // split mode (p_eff >= 5): chunks of the LPT queue; per chunk, enum_kernel
            // writes every frame to the frame arena and pushes the split-level nodes,
            // then sub_kernel drains them heaviest first with every warp.
            // sub-tasks at level 2, or at level 3 when p_eff > 6 and there are too few heavy
            // tasks to fill the GPU at level 2 (C4: three planted cores, 2.8 vs 6.4 ms;
            // C5H: 2.9e5 heavy tasks, level 2 is 7% faster than 3)
            const int split_level = s.p_eff <= 6 || n_heavy >= 65536 ? 2 : 3;
            const int budget = 1024;
            const size_t smem = (size_t)wpb * (budget + map_w + LEAF_WORDS) * 4;
            const EnumVariant ev{instr, false, true, false};
            const size_t ssmem = (size_t)wpb * (budget + LEAF_WORDS) * 4;
            const int64_t blocks = (int64_t)sms * eblocks(ev, smem);
            const int64_t sblocks = std::min<int64_t>(
                (int64_t)sms * (compact ? sub_blocks_per_sm_c1(instr, ssmem)
                                        : sub_blocks_per_sm_c0(instr, ssmem)),
                blocks);
            A.budget_words = budget;
            DBuf<uint32_t> gs;
            if (max_scr > budget) {
              A.gscratch_words = (max_scr + 31) & ~int64_t(31);
              gs.alloc((size_t)blocks * wpb * A.gscratch_words, st);
              A.gscratch = gs.p;
            }
            const int64_t arena_limit = int64_t(1) << 29;  // words per arena (2 GiB)
            DBuf<int64_t> ro, sub, foff, soff;
            ro.alloc(n_heavy + 1, st);
            sub.alloc(n_heavy + 1, st);
            foff.alloc(n_heavy + 1, st);
            soff.alloc(n_heavy + 1, st);
            ro.zero();
            sub.zero();
            split_sizes<<<(unsigned)((n_heavy + 255) / 256), 256, 0, st>>>(
                info.p, hq_p, hcap_p, 0, n_heavy, instr, compact, split_level, ro.p, sub.p);
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
              dt.mark("split chunk setup");
              elaunch(ev, (unsigned)blocks, smem, P, A);
              unsigned long long hn = 0;
              copy_d2h(&hn, ctr.p + CTR_SUB_N, sizeof hn, st);
              BC_CUDA(cudaStreamSynchronize(st));
              const int64_t n_sub = std::min<int64_t>((int64_t)hn, cap);
              launches += 1;
              if (dt.on)
                fprintf(stderr, "[bc search] split chunk [%lld, %lld): frames %lld words, %lld sub-tasks\n",
                        (long long)q0, (long long)q1, (long long)fw, (long long)n_sub);
              dt.mark("split enum");
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
                if (dt.on) {
                  uint32_t top[4] = {0, 0, 0, 0};
                  copy_d2h(top, k1.p, sizeof(uint32_t) * std::min<int64_t>(4, n_sub), st);
                  const unsigned long long ksum = sum_device(k1.p, n_sub, st);
                  fprintf(stderr, "[bc search]   sub keys top %u %u %u %u sum %llu\n", top[0], top[1],
                          top[2], top[3], ksum);
                }
                cudaEvent_t k0e, k1e;
                if (dt.on) {
                  BC_CUDA(cudaEventCreate(&k0e));
                  BC_CUDA(cudaEventCreate(&k1e));
                  BC_CUDA(cudaEventRecord(k0e, st));
                }
                if (compact) sub_launch_c1(instr, (unsigned)sblocks, ssmem, st, P, A, n_sub);
                else sub_launch_c0(instr, (unsigned)sblocks, ssmem, st, P, A, n_sub);
                if (dt.on) {
                  BC_CUDA(cudaEventRecord(k1e, st));
                  BC_CUDA(cudaEventSynchronize(k1e));
                  float kms = 0;
                  BC_CUDA(cudaEventElapsedTime(&kms, k0e, k1e));
                  fprintf(stderr, "[bc search]   sub_kernel %.3f ms (events)\n", kms);
                  cudaEventDestroy(k0e);
                  cudaEventDestroy(k1e);
                }
                dt.mark("split sub");
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
  if (want_claims) copy_d2h(cfg.task_claims, claims.p, n_tasks * sizeof(uint32_t), st);
  BC_CUDA(cudaStreamSynchronize(st));
  float t1 = 0, t2 = 0;
  BC_CUDA(cudaEventElapsedTime(&t1, e0, e1));
  BC_CUDA(cudaEventElapsedTime(&t2, e1, e2));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  if (h_ovf == 2) throw Error(BC_ECUDA, "enumeration frame exceeded its scratch sizing");
  if (h_ctr[CTR_NEST_BAD])
    throw Error(BC_EASSERT, "check_nesting: " + std::to_string(h_ctr[CTR_NEST_BAD]) + " of " +
                                std::to_string(h_ctr[CTR_NEST_CHECKED]) +
                                " child C_L ids are outside dir2(root)");
  out.count_lo = h_acc[0];
  out.count_hi = h_acc[1];
  out.overflow = h_ovf ? 1 : 0;
  out.tasks_consumed = (int64_t)h_ctr[CTR_CONSUMED];
  out.nesting_checked = (int64_t)h_ctr[CTR_NEST_CHECKED];
  out.level1_entries = l1_entries;
  out.tasks_alive = n_alive;
  out.tasks_split = n_split;
  out.tasks_stolen = (int64_t)h_ctr[CTR_STOLEN];
  out.batches_executed = (s.p_eff >= 2 ? nloc : 0) + (int64_t)h_ctr[CTR_BATCHES];
  out.intersections = (int64_t)h_ctr[CTR_INTER];
  out.operand_words = (int64_t)h_ctr[CTR_OPW];
  out.level1_operand_words = (int64_t)h_ctr[CTR_OPW_L1];
  out.min_words = (int64_t)h_ctr[CTR_MINW];
  out.time_level1 = t1 * 1e-3;
  out.time_enum = t2 * 1e-3;
  out.kernel_launches += launches;
  (void)n_sub_total;
}

}  // namespace bc
