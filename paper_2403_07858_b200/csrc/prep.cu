// prep.cu -- device preprocessing for the (p,q)-biclique path (sm_100a).
//
// Restates, on device, prepare_structures (reference engine.py:115-144) and
// pre_runtime_tasks (engine.py:147-173):
//   anchor choice    graph.py:246-269   wedge mass per layer (computed at graph upload)
//   2-hop index      graph.py:192-215   CTA per anchor vertex, packed u16 counters in smem
//   priority         graph.py:227-243   radix sort on (|N2|, id)
//   directed filter  graph.py:218-224   warp per vertex, order-preserving ballot compaction
//   HTB              htb.py:89-115      warp per set, run boundaries by ballot
//   tasks            engine.py:147-173  scan over the priority order
// Every array is bit-identical to the reference's (tests/test_gpu_parity.py).
#include <cub/cub.cuh>

#include <cstdlib>
#include <ctime>

#include "engine.h"

namespace bc {

namespace {

template <typename T>
void exclusive_scan(const T *in, T *out, int64_t n, cudaStream_t st) {
  size_t tmp = 0;
  BC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, st));
  DBuf<char> t;
  t.alloc(tmp, st);
  BC_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, n, st));
}

template <typename T>
T d2h_scalar(const T *p, cudaStream_t st) {
  T v;
  copy_d2h(&v, p, sizeof(T), st);
  BC_CUDA(cudaStreamSynchronize(st));
  return v;
}

// ---------------------------------------------------------------------------
// 2-hop index: one CTA per anchor vertex u (dynamic queue, heaviest first).
// Counters for ids of the current tile live in shared memory (two u16 per
// u32 word, or one u32 per id when WIDE), next to a "touched" bitmap with one
// bit per id and a summary bitmap with one bit per touched 32-id word.
// The wedges u - v - w (v in N(u), w in N(v)) are walked as one flattened
// range per batch of TH_THREADS neighbours (block scan of the row lengths,
// owner by bisection in shared memory), so hub rows do not leave the other
// warps waiting at the barrier.  Increments stop once a counter reaches k (the
// reads are racy but monotone: a stale read costs one extra increment, at most
// blockDim per id, which keeps u16 counters exact below k <= 60000).  The first
// increment of an id sets its touched bit (and, for a word's first id, its
// summary bit); the summary is compacted into the ascending list of touched
// words, pass 1 turns each into its kept mask (count >= k, id != u) and clears
// the counters, pass 2 writes the kept ids in ascending order with a block-wide
// exclusive scan.  Cost per vertex is O(pool + n/1024), not O(n).
// ---------------------------------------------------------------------------
#ifndef TH_THREADS_DEF
#define TH_THREADS_DEF 1024
#endif
constexpr int TH_THREADS = TH_THREADS_DEF;

template <bool WIDE>
__device__ __forceinline__ uint32_t ctr_get(const uint32_t *c, int64_t i) {
  if (WIDE) return c[i];
  return (c[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
}

// shared-memory words per tile: counters, touched bits, summary bits, touched-word list
__host__ __device__ __forceinline__ int64_t th_ctr_words(int64_t tile, bool wide) {
  return wide ? tile : (tile + 1) / 2;
}
__host__ __device__ __forceinline__ int64_t th_smem_words(int64_t tile, bool wide) {
  const int64_t nt = (tile + 31) / 32;
  return th_ctr_words(tile, wide) + nt + (nt + 31) / 32 + nt;
}

template <bool WIDE, bool SUMMARY>
__global__ void __launch_bounds__(TH_THREADS) twohop_kernel(
    const int64_t *__restrict__ aoff, const int32_t *__restrict__ aidx,
    const int64_t *__restrict__ boff, const int32_t *__restrict__ bidx,
    const int32_t *__restrict__ vorder, int64_t n_claim, int64_t n, uint32_t k, int64_t tile,
    int ntiles, int *next, int64_t *__restrict__ und_size, int64_t *__restrict__ seg_start,
    int32_t *__restrict__ seg_len, int32_t *__restrict__ out_ids, int64_t out_cap,
    unsigned long long *out_used, int *overflow) {
  typedef cub::BlockScan<int, TH_THREADS> Scan;
  typedef cub::BlockReduce<int, TH_THREADS> Reduce;
  __shared__ union {
    typename Scan::TempStorage scan;
    typename Reduce::TempStorage reduce;
  } tmp;
  __shared__ int64_t s_rstart[TH_THREADS];
  __shared__ int s_roff[TH_THREADS + 1];
  extern __shared__ uint32_t sm[];
  const int64_t nctr = th_ctr_words(tile, WIDE);
  const int64_t nbits = (tile + 31) / 32;
  const int64_t nsum = (nbits + 31) / 32;
  uint32_t *ctr = sm;
  uint32_t *touched = sm + nctr;
  uint32_t *summary = touched + nbits;
  int *wlist = (int *)(summary + nsum);
  __shared__ int64_t s_u, s_base;
  __shared__ int s_total, s_nw;
  const int tid = threadIdx.x;
  for (int64_t i = tid; i < nctr + nbits + nsum; i += TH_THREADS) sm[i] = 0;
  __syncthreads();
  for (;;) {
    if (tid == 0) {
      int j = atomicAdd(next, 1);
      s_u = j < n_claim ? vorder[j] : -1;
    }
    __syncthreads();
    const int64_t u = s_u;
    if (u < 0) break;
    const int64_t e0 = aoff[u], e1 = aoff[u + 1];
    int64_t total = 0;
    for (int ti = 0; ti < ntiles; ti++) {
      const int64_t t0 = (int64_t)ti * tile;
      const int64_t t1 = t0 + tile < n ? t0 + tile : n;
      // count phase: the wedges of TH_THREADS neighbours at a time, spread evenly
      for (int64_t b = e0; b < e1; b += TH_THREADS) {
        int len = 0;
        int64_t st = 0;
        if (b + tid < e1) {
          const int32_t v = __ldg(aidx + b + tid);
          int64_t lo = __ldg(boff + v), hi = __ldg(boff + v + 1);
          const int64_t end = hi;
          const int32_t key = (int32_t)(u >= t0 ? u + 1 : t0);  // first id counted: > u, in tile
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (__ldg(bidx + mid) < key) lo = mid + 1;
            else hi = mid;
          }
          st = lo;
          len = (int)(end - lo);
        }
        int off, sum;
        Scan(tmp.scan).ExclusiveSum(len, off, sum);
        s_rstart[tid] = st;
        s_roff[tid] = off;
        if (tid == 0) s_roff[TH_THREADS] = sum;
        __syncthreads();
        for (int pos = tid; pos < sum; pos += TH_THREADS) {
          int lo = 0, hi = TH_THREADS - 1;  // last row whose offset is <= pos
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_roff[mid] <= pos) lo = mid;
            else hi = mid - 1;
          }
          const int64_t w = __ldg(bidx + s_rstart[lo] + (pos - s_roff[lo]));
          if (w < t0 || w >= t1) continue;
          const int64_t l = w - t0;
          bool first;
          if (WIDE) {
            if (((volatile uint32_t *)ctr)[l] >= k) continue;
            first = atomicAdd(&ctr[l], 1u) == 0;
          } else {
            const int sh = (int)(l & 1) * 16;
            if (((((volatile uint32_t *)ctr)[l >> 1] >> sh) & 0xffffu) >= k) continue;
            first = ((atomicAdd(&ctr[l >> 1], 1u << sh) >> sh) & 0xffffu) == 0;
          }
          if (first) {
            const uint32_t old = atomicOr(&touched[l >> 5], 1u << (l & 31));
            if (SUMMARY && old == 0) atomicOr(&summary[l >> 10], 1u << ((l >> 5) & 31));
          }
        }
        __syncthreads();
      }
      // the touched words, ascending: compaction of the summary bitmap (SUMMARY, for
      // vertices whose pool is small against the tile), else every word of the tile
      int nw = 0;
      const int64_t ntw = (t1 - t0 + 31) / 32;
      if (!SUMMARY) nw = (int)ntw;
      for (int64_t r0 = 0; SUMMARY && r0 < nsum; r0 += TH_THREADS) {
        const int64_t si = r0 + tid;
        uint32_t sw = si < nsum ? summary[si] : 0u;
        int off, round;
        Scan(tmp.scan).ExclusiveSum(__popc(sw), off, round);
        if (sw) summary[si] = 0;
        int o = nw + off;
        while (sw) {
          const int bb = __ffs(sw) - 1;
          sw &= sw - 1;
          wlist[o++] = (int)(si * 32 + bb);
        }
        nw += round;
        __syncthreads();
      }
      // pass 1: touched words -> kept masks, counters cleared
      int mine = 0;
      for (int i = tid; i < nw; i += TH_THREADS) {
        const int64_t wi = SUMMARY ? wlist[i] : i;
        const uint32_t t = touched[wi];
        if (!SUMMARY && !t) continue;
        uint32_t km = 0, m = t;
        while (m) {
          const int bb = __ffs(m) - 1;
          m &= m - 1;
          const int64_t l = wi * 32 + bb;
          if (ctr_get<WIDE>(ctr, l) >= k && t0 + l != u) km |= 1u << bb;
        }
        if (WIDE) {
          m = t;
          while (m) {
            const int bb = __ffs(m) - 1;
            m &= m - 1;
            ctr[wi * 32 + bb] = 0;
          }
        } else {
          for (int h = 0; h < 16; h++)
            if ((t >> (2 * h)) & 3u) ctr[wi * 16 + h] = 0;
        }
        touched[wi] = km;
        mine += __popc(km);
      }
      const int kept = Reduce(tmp.reduce).Sum(mine);
      if (tid == 0) {
        int64_t base = -1;
        if (kept) {
          unsigned long long bq = atomicAdd(out_used, (unsigned long long)kept);
          if ((int64_t)bq + kept > out_cap) atomicExch(overflow, 1);
          else base = (int64_t)bq;
        }
        s_base = base;
        s_total = kept;
        seg_start[u * ntiles + ti] = base;
        seg_len[u * ntiles + ti] = kept;
      }
      __syncthreads();
      total += s_total;
      const int64_t base = s_base;
      // pass 2: ordered emit of the kept ids, bitmap cleared
      int64_t pos = 0;
      if (s_total) {
        for (int r0 = 0; r0 < nw; r0 += TH_THREADS) {
          const int i = r0 + tid;
          const int64_t wi = i < nw ? (SUMMARY ? wlist[i] : i) : 0;
          uint32_t km = i < nw ? touched[wi] : 0u;
          int off, round;
          Scan(tmp.scan).ExclusiveSum(__popc(km), off, round);
          if (i < nw) touched[wi] = 0;
          if (km && base >= 0) {
            int64_t o = base + pos + off;
            while (km) {
              const int bb = __ffs(km) - 1;
              km &= km - 1;
              out_ids[o++] = (int32_t)(t0 + wi * 32 + bb);
            }
          }
          pos += round;
          __syncthreads();
        }
      } else {
        for (int i = tid; i < nw; i += TH_THREADS) touched[SUMMARY ? wlist[i] : i] = 0;
      }
      __syncthreads();
    }
    if (tid == 0) und_size[u] = total;  // the upper part |{w > u}|; lower parts added later
    __syncthreads();
  }
}

// upper bound on the 2-hop output: per anchor u, the kept ids (multiplicity >= k)
// number at most min(n - 1, pool(u) / k), pool(u) = sum_{v in N(u)} deg(v)
// opposite-layer degrees as int32 (an L2-resident gather table: C5's 8.96 M opposite
// vertices are 36 MB, against 72 MB of int64 offsets read twice per wedge)
__global__ void opp_degrees(const int64_t *__restrict__ boff, int64_t m, int32_t *__restrict__ deg) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v < m) {
    const int64_t d = boff[v + 1] - boff[v];
    deg[v] = d < INT32_MAX ? (int32_t)d : INT32_MAX;
  }
}

__global__ void twohop_bound(const int64_t *__restrict__ aoff, const int32_t *__restrict__ aidx,
                             const int32_t *__restrict__ bdeg, int64_t n, uint32_t k,
                             unsigned long long *out, int32_t *__restrict__ pool_of) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long tot = 0, ptot = 0;
  for (int64_t u = gw; u < n; u += nw) {
    unsigned long long pool = 0;
    for (int64_t e = aoff[u] + lane; e < aoff[u + 1]; e += 32)
      pool += (unsigned long long)__ldg(bdeg + __ldg(aidx + e));
    pool = warp_sum(pool);
    if (lane == 0) pool_of[u] = pool < 0x7fffffffull ? (int32_t)pool : 0x7fffffff;
    const unsigned long long b = pool / k;
    tot += b < (unsigned long long)(n - 1) ? b : (unsigned long long)(n - 1);
    ptot += pool;
  }
  if (lane == 0 && tot) atomicAdd(out, tot);
  if (lane == 0 && ptot) atomicAdd(out + 1, ptot);
}

// Output bound of the anchors one rank owns (sharded preprocessing): the same
// sum_u min(n - 1, pool(u) / k) over the selected light and heavy ids only, so a rank
// allocates its slice's share, not the whole graph's 2-hop output.
__global__ void owned_bound(const int32_t *__restrict__ ids_a, int64_t na,
                            const int32_t *__restrict__ ids_b, int64_t nb,
                            const int32_t *__restrict__ pool_of, int64_t n, uint32_t k,
                            unsigned long long *out) {
  unsigned long long tot = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < na + nb;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = i < na ? ids_a[i] : ids_b[i - na];
    const unsigned long long b = (unsigned long long)pool_of[u] / k;
    tot += b < (unsigned long long)(n - 1) ? b : (unsigned long long)(n - 1);
  }
  tot = warp_sum(tot);
  if ((threadIdx.x & 31) == 0 && tot) atomicAdd(out, tot);
}

// Light anchors (pool <= LIGHT_POOL wedges, most vertices of a power-law graph) skip
// the block kernel's tile counters and its ~10 block barriers per vertex: one warp
// gathers the vertex's upper wedge ids (w > u) into shared memory, bitonic-sorts them,
// and keeps every id whose run is >= k long (sorted: buf[i + k - 1] == buf[i]); the
// kept ids are already ascending.  Same outputs as the block kernel (one segment).
#ifndef LIGHT_POOL_DEF
#define LIGHT_POOL_DEF 1024
#endif
#ifndef LIGHT_WARPS_DEF
#define LIGHT_WARPS_DEF 8
#endif
constexpr int LIGHT_POOL = LIGHT_POOL_DEF;
constexpr int LIGHT_WARPS = LIGHT_WARPS_DEF;

__global__ void __launch_bounds__(LIGHT_WARPS * 32) twohop_light(
    const int64_t *__restrict__ aoff, const int32_t *__restrict__ aidx,
    const int64_t *__restrict__ boff, const int32_t *__restrict__ bidx,
    const int32_t *__restrict__ light, int64_t n_light, uint32_t k, int ntiles,
    int64_t *__restrict__ und_size, int64_t *__restrict__ seg_start, int32_t *__restrict__ seg_len,
    int32_t *__restrict__ out_ids, int64_t out_cap, unsigned long long *out_used, int *overflow) {
  extern __shared__ int32_t lbuf[];
  const int lane = threadIdx.x & 31;
  int32_t *buf = lbuf + (threadIdx.x >> 5) * LIGHT_POOL;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = gw; j < n_light; j += nw) {
    const int64_t u = light[j];
    const int64_t e1 = aoff[u + 1];
    int cnt = 0;
    for (int64_t e0 = aoff[u]; e0 < e1; e0 += 32) {
      int64_t st = 0;
      int len = 0;
      if (e0 + lane < e1) {
        const int32_t c = __ldg(aidx + e0 + lane);
        int64_t lo = __ldg(boff + c), hi = __ldg(boff + c + 1);
        const int64_t end = hi;
        while (lo < hi) {  // first id > u
          const int64_t mid = (lo + hi) >> 1;
          if (__ldg(bidx + mid) <= u) lo = mid + 1;
          else hi = mid;
        }
        st = lo;
        len = (int)(end - lo);
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
        int sl = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const int c = sl + step;
          const int e = __shfl_sync(FULL, excl, c < 32 ? c : 31);
          if (c < 32 && e <= pos) sl = c;
        }
        const int64_t so = __shfl_sync(FULL, st, sl);
        const int eo = __shfl_sync(FULL, excl, sl);
        if (pos < T) buf[cnt + pos] = __ldg(bidx + so + (pos - eo));
      }
      cnt += T;
    }
    int P = 32;
    while (P < cnt) P <<= 1;
    for (int i = cnt + lane; i < P; i += 32) buf[i] = 0x7fffffff;
    __syncwarp();
    for (int size = 2; size <= P; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = lane; i < (P >> 1); i += 32) {
          const int a = 2 * stride * (i / stride) + (i % stride), b = a + stride;
          const int x = buf[a], y = buf[b];
          const bool up = (a & size) == 0;
          if ((x > y) == up) {
            buf[a] = y;
            buf[b] = x;
          }
        }
        __syncwarp();
      }
    int kept = 0;
    for (int b0 = 0; b0 < cnt; b0 += 32) {
      const int i = b0 + lane;
      const bool keep = i < cnt && (i == 0 || buf[i] != buf[i - 1]) && i + (int)k - 1 < cnt &&
                        buf[i + k - 1] == buf[i];
      kept += __popc(__ballot_sync(FULL, keep));
    }
    long long base = -1;
    if (lane == 0 && kept) {
      const unsigned long long bq = atomicAdd(out_used, (unsigned long long)kept);
      if ((int64_t)bq + kept > out_cap) atomicExch(overflow, 1);
      else base = (long long)bq;
    }
    base = __shfl_sync(FULL, base, 0);
    if (base >= 0) {
      int pos = 0;
      for (int b0 = 0; b0 < cnt; b0 += 32) {
        const int i = b0 + lane;
        const bool keep = i < cnt && (i == 0 || buf[i] != buf[i - 1]) && i + (int)k - 1 < cnt &&
                          buf[i + k - 1] == buf[i];
        const unsigned m = __ballot_sync(FULL, keep);
        if (keep) out_ids[base + pos + __popc(m & lanemask_lt())] = buf[i];
        pos += __popc(m);
      }
    }
    for (int ti = lane; ti < ntiles; ti += 32) {
      seg_start[u * ntiles + ti] = ti == 0 ? base : -1;
      seg_len[u * ntiles + ti] = ti == 0 ? kept : 0;
    }
    if (lane == 0) und_size[u] = kept;
    __syncwarp();
  }
}

// light / heavy split of the LPT order; with nshards > 1 only the anchors this shard owns
// (snake order over the LPT positions, so every shard gets a like share of hubs)
__global__ void light_flags(const int32_t *__restrict__ vorder, const int32_t *__restrict__ pool_of,
                            int64_t n, int use_light, int shard, int nshards,
                            uint8_t *__restrict__ is_light, uint8_t *__restrict__ is_heavy) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) {
    const int64_t r = j % (2 * nshards);
    const bool own = (r < nshards ? r : 2 * nshards - 1 - r) == shard;
    const bool l = use_light && pool_of[vorder[j]] <= LIGHT_POOL;
    is_light[j] = own && l;
    is_heavy[j] = own && !l;
  }
}

// injected upper lists -> the per-(anchor, tile) segments the consumers read (one tile)
__global__ void segs_from_off(const int64_t *__restrict__ off, int64_t n, int64_t *__restrict__ seg_start,
                              int32_t *__restrict__ seg_len, int64_t *__restrict__ und_size) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u < n) {
    seg_start[u] = off[u];
    seg_len[u] = (int32_t)(off[u + 1] - off[u]);
    und_size[u] = off[u + 1] - off[u];
  }
}

// slice export: upper-list length per anchor, then the ids in anchor order
__global__ void slice_lens_k(const int32_t *__restrict__ seg_len, int64_t n, int ntiles,
                             int32_t *__restrict__ lens, int64_t *__restrict__ lens64) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u < n) {
    int64_t t = 0;
    for (int ti = 0; ti < ntiles; ti++) t += seg_len[u * ntiles + ti];
    lens[u] = (int32_t)t;
    lens64[u] = t;
  }
}

__global__ void slice_copy(const int64_t *__restrict__ seg_start, const int32_t *__restrict__ seg_len,
                           int64_t n, int ntiles, const int32_t *__restrict__ up_ids,
                           const int64_t *__restrict__ pos, int32_t *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = gw; u < n; u += nw) {
    int64_t o = pos[u];
    for (int ti = 0; ti < ntiles; ti++) {
      const int64_t st = seg_start[u * ntiles + ti];
      const int32_t ln = seg_len[u * ntiles + ti];
      for (int32_t i = lane; i < ln; i += 32) out[o + i] = up_ids[st + i];
      o += ln;
    }
  }
}

// The 2-hop relation is symmetric (|N(u) & N(w)| both ways), so the kernel above
// counts only w > u: half the wedges.  und(u) = {w < u : u in up(w)} ++ up(u).
// lower_counts: |{w < u : u in up(w)}| per u (warp per w walking up(w)'s tiles).
__global__ void lower_counts(const int64_t *__restrict__ seg_start, const int32_t *__restrict__ seg_len,
                             int ntiles, const int32_t *__restrict__ up_ids, int64_t n,
                             int64_t *__restrict__ cnt_low) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = gw; w < n; w += nw)
    for (int ti = 0; ti < ntiles; ti++) {
      const int64_t st = seg_start[w * ntiles + ti];
      const int32_t ln = seg_len[w * ntiles + ti];
      for (int32_t i = lane; i < ln; i += 32) atomicAdd((unsigned long long *)(cnt_low + up_ids[st + i]), 1ull);
    }
}

// directed lists from the upper pairs (u, w), u < w: w in dir2(u) iff rank[w] < rank[u],
// else u in dir2(w) (graph.py:223).  dup[u]: upper entries kept in dir2(u); dlow[w]:
// entries of dir2(w) that come from other rows.  The upper segments are cut into work
// items of DIR_CHUNK pairs (a hub's list of ~20K pairs is ~80 items, not one warp's
// serial walk): item_seg[i] = segment of item i, item_off[s] = first item of segment s.
constexpr int DIR_CHUNK = 256;

__global__ void dir_items(const int32_t *__restrict__ seg_len, int64_t nseg,
                          int64_t *__restrict__ nitems) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < nseg) nitems[s] = (seg_len[s] + DIR_CHUNK - 1) / DIR_CHUNK;
}

__global__ void dir_item_owner(const int64_t *__restrict__ item_off, int64_t nseg,
                               int32_t *__restrict__ item_seg) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < nseg)
    for (int64_t i = item_off[s]; i < item_off[s + 1]; i++) item_seg[i] = (int32_t)s;
}

__global__ void dir_counts(const int64_t *__restrict__ seg_start, const int32_t *__restrict__ seg_len,
                           int ntiles, const int32_t *__restrict__ up_ids,
                           const int64_t *__restrict__ rank, const int64_t *__restrict__ item_off,
                           const int32_t *__restrict__ item_seg, int64_t nseg,
                           int64_t *__restrict__ dup, int64_t *__restrict__ dlow,
                           int64_t *__restrict__ item_mine) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nitems = item_off[nseg];
  for (int64_t it = gw; it < nitems; it += nw) {
    const int64_t sg = item_seg[it];
    const int64_t u = sg / ntiles;
    const int64_t ru = rank[u];
    const int64_t b0 = (it - item_off[sg]) * DIR_CHUNK;
    const int64_t rest = seg_len[sg] - b0;
    const int32_t ln = (int32_t)(rest < DIR_CHUNK ? rest : DIR_CHUNK);
    const int64_t st = seg_start[sg] + b0;
    int c = 0;
    for (int32_t i = lane; i < ln; i += 32) {
      const int32_t w = up_ids[st + i];
      if (__ldg(rank + w) < ru) c++;
      else atomicAdd((unsigned long long *)(dlow + w), 1ull);
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) {
      item_mine[it] = c;
      if (c) atomicAdd((unsigned long long *)(dup + u), (unsigned long long)c);
    }
  }
}

// item_pre: exclusive scan of item_mine; an item's kept upper entries start at
// dir_off[u] + dlow[u] + (item_pre[it] - item_pre[first item of u]).
__global__ void dir_fill(const int64_t *__restrict__ seg_start, const int32_t *__restrict__ seg_len,
                         int ntiles, const int32_t *__restrict__ up_ids,
                         const int64_t *__restrict__ rank, const int64_t *__restrict__ item_off,
                         const int32_t *__restrict__ item_seg, const int64_t *__restrict__ item_pre,
                         int64_t nseg, const int64_t *__restrict__ dir_off,
                         const int64_t *__restrict__ dlow, unsigned long long *__restrict__ cur,
                         int32_t *__restrict__ low_buf, int32_t *__restrict__ dir_idx) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nitems = item_off[nseg];
  for (int64_t it = gw; it < nitems; it += nw) {
    const int64_t sg = item_seg[it];
    const int64_t u = sg / ntiles;
    const int64_t ru = rank[u];
    const int64_t b0 = (it - item_off[sg]) * DIR_CHUNK;
    const int64_t rest = seg_len[sg] - b0;
    const int32_t ln = (int32_t)(rest < DIR_CHUNK ? rest : DIR_CHUNK);
    const int64_t st = seg_start[sg] + b0;
    int64_t pos = dir_off[u] + dlow[u] + item_pre[it] - item_pre[item_off[u * ntiles]];
    for (int32_t b = 0; b < ln; b += 32) {
      const int32_t i = b + lane;
      int32_t w = 0;
      bool mine = false;
      if (i < ln) {
        w = up_ids[st + i];
        mine = __ldg(rank + w) < ru;
        if (!mine) low_buf[dir_off[w] + (int64_t)atomicAdd(cur + w, 1ull)] = (int32_t)u;
      }
      const unsigned m = __ballot_sync(0xffffffffu, mine);
      if (mine) dir_idx[pos + __popc(m & ((1u << lane) - 1u))] = w;
      pos += __popc(m);
    }
  }
}

__global__ void add_sizes(const int64_t *__restrict__ a, const int64_t *__restrict__ b, int64_t n,
                          int64_t *__restrict__ out, int64_t *__restrict__ low_end,
                          const int64_t *__restrict__ off) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    out[i] = a[i] + b[i];
    if (off) low_end[i] = off[i] + b[i];
  }
}

// vertices by descending degree (LPT order for the 2-hop CTAs)
__global__ void degree_keys(const int64_t *off, int64_t n, unsigned long long *keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    unsigned long long d = (unsigned long long)(off[i + 1] - off[i]);
    keys[i] = ((~d & 0xffffffffull) << 32) | (unsigned long long)i;  // ascending key = descending degree
  }
}

__global__ void low_bits(const unsigned long long *keys, int64_t n, int32_t *out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int32_t)(keys[i] & 0xffffffffull);
}

// vertex_priority (graph.py:227-243): ascending (size, id) -> rank n..1
__global__ void priority_keys(const int64_t *size, int64_t n, unsigned long long *keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) keys[i] = ((unsigned long long)size[i] << 32) | (unsigned long long)i;
}

__global__ void priority_rank(const unsigned long long *sorted, int64_t n, int64_t *rank,
                              int64_t *order) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    int64_t id = (int64_t)(sorted[i] & 0xffffffffull);
    order[i] = id;
    rank[id] = n - i;
  }
}

__global__ void iota64(int64_t *a, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

__global__ void adjacent_dupes(const int64_t *sorted, int64_t n, int *flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > 0 && i < n && sorted[i] == sorted[i - 1]) atomicExch(flag, 1);
}

// HTB (htb.py:89-115): per set, idx = distinct id>>5, val = OR of 1<<(id&31).
template <bool WRITE>
__global__ void htb_build(const int64_t *__restrict__ off, const int32_t *__restrict__ idx,
                          int64_t n, int64_t *__restrict__ words, const int64_t *__restrict__ hoff,
                          uint32_t *__restrict__ hidx, uint32_t *__restrict__ hval) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = gw; u < n; u += nw) {
    const int64_t a = off[u], b = off[u + 1];
    int64_t pos = WRITE ? hoff[u] : 0;
    for (int64_t c = a; c < b; c += 32) {
      const int64_t i = c + lane;
      bool start = false;
      uint32_t word = 0;
      if (i < b) {
        word = (uint32_t)__ldg(idx + i) >> 5;
        start = (i == a) || (((uint32_t)__ldg(idx + i - 1) >> 5) != word);
      }
      const unsigned m = __ballot_sync(FULL, start);
      if (WRITE && start) {
        uint32_t v = 0;
        for (int64_t j = i; j < b; j++) {
          const uint32_t id = (uint32_t)__ldg(idx + j);
          if ((id >> 5) != word) break;
          v |= 1u << (id & 31);
        }
        const int64_t o = pos + __popc(m & lanemask_lt());
        hidx[o] = word;
        hval[o] = v;
      }
      pos += __popc(m);
    }
    if (!WRITE && lane == 0) words[u] = pos - (WRITE ? hoff[u] : 0);
  }
}

// Flat HTB build (no per-row tails: a hub row is spread over many threads like any
// other): flag[i] = entry i starts a word (first of its row, or a new id >> 5), an
// exclusive scan gives every word its slot, and each word's first entry ORs its run.
__global__ void htb_rowmark(const int64_t *__restrict__ off, int64_t n, uint8_t *__restrict__ rs) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u < n && off[u] < off[u + 1]) rs[off[u]] = 1;
}

__global__ void htb_flags(const int32_t *__restrict__ idx, int64_t E, const uint8_t *__restrict__ rs,
                          int32_t *__restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < E)
    flag[i] = rs[i] || (((uint32_t)idx[i] >> 5) != ((uint32_t)idx[i - 1] >> 5)) ? 1 : 0;
  else if (i == E)
    flag[i] = 0;
}

__global__ void htb_rowoff(const int64_t *__restrict__ off, int64_t n, const int32_t *__restrict__ wpos,
                           int64_t *__restrict__ hoff, int64_t *__restrict__ words) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u <= n) hoff[u] = wpos[off[u]];
  if (u < n) words[u] = (int64_t)wpos[off[u + 1]] - wpos[off[u]];
}

__global__ void htb_fill(const int32_t *__restrict__ idx, int64_t E, const int32_t *__restrict__ flag,
                         const int32_t *__restrict__ wpos, uint32_t *__restrict__ hidx,
                         uint32_t *__restrict__ hval) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= E || !flag[i]) return;
  const uint32_t word = (uint32_t)idx[i] >> 5;
  uint32_t v = 1u << (idx[i] & 31);
  for (int64_t j = i + 1; j < E && !flag[j]; j++) v |= 1u << (idx[j] & 31);
  hidx[wpos[i]] = word;
  hval[wpos[i]] = v;
}

// dense hub rows: histogram of rows with more than 16 << i words
constexpr int DENSE_NT = 12;
__global__ void dense_hist(const int64_t *hoff, int64_t n, unsigned long long *hist) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t w = hoff[i + 1] - hoff[i];
  for (int t = 0; t < DENSE_NT; t++)
    if (w > (int64_t(16) << t)) atomicAdd(hist + t, 1ull);
}

__global__ void dense_flags(const int64_t *hoff, int64_t n, int64_t T, int32_t *flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) flag[i] = (hoff[i + 1] - hoff[i]) > T ? 1 : 0;
}

__global__ void dense_ids(const int32_t *flag, const int32_t *slot, int64_t n, int32_t *id) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) id[i] = flag[i] ? slot[i] : -1;
}

__global__ void dense_fill(const int64_t *__restrict__ hoff, const uint32_t *__restrict__ hidx,
                           const uint32_t *__restrict__ hval, int64_t n,
                           const int32_t *__restrict__ id, uint32_t *__restrict__ dense,
                           int64_t mw) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = gw; x < n; x += nw) {
    const int32_t sl = id[x];
    if (sl < 0) continue;
    uint32_t *row = dense + (int64_t)sl * mw;
    for (int64_t j = hoff[x] + lane; j < hoff[x + 1]; j += 32) row[hidx[j]] = hval[j];
  }
}

__global__ void set_mask(const int32_t *roots, int64_t nr, int64_t n, uint8_t *mask) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nr) {
    int64_t r = roots[i];
    if (r >= 0 && r < n) mask[r] = 1;
  }
}

// pre_runtime_tasks (engine.py:147-173): per priority position, task count.
__global__ void task_counts(const int64_t *__restrict__ order, const int64_t *__restrict__ und_size,
                            const int64_t *__restrict__ dir_off, const uint8_t *__restrict__ mask,
                            int64_t n, int p_eff, int64_t *__restrict__ cnt,
                            unsigned long long *filtered) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t r = order[i];
  int64_t c = 0;
  if (!mask || mask[r]) {
    if (und_size[r] < p_eff - 1) atomicAdd(filtered, 1ull);
    else c = p_eff == 1 ? 1 : dir_off[r + 1] - dir_off[r];
  }
  cnt[i] = c;
}

__global__ void task_write(const int64_t *__restrict__ order, const int64_t *__restrict__ toff,
                           const int64_t *__restrict__ cnt, const int64_t *__restrict__ dir_off,
                           const int32_t *__restrict__ dir_idx, int64_t n, int p_eff,
                           int2 *__restrict__ tasks) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < n; i += nw) {
    const int64_t c = cnt[i];
    if (!c) continue;
    const int32_t r = (int32_t)order[i];
    const int64_t o = toff[i];
    if (p_eff == 1) {
      if (lane == 0) tasks[o] = make_int2(r, -1);
      continue;
    }
    const int64_t d0 = dir_off[r];
    for (int64_t j = lane; j < c; j += 32) tasks[o + j] = make_int2(r, dir_idx[d0 + j]);
  }
}

__global__ void root_task_off(const int64_t *__restrict__ order, const int64_t *__restrict__ toff,
                              const int64_t *__restrict__ cnt, int64_t n, int64_t *__restrict__ troot) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) troot[order[i]] = cnt[i] ? toff[i] : -1;
}

__global__ void max_reduce(const int64_t *a, int64_t n, unsigned long long *out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long v = i < n ? (unsigned long long)a[i] : 0;
  v = __reduce_max_sync(FULL, (unsigned)v);  // words per slice < 2^32
  if ((threadIdx.x & 31) == 0 && v) atomicMax(out, v);
}


inline unsigned blocks_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return (unsigned)(b < 1 ? 1 : b);
}

inline unsigned warp_blocks(int64_t n_items, int sms) {
  int64_t b = (n_items * 32 + 255) / 256;
  int64_t cap = (int64_t)sms * 16;
  if (b > cap) b = cap;
  return (unsigned)(b < 1 ? 1 : b);
}

// (r << ib) | id keys of every directed pair (warp per root): lower part from low_buf,
// upper part from dir_idx
__global__ void dir_sort_keys(const int64_t *__restrict__ doff, const int64_t *__restrict__ low_end,
                              const int32_t *__restrict__ low_buf, const int32_t *__restrict__ didx,
                              int64_t n, int ib, unsigned long long *__restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw; r < n; r += nw) {
    const int64_t le = low_end[r];
    for (int64_t i = doff[r] + lane; i < doff[r + 1]; i += 32)
      keys[i] = ((unsigned long long)r << ib) | (unsigned long long)(i < le ? low_buf[i] : didx[i]);
  }
}

__global__ void key_low_ids(const unsigned long long *__restrict__ keys, int64_t m, int ib,
                            int32_t *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) out[i] = (int32_t)(keys[i] & ((1ull << ib) - 1ull));
}

// HTB of a CSR family into (off, idx, val)
void build_htb(const int64_t *off, const int32_t *idx, int64_t n, int64_t E, DBuf<int64_t> &hoff,
               DBuf<uint32_t> &hidx, DBuf<uint32_t> &hval, int64_t &total, int64_t &max_slice,
               int sms, cudaStream_t st, int64_t &launches) {
  DBuf<int64_t> words;
  words.alloc(n + 1, st);
  words.zero();
  DBuf<int32_t> flag, wpos;
  // small families keep the per-row kernels (fewer launches); large ones go flat
  const int64_t flat_min = int64_t(1) << 17;
  const bool flat = E >= flat_min && E < (int64_t(1) << 31) - 1;
  if (flat) {  // word slots by one scan over the entries
    DBuf<uint8_t> rs;
    rs.alloc(E + 1, st);
    rs.zero();
    flag.alloc(E + 1, st);
    wpos.alloc(E + 1, st);
    htb_rowmark<<<blocks_for(n, 256), 256, 0, st>>>(off, n, rs.p);
    htb_flags<<<blocks_for(E + 1, 256), 256, 0, st>>>(idx, E, rs.p, flag.p);
    exclusive_scan(flag.p, wpos.p, E + 1, st);
    hoff.alloc(n + 1, st);
    htb_rowoff<<<blocks_for(n + 1, 256), 256, 0, st>>>(off, n, wpos.p, hoff.p, words.p);
    BC_CHECK_LAUNCH();
    launches += 4;
  } else {
    htb_build<false><<<warp_blocks(n, sms), 256, 0, st>>>(off, idx, n, words.p, nullptr, nullptr,
                                                        nullptr);
    BC_CHECK_LAUNCH();
    hoff.alloc(n + 1, st);
    exclusive_scan(words.p, hoff.p, n + 1, st);
  }
  DBuf<unsigned long long> mx;
  mx.alloc(1, st);
  mx.zero();
  max_reduce<<<blocks_for(n, 256), 256, 0, st>>>(words.p, n, mx.p);
  BC_CHECK_LAUNCH();
  total = d2h_scalar(hoff.p + n, st);
  max_slice = (int64_t)d2h_scalar(mx.p, st);
  hidx.alloc(total, st);
  hval.alloc(total, st);
  if (flat)
    htb_fill<<<blocks_for(E, 256), 256, 0, st>>>(idx, E, flag.p, wpos.p, hidx.p, hval.p);
  else
    htb_build<true><<<warp_blocks(n, sms), 256, 0, st>>>(off, idx, n, nullptr, hoff.p, hidx.p,
                                                       hval.p);
  BC_CHECK_LAUNCH();
  launches += 4;
}

}  // namespace

int num_sms(int device) {
  int v = 0;
  BC_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  return v;
}

// BC_DEBUG=1: per-stage wall time of the preprocessing on stderr (development).
struct StageTimer {
  bool on;
  cudaStream_t st;
  double t0;
  explicit StageTimer(cudaStream_t s) : on(getenv("BC_DEBUG") != nullptr), st(s), t0(now()) {}
  static double now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
  }
  void mark(const char *what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const double t = now();
    fprintf(stderr, "[bc prep] %-10s %8.3f ms\n", what, 1e3 * (t - t0));
    t0 = t;
  }
};

// Whole upper CSR from `world` gathered slices (rank r: lens_all[r * n + u], ids at
// ids_all[r * stride ...] in anchor order); each anchor's list is in exactly one slice.
__global__ void up_glens(const int32_t *__restrict__ lens_all, int world, int64_t n,
                         int64_t *__restrict__ glens, int64_t *__restrict__ flat) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u < n) {
    int64_t t = 0;
    for (int r = 0; r < world; r++) {
      const int32_t l = lens_all[(int64_t)r * n + u];
      flat[(int64_t)r * n + u] = l;
      t += l;
    }
    glens[u] = t;
  }
}

__global__ void up_copy(const int32_t *__restrict__ lens_all, const int32_t *__restrict__ ids_all,
                        int64_t stride, int world, int64_t n, const int64_t *__restrict__ pos_flat,
                        const int64_t *__restrict__ off, int32_t *__restrict__ ids_out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = gw; u < n; u += nw) {
    const int64_t len = off[u + 1] - off[u];
    if (!len) continue;
    int r = 0;
    while (r < world - 1 && lens_all[(int64_t)r * n + u] == 0) r++;
    const int32_t *src = ids_all + (int64_t)r * stride + (pos_flat[(int64_t)r * n + u] - pos_flat[(int64_t)r * n]);
    for (int64_t i = lane; i < len; i += 32) ids_out[off[u] + i] = src[i];
  }
}

int64_t assemble_upper(int world, int64_t n, const int32_t *lens_all, const int32_t *ids_all,
                       int64_t stride, int64_t *off_out, int32_t *ids_out, int64_t ids_cap,
                       cudaStream_t st, int sms) {
  DBuf<int64_t> glens, flat, pos;
  glens.alloc(n + 1, st);
  flat.alloc((size_t)world * n + 1, st);
  pos.alloc((size_t)world * n + 1, st);
  glens.zero();
  flat.zero();
  up_glens<<<blocks_for(n, 256), 256, 0, st>>>(lens_all, world, n, glens.p, flat.p);
  exclusive_scan(glens.p, off_out, n + 1, st);
  exclusive_scan(flat.p, pos.p, (int64_t)world * n + 1, st);
  const int64_t total = d2h_scalar(off_out + n, st);
  if (total > ids_cap) throw Error(BC_EINVAL, "upper ids buffer too small");
  up_copy<<<warp_blocks(n, sms), 256, 0, st>>>(lens_all, ids_all, stride, world, n, pos.p, off_out,
                                                ids_out);
  BC_CHECK_LAUNCH();
  BC_CUDA(cudaStreamSynchronize(st));
  return total;
}

void prepare(const DevGraph &g, int p, int q, const bc_config &cfg, DevStructs &s,
             const UpperPairs *upper, const SliceSpec *slice) {
  if (p < 1 || q < 1) throw Error(BC_EINVAL, "p and q must be >= 1");
  cudaStream_t st = g.stream;
  StageTimer tm(st);
  s.stream = st;
  const int sms = num_sms(g.device);
  int64_t &L = s.launches;
  // select_anchor_layer (graph.py:252-269): U iff wedge(V) <= wedge(U); V swaps p, q
  int layer;
  if (cfg.anchor < 0) layer = g.wedge_v <= g.wedge_u ? 0 : 1;
  else if (cfg.anchor <= 1) layer = cfg.anchor;
  else throw Error(BC_EINVAL, "anchor must be one of ('auto', 'U', 'V')");
  s.anchor = layer;
  s.p_eff = layer == 0 ? p : q;
  s.q_eff = layer == 0 ? q : p;
  s.n = layer == 0 ? g.n_u : g.n_v;
  s.m = layer == 0 ? g.n_v : g.n_u;
  s.aoff = layer == 0 ? g.u_off : g.v_off;
  s.aidx = layer == 0 ? g.u_idx : g.v_idx;
  s.boff = layer == 0 ? g.v_off : g.u_off;
  s.bidx = layer == 0 ? g.v_idx : g.u_idx;
  s.max_deg_anchor = layer == 0 ? g.max_deg_u : g.max_deg_v;
  const int64_t n = s.n;
  if (cfg.rank_override && cfg.n_rank != n)
    throw Error(BC_EINVAL, "rank override must give one distinct value per anchor vertex");

  // ---- 2-hop index, k = q_eff (engine.py:127) ----
  s.und_size.alloc(n ? n : 1, st);
  s.und_size.zero();
  const uint32_t k = (uint32_t)s.q_eff;
  const bool wide = k > 60000;
  int ntiles = 1;
  int64_t tile = n ? n : 1;
  DBuf<int64_t> seg_start;
  DBuf<int32_t> seg_len;
  DBuf<int32_t> und_ids;
  const int32_t *up_ids = nullptr;  // the upper lists (built here, or injected)
  if (upper && n > 0) {
    seg_start.alloc(n, st);
    seg_len.alloc(n, st);
    segs_from_off<<<blocks_for(n, 256), 256, 0, st>>>(upper->off, n, seg_start.p, seg_len.p,
                                                       s.und_size.p);
    up_ids = upper->ids;
    DBuf<int64_t> low;
    low.alloc(n, st);
    low.zero();
    lower_counts<<<warp_blocks(n, sms), 256, 0, st>>>(seg_start.p, seg_len.p, 1, up_ids, n, low.p);
    add_sizes<<<blocks_for(n, 256), 256, 0, st>>>(s.und_size.p, low.p, n, s.und_size.p, nullptr,
                                                   nullptr);
    BC_CHECK_LAUNCH();
    s.und_pairs = 2 * upper->pairs;
    L += 3;
  } else if (n > 0 && (int64_t)k <= s.max_deg_anchor) {
    int smem_optin = 0;
    BC_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g.device));
    // counters + touched bitmap per tile id: 2 B + 1/8 B (u16) or 4 B + 1/8 B (u32)
    // counters (16 or 32 bits) + touched bit + touched-word list (32 bits per word) + summary
    const int64_t budget_bits = (int64_t)(smem_optin - 16384) * 8;
    int64_t max_tile = wide ? budget_bits / 34 : budget_bits / 18;
    max_tile &= ~int64_t(63);
    ntiles = (int)((n + max_tile - 1) / max_tile);
    tile = (n + ntiles - 1) / ntiles;
    tile = (tile + 63) & ~int64_t(63);
    const size_t smem = (size_t)th_smem_words(tile, wide) * 4;
    // LPT vertex order: descending anchor degree
    DBuf<unsigned long long> keys, keys2;
    keys.alloc(n, st);
    keys2.alloc(n, st);
    degree_keys<<<blocks_for(n, 256), 256, 0, st>>>(s.aoff, n, keys.p);
    size_t tmp = 0;
    BC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.p, keys2.p, n, 0, 64, st));
    {
      DBuf<char> t;
      t.alloc(tmp, st);
      BC_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, keys.p, keys2.p, n, 0, 64, st));
    }
    DBuf<int32_t> vorder;
    vorder.alloc(n, st);
    low_bits<<<blocks_for(n, 256), 256, 0, st>>>(keys2.p, n, vorder.p);
    L += 3;
    seg_start.alloc((size_t)n * ntiles, st);
    seg_len.alloc((size_t)n * ntiles, st);
    seg_len.zero();  // anchors of other shards keep empty segments
    // output capacity: the pool bound (exact upper bound; int32 offsets cap it at 2^31,
    // an overflow past that is retried at the exact size)
    DBuf<int> ctrs;  // [0] next vertex, [1] overflow
    DBuf<unsigned long long> used;
    ctrs.alloc(2, st);
    used.alloc(2, st);
    used.zero();
    DBuf<int32_t> light_ids, heavy_ids;
    DBuf<int32_t> &pool_of = s.pool;  // kept: level 1 sums it for its mode choice
    pool_of.alloc(n, st);
    {
      DBuf<int32_t> bdeg;
      bdeg.alloc(s.m, st);
      opp_degrees<<<blocks_for(s.m, 256), 256, 0, st>>>(s.boff, s.m, bdeg.p);
      twohop_bound<<<warp_blocks(n, sms), 256, 0, st>>>(s.aoff, s.aidx, bdeg.p, n, k, used.p,
                                                        pool_of.p);
      L++;
    }
    BC_CHECK_LAUNCH();
    L++;
    // light anchors (small wedge pools) go to the warp-per-vertex kernel, the rest keep
    // the LPT order of the block kernel
    const bool use_light = !wide;
    const bool select = use_light || slice;
    int64_t n_light = 0, n_heavy = n;
    DBuf<int64_t> nsel;
    if (select) {
      DBuf<uint8_t> fl, fh;
      fl.alloc(n, st);
      fh.alloc(n, st);
      light_ids.alloc(n, st);
      heavy_ids.alloc(n, st);
      nsel.alloc(2, st);
      light_flags<<<blocks_for(n, 256), 256, 0, st>>>(vorder.p, pool_of.p, n, use_light ? 1 : 0,
                                                      slice ? slice->shard : 0,
                                                      slice ? slice->nshards : 1, fl.p, fh.p);
      size_t stmp = 0;
      BC_CUDA(cub::DeviceSelect::Flagged(nullptr, stmp, vorder.p, fl.p, light_ids.p, nsel.p, n, st));
      DBuf<char> t;
      t.alloc(stmp, st);
      BC_CUDA(cub::DeviceSelect::Flagged(t.p, stmp, vorder.p, fl.p, light_ids.p, nsel.p, n, st));
      BC_CUDA(cub::DeviceSelect::Flagged(t.p, stmp, vorder.p, fh.p, heavy_ids.p, nsel.p + 1, n, st));
      L += 3;
    }
    unsigned long long hb[2];
    copy_d2h(hb, used.p, sizeof hb, st);
    if (select) {
      int64_t hn[2];
      copy_d2h(hn, nsel.p, sizeof hn, st);
      BC_CUDA(cudaStreamSynchronize(st));
      n_light = hn[0];
      n_heavy = hn[1];
    }
    BC_CUDA(cudaStreamSynchronize(st));
    if (slice) {  // size the output by the owned anchors only
      DBuf<unsigned long long> ob;
      ob.alloc(1, st);
      ob.zero();
      owned_bound<<<sms * 4, 256, 0, st>>>(light_ids.p, n_light, heavy_ids.p, n_heavy, pool_of.p,
                                           n, k, ob.p);
      BC_CHECK_LAUNCH();
      L++;
      unsigned long long hob = 0;
      copy_d2h(&hob, ob.p, sizeof hob, st);
      BC_CUDA(cudaStreamSynchronize(st));
      hb[0] = hob;
    }
    int64_t cap = std::min<int64_t>((int64_t)hb[0], int64_t(1) << 31);
    cap = std::max<int64_t>(cap, 1);
    // touched-word lists when a vertex's pool is small against the tile's words
    bool summary = (double)hb[1] / (double)n < (double)((tile + 31) / 32);
    auto kern = wide ? (summary ? twohop_kernel<true, true> : twohop_kernel<true, false>)
                     : (summary ? twohop_kernel<false, true> : twohop_kernel<false, false>);
    BC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    BC_CUDA(cudaFuncSetAttribute(twohop_light, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 LIGHT_WARPS * LIGHT_POOL * 4));
    int per_sm = 0;
    BC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TH_THREADS, smem));
    if (per_sm < 1) per_sm = 1;
    for (int attempt = 0; attempt < 2; attempt++) {
      und_ids.alloc(cap, st);
      ctrs.zero();
      used.zero();
      if (n_light > 0) {
        const size_t lsmem = (size_t)LIGHT_WARPS * LIGHT_POOL * 4;
        twohop_light<<<(unsigned)std::min<int64_t>((n_light + LIGHT_WARPS - 1) / LIGHT_WARPS,
                                                   (int64_t)sms * 8),
                       LIGHT_WARPS * 32, lsmem, st>>>(s.aoff, s.aidx, s.boff, s.bidx, light_ids.p,
                                                      n_light, k, ntiles, s.und_size.p,
                                                      seg_start.p, seg_len.p, und_ids.p, cap,
                                                      used.p, ctrs.p + 1);
        L++;
      }
      if (n_heavy > 0) {
        kern<<<sms * per_sm, TH_THREADS, smem, st>>>(s.aoff, s.aidx, s.boff, s.bidx,
                                                     select ? heavy_ids.p : vorder.p, n_heavy,
                                                     n, k, tile, ntiles, ctrs.p, s.und_size.p,
                                                     seg_start.p, seg_len.p, und_ids.p, cap,
                                                     used.p, ctrs.p + 1);
        L++;
      }
      BC_CHECK_LAUNCH();
      int ovf = d2h_scalar(ctrs.p + 1, st);
      unsigned long long need = d2h_scalar(used.p, st);
      if (!ovf) break;
      if (attempt == 1) throw Error(BC_ECUDA, "2-hop output overflow after exact resize");
      cap = (int64_t)need;
    }
    up_ids = und_ids.p;
    if (slice) {  // export this shard's upper lists and stop
      DBuf<int64_t> l64, pos;
      s.slice_lens.alloc(n, st);
      l64.alloc(n + 1, st);
      pos.alloc(n + 1, st);
      l64.zero();
      slice_lens_k<<<blocks_for(n, 256), 256, 0, st>>>(seg_len.p, n, ntiles, s.slice_lens.p, l64.p);
      exclusive_scan(l64.p, pos.p, n + 1, st);
      s.slice_n_ids = d2h_scalar(pos.p + n, st);
      s.slice_ids.alloc(s.slice_n_ids ? s.slice_n_ids : 1, st);
      slice_copy<<<warp_blocks(n, sms), 256, 0, st>>>(seg_start.p, seg_len.p, n, ntiles, up_ids,
                                                       pos.p, s.slice_ids.p);
      BC_CHECK_LAUNCH();
      BC_CUDA(cudaStreamSynchronize(st));
      L += 4;
      return;
    }
    // |und(u)| = |up(u)| + |{w < u : u in up(w)}| (the relation is symmetric); the
    // directed lists are built from the upper pairs after the priority (below)
    {
      DBuf<int64_t> low;
      low.alloc(n, st);
      low.zero();
      lower_counts<<<warp_blocks(n, sms), 256, 0, st>>>(seg_start.p, seg_len.p, ntiles, up_ids,
                                                        n, low.p);
      add_sizes<<<blocks_for(n, 256), 256, 0, st>>>(s.und_size.p, low.p, n, s.und_size.p,
                                                     nullptr, nullptr);
      BC_CHECK_LAUNCH();
      s.und_pairs = 2 * (int64_t)d2h_scalar(used.p, st);
      L += 2;
    }
  } else {
    s.und_pairs = 0;
    seg_start.alloc((size_t)(n ? n : 1), st);
    seg_len.alloc((size_t)(n ? n : 1), st);
    seg_len.zero();
    seg_start.zero();
    und_ids.alloc(1, st);
    up_ids = und_ids.p;
    ntiles = 1;
    if (slice) {
      s.slice_lens.alloc(n ? n : 1, st);
      s.slice_lens.zero();
      s.slice_n_ids = 0;
      s.slice_ids.alloc(1, st);
      return;
    }
  }

  tm.mark("2-hop");
  // ---- priority (graph.py:227-243) or rank override (engine.py:130-134) ----
  s.rank.alloc(n ? n : 1, st);
  s.order.alloc(n ? n : 1, st);
  if (n > 0) {
    if (!cfg.rank_override) {
      DBuf<unsigned long long> keys, sorted;
      keys.alloc(n, st);
      sorted.alloc(n, st);
      priority_keys<<<blocks_for(n, 256), 256, 0, st>>>(s.und_size.p, n, keys.p);
      size_t tmp = 0;
      BC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.p, sorted.p, n, 0, 64, st));
      DBuf<char> t;
      t.alloc(tmp, st);
      BC_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, keys.p, sorted.p, n, 0, 64, st));
      priority_rank<<<blocks_for(n, 256), 256, 0, st>>>(sorted.p, n, s.rank.p, s.order.p);
      L += 3;
    } else {
      copy_h2d(s.rank.p, cfg.rank_override, n * sizeof(int64_t), st);
      DBuf<int64_t> ids, skeys;
      ids.alloc(n, st);
      skeys.alloc(n, st);
      iota64<<<blocks_for(n, 256), 256, 0, st>>>(ids.p, n);
      size_t tmp = 0;
      BC_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, s.rank.p, skeys.p, ids.p,
                                                        s.order.p, n, 0, 64, st));
      DBuf<char> t;
      t.alloc(tmp, st);
      BC_CUDA(cub::DeviceRadixSort::SortPairsDescending(t.p, tmp, s.rank.p, skeys.p, ids.p,
                                                        s.order.p, n, 0, 64, st));
      DBuf<int> dup;
      dup.alloc(1, st);
      dup.zero();
      adjacent_dupes<<<blocks_for(n, 256), 256, 0, st>>>(skeys.p, n, dup.p);
      L += 3;
      if (d2h_scalar(dup.p, st))
        throw Error(BC_EINVAL, "rank override must give one distinct value per anchor vertex");
    }
  }

  tm.mark("priority");
  // ---- directed 2-hop lists (graph.py:218-224) from the upper pairs: a pair (u, w),
  // u < w, goes to dir2(u) if rank[w] < rank[u], else to dir2(w); dir2(v) is its lower
  // entries (from other rows, sorted here) followed by its upper ones (already ascending)
  {
    DBuf<int64_t> dup, dlow, dsize, low_end;
    DBuf<unsigned long long> cur;
    dup.alloc(n + 1, st);
    dlow.alloc(n + 1, st);
    dsize.alloc(n + 1, st);
    low_end.alloc(n + 1, st);
    cur.alloc(n + 1, st);
    dup.zero();
    dlow.zero();
    dsize.zero();
    cur.zero();
    // work items: DIR_CHUNK upper pairs each
    const int64_t nseg = n * ntiles;
    const int64_t max_items = nseg + s.und_pairs / 2 / DIR_CHUNK + 1;
    DBuf<int64_t> item_n, item_off, item_mine, item_pre;
    DBuf<int32_t> item_seg;
    item_n.alloc(nseg + 1, st);
    item_off.alloc(nseg + 1, st);
    item_seg.alloc(max_items, st);
    item_mine.alloc(max_items + 1, st);
    item_pre.alloc(max_items + 1, st);
    item_n.zero();
    item_mine.zero();
    if (n > 0) {
      dir_items<<<blocks_for(nseg, 256), 256, 0, st>>>(seg_len.p, nseg, item_n.p);
      exclusive_scan(item_n.p, item_off.p, nseg + 1, st);
      dir_item_owner<<<blocks_for(nseg, 256), 256, 0, st>>>(item_off.p, nseg, item_seg.p);
      dir_counts<<<(unsigned)sms * 16, 256, 0, st>>>(seg_start.p, seg_len.p, ntiles, up_ids,
                                                     s.rank.p, item_off.p, item_seg.p, nseg, dup.p,
                                                     dlow.p, item_mine.p);
      exclusive_scan(item_mine.p, item_pre.p, max_items + 1, st);
      L += 5;
    }
    add_sizes<<<blocks_for(n, 256), 256, 0, st>>>(dup.p, dlow.p, n, dsize.p, nullptr, nullptr);
    s.dir_off.alloc(n + 1, st);
    exclusive_scan(dsize.p, s.dir_off.p, n + 1, st);
    s.dir2_pairs = d2h_scalar(s.dir_off.p + n, st);
    s.dir_idx.alloc(s.dir2_pairs, st);
    DBuf<int32_t> low_buf;
    low_buf.alloc(s.dir2_pairs ? s.dir2_pairs : 1, st);
    if (n > 0) {
      add_sizes<<<blocks_for(n, 256), 256, 0, st>>>(dsize.p, dlow.p, n, dsize.p, low_end.p,
                                                     s.dir_off.p);
      dir_fill<<<(unsigned)sms * 16, 256, 0, st>>>(seg_start.p, seg_len.p, ntiles, up_ids,
                                                   s.rank.p, item_off.p, item_seg.p, item_pre.p,
                                                   nseg, s.dir_off.p, dlow.p, cur.p, low_buf.p,
                                                   s.dir_idx.p);
      BC_CHECK_LAUNCH();
    }
    if (s.dir2_pairs > 0) {
      // the lower parts (ids < r, from the other endpoints' upper lists) arrive unordered;
      // every list is ordered by one radix sort of (r, id) keys over all pairs (upper
      // parts are already ascending and above r, so only the lower parts move)
      int ib = 1;
      while ((int64_t(1) << ib) < n) ib++;
      DBuf<unsigned long long> k0, k1;
      k0.alloc(s.dir2_pairs, st);
      k1.alloc(s.dir2_pairs, st);
      dir_sort_keys<<<warp_blocks(n, sms), 256, 0, st>>>(s.dir_off.p, low_end.p, low_buf.p,
                                                         s.dir_idx.p, n, ib, k0.p);
      size_t tmp = 0;
      BC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, k0.p, k1.p, s.dir2_pairs, 0, 2 * ib, st));
      DBuf<char> t;
      t.alloc(tmp, st);
      BC_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, k0.p, k1.p, s.dir2_pairs, 0, 2 * ib, st));
      key_low_ids<<<blocks_for(s.dir2_pairs, 256), 256, 0, st>>>(k1.p, s.dir2_pairs, ib,
                                                                 s.dir_idx.p);
      BC_CHECK_LAUNCH();
      L += 2;
    }
    L += 6;
  }
  tm.mark("directed");
  // ---- HTB encodings (htb.py:104-115) ----
  build_htb(s.aoff, s.aidx, n, g.n_e, s.hadj_off, s.hadj_idx, s.hadj_val, s.adj_words, s.max_adj_slice,
            sms, st, L);
  build_htb(s.dir_off.p, s.dir_idx.p, n, s.dir2_pairs, s.hdir_off, s.hdir_idx, s.hdir_val, s.dir2_words,
            s.max_dir_slice, sms, st, L);

  tm.mark("htb");
  // ---- dense bitmaps of the longest adjacency rows (probe = one load) ----
  s.dense_id.alloc(n ? n : 1, st);
  BC_CUDA(cudaMemsetAsync(s.dense_id.p, 0xff, (n ? n : 1) * sizeof(int32_t), st));
  s.dense_mw = (s.m + 31) / 32;
  if (n > 0 && s.m > 0) {
    DBuf<unsigned long long> hist;
    hist.alloc(DENSE_NT, st);
    hist.zero();
    dense_hist<<<blocks_for(n, 256), 256, 0, st>>>(s.hadj_off.p, n, hist.p);
    unsigned long long h[DENSE_NT];
    copy_d2h(h, hist.p, sizeof h, st);
    BC_CUDA(cudaStreamSynchronize(st));
    const int64_t budget = int64_t(64) << 20;  // bytes of dense rows (L2-sized)
    int pick = -1;
    for (int t = 0; t < DENSE_NT; t++) {
      const int64_t T = int64_t(16) << t;
      if (T >= s.dense_mw / 4) break;  // a row that long is already dense-ish: no gain
      if (h[t] > 0 && (int64_t)h[t] * s.dense_mw * 4 <= budget) {
        pick = t;
        break;
      }
    }
    L += 1;
    if (pick >= 0) {
      s.dense_T = 16 << pick;
      s.dense_rows = (int64_t)h[pick];
      DBuf<int32_t> flag, slot;
      flag.alloc(n, st);
      slot.alloc(n, st);
      dense_flags<<<blocks_for(n, 256), 256, 0, st>>>(s.hadj_off.p, n, s.dense_T, flag.p);
      exclusive_scan(flag.p, slot.p, n, st);
      dense_ids<<<blocks_for(n, 256), 256, 0, st>>>(flag.p, slot.p, n, s.dense_id.p);
      s.dense.alloc((size_t)s.dense_rows * s.dense_mw, st);
      s.dense.zero();
      dense_fill<<<warp_blocks(n, sms), 256, 0, st>>>(s.hadj_off.p, s.hadj_idx.p, s.hadj_val.p, n,
                                                      s.dense_id.p, s.dense.p, s.dense_mw);
      BC_CHECK_LAUNCH();
      L += 4;
    }
  }

  tm.mark("dense");
  // ---- tasks (engine.py:147-173) ----
  {
    DBuf<uint8_t> mask;
    if (cfg.roots) {
      mask.alloc(n ? n : 1, st);
      mask.zero();
      if (cfg.n_roots > 0) {
        DBuf<int32_t> r;
        r.alloc(cfg.n_roots, st);
        copy_h2d(r.p, cfg.roots, cfg.n_roots * sizeof(int32_t), st);
        set_mask<<<blocks_for(cfg.n_roots, 256), 256, 0, st>>>(r.p, cfg.n_roots, n, mask.p);
        L++;
      }
    }
    DBuf<int64_t> cnt, toff;
    DBuf<unsigned long long> filt;
    cnt.alloc(n + 1, st);
    cnt.zero();
    toff.alloc(n + 1, st);
    filt.alloc(1, st);
    filt.zero();
    if (n > 0)
      task_counts<<<blocks_for(n, 256), 256, 0, st>>>(s.order.p, s.und_size.p, s.dir_off.p,
                                                       cfg.roots ? mask.p : nullptr, n, s.p_eff,
                                                       cnt.p, filt.p);
    exclusive_scan(cnt.p, toff.p, n + 1, st);
    s.emitted = d2h_scalar(toff.p + n, st);
    s.filtered = (int64_t)d2h_scalar(filt.p, st);
    s.tasks.alloc(s.emitted, st);
    if (n > 0 && s.emitted)
      task_write<<<warp_blocks(n, sms), 256, 0, st>>>(s.order.p, toff.p, cnt.p, s.dir_off.p,
                                                      s.dir_idx.p, n, s.p_eff, s.tasks.p);
    s.troot.alloc(n ? n : 1, st);
    if (n > 0)
      root_task_off<<<blocks_for(n, 256), 256, 0, st>>>(s.order.p, toff.p, cnt.p, n, s.troot.p);
    L += 4;
  }
  tm.mark("tasks");
  (void)p;
}

}  // namespace bc
