// border.cu -- Border column reordering on the device.
//
// Restates the reference's greedy 1-block reduction, reorder.py:146-179: each round
// takes the column owning the most 1-blocks (a stored (row, 32-column block) word
// with exactly one bit, reorder.py:67-79), the columns sharing the fewest rows with
// it (reorder.py:182-188), and swaps it with the first of those whose swap removes
// the most 1-blocks (reorder.py:82-110); it stops when no swap helps.  Ties follow
// the reference exactly (numpy argmax = first maximum; strict '>' over ascending
// partner ids = smallest id), so permutation and history are bit-identical.
//
// Device layout (B200-first, not the reference's dict):
//   * the block matrix is an open-addressing hash table of (row * nblocks + block)
//     -> mask, load <= 1/2, keys u64, values u32; zero masks stay as entries (the
//     reference deletes them; every count treats the two the same);
//   * per-column 1-block counts are kept incrementally by the swap kernel instead of
//     re-scanning the table every round (reorder.py:71-79 recounts);
//   * the swap profit of a partner n is decomposed (algebra below) so a round costs
//     sum_{r in rows(m)} deg(r) + sum over partners of deg(n) hash probes, spread over
//     the whole GPU, and a round is ~11 back-to-back launches with no host sync (the
//     host checks the stop flag and table headroom after rounds 1, 2, 4, .., 64 and
//     then every 64).
//
// Profit decomposition.  one(w) = [popc(w) == 1].  For the chosen column m at
// position (bm, jm) and a partner n at (bn, jn), bm != bn:
//   rows r in rows(m) only:  [one(wm) - one(wm & ~bit_m)] + [one(wn) - one(wn | bit_n)]
//     with bit_n clear in wn, the second bracket is g(wn) = [popc(wn)==1] - [wn==0],
//     so sum_r = dm_sum + cnt1[bn] + cntnz[bn] - deg(m), where dm_sum = sum of the
//     first brackets and cnt1 / cntnz count rows of m whose block-b word has one bit /
//     is non-zero (computed once per round for all blocks);
//   rows in rows(m) and rows(n): excluded by the reference; the term above counted
//     them with their actual words, so they are subtracted again;
//   rows in rows(n) only: evaluated directly (two probes).
#include <algorithm>
#include <vector>

#include "engine.h"

namespace bc {

namespace {

constexpr unsigned long long EMPTY = ~0ull;

struct BorderState {
  unsigned long long vm_key;   // argmax: (count << 32) | ~column
  unsigned long long best;     // best partner: (profit << 32) | ~column
  long long floor;             // min overlap over partners
  long long dm_sum;            // sum over rows(m) of the m-side bracket, minus deg(m)
  long long total;             // current number of 1-blocks
  long long nh;                // history entries written
  unsigned long long used;     // occupied table slots
  int done;
};

struct BorderArgs {
  const int64_t *coff;  // column -> rows (rows_of, reorder.py:61)
  const int32_t *cidx;
  const int64_t *roff;  // row -> columns (row_cols, reorder.py:62)
  const int32_t *ridx;
  int64_t ncols, nrows, nblocks;
  int32_t *pos, *colv;
  unsigned long long *key;
  uint32_t *val;
  unsigned long long cap;  // power of two
  int32_t *per;            // 1-blocks owned per column
  int32_t *ov;             // overlap with m per column
  int32_t *cnt1, *cntnz;   // per block
  uint8_t *flag;           // per row: 1 = row of m, 2 = row of n
  BorderState *st;
  int64_t *hist;
  int64_t hist_cap;
};

__device__ __forceinline__ unsigned long long hmix(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  return k;
}

__device__ __forceinline__ int one(uint32_t w) { return __popc(w) == 1; }

__device__ __forceinline__ uint32_t probe(const BorderArgs &A, int64_t r, int64_t b) {
  const unsigned long long k = (unsigned long long)r * A.nblocks + b;
  unsigned long long i = hmix(k) & (A.cap - 1);
  for (;;) {
    const unsigned long long x = A.key[i];
    if (x == k) return A.val[i];
    if (x == EMPTY) return 0u;
    i = (i + 1) & (A.cap - 1);
  }
}

// slot of key (row, block), inserted if absent
__device__ __forceinline__ uint32_t *slot(const BorderArgs &A, int64_t r, int64_t b) {
  const unsigned long long k = (unsigned long long)r * A.nblocks + b;
  unsigned long long i = hmix(k) & (A.cap - 1);
  for (;;) {
    unsigned long long x = A.key[i];
    if (x == EMPTY) {
      x = atomicCAS(A.key + i, EMPTY, k);
      if (x == EMPTY) {
        atomicAdd(&A.st->used, 1ull);
        return A.val + i;
      }
    }
    if (x == k) return A.val + i;
    i = (i + 1) & (A.cap - 1);
  }
}

__device__ __forceinline__ int64_t gtid() { return blockIdx.x * (int64_t)blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gthreads() { return (int64_t)gridDim.x * blockDim.x; }

// build_block_matrix (reorder.py:44-64): one thread per (column, row) edge
__global__ void bd_build(BorderArgs A) {
  for (int64_t c = gtid() >> 5; c < A.ncols; c += gthreads() >> 5) {
    const int64_t b = c >> 5;
    const uint32_t bit = 1u << (c & 31);
    for (int64_t e = A.coff[c] + lane_id(); e < A.coff[c + 1]; e += 32)
      atomicOr(slot(A, A.cidx[e], b), bit);
  }
  for (int64_t c = gtid(); c < A.ncols; c += gthreads()) {
    A.pos[c] = (int32_t)c;
    A.colv[c] = (int32_t)c;
  }
}

// initial 1-block total and per-column attribution (reorder.py:67-79)
__global__ void bd_count(BorderArgs A) {
  long long local = 0;
  for (int64_t i = gtid(); i < (int64_t)A.cap; i += gthreads()) {
    const unsigned long long k = A.key[i];
    const uint32_t w = A.val[i];
    if (k == EMPTY || !one(w)) continue;
    local++;
    const int64_t b = (int64_t)(k % (unsigned long long)A.nblocks);
    atomicAdd(A.per + A.colv[b * 32 + __ffs(w) - 1], 1);
  }
  local = warp_sum(local);
  if (lane_id() == 0 && local) atomicAdd((unsigned long long *)&A.st->total, (unsigned long long)local);
}

__global__ void bd_history0(BorderArgs A) {
  A.hist[0] = A.st->total;
  A.st->nh = 1;
  A.st->vm_key = 0;
  A.st->best = 0;
  A.st->floor = LLONG_MAX;
  A.st->dm_sum = 0;
}

// argmax of the per-column counts, first maximum (reorder.py:163-164)
__global__ void bd_argmax(BorderArgs A) {
  if (A.st->done) return;
  unsigned long long best = 0;
  for (int64_t c = gtid(); c < A.ncols; c += gthreads()) {
    const unsigned long long k =
        ((unsigned long long)(uint32_t)A.per[c] << 32) | (0xffffffffull - (unsigned long long)c);
    best = k > best ? k : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(FULL, best, o);
    best = t > best ? t : best;
  }
  if (lane_id() == 0) atomicMax(&A.st->vm_key, best);
}

__device__ __forceinline__ int64_t vm_of(const BorderArgs &A) {
  return (int64_t)(0xffffffffull - (A.st->vm_key & 0xffffffffull));
}

// Rows of m: flags, overlap counts (reorder.py:182-188), the per-block counts of the
// decomposition and dm_sum.  One warp per row of m, lanes over the row's columns.
__global__ void bd_rows_m(BorderArgs A) {
  if (A.st->done) return;
  const int64_t m = vm_of(A);
  const int64_t pm = A.pos[m], bm = pm >> 5;
  const uint32_t bit_m = 1u << (pm & 31);
  const int64_t e0 = A.coff[m], e1 = A.coff[m + 1];
  long long dm = 0;
  for (int64_t e = e0 + (gtid() >> 5); e < e1; e += gthreads() >> 5) {
    const int64_t r = A.cidx[e];
    if (lane_id() == 0) {
      A.flag[r] = 1;
      const uint32_t wm = probe(A, r, bm);
      dm += one(wm) - one(wm & ~bit_m) - 1;  // the -1: the -deg(m) of the decomposition
    }
    for (int64_t f = A.roff[r] + lane_id(); f < A.roff[r + 1]; f += 32) {
      const int64_t c = A.ridx[f];
      atomicAdd(A.ov + c, 1);
      const int32_t pc = A.pos[c];
      const uint32_t w = probe(A, r, pc >> 5);
      if (__ffs(w) - 1 == (pc & 31)) {  // count each (row, block) word once
        atomicAdd(A.cntnz + (pc >> 5), 1);
        if (one(w)) atomicAdd(A.cnt1 + (pc >> 5), 1);
      }
    }
  }
  dm = warp_sum(dm);
  if (lane_id() == 0 && dm) atomicAdd((unsigned long long *)&A.st->dm_sum, (unsigned long long)dm);
}

// floor = min overlap over the other columns (reorder.py:166-167)
__global__ void bd_floor(BorderArgs A) {
  if (A.st->done) return;
  const int64_t m = vm_of(A);
  long long lo = LLONG_MAX;
  for (int64_t c = gtid(); c < A.ncols; c += gthreads())
    if (c != m && A.ov[c] < lo) lo = A.ov[c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long t = __shfl_xor_sync(FULL, lo, o);
    lo = t < lo ? t : lo;
  }
  if (lane_id() == 0 && lo != LLONG_MAX) atomicMin(&A.st->floor, lo);
}

// swap profit of every minimum-overlap partner (reorder.py:168-174); one warp per
// partner, lanes over its rows.
__global__ void bd_profit(BorderArgs A) {
  if (A.st->done) return;
  const int64_t m = vm_of(A);
  const int64_t pm = A.pos[m], bm = pm >> 5;
  const uint32_t bit_m = 1u << (pm & 31);
  const long long fl = A.st->floor, base = A.st->dm_sum;
  unsigned long long best = 0;
  for (int64_t n = gtid() >> 5; n < A.ncols; n += gthreads() >> 5) {
    if (n == m || A.ov[n] != fl) continue;
    const int64_t pn = A.pos[n], bn = pn >> 5;
    if (bn == bm) continue;  // profit 0 (reorder.py:94-95)
    const uint32_t bit_n = 1u << (pn & 31);
    long long pr = 0;
    for (int64_t e = A.coff[n] + lane_id(); e < A.coff[n + 1]; e += 32) {
      const int64_t r = A.cidx[e];
      const uint32_t wm = probe(A, r, bm), wn = probe(A, r, bn);
      if (A.flag[r] & 1) {  // shared row: remove what the per-block term counted
        pr -= one(wm) - one(wm & ~bit_m) + one(wn);
      } else {
        pr += one(wm) + one(wn) - one(wm | bit_m) - one(wn & ~bit_n);
      }
    }
    pr = warp_sum(pr);
    pr += base + A.cnt1[bn] + A.cntnz[bn];
    if (pr > 0) {
      const unsigned long long k = ((unsigned long long)pr << 32) | (0xffffffffull - (unsigned long long)n);
      best = k > best ? k : best;
    }
  }
  if (lane_id() == 0 && best) atomicMax(&A.st->best, best);
}

__device__ __forceinline__ int64_t vn_of(const BorderArgs &A) {
  return (int64_t)(0xffffffffull - (A.st->best & 0xffffffffull));
}

// mark the rows of the chosen partner (or stop: no profitable swap, reorder.py:175-176)
__global__ void bd_rows_n(BorderArgs A) {
  if (A.st->done) return;
  if (A.st->best == 0) return;
  const int64_t n = vn_of(A);
  for (int64_t e = A.coff[n] + gtid(); e < A.coff[n + 1]; e += gthreads()) A.flag[A.cidx[e]] |= 2;
}

// apply_swap (reorder.py:113-134) on the rows of the symmetric difference, with the
// per-column 1-block counts moved along: a changed word releases its old owner and
// credits the new one; in rows holding both columns the words keep their bits but
// trade owners.
__device__ __forceinline__ void own_dec(const BorderArgs &A, int64_t blk, uint32_t w) {
  if (one(w)) atomicSub(A.per + A.colv[blk * 32 + __ffs(w) - 1], 1);
}

__global__ void bd_apply(BorderArgs A) {
  if (A.st->done || A.st->best == 0) return;
  const int64_t m = vm_of(A), n = vn_of(A);
  const int64_t pm = A.pos[m], pn = A.pos[n];
  const int64_t bm = pm >> 5, bn = pn >> 5;
  const uint32_t bit_m = 1u << (pm & 31), bit_n = 1u << (pn & 31);
  auto colv_new = [&](int64_t p) -> int64_t { return p == pm ? n : p == pn ? m : A.colv[p]; };
  auto own_inc = [&](int64_t blk, uint32_t w) {
    if (one(w)) atomicAdd(A.per + colv_new(blk * 32 + __ffs(w) - 1), 1);
  };
  const int64_t dm = A.coff[m + 1] - A.coff[m], dn = A.coff[n + 1] - A.coff[n];
  for (int64_t i = gtid(); i < dm + dn; i += gthreads()) {
    const bool from_m = i < dm;
    const int64_t r = from_m ? A.cidx[A.coff[m] + i] : A.cidx[A.coff[n] + i - dm];
    const int f = A.flag[r];
    if (f == 3) {
      if (!from_m) continue;
      // both columns in row r: bits stay, owners of 1-blocks at pm / pn swap
      const uint32_t wm = probe(A, r, bm), wn = probe(A, r, bn);
      if (one(wm)) {
        atomicSub(A.per + m, 1);
        atomicAdd(A.per + n, 1);
      }
      if (one(wn)) {
        atomicSub(A.per + n, 1);
        atomicAdd(A.per + m, 1);
      }
      continue;
    }
    const int64_t sb = from_m ? bm : bn, db = from_m ? bn : bm;
    const uint32_t sbit = from_m ? bit_m : bit_n, dbit = from_m ? bit_n : bit_m;
    uint32_t *s = slot(A, r, sb), *d = slot(A, r, db);
    const uint32_t ws = *s, wd = *d;
    own_dec(A, sb, ws);
    own_dec(A, db, wd);
    *s = ws & ~sbit;
    *d = wd | dbit;
    own_inc(sb, ws & ~sbit);
    own_inc(db, wd | dbit);
  }
}

// finish the round: positions, history, reset the per-round reductions
__global__ void bd_finish(BorderArgs A) {
  BorderState *S = A.st;
  if (S->done) return;
  if (S->best == 0) {
    S->done = 1;
    return;
  }
  const int64_t m = vm_of(A), n = vn_of(A);
  const int32_t pm = A.pos[m], pn = A.pos[n];
  A.pos[m] = pn;
  A.pos[n] = pm;
  A.colv[pm] = (int32_t)n;
  A.colv[pn] = (int32_t)m;
  S->total -= (long long)(S->best >> 32);
  if (S->nh < A.hist_cap) A.hist[S->nh] = S->total;
  S->nh++;
  S->vm_key = 0;
  S->best = 0;
  S->floor = LLONG_MAX;
  S->dm_sum = 0;
}

__global__ void bd_rehash(BorderArgs A, const unsigned long long *okey, const uint32_t *oval,
                          unsigned long long ocap) {
  for (int64_t i = gtid(); i < (int64_t)ocap; i += gthreads()) {
    const unsigned long long k = okey[i];
    if (k == EMPTY) continue;
    const int64_t r = (int64_t)(k / (unsigned long long)A.nblocks), b = (int64_t)(k % A.nblocks);
    *slot(A, r, b) = oval[i];
  }
}

unsigned long long pow2_at_least(unsigned long long x) {
  unsigned long long c = 1024;
  while (c < x) c <<= 1;
  return c;
}

}  // namespace

int64_t border_reorder(const DevGraph &g, int layer, int64_t iterations, int64_t *perm_out,
                       int64_t *hist_out, int64_t &launches) {
  cudaStream_t s = g.stream;
  BorderArgs A{};
  A.coff = layer == 0 ? g.u_off : g.v_off;
  A.cidx = layer == 0 ? g.u_idx : g.v_idx;
  A.roff = layer == 0 ? g.v_off : g.u_off;
  A.ridx = layer == 0 ? g.v_idx : g.u_idx;
  A.ncols = layer == 0 ? g.n_u : g.n_v;
  A.nrows = layer == 0 ? g.n_v : g.n_u;
  if (A.ncols >= (int64_t(1) << 31) - 1) throw Error(BC_EINVAL, "border: layer too large");
  A.nblocks = std::max<int64_t>((A.ncols + 31) / 32, 1);
  const int64_t maxdeg = std::max(layer == 0 ? g.max_deg_u : g.max_deg_v, 1);
  constexpr int64_t CHECK = 64;  // rounds between host checks
  const int64_t headroom = CHECK * 2 * maxdeg;
  A.cap = pow2_at_least(2 * (unsigned long long)(g.n_e + headroom));
  DBuf<unsigned long long> key;
  DBuf<uint32_t> val;
  DBuf<int32_t> pos, colv, per, ov, cnt1, cntnz;
  DBuf<uint8_t> flag;
  DBuf<BorderState> st;
  DBuf<int64_t> hist;
  key.alloc(A.cap, s);
  val.alloc(A.cap, s);
  BC_CUDA(cudaMemsetAsync(key.p, 0xff, A.cap * 8, s));
  val.zero();
  pos.alloc(A.ncols, s);
  colv.alloc(A.ncols, s);
  per.alloc(A.ncols, s);
  ov.alloc(A.ncols, s);
  cnt1.alloc(A.nblocks, s);
  cntnz.alloc(A.nblocks, s);
  flag.alloc(std::max<int64_t>(A.nrows, 1), s);
  st.alloc(1, s);
  hist.alloc(iterations + 1, s);
  per.zero();
  st.zero();
  A.key = key.p;
  A.val = val.p;
  A.pos = pos.p;
  A.colv = colv.p;
  A.per = per.p;
  A.ov = ov.p;
  A.cnt1 = cnt1.p;
  A.cntnz = cntnz.p;
  A.flag = flag.p;
  A.st = st.p;
  A.hist = hist.p;
  A.hist_cap = iterations + 1;
  int sms = 148;
  BC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g.device));
  const unsigned grid = (unsigned)sms * 8, tpb = 256;
  bd_build<<<grid, tpb, 0, s>>>(A);
  bd_count<<<grid, tpb, 0, s>>>(A);
  bd_history0<<<1, 1, 0, s>>>(A);
  launches += 3;
  BC_CHECK_LAUNCH();
  if (A.ncols >= 2) {
    for (int64_t it = 0; it < iterations; it++) {
      if (it > 0 && (it % CHECK == 0 || (it & (it - 1)) == 0)) {  // 1, 2, 4, .. then every 64
        BorderState h{};
        copy_d2h(&h, st.p, sizeof h, s);
        BC_CUDA(cudaStreamSynchronize(s));
        if (h.done) break;
        if (2 * (h.used + (unsigned long long)headroom) > A.cap) {  // grow the table
          DBuf<unsigned long long> okey = std::move(key);
          DBuf<uint32_t> oval = std::move(val);
          const unsigned long long ocap = A.cap;
          A.cap = pow2_at_least(2 * (h.used + 2 * (unsigned long long)headroom));
          key.alloc(A.cap, s);
          val.alloc(A.cap, s);
          BC_CUDA(cudaMemsetAsync(key.p, 0xff, A.cap * 8, s));
          val.zero();
          A.key = key.p;
          A.val = val.p;
          BC_CUDA(cudaMemsetAsync(&st.p->used, 0, sizeof(unsigned long long), s));
          bd_rehash<<<grid, tpb, 0, s>>>(A, okey.p, oval.p, ocap);
          launches++;
        }
      }
      BC_CUDA(cudaMemsetAsync(ov.p, 0, A.ncols * 4, s));
      BC_CUDA(cudaMemsetAsync(cnt1.p, 0, A.nblocks * 4, s));
      BC_CUDA(cudaMemsetAsync(cntnz.p, 0, A.nblocks * 4, s));
      BC_CUDA(cudaMemsetAsync(flag.p, 0, std::max<int64_t>(A.nrows, 1), s));
      bd_argmax<<<grid, tpb, 0, s>>>(A);
      bd_rows_m<<<grid, tpb, 0, s>>>(A);
      bd_floor<<<grid, tpb, 0, s>>>(A);
      bd_profit<<<grid, tpb, 0, s>>>(A);
      bd_rows_n<<<grid, tpb, 0, s>>>(A);
      bd_apply<<<grid, tpb, 0, s>>>(A);
      bd_finish<<<1, 1, 0, s>>>(A);
      launches += 7;
    }
    BC_CHECK_LAUNCH();
  }
  BorderState h{};
  copy_d2h(&h, st.p, sizeof h, s);
  BC_CUDA(cudaStreamSynchronize(s));
  const int64_t nh = std::min<int64_t>(h.nh, iterations + 1);
  copy_d2h(hist_out, hist.p, nh * 8, s);
  std::vector<int32_t> p32(A.ncols);
  copy_d2h(p32.data(), pos.p, A.ncols * 4, s);
  BC_CUDA(cudaStreamSynchronize(s));
  for (int64_t c = 0; c < A.ncols; c++) perm_out[c] = p32[c];
  return nh;
}

}  // namespace bc
