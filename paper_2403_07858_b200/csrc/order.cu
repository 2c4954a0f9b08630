// order.cu -- "fast" order mode on device (north-star K2, K4a).
//
// a3  (q_eff, p_eff)-core pruning of the work graph: repeatedly drop anchor
//     vertices with fewer than q_eff neighbours and opposite vertices with fewer
//     than p_eff, to the fixpoint.  Every vertex of a (p_eff, q_eff)-biclique has
//     at least that many neighbours inside the biclique, so the count is unchanged
//     (not in the reference; its counters differ from the reference order's).
// a4  degree reorder (reorder.py:137-143 degree_order + graph.py:169-183 relabel):
//     both layers renumbered by (degree descending, id), dead vertices dropped,
//     rows re-sorted.  Count-invariant (test_reorder.py:147-154); hubs share the
//     low HTB words, so candidate sets and their local universes pack tighter.
//
// The peel is frontier-driven: each round marks the vertices that fell below
// their threshold and only their adjacency is walked to decrement the survivors'
// degrees, so the total work is O(E) over all rounds.
#include <cub/cub.cuh>

#include "engine.h"

namespace bc {

namespace {

__global__ void deg_init(const int64_t *__restrict__ off, int64_t n, int32_t *__restrict__ deg) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) deg[i] = (int32_t)(off[i + 1] - off[i]);
}

// alive vertices under the threshold die this round and join the frontier
__global__ void peel_mark(const int32_t *__restrict__ deg, uint8_t *__restrict__ dead, int64_t n,
                          int thr, int32_t *__restrict__ frontier, int *__restrict__ nf) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && !dead[i] && deg[i] < thr) {
    dead[i] = 1;
    frontier[atomicAdd(nf, 1)] = (int32_t)i;
  }
}

// warp per frontier vertex: its alive neighbours lose one degree
__global__ void peel_push(const int32_t *__restrict__ frontier, int nf,
                          const int64_t *__restrict__ off, const int32_t *__restrict__ idx,
                          const uint8_t *__restrict__ dead_other, int32_t *__restrict__ deg_other) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t f = gw; f < nf; f += nw) {
    const int u = frontier[f];
    for (int64_t e = off[u] + lane; e < off[u + 1]; e += 32) {
      const int w = idx[e];
      if (!dead_other[w]) atomicSub(deg_other + w, 1);
    }
  }
}

__global__ void max_alive_deg(const int32_t *__restrict__ deg, const uint8_t *__restrict__ dead,
                              int64_t n, int *out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int d = i < n && !dead[i] ? deg[i] : 0;
  d = (int)__reduce_max_sync(0xffffffffu, (unsigned)d);
  if ((threadIdx.x & 31) == 0 && d) atomicMax(out, d);
}

// new id of each alive vertex (dead: -1), given the alive vertices in new order
__global__ void scatter_ids(const int32_t *__restrict__ order, int64_t n_alive,
                            int32_t *__restrict__ newid) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n_alive) newid[order[i]] = (int32_t)i;
}

// sort keys (degree descending, id ascending) of the alive vertices; dead ones last
__global__ void order_keys(const int32_t *__restrict__ deg, const uint8_t *__restrict__ dead,
                           int64_t n, bool by_degree, unsigned long long *__restrict__ keys,
                           int32_t *__restrict__ ids) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long d = dead[i] ? 0ull : (unsigned long long)(by_degree ? deg[i] : 1) + 1;
  keys[i] = ((~d & 0xffffffffull) << 32) | (unsigned long long)i;  // ascending: big degree first
  ids[i] = (int32_t)i;
}

// row lengths of the pruned, relabelled view: new row newa[u] keeps the alive neighbours
__global__ void row_counts(const int64_t *__restrict__ off, const int32_t *__restrict__ idx,
                           int64_t n, const int32_t *__restrict__ newa,
                           const int32_t *__restrict__ newb, int64_t *__restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = gw; u < n; u += nw) {
    const int nu = newa[u];
    if (nu < 0) continue;
    int c = 0;
    for (int64_t e = off[u] + lane; e < off[u + 1]; e += 32) c += newb[idx[e]] >= 0;
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) cnt[nu] = c;
  }
}

// write the alive neighbours' new ids (order kept); rows re-sorted afterwards if relabelled
__global__ void row_write(const int64_t *__restrict__ off, const int32_t *__restrict__ idx,
                          int64_t n, const int32_t *__restrict__ newa,
                          const int32_t *__restrict__ newb, const int64_t *__restrict__ noff,
                          int32_t *__restrict__ nidx) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = gw; u < n; u += nw) {
    const int nu = newa[u];
    if (nu < 0) continue;
    int64_t pos = noff[nu];
    for (int64_t b = off[u]; b < off[u + 1]; b += 32) {
      const int64_t e = b + lane;
      int w = -1;
      if (e < off[u + 1]) w = newb[idx[e]];
      const unsigned m = __ballot_sync(0xffffffffu, w >= 0);
      if (w >= 0) nidx[pos + __popc(m & ((1u << lane) - 1u))] = w;
      pos += __popc(m);
    }
  }
}

inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t > 0 ? (n + t - 1) / t : 1); }

template <typename T>
void scan_excl(const T *in, T *out, int64_t n, cudaStream_t st) {
  size_t tmp = 0;
  BC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, st));
  DBuf<char> t;
  t.alloc(tmp, st);
  BC_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, n, st));
}

// one view of the new graph: rows of the alive `a` vertices, ids mapped through newb
void build_view(const int64_t *off, const int32_t *idx, int64_t n, const int32_t *newa,
                int64_t na, const int32_t *newb, bool resort, int64_t **noff_out,
                int32_t **nidx_out, int64_t &ne, int sms, cudaStream_t st, int64_t &L) {
  DBuf<int64_t> cnt;
  cnt.alloc(na + 1, st);
  cnt.zero();
  const unsigned wb = (unsigned)std::min<int64_t>(((n * 32) + 255) / 256 + 1, (int64_t)sms * 16);
  row_counts<<<wb, 256, 0, st>>>(off, idx, n, newa, newb, cnt.p);
  BC_CHECK_LAUNCH();
  int64_t *noff;
  BC_CUDA(pool_malloc((void **)&noff, (na + 1) * 8, st));
  scan_excl(cnt.p, noff, na + 1, st);
  BC_CUDA(cudaMemcpyAsync(&ne, noff + na, 8, cudaMemcpyDeviceToHost, st));
  BC_CUDA(cudaStreamSynchronize(st));
  int32_t *nidx;
  BC_CUDA(pool_malloc((void **)&nidx, (ne ? ne : 1) * 4, st));
  row_write<<<wb, 256, 0, st>>>(off, idx, n, newa, newb, noff, nidx);
  BC_CHECK_LAUNCH();
  L += 3;
  if (resort && ne > 0 && na > 0) {  // relabelled neighbours: sort every row
    DBuf<int32_t> sorted;
    sorted.alloc(ne, st);
    size_t tmp = 0;
    BC_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, nidx, sorted.p, ne, na, noff,
                                                noff + 1, st));
    DBuf<char> t;
    t.alloc(tmp, st);
    BC_CUDA(cub::DeviceSegmentedSort::SortKeys(t.p, tmp, nidx, sorted.p, ne, na, noff, noff + 1,
                                                st));
    BC_CUDA(cudaMemcpyAsync(nidx, sorted.p, ne * 4, cudaMemcpyDeviceToDevice, st));
    L += 1;
  }
  *noff_out = noff;
  *nidx_out = nidx;
}

}  // namespace

// Work graph of the fast order: `layer` is the anchor (0 = U); out.u = anchor view.
void fast_order(const DevGraph &g, int layer, int p_eff, int q_eff, bool reorder, DevGraph &out,
                int64_t &launches) {
  cudaStream_t st = g.stream;
  const int sms = num_sms(g.device);
  const int64_t n = layer == 0 ? g.n_u : g.n_v, m = layer == 0 ? g.n_v : g.n_u;
  const int64_t *aoff = layer == 0 ? g.u_off : g.v_off, *boff = layer == 0 ? g.v_off : g.u_off;
  const int32_t *aidx = layer == 0 ? g.u_idx : g.v_idx, *bidx = layer == 0 ? g.v_idx : g.u_idx;
  int64_t &L = launches;
  DBuf<int32_t> dega, degb, fa, fb;
  DBuf<uint8_t> deada, deadb;
  DBuf<int> nf;
  dega.alloc(n ? n : 1, st);
  degb.alloc(m ? m : 1, st);
  deada.alloc(n ? n : 1, st);
  deadb.alloc(m ? m : 1, st);
  fa.alloc(n ? n : 1, st);
  fb.alloc(m ? m : 1, st);
  nf.alloc(2, st);
  deada.zero();
  deadb.zero();
  deg_init<<<nblk(n), 256, 0, st>>>(aoff, n, dega.p);
  deg_init<<<nblk(m), 256, 0, st>>>(boff, m, degb.p);
  BC_CHECK_LAUNCH();
  L += 2;
  // ---- a3: peel to the (q_eff, p_eff)-core ----
  int64_t dead_a = 0, dead_b = 0;
  for (int round = 0;; round++) {
    nf.zero();
    peel_mark<<<nblk(n), 256, 0, st>>>(dega.p, deada.p, n, q_eff, fa.p, nf.p);
    peel_mark<<<nblk(m), 256, 0, st>>>(degb.p, deadb.p, m, p_eff, fb.p, nf.p + 1);
    BC_CHECK_LAUNCH();
    int h[2];
    BC_CUDA(cudaMemcpyAsync(h, nf.p, 8, cudaMemcpyDeviceToHost, st));
    BC_CUDA(cudaStreamSynchronize(st));
    L += 2;
    if (!h[0] && !h[1]) break;
    dead_a += h[0];
    dead_b += h[1];
    const unsigned g1 = (unsigned)std::min<int64_t>((int64_t)h[0] / 8 + 1, (int64_t)sms * 16);
    const unsigned g2 = (unsigned)std::min<int64_t>((int64_t)h[1] / 8 + 1, (int64_t)sms * 16);
    if (h[0]) peel_push<<<g1, 256, 0, st>>>(fa.p, h[0], aoff, aidx, deadb.p, degb.p);
    if (h[1]) peel_push<<<g2, 256, 0, st>>>(fb.p, h[1], boff, bidx, deada.p, dega.p);
    BC_CHECK_LAUNCH();
    L += 2;
  }
  // ---- new ids: alive vertices, by (degree desc, id) with a4, else by id ----
  DBuf<int32_t> newa, newb;
  newa.alloc(n ? n : 1, st);
  newb.alloc(m ? m : 1, st);
  int64_t na = 0, nb = 0;
  for (int side = 0; side < 2; side++) {
    const int64_t cnt = side == 0 ? n : m;
    DBuf<unsigned long long> keys, skeys;
    DBuf<int32_t> ids, sids;
    keys.alloc(cnt ? cnt : 1, st);
    skeys.alloc(cnt ? cnt : 1, st);
    ids.alloc(cnt ? cnt : 1, st);
    sids.alloc(cnt ? cnt : 1, st);
    int32_t *nid = side == 0 ? newa.p : newb.p;
    BC_CUDA(cudaMemsetAsync(nid, 0xff, (cnt ? cnt : 1) * 4, st));
    if (cnt == 0) continue;
    order_keys<<<nblk(cnt), 256, 0, st>>>(side == 0 ? dega.p : degb.p,
                                          side == 0 ? deada.p : deadb.p, cnt, reorder, keys.p,
                                          ids.p);
    size_t tmp = 0;
    BC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys.p, skeys.p, ids.p, sids.p, cnt, 0,
                                            64, st));
    DBuf<char> t;
    t.alloc(tmp, st);
    BC_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, keys.p, skeys.p, ids.p, sids.p, cnt, 0, 64,
                                            st));
    const int64_t nal = cnt - (side == 0 ? dead_a : dead_b);  // alive ones sort first
    scatter_ids<<<nblk(nal), 256, 0, st>>>(sids.p, nal, nid);
    BC_CHECK_LAUNCH();
    L += 3;
    (side == 0 ? na : nb) = nal;
  }
  // ---- the pruned (and relabelled) views ----
  out = DevGraph();
  out.device = g.device;
  out.stream = st;
  out.n_u = na;
  out.n_v = nb;
  int64_t ea = 0, eb = 0;
  build_view(aoff, aidx, n, newa.p, na, newb.p, reorder, &out.u_off, &out.u_idx, ea, sms, st, L);
  build_view(boff, bidx, m, newb.p, nb, newa.p, reorder, &out.v_off, &out.v_idx, eb, sms, st, L);
  if (ea != eb) throw Error(BC_ECUDA, "fast order: views disagree after pruning");
  out.n_e = ea;
  DBuf<int> md;
  md.alloc(2, st);
  md.zero();
  max_alive_deg<<<nblk(n), 256, 0, st>>>(dega.p, deada.p, n, md.p);
  max_alive_deg<<<nblk(m), 256, 0, st>>>(degb.p, deadb.p, m, md.p + 1);
  BC_CHECK_LAUNCH();
  int hm[2];
  BC_CUDA(cudaMemcpyAsync(hm, md.p, 8, cudaMemcpyDeviceToHost, st));
  BC_CUDA(cudaStreamSynchronize(st));
  out.max_deg_u = hm[0];
  out.max_deg_v = hm[1];
  L += 2;
}

void free_graph(DevGraph &g) {
  if (g.u_off) cudaFreeAsync(g.u_off, g.stream);
  if (g.u_idx) cudaFreeAsync(g.u_idx, g.stream);
  if (g.v_off) cudaFreeAsync(g.v_off, g.stream);
  if (g.v_idx) cudaFreeAsync(g.v_idx, g.stream);
  g.u_off = g.v_off = nullptr;
  g.u_idx = g.v_idx = nullptr;
}

}  // namespace bc
