// engine.h -- host-side orchestration types shared by prep.cu, search.cu, abi.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace bc {

// Device-resident CSR of both views (BipartiteGraph, graph.py:15-49).
struct DevGraph {
  int device = 0;
  int64_t n_u = 0, n_v = 0, n_e = 0;
  int64_t *u_off = nullptr;
  int32_t *u_idx = nullptr;
  int64_t *v_off = nullptr;
  int32_t *v_idx = nullptr;
  cudaStream_t stream = nullptr;
  int max_deg_u = 0, max_deg_v = 0;
  int64_t wedge_u = 0, wedge_v = 0;  // sum C(d,2) per layer (graph.py:246-249)
};

// The library's own stream-ordered pool on each device (created on first use, release
// threshold UINT64_MAX so freed scratch stays cached between calls).  Private, so the
// caching never changes the device's default pool that PyTorch or NCCL allocate from.
cudaMemPool_t lib_pool(int device);
cudaMemPool_t lib_pool_if_created(int device);  // null until the first allocation
inline cudaError_t pool_malloc(void **p, size_t bytes, cudaStream_t st) {
  int d = 0;
  cudaError_t e = cudaGetDevice(&d);
  if (e != cudaSuccess) return e;
  return cudaMallocFromPoolAsync(p, bytes, lib_pool(d), st);
}

// Stream-ordered device buffer.
template <typename T>
struct DBuf {
  T *p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  DBuf(DBuf &&o) noexcept { *this = std::move(o); }
  DBuf &operator=(DBuf &&o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    BC_CUDA(pool_malloc((void **)&p, (count ? count : 1) * sizeof(T), stream));
  }
  void zero() { if (n) BC_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s)); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
};

// Host<->device traffic of the current call (reported in bc_report).
extern thread_local int64_t t_h2d_bytes, t_d2h_bytes;

inline void copy_h2d(void *dst, const void *src, size_t n, cudaStream_t st) {
  if (!n) return;
  BC_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st));
  t_h2d_bytes += (int64_t)n;
}

inline void copy_d2h(void *dst, const void *src, size_t n, cudaStream_t st) {
  if (!n) return;
  BC_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st));
  t_d2h_bytes += (int64_t)n;
}

// Prepared structures on device (SearchStructures, engine.py:82-92).
struct DevStructs {
  int anchor = 0, p_eff = 0, q_eff = 0;
  int64_t n = 0, m = 0;  // anchor-layer and opposite-layer sizes
  // borrowed from DevGraph: work.u_adj / work.v_adj (engine.py:126)
  const int64_t *aoff = nullptr;
  const int32_t *aidx = nullptr;
  const int64_t *boff = nullptr;
  const int32_t *bidx = nullptr;
  int max_deg_anchor = 0;
  DBuf<int64_t> und_size, rank, order;
  DBuf<int64_t> dir_off;
  DBuf<int32_t> dir_idx;
  DBuf<int64_t> hadj_off, hdir_off;
  DBuf<uint32_t> hadj_idx, hadj_val, hdir_idx, hdir_val;
  DBuf<int2> tasks;  // (root, second) in emission order
  // first task id of each anchor vertex's tasks (-1 if it roots none): the tasks of
  // root r are troot[r] + j for its j-th dir2 entry (engine.py:160-172)
  DBuf<int64_t> troot;
  // dense bitmaps of the longest adjacency rows (hubs): dense[slot * dense_mw + w] is the
  // HTB Val of word w (0 if absent); dense_id[x] = slot or -1
  DBuf<int32_t> dense_id;
  DBuf<uint32_t> dense;
  int64_t dense_mw = 0, dense_rows = 0;
  int dense_T = 0;
  int64_t emitted = 0, filtered = 0;
  int64_t und_pairs = 0, dir2_pairs = 0, adj_words = 0, dir2_words = 0;
  int64_t max_adj_slice = 0, max_dir_slice = 0;
  int64_t launches = 0;
  cudaStream_t stream = nullptr;
  // 2-hop slice (sharded preprocessing): upper-list lengths of every anchor (0 unless
  // owned) and the owned anchors' upper ids in vertex order
  DBuf<int32_t> slice_lens, slice_ids;
  // wedge pool sum_{v in N(u)} deg(v) per anchor (saturated at 2^31 - 1) when the 2-hop
  // construction ran here (null when the upper lists were injected)
  DBuf<int32_t> pool;
  int64_t slice_n_ids = -1;
};

// Sharded preprocessing (multi-GPU): each rank builds the upper 2-hop lists of the
// anchors it owns; after an all-gather, every rank passes the whole upper CSR back in
// and prepare() skips the 2-hop construction.
struct UpperPairs {
  const int64_t *off;  // device int64[n + 1]
  const int32_t *ids;  // device int32[pairs], each list ascending, ids > its anchor
  int64_t pairs;
};
struct SliceSpec {
  int shard, nshards;
};

// Whole upper CSR from gathered slices (device pointers); returns the pair count.
int64_t assemble_upper(int world, int64_t n, const int32_t *lens_all, const int32_t *ids_all,
                       int64_t stride, int64_t *off_out, int32_t *ids_out, int64_t ids_cap,
                       cudaStream_t st, int sms);
int num_sms(int device);

// Preprocessing: anchor choice .. task emission (prep.cu).  With `slice`, stops after
// the owned anchors' upper 2-hop lists (s.slice_*); with `upper`, takes them as given.
void prepare(const DevGraph &g, int p, int q, const bc_config &cfg, DevStructs &s,
             const UpperPairs *upper = nullptr, const SliceSpec *slice = nullptr);

// Enumeration: level-1 pass + hybrid search (search.cu). Fills counters in out.
void search(const DevStructs &s, const bc_config &cfg, bc_report &out);

int num_sms(int device);

// Enumeration mode (emit.cu): leaf records [L (p_eff ids), |C_R|, C_R ids] of every task,
// copied to host_out when they fit cap_words; returns the words needed.
// border.cu: reorder.py:146-179 on the device; returns the history length
int64_t border_reorder(const DevGraph &g, int layer, int64_t iterations, int64_t *perm_out,
                       int64_t *hist_out, int64_t &launches);

int64_t enumerate_records(const DevStructs &s, int32_t *host_out, int64_t cap_words,
                          int64_t &launches);

// "fast" order mode (order.cu): the (q_eff, p_eff)-core of the work graph (anchor
// `layer` becomes U), optionally relabelled by degree; frees with free_graph.
void fast_order(const DevGraph &g, int layer, int p_eff, int q_eff, bool reorder, DevGraph &out,
                int64_t &launches);
void free_graph(DevGraph &g);

// BC_PHASE_PROF builds: per-phase SM cycles of the last enumeration (reset on read).
int64_t debug_phase_cycles(uint64_t *out, int n);

}  // namespace bc
