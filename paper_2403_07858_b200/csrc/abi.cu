// abi.cu -- the C-ABI declared in include/bicount_b200.h.
//
// bc_count replaces the reference's count_bicliques (engine.py:419-500):
// validate like EngineConfig.validate / _build_shared (engine.py:53-61,
// 387-391), upload the CSR, run preprocessing (prep.cu) and the search
// (search.cu), and return the exact count and CountReport fields.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "engine.h"

namespace bc {
thread_local int64_t t_h2d_bytes = 0, t_d2h_bytes = 0;
}

namespace bc {

static std::mutex g_pool_mu;
static cudaMemPool_t g_pools[64] = {};

cudaMemPool_t lib_pool_if_created(int device) {
  if (device < 0 || device >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  return g_pools[device];
}

cudaMemPool_t lib_pool(int device) {
  cudaMemPool_t *pools = g_pools;
  if (device < 0 || device >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!pools[device]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[device] = p;
  }
  return pools[device];
}

}  // namespace bc

namespace {

thread_local std::string g_err;
thread_local int64_t g_last_launches = 0;  // kernels of the last bc_graph_border call
// One lock per device: calls on the same device serialise (they share its stream-ordered
// pool and the pool reservation below); calls on different devices run concurrently, so
// one process can drive several GPUs from several host threads (EngineConfig.devices).
std::mutex g_dev_mu[64];
std::mutex &dev_mu(int device) { return g_dev_mu[(unsigned)device & 63u]; }

// Stream-ordered pool reservation.  Every count allocates its scratch (2-hop ids,
// C_R1 lists, frame arenas: GBs at the FR-scale config) from the device's default
// pool; letting the pool grow piecemeal makes later large allocations remap
// physical memory (seen as 0.1-2 s stalls).  Before a count the pool is grown once,
// as one contiguous block, to the larger of an edge-count estimate and 1.5x the
// highest use seen so far on this device (regrown only when use comes within 10%
// of it); freed blocks then coalesce in place.
size_t g_pool_reserved[64];
size_t g_pool_high[64];

void pool_reserve(int device, int64_t n_edges, cudaStream_t st) {
  if (device < 0 || device >= 64) return;
  const size_t base = (size_t)n_edges * 160 + (size_t(256) << 20), high = g_pool_high[device];
  if (g_pool_reserved[device] >= std::max(base, high + high / 10)) return;
  const size_t want = std::max(base, high + high / 2);
  cudaMemPool_t pool = bc::lib_pool(device);
  if (!pool) return;
  cudaStreamSynchronize(st);
  cudaMemPoolTrimTo(pool, 0);
  void *p = nullptr;
  if (cudaMallocFromPoolAsync(&p, want, pool, st) == cudaSuccess) {
    cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    g_pool_reserved[device] = want;
  }
  unsigned long long zero = 0;  // the watermark tracks the counts' own use, not this block
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero);
  cudaGetLastError();  // a failed reservation (too little free memory) is not an error
}

void pool_record(int device) {
  if (device < 0 || device >= 64) return;
  cudaMemPool_t pool = bc::lib_pool(device);
  if (!pool) return;
  unsigned long long high = 0;
  if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &high) == cudaSuccess &&
      (size_t)high > g_pool_high[device])
    g_pool_high[device] = (size_t)high;
  cudaGetLastError();
}

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

__global__ void degree_stats(const int64_t *off, int64_t n, unsigned long long *wedge,
                             int *maxdeg) {
  unsigned long long w = 0;
  int md = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = off[i + 1] - off[i];
    w += (unsigned long long)(d * (d - 1) / 2);
    md = d > md ? (int)d : md;
  }
  w = bc::warp_sum(w);
  md = __reduce_max_sync(bc::FULL, (unsigned)md);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(wedge, w);
    atomicMax(maxdeg, md);
  }
}

void validate_config(const bc_config &c) {
  using bc::Error;
  if (c.batch_words < 1) throw Error(BC_EINVAL, "batch_buffer_capacity must be >= 1");
  if (c.mode != 0 && c.mode != 1) throw Error(BC_EINVAL, "mode must be one of ('dfs', 'hybrid')");
  if (c.anchor < -1 || c.anchor > 1) throw Error(BC_EINVAL, "anchor must be one of ('auto', 'U', 'V')");
  if (c.shard_count < 1 || c.shard_index < 0 || c.shard_index >= c.shard_count)
    throw Error(BC_EINVAL, "invalid shard_index / shard_count");
  if (c.order_mode < 0 || c.order_mode > 2)
    throw Error(BC_EINVAL, "order_mode must be one of ('reference', 'fast', 'fast-reorder')");
  if (c.order_mode != 0 && c.rank_override)
    throw Error(BC_EINVAL, "a rank override needs order_mode 'reference'");
  if (c.order_mode != 0 && c.roots)
    throw Error(BC_EINVAL, "roots= needs order_mode 'reference'");
}

void fill_from_structs(const bc::DevStructs &s, bc_report &out) {
  out.anchor = s.anchor;
  out.p_eff = s.p_eff;
  out.q_eff = s.q_eff;
  out.tasks_emitted = s.emitted;
  out.roots_filtered = s.filtered;
  out.und_pairs = s.und_pairs;
  out.dir2_pairs = s.dir2_pairs;
  out.adj_words = s.adj_words;
  out.dir2_words = s.dir2_words;
  out.max_slice_words = s.max_adj_slice > s.max_dir_slice ? s.max_adj_slice : s.max_dir_slice;
  out.kernel_launches += s.launches;
}

}  // namespace

struct bc_graph {
  bc::DevGraph g;
};

struct bc_structs {
  bc::DevGraph *g = nullptr;
  bc::DevStructs s;
};

extern "C" {

int bc_abi_version(void) { return BC_ABI_VERSION; }

const char *bc_last_error(void) { return g_err.c_str(); }

int64_t bc_last_launch_count(void) { return g_last_launches; }

int bc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

static int graph_create(const int64_t *u_off, const int32_t *u_idx, int64_t n_u,
                        const int64_t *v_off, const int32_t *v_idx, int64_t n_v, int32_t device,
                        bool on_device, bc_graph **out) {
  std::lock_guard<std::mutex> lk(dev_mu(device));
  g_err.clear();
  *out = nullptr;
  if (n_u < 0 || n_v < 0 || !u_off || !v_off) return fail(BC_EINVAL, "invalid graph arrays");
  if (n_u >= (int64_t(1) << 31) || n_v >= (int64_t(1) << 31))
    return fail(BC_EINVAL, "layer sizes must be < 2^31");
  int64_t e = 0, ev = 0;
  if (on_device) {
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaMemcpy(&e, u_off + n_u, 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(&ev, v_off + n_v, 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
      cudaGetLastError();
      return fail(BC_ECUDA, "cannot read device CSR offsets");
    }
  } else {
    e = u_off[n_u];
    ev = v_off[n_v];
  }
  if (ev != e) return fail(BC_EINVAL, "U and V views disagree on the edge count");
  bc_graph *h = new bc_graph();
  try {
    bc::DevGraph &g = h->g;
    g.device = device;
    BC_CUDA(cudaSetDevice(device));
    if (!bc::lib_pool(device)) throw bc::Error(BC_ECUDA, "cannot create the device memory pool");
    BC_CUDA(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
    g.n_u = n_u;
    g.n_v = n_v;
    g.n_e = e;
    cudaStream_t st = g.stream;
    BC_CUDA(bc::pool_malloc((void **)&g.u_off, (n_u + 1) * 8, st));
    BC_CUDA(bc::pool_malloc((void **)&g.v_off, (n_v + 1) * 8, st));
    BC_CUDA(bc::pool_malloc((void **)&g.u_idx, (e ? e : 1) * 4, st));
    BC_CUDA(bc::pool_malloc((void **)&g.v_idx, (e ? e : 1) * 4, st));
    if (on_device) {  // device-resident input (e.g. a torch CUDA tensor): D2D copy
      BC_CUDA(cudaMemcpyAsync(g.u_off, u_off, (n_u + 1) * 8, cudaMemcpyDeviceToDevice, st));
      BC_CUDA(cudaMemcpyAsync(g.v_off, v_off, (n_v + 1) * 8, cudaMemcpyDeviceToDevice, st));
      if (e) {
        BC_CUDA(cudaMemcpyAsync(g.u_idx, u_idx, e * 4, cudaMemcpyDeviceToDevice, st));
        BC_CUDA(cudaMemcpyAsync(g.v_idx, v_idx, e * 4, cudaMemcpyDeviceToDevice, st));
      }
    } else {
      bc::copy_h2d(g.u_off, u_off, (n_u + 1) * 8, st);
      bc::copy_h2d(g.v_off, v_off, (n_v + 1) * 8, st);
      if (e) {
        bc::copy_h2d(g.u_idx, u_idx, e * 4, st);
        bc::copy_h2d(g.v_idx, v_idx, e * 4, st);
      }
    }
    // wedge mass + max degree per layer (graph.py:246-249), once per graph
    unsigned long long *dw;
    int *dm;
    BC_CUDA(bc::pool_malloc((void **)&dw, 16, st));
    BC_CUDA(bc::pool_malloc((void **)&dm, 8, st));
    BC_CUDA(cudaMemsetAsync(dw, 0, 16, st));
    BC_CUDA(cudaMemsetAsync(dm, 0, 8, st));
    const int sms = bc::num_sms(device);
    degree_stats<<<sms * 4, 256, 0, st>>>(g.u_off, n_u, dw, dm);
    degree_stats<<<sms * 4, 256, 0, st>>>(g.v_off, n_v, dw + 1, dm + 1);
    BC_CHECK_LAUNCH();
    unsigned long long hw[2];
    int hm[2];
    bc::copy_d2h(hw, dw, 16, st);
    bc::copy_d2h(hm, dm, 8, st);
    BC_CUDA(cudaFreeAsync(dw, st));
    BC_CUDA(cudaFreeAsync(dm, st));
    BC_CUDA(cudaStreamSynchronize(st));
    g.wedge_u = (int64_t)hw[0];
    g.wedge_v = (int64_t)hw[1];
    g.max_deg_u = hm[0];
    g.max_deg_v = hm[1];
  } catch (const bc::Error &err) {
    bc_graph_destroy(h);
    return fail(err.code, err.what());
  }
  *out = h;
  return BC_OK;
}

int bc_graph_create(const int64_t *u_off, const int32_t *u_idx, int64_t n_u,
                    const int64_t *v_off, const int32_t *v_idx, int64_t n_v, int32_t device,
                    bc_graph **out) {
  return graph_create(u_off, u_idx, n_u, v_off, v_idx, n_v, device, false, out);
}

int bc_graph_create_device(const int64_t *u_off, const int32_t *u_idx, int64_t n_u,
                           const int64_t *v_off, const int32_t *v_idx, int64_t n_v,
                           int32_t device, bc_graph **out) {
  return graph_create(u_off, u_idx, n_u, v_off, v_idx, n_v, device, true, out);
}

void bc_graph_destroy(bc_graph *h) {
  if (!h) return;
  bc::DevGraph &g = h->g;
  cudaSetDevice(g.device);
  if (g.stream) {
    cudaFreeAsync(g.u_off, g.stream);
    cudaFreeAsync(g.v_off, g.stream);
    cudaFreeAsync(g.u_idx, g.stream);
    cudaFreeAsync(g.v_idx, g.stream);
    cudaStreamSynchronize(g.stream);
    cudaStreamDestroy(g.stream);
  }
  delete h;
}

// temporary work graph of the fast order modes, freed on every exit path
struct WorkGraph {
  bc::DevGraph g;
  ~WorkGraph() { bc::free_graph(g); }
};

static int count_impl(bc_graph *h, int32_t p, int32_t q, const bc_config *cfg, bc_report *out,
                      const bc::UpperPairs *upper = nullptr) {
  try {
    if (!h || !cfg || !out) throw bc::Error(BC_EINVAL, "null argument");
    validate_config(*cfg);
    if (p < 1 || q < 1) throw bc::Error(BC_EINVAL, "p and q must be >= 1");
    BC_CUDA(cudaSetDevice(h->g.device));
    pool_reserve(h->g.device, h->g.n_e, h->g.stream);
    const double t0 = now_s();
    bc::DevStructs s;
    cudaEvent_t a, b;
    BC_CUDA(cudaEventCreate(&a));
    BC_CUDA(cudaEventCreate(&b));
    BC_CUDA(cudaEventRecord(a, h->g.stream));
    // "fast" order modes: anchor choice on the input graph (graph.py:252-269), then the
    // (q_eff, p_eff)-core of the work graph (optionally degree-relabelled) with that
    // anchor as U; the count is the same, the structures and counters are not
    WorkGraph work;
    const bc::DevGraph *gp = &h->g;
    bc_config c2 = *cfg;
    int layer = -1, pp = p, qq = q;
    if (cfg->order_mode != 0) {
      layer = cfg->anchor < 0 ? (h->g.wedge_v <= h->g.wedge_u ? 0 : 1) : cfg->anchor;
      pp = layer == 0 ? p : q;
      qq = layer == 0 ? q : p;
      int64_t L = 0;
      bc::fast_order(h->g, layer, pp, qq, cfg->order_mode == 2, work.g, L);
      out->kernel_launches += L;
      c2.anchor = 0;
      gp = &work.g;
    }
    if (upper && cfg->order_mode != 0)
      throw bc::Error(BC_EINVAL, "injected 2-hop lists need order_mode 'reference'");
    bc::prepare(*gp, pp, qq, c2, s, upper);
    BC_CUDA(cudaEventRecord(b, h->g.stream));
    // _build_shared capacity check (engine.py:382-391)
    const int64_t max_words = s.max_adj_slice > s.max_dir_slice ? s.max_adj_slice : s.max_dir_slice;
    if (cfg->batch_words < max_words)
      throw bc::Error(BC_EINVAL, "batch_buffer_capacity " + std::to_string(cfg->batch_words) +
                                     " words is below the largest candidate slice (" +
                                     std::to_string(max_words) +
                                     " words); raise --batch-words");
    fill_from_structs(s, *out);
    if (layer >= 0) out->anchor = layer;
    bc::search(s, c2, *out);
    float ms = 0;
    BC_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    out->time_prep = ms * 1e-3;
    out->time_total = now_s() - t0;
    pool_record(h->g.device);
    if (out->overflow) throw bc::Error(BC_EOVERFLOW, "biclique count exceeds 128 bits");
  } catch (const bc::Error &err) {
    cudaStreamSynchronize(h ? h->g.stream : 0);
    return fail(err.code, err.what());
  }
  return BC_OK;
}

int bc_graph_count(bc_graph *h, int32_t p, int32_t q, const bc_config *cfg, bc_report *out) {
  std::lock_guard<std::mutex> lk(dev_mu(h ? h->g.device : 0));
  g_err.clear();
  if (out) std::memset(out, 0, sizeof *out);
  bc::t_h2d_bytes = bc::t_d2h_bytes = 0;
  const int rc = count_impl(h, p, q, cfg, out);
  if (out) {
    out->h2d_bytes = bc::t_h2d_bytes;
    out->d2h_bytes = bc::t_d2h_bytes;
  }
  return rc;
}

int bc_graph_count_upper(bc_graph *h, int32_t p, int32_t q, const bc_config *cfg,
                         const int64_t *upper_off, const int32_t *upper_ids, int64_t n_pairs,
                         bc_report *out) {
  std::lock_guard<std::mutex> lk(dev_mu(h ? h->g.device : 0));
  g_err.clear();
  if (out) std::memset(out, 0, sizeof *out);
  if (!upper_off || (n_pairs > 0 && !upper_ids) || n_pairs < 0)
    return fail(BC_EINVAL, "null or negative upper 2-hop arguments");
  bc::t_h2d_bytes = bc::t_d2h_bytes = 0;
  const bc::UpperPairs up{upper_off, upper_ids, n_pairs};
  const int rc = count_impl(h, p, q, cfg, out, &up);
  if (out) {
    out->h2d_bytes = bc::t_h2d_bytes;
    out->d2h_bytes = bc::t_d2h_bytes;
  }
  return rc;
}

int bc_assemble_upper(int32_t device, int32_t world, int64_t n, const int32_t *lens_all,
                      const int32_t *ids_all, int64_t ids_stride, int64_t *upper_off,
                      int32_t *upper_ids, int64_t ids_cap, int64_t *n_pairs) {
  std::lock_guard<std::mutex> lk(dev_mu(device));
  g_err.clear();
  try {
    if (!lens_all || !upper_off || !n_pairs || world < 1 || n < 0)
      throw bc::Error(BC_EINVAL, "bad argument");
    BC_CUDA(cudaSetDevice(device));
    cudaStream_t st = nullptr;
    BC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    try {
      *n_pairs = bc::assemble_upper(world, n, lens_all, ids_all, ids_stride, upper_off, upper_ids,
                                    ids_cap, st, bc::num_sms(device));
    } catch (...) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
      throw;
    }
    BC_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
  } catch (const bc::Error &err) {
    return fail(err.code, err.what());
  }
  return BC_OK;
}

int bc_graph_twohop_slice(bc_graph *h, int32_t p, int32_t q, const bc_config *cfg, int32_t shard,
                          int32_t nshards, bc_structs **out) {
  std::lock_guard<std::mutex> lk(dev_mu(h ? h->g.device : 0));
  g_err.clear();
  try {
    if (!h || !cfg || !out) throw bc::Error(BC_EINVAL, "null argument");
    *out = nullptr;
    if (nshards < 1 || shard < 0 || shard >= nshards) throw bc::Error(BC_EINVAL, "bad shard");
    if (cfg->order_mode != 0) throw bc::Error(BC_EINVAL, "2-hop slices need order_mode 'reference'");
    if (p < 1 || q < 1) throw bc::Error(BC_EINVAL, "p and q must be >= 1");
    BC_CUDA(cudaSetDevice(h->g.device));
    auto *r = new bc_structs;
    r->g = &h->g;
    const bc::SliceSpec sl{shard, nshards};
    try {
      bc::prepare(h->g, p, q, *cfg, r->s, nullptr, &sl);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
  } catch (const bc::Error &err) {
    cudaStreamSynchronize(h ? h->g.stream : 0);
    return fail(err.code, err.what());
  }
  return BC_OK;
}

int bc_count(const int64_t *u_off, const int32_t *u_idx, int64_t n_u, const int64_t *v_off,
             const int32_t *v_idx, int64_t n_v, int32_t p, int32_t q, const bc_config *cfg,
             bc_report *out) {
  if (out) std::memset(out, 0, sizeof *out);
  const double t0 = now_s();
  bc_graph *h = nullptr;
  bc::t_h2d_bytes = bc::t_d2h_bytes = 0;
  int rc = bc_graph_create(u_off, u_idx, n_u, v_off, v_idx, n_v, cfg ? cfg->device : 0, &h);
  if (rc != BC_OK) return rc;
  const double t1 = now_s();
  {
    std::lock_guard<std::mutex> lk(dev_mu(h->g.device));
    g_err.clear();
    rc = count_impl(h, p, q, cfg, out);
  }
  const double t2 = now_s();
  bc_graph_destroy(h);
  if (out) {
    out->time_h2d = t1 - t0;
    out->time_total = now_s() - t0;
    out->h2d_bytes = bc::t_h2d_bytes;
    out->d2h_bytes = bc::t_d2h_bytes;
    (void)t2;
  }
  return rc;
}

int bc_graph_enumerate(bc_graph *h, int32_t p, int32_t q, const bc_config *cfg,
                       int32_t *records, int64_t cap_words, int64_t *words_needed,
                       bc_report *out) {
  std::lock_guard<std::mutex> lk(dev_mu(h ? h->g.device : 0));
  g_err.clear();
  if (out) std::memset(out, 0, sizeof *out);
  try {
    if (!h || !cfg || !words_needed) throw bc::Error(BC_EINVAL, "null argument");
    validate_config(*cfg);
    if (cfg->order_mode != 0)
      throw bc::Error(BC_EINVAL, "enumeration needs order_mode 'reference'");
    if (p < 1 || q < 1) throw bc::Error(BC_EINVAL, "p and q must be >= 1");
    if (cap_words > 0 && !records) throw bc::Error(BC_EINVAL, "null record buffer");
    BC_CUDA(cudaSetDevice(h->g.device));
    bc::DevStructs s;
    bc::prepare(h->g, p, q, *cfg, s);
    const int64_t max_words = std::max(s.max_adj_slice, s.max_dir_slice);
    if (cfg->batch_words < max_words)
      throw bc::Error(BC_EINVAL, "batch_buffer_capacity " + std::to_string(cfg->batch_words) +
                                     " words is below the largest candidate slice (" +
                                     std::to_string(max_words) + " words); raise --batch-words");
    int64_t launches = 0;
    *words_needed = bc::enumerate_records(s, records, cap_words, launches);
    if (out) {
      fill_from_structs(s, *out);
      out->kernel_launches += launches;
    }
  } catch (const bc::Error &err) {
    cudaStreamSynchronize(h ? h->g.stream : 0);
    return fail(err.code, err.what());
  }
  return BC_OK;
}

int bc_graph_border(bc_graph *h, int32_t layer, int64_t iterations, int64_t *perm,
                    int64_t *history, int64_t *n_history) {
  std::lock_guard<std::mutex> lk(dev_mu(h ? h->g.device : 0));
  g_err.clear();
  try {
    if (!h || !history || !n_history) throw bc::Error(BC_EINVAL, "null argument");
    if (iterations < 0) throw bc::Error(BC_EINVAL, "iterations must be >= 0");
    if (layer != 0 && layer != 1) throw bc::Error(BC_EINVAL, "layer must be 0 (U) or 1 (V)");
    if (!perm && (layer == 0 ? h->g.n_u : h->g.n_v) > 0) throw bc::Error(BC_EINVAL, "null perm");
    BC_CUDA(cudaSetDevice(h->g.device));
    int64_t launches = 0;
    *n_history = bc::border_reorder(h->g, layer, iterations, perm, history, launches);
    g_last_launches = launches;
  } catch (const bc::Error &err) {
    cudaStreamSynchronize(h ? h->g.stream : 0);
    return fail(err.code, err.what());
  }
  return BC_OK;
}

int bc_prepare(bc_graph *h, int32_t p, int32_t q, const bc_config *cfg, bc_structs **out) {
  std::lock_guard<std::mutex> lk(dev_mu(h ? h->g.device : 0));
  g_err.clear();
  *out = nullptr;
  bc_structs *r = new bc_structs();
  try {
    if (!h || !cfg) throw bc::Error(BC_EINVAL, "null argument");
    validate_config(*cfg);
    if (cfg->order_mode != 0)
      throw bc::Error(BC_EINVAL, "structure export needs order_mode 'reference'");
    BC_CUDA(cudaSetDevice(h->g.device));
    r->g = &h->g;
    bc::prepare(h->g, p, q, *cfg, r->s);
    BC_CUDA(cudaStreamSynchronize(h->g.stream));
  } catch (const bc::Error &err) {
    delete r;
    return fail(err.code, err.what());
  }
  *out = r;
  return BC_OK;
}

int64_t bc_export_len(const bc_structs *r, int32_t what) {
  if (!r) return -1;
  const bc::DevStructs &s = r->s;
  const int64_t n = s.n;
  switch (what) {
    case BC_X_UND_SIZE:
    case BC_X_RANK:
    case BC_X_ORDER: return n;
    case BC_X_DIR_OFF:
    case BC_X_HADJ_OFF:
    case BC_X_HDIR_OFF: return n + 1;
    case BC_X_DIR_IDX: return s.dir2_pairs;
    case BC_X_HADJ_IDX:
    case BC_X_HADJ_VAL: return s.adj_words;
    case BC_X_HDIR_IDX:
    case BC_X_HDIR_VAL: return s.dir2_words;
    case BC_X_TASKS: return 2 * s.emitted;
    case BC_X_META: return 4;
    case BC_X_SLICE_LENS: return s.slice_n_ids >= 0 ? n : -1;
    case BC_X_SLICE_IDS: return s.slice_n_ids;
  }
  return -1;
}

// source pointer and element size of an export (device memory)
static const void *export_src(const bc::DevStructs &s, int32_t what, size_t &el) {
  el = 8;
  switch (what) {
    case BC_X_UND_SIZE: return s.und_size.p;
    case BC_X_RANK: return s.rank.p;
    case BC_X_ORDER: return s.order.p;
    case BC_X_DIR_OFF: return s.dir_off.p;
    case BC_X_DIR_IDX: el = 4; return s.dir_idx.p;
    case BC_X_HADJ_OFF: return s.hadj_off.p;
    case BC_X_HADJ_IDX: el = 4; return s.hadj_idx.p;
    case BC_X_HADJ_VAL: el = 4; return s.hadj_val.p;
    case BC_X_HDIR_OFF: return s.hdir_off.p;
    case BC_X_HDIR_IDX: el = 4; return s.hdir_idx.p;
    case BC_X_HDIR_VAL: el = 4; return s.hdir_val.p;
    case BC_X_TASKS: el = 4; return s.tasks.p;
    case BC_X_SLICE_LENS: el = 4; return s.slice_lens.p;
    case BC_X_SLICE_IDS: el = 4; return s.slice_ids.p;
  }
  return nullptr;
}

int bc_export_device(const bc_structs *r, int32_t what, void *device_dst) {
  std::lock_guard<std::mutex> lk(dev_mu(r ? r->g->device : 0));
  g_err.clear();
  try {
    if (!r) throw bc::Error(BC_EINVAL, "null argument");
    const int64_t len = bc_export_len(r, what);
    if (len < 0 || what == BC_X_META) throw bc::Error(BC_EINVAL, "unknown export id");
    if (len > 0 && !device_dst) throw bc::Error(BC_EINVAL, "null destination");
    BC_CUDA(cudaSetDevice(r->g->device));
    size_t el = 8;
    const void *src = export_src(r->s, what, el);
    if (len > 0) {
      BC_CUDA(cudaMemcpyAsync(device_dst, src, (size_t)len * el, cudaMemcpyDeviceToDevice,
                              r->s.stream));
      BC_CUDA(cudaStreamSynchronize(r->s.stream));
    }
  } catch (const bc::Error &err) {
    return fail(err.code, err.what());
  }
  return BC_OK;
}

int bc_export(const bc_structs *r, int32_t what, void *dst) {
  std::lock_guard<std::mutex> lk(dev_mu(r ? r->g->device : 0));
  g_err.clear();
  try {
    if (!r || !dst) throw bc::Error(BC_EINVAL, "null argument");
    const bc::DevStructs &s = r->s;
    BC_CUDA(cudaSetDevice(r->g->device));
    const int64_t len = bc_export_len(r, what);
    if (len < 0) throw bc::Error(BC_EINVAL, "unknown export id");
    const void *src = nullptr;
    size_t el = 8;
    switch (what) {
      case BC_X_UND_SIZE: src = s.und_size.p; break;
      case BC_X_RANK: src = s.rank.p; break;
      case BC_X_ORDER: src = s.order.p; break;
      case BC_X_DIR_OFF: src = s.dir_off.p; break;
      case BC_X_DIR_IDX: src = s.dir_idx.p; el = 4; break;
      case BC_X_HADJ_OFF: src = s.hadj_off.p; break;
      case BC_X_HADJ_IDX: src = s.hadj_idx.p; el = 4; break;
      case BC_X_HADJ_VAL: src = s.hadj_val.p; el = 4; break;
      case BC_X_HDIR_OFF: src = s.hdir_off.p; break;
      case BC_X_HDIR_IDX: src = s.hdir_idx.p; el = 4; break;
      case BC_X_HDIR_VAL: src = s.hdir_val.p; el = 4; break;
      case BC_X_TASKS: src = s.tasks.p; el = 4; break;
      case BC_X_SLICE_LENS: src = s.slice_lens.p; el = 4; break;
      case BC_X_SLICE_IDS: src = s.slice_ids.p; el = 4; break;
      case BC_X_META: {
        int64_t *d = (int64_t *)dst;
        d[0] = s.anchor; d[1] = s.p_eff; d[2] = s.q_eff; d[3] = s.n;
        return BC_OK;
      }
    }
    if (len > 0) {
      bc::copy_d2h(dst, src, (size_t)len * el, s.stream);
      BC_CUDA(cudaStreamSynchronize(s.stream));
    }
  } catch (const bc::Error &err) {
    return fail(err.code, err.what());
  }
  return BC_OK;
}

void bc_structs_destroy(bc_structs *r) {
  if (!r) return;
  cudaSetDevice(r->g->device);
  cudaStream_t st = r->s.stream;
  delete r;  // DBuf destructors free stream-ordered
  if (st) cudaStreamSynchronize(st);
}

void bc_shutdown(void) {
  // hand the library pools' cached memory back to the device (graphs and structures the
  // caller still holds keep their own allocations) and forget the reservations
  for (int d = 0; d < 64; d++) {
    std::lock_guard<std::mutex> lk(dev_mu(d));
    if (!bc::lib_pool_if_created(d)) continue;
    cudaSetDevice(d);
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(bc::lib_pool_if_created(d), 0);
    g_pool_reserved[d] = 0;
    g_pool_high[d] = 0;
  }
  cudaGetLastError();
}

int bc_debug_phase_cycles(uint64_t *out, int32_t n) {
  try {
    return (int)bc::debug_phase_cycles(out, n);
  } catch (const bc::Error &err) {
    return fail(err.code, err.what());
  }
}

}  // extern "C"
