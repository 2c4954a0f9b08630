// emit.cu -- enumeration mode (EngineConfig.enumerate_results).
//
// Restates the reference's enumerating search (engine.py:265-304, 315-374, _emit at
// 301-304): one thread per (root, second) task walks the same hybrid search on the HTB
// slices -- C_R = C_R & N(u), C_L = C_L & dir2(u) as sorted-merge intersections
// (htb.py:122-154) -- with prune_keep (engine.py:110-112), and every leaf with
// |C_R| >= q_eff writes one record [L members (p_eff ids), |C_R|, C_R ids] to a global
// buffer.  The host expands each record into its combinations(C_R, q_eff) pairs,
// normalises V-anchored pairs and sorts (engine.py:480-483).  Output-bound by nature, so
// it favours simplicity over the counting kernels' machinery; the count path is untouched.
#include "engine.h"

namespace bc {

namespace {

// sorted merge of two HTB slices into (idx, val) words; returns the word count
__device__ int htb_and(const uint32_t *__restrict__ aidx, const uint32_t *__restrict__ aval,
                       int64_t a0, int64_t a1, const uint32_t *bidx, const uint32_t *bval,
                       int64_t b0, int64_t b1, uint32_t *oidx, uint32_t *oval) {
  int n = 0;
  while (a0 < a1 && b0 < b1) {
    const uint32_t x = aidx[a0], y = bidx[b0];
    if (x < y) a0++;
    else if (y < x) b0++;
    else {
      const uint32_t v = aval[a0] & bval[b0];
      if (v) {
        oidx[n] = x;
        oval[n] = v;
        n++;
      }
      a0++;
      b0++;
    }
  }
  return n;
}

__device__ int card(const uint32_t *val, int n) {
  int c = 0;
  for (int i = 0; i < n; i++) c += __popc(val[i]);
  return c;
}

struct EmitArgs {
  const int64_t *aoff;  // adjacency HTB (htb.py:64-86)
  const uint32_t *aidx, *aval;
  const int64_t *doff;  // dir2 HTB
  const uint32_t *didx, *dval;
  const int2 *tasks;
  int64_t t0, n_tasks;   // this launch: tasks [t0, t0 + n_tasks)
  int p_eff, q_eff;
  int64_t mw, ml;        // scratch words per level (max adjacency / dir2 slice words)
  uint32_t *scratch;     // per thread: p_eff levels x (2 mw + 2 ml) words
  int32_t *out;          // records
  int64_t cap;
  unsigned long long *used;
};

__device__ void emit_record(const EmitArgs &A, const int *chain, int nchain,
                            const uint32_t *ridx, const uint32_t *rval, int rw, int c) {
  const unsigned long long need = (unsigned long long)(nchain + 1 + c);
  const unsigned long long at = atomicAdd(A.used, need);
  if ((int64_t)(at + need) > A.cap) return;  // the host retries with the exact size
  int32_t *o = A.out + at;
  for (int i = 0; i < nchain; i++) *o++ = chain[i];
  *o++ = c;
  for (int k = 0; k < rw; k++) {
    uint32_t v = rval[k];
    while (v) {
      *o++ = (int32_t)(ridx[k] * 32 + __ffs(v) - 1);
      v &= v - 1;
    }
  }
}

__global__ void emit_kernel(EmitArgs A) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= A.n_tasks) return;
  const int64_t t = A.t0 + i;
  const int p = A.p_eff, q = A.q_eff;
  const int r = A.tasks[t].x, s = A.tasks[t].y;
  int chain[64];
  chain[0] = r;
  // per level: C_R words (idx, val) and C_L words (idx, val); level 1 at slot 0
  uint32_t *base = A.scratch + i * (int64_t)p * (2 * A.mw + 2 * A.ml);
  auto Ri = [&](int l) { return base + (int64_t)l * (2 * A.mw + 2 * A.ml); };
  auto Rv = [&](int l) { return Ri(l) + A.mw; };
  auto Li = [&](int l) { return Ri(l) + 2 * A.mw; };
  auto Lv = [&](int l) { return Ri(l) + 2 * A.mw + A.ml; };
  if (p == 1) {  // engine.py:267-275: every neighbour set of size >= q
    const int64_t a0 = A.aoff[r], a1 = A.aoff[r + 1];
    const int c = card(A.aval + a0, (int)(a1 - a0));
    if (c >= q) emit_record(A, chain, 1, A.aidx + a0, A.aval + a0, (int)(a1 - a0), c);
    return;
  }
  chain[1] = s;
  int rw[64], lw[64], pos[64];
  rw[0] = htb_and(A.aidx, A.aval, A.aoff[r], A.aoff[r + 1], A.aidx, A.aval, A.aoff[s],
                  A.aoff[s + 1], Ri(0), Rv(0));
  const int c1 = card(Rv(0), rw[0]);
  if (c1 < q) return;
  if (p == 2) {
    emit_record(A, chain, 2, Ri(0), Rv(0), rw[0], c1);
    return;
  }
  lw[0] = htb_and(A.didx, A.dval, A.doff[r], A.doff[r + 1], A.didx, A.dval, A.doff[s],
                  A.doff[s + 1], Li(0), Lv(0));
  if (card(Lv(0), lw[0]) < p - 2) return;  // prune_keep(cr, cl, 1)
  // DFS over the candidates of each level's C_L, ascending (engine.py:315-374)
  int level = 1;  // node at `level` has its sets in slot level - 1
  pos[0] = 0;
  while (level >= 1) {
    const int li = level - 1;
    // next candidate u of this node: the pos[li]-th id of C_L
    int u = -1;
    {
      int k = pos[li], seen = 0;
      for (int w = 0; w < lw[li] && u < 0; w++) {
        const int c = __popc(Lv(li)[w]);
        if (k < seen + c) {
          u = (int)(Li(li)[w] * 32 + __fns(Lv(li)[w], 0, k - seen + 1));
        }
        seen += c;
      }
    }
    if (u < 0) {
      level--;
      continue;
    }
    pos[li]++;
    const int child = level + 1;  // the child's L has child + 1 members
    chain[child] = u;
    const int cw = htb_and(Ri(li), Rv(li), 0, rw[li], A.aidx, A.aval, A.aoff[u], A.aoff[u + 1],
                           Ri(child - 1), Rv(child - 1));
    const int cc = card(Rv(child - 1), cw);
    if (cc < q) continue;
    if (child == p - 1) {  // a leaf: L = chain[0..p)
      emit_record(A, chain, p, Ri(child - 1), Rv(child - 1), cw, cc);
      continue;
    }
    const int lwn = htb_and(Li(li), Lv(li), 0, lw[li], A.didx, A.dval, A.doff[u], A.doff[u + 1],
                            Li(child - 1), Lv(child - 1));
    if (card(Lv(child - 1), lwn) < p - child - 1) continue;  // prune_keep(cr, cl, child)
    rw[child - 1] = cw;
    lw[child - 1] = lwn;
    pos[child - 1] = 0;
    level = child;
  }
}

}  // namespace

int64_t enumerate_records(const DevStructs &s, int32_t *host_out, int64_t cap_words,
                          int64_t &launches) {
  cudaStream_t st = s.stream;
  if (s.p_eff > 62) throw Error(BC_EINVAL, "enumeration supports p_eff <= 62");
  EmitArgs A{};
  A.aoff = s.hadj_off.p;
  A.aidx = s.hadj_idx.p;
  A.aval = s.hadj_val.p;
  A.doff = s.hdir_off.p;
  A.didx = s.hdir_idx.p;
  A.dval = s.hdir_val.p;
  A.tasks = s.tasks.p;
  A.p_eff = s.p_eff;
  A.q_eff = s.q_eff;
  A.mw = std::max<int64_t>(s.max_adj_slice, 1);
  A.ml = std::max<int64_t>(s.max_dir_slice, 1);
  const int64_t per = (int64_t)s.p_eff * (2 * A.mw + 2 * A.ml);
  constexpr int64_t CHUNK = 1 << 16;  // tasks per launch (scratch reused)
  DBuf<uint32_t> scratch;
  DBuf<int32_t> out;
  DBuf<unsigned long long> used;
  scratch.alloc((size_t)std::max<int64_t>(std::min(s.emitted, CHUNK), 1) * per, st);
  out.alloc((size_t)std::max<int64_t>(cap_words, 1), st);
  used.alloc(1, st);
  used.zero();
  A.scratch = scratch.p;
  A.out = out.p;
  A.cap = cap_words;
  A.used = used.p;
  for (int64_t t0 = 0; t0 < s.emitted; t0 += CHUNK) {
    A.t0 = t0;
    A.n_tasks = std::min(CHUNK, s.emitted - t0);
    emit_kernel<<<(unsigned)((A.n_tasks + 127) / 128), 128, 0, st>>>(A);
    BC_CHECK_LAUNCH();
    launches++;
  }
  unsigned long long n = 0;
  copy_d2h(&n, used.p, sizeof n, st);
  BC_CUDA(cudaStreamSynchronize(st));
  if ((int64_t)n <= cap_words && n > 0) {
    copy_d2h(host_out, out.p, n * sizeof(int32_t), st);
    BC_CUDA(cudaStreamSynchronize(st));
  }
  return (int64_t)n;
}

}  // namespace bc
