/*
 * bicount_b200.h -- C-ABI of the B200 (sm_100a) (p,q)-biclique counting path.
 *
 * The reference exposes this path as one Python call,
 *   count_bicliques(g, p, q, cfg, *, structures=None, roots=None) -> CountReport
 * (/root/reference/pkg/src/bicount/engine.py:419-500), with preprocessing in
 * prepare_structures (engine.py:115-144).  This library is the compiled side
 * of that call: plain pointers and sizes, no torch types, bound from Python
 * with ctypes (paper_2403_07858_b200/_abi.py).  See INTEGRATION.md for the
 * binding a reference maintainer would add.
 *
 * Ownership: every input pointer is borrowed, read-only, for the duration
 * of the call.  Output structs are caller-allocated.  Device memory is owned
 * by the library: bc_count frees everything before returning; a bc_graph
 * handle owns its device-resident CSR until bc_graph_destroy.
 *
 * Errors: 0 = ok, < 0 = error code below; message via bc_last_error()
 * (thread-local).  The Python shim maps BC_EINVAL -> ValueError, the rest
 * -> RuntimeError, mirroring the reference's exceptions
 * (engine.py:53-61, 123-124, 132-133, 387-391).  An exact count that would
 * exceed 2^128 is BC_EOVERFLOW, never a wrapped value.
 */
#ifndef BICOUNT_B200_H
#define BICOUNT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BC_OK 0
#define BC_EINVAL (-1)
#define BC_ECUDA (-2)
#define BC_ENCCL (-3)
#define BC_EOOM (-4)
#define BC_EOVERFLOW (-5)
#define BC_EASSERT (-6)     /* BC_FLAG_CHECK_NESTING found a violation (the reference's
                               AssertionError, engine.py:365-366) */

#define BC_ABI_VERSION 3

/* EngineConfig (engine.py:43-61) plus the device-side knobs. */
typedef struct bc_config {
  int32_t batch_words;    /* EngineConfig.batch_buffer_capacity: validated against the
                             largest HTB slice (engine.py:382-391) and used for the
                             reference batch accounting (engine.py:306-313) */
  int32_t mode;           /* 0 = "dfs", 1 = "hybrid" (EngineConfig.mode) */
  int32_t anchor;         /* -1 = "auto", 0 = "U", 1 = "V" (EngineConfig.anchor) */
  int32_t order_mode;     /* 0 = reference order (rank == vertex_priority, counters
                             match the reference); 1 = fast ((q,p)-core pruning) */
  int32_t device;         /* CUDA device ordinal */
  int32_t shard_index;    /* multi-GPU sharding (roots, degree-balanced): this rank */
  int32_t shard_count;    /* number of ranks (1 = whole job) */
  int32_t flags;          /* BC_FLAG_* */
  const int64_t *rank_override; /* NULL or one distinct value per anchor vertex
                                   (prepare_structures(rank=...), engine.py:130-134) */
  int64_t n_rank;
  const int32_t *roots;   /* NULL = every anchor vertex may root tasks, else the
                             allowed root ids (count_bicliques(roots=...)) */
  int64_t n_roots;
  uint64_t *task_counts;  /* BC_FLAG_TASK_COUNTS: [2 * tasks_emitted] u128 (lo, hi) per
                             task, tasks in reference emission order (engine.py:160-172);
                             capacity in tasks given by task_counts_cap */
  int64_t task_counts_cap;
  uint32_t *task_claims;  /* BC_FLAG_TRACK_TASKS: [tasks_emitted] how many times each task
                             (reference emission order) was claimed by a warp; every entry
                             of this shard's tasks must read 1 (EngineConfig.track_tasks,
                             engine.py:446,462,473,498-499: task_tally is built from it) */
  int64_t task_claims_cap;
} bc_config;

#define BC_FLAG_TASK_COUNTS 1   /* fill cfg->task_counts */
#define BC_FLAG_INSTRUMENT 2    /* tally reference-equivalent intersections / operand
                                   words (B_enum, B_min) on device */
#define BC_FLAG_NO_SPLIT 4      /* disable heavy-task splitting (tests) */
#define BC_FLAG_L1_SCATTER 8    /* level 1 by root-grouped wedge scatter (default: chosen
                                   by a cost estimate) */
#define BC_FLAG_L1_PROBE 16     /* level 1 by per-task HTB intersections */
#define BC_FLAG_ROWR_SCATTER 32 /* candidate rows by wedge scatter where a slot map exists */
#define BC_FLAG_ROWR_PROBE 64   /* candidate rows by per-candidate intersections */
#define BC_FLAG_TASK_SHARD 128  /* multi-GPU: tasks interleaved (t % shard_count) instead of
                                   whole roots dealt degree-balanced (the default) */
#define BC_FLAG_TRACK_TASKS 256 /* fill cfg->task_claims (EngineConfig.track_tasks) */
#define BC_FLAG_CHECK_NESTING 512 /* EngineConfig.check_nesting (engine.py:296-297,365-366):
                                   for every task that descends, recompute every child
                                   C_L = C_L1 & dir2(u) from the HTB arenas and check each id
                                   against the root's directed 2-hop list; BC_EASSERT on a
                                   violation */
#define BC_FLAG_FULL_ROWS 1024  /* wedge-scatter frames walk whole opposite-layer rows N(v)
                                   instead of the root-restricted rows N(v) & dir2(r) (tests) */
#define BC_FLAG_FORCE_TRIAGE 2048 /* p_eff >= 5: run the survivor filter + triage path even
                                     when every task's frame would fit the split arena (it is
                                     chosen by size otherwise: C5-scale task counts; tests) */

/* CountReport (engine.py:64-79) plus device measurements. */
typedef struct bc_report {
  uint64_t count_lo, count_hi;   /* exact 128-bit count of this shard */
  int32_t overflow;              /* 1 if the exact count does not fit 128 bits */
  int32_t anchor;                /* 0 = 'U', 1 = 'V' */
  int32_t p_eff, q_eff;
  int64_t tasks_emitted;         /* whole job, as engine.py:147-173 */
  int64_t tasks_consumed;        /* tasks this shard claimed (device counter) */
  int64_t tasks_stolen;          /* dynamic-queue claims beyond each warp's first */
  int64_t roots_filtered;
  int64_t batches_executed;      /* reference hybrid/dfs batch accounting */
  int64_t tasks_alive;           /* tasks surviving level 1 (prune_keep) */
  int64_t tasks_split;           /* heavy tasks split across warps */
  int64_t und_pairs, dir2_pairs, adj_words, dir2_words, max_slice_words;
  int64_t intersections, operand_words, min_words;   /* BC_FLAG_INSTRUMENT */
  int64_t kernel_launches;       /* device kernels this call launched */
  int64_t h2d_bytes, d2h_bytes;  /* host<->device bytes this call moved */
  double time_h2d;               /* s: host->device copy of the CSR (bc_count only) */
  double time_prep;              /* s: device preprocessing (anchor .. task emission) */
  double time_level1;            /* s: level-1 pass (time_1hop analogue) */
  double time_enum;              /* s: enumeration (time_2hop analogue) */
  double time_total;             /* s: whole call */
  int64_t level1_operand_words;  /* BC_FLAG_INSTRUMENT: the level-1 share of operand_words */
  int64_t nesting_checked;       /* BC_FLAG_CHECK_NESTING: child C_L ids checked */
  int64_t level1_entries;        /* C_R1 list entries written by the wedge-scatter level 1
                                    (0 on the probe path): the level-1 lists' size / 4 B */
} bc_report;

/* Export ids for bc_export (device structures, for parity tests). */
enum bc_export_what {
  BC_X_UND_SIZE = 0,  /* int64[n]   |N2^q(u)| (graph.py:192-215) */
  BC_X_RANK = 1,      /* int64[n]   vertex_priority rank (graph.py:227-243) */
  BC_X_ORDER = 2,     /* int64[n]   highest priority first */
  BC_X_DIR_OFF = 3,   /* int64[n+1] directed 2-hop CSR (graph.py:218-224) */
  BC_X_DIR_IDX = 4,   /* int32[]    */
  BC_X_HADJ_OFF = 5,  /* int64[n+1] adjacency HTB (htb.py:104-115) */
  BC_X_HADJ_IDX = 6,  /* uint32[]   */
  BC_X_HADJ_VAL = 7,  /* uint32[]   */
  BC_X_HDIR_OFF = 8,  /* int64[n+1] directed 2-hop HTB */
  BC_X_HDIR_IDX = 9,  /* uint32[]   */
  BC_X_HDIR_VAL = 10, /* uint32[]   */
  BC_X_TASKS = 11,    /* int32[2*emitted] (root, second) in emission order (engine.py:147-173) */
  BC_X_META = 12,     /* int64[4]   anchor, p_eff, q_eff, n */
  BC_X_SLICE_LENS = 13, /* int32[n] upper 2-hop list length per anchor (bc_graph_twohop_slice;
                           0 for anchors of other shards) */
  BC_X_SLICE_IDS = 14,  /* int32[]  the owned anchors' upper lists, anchor order */
  BC_X_COUNT = 15
};

typedef struct bc_graph bc_graph;       /* device-resident CSR (both views) */
typedef struct bc_structs bc_structs;   /* device-resident prepared structures */

/* Library / ABI identification and device presence. */
int bc_abi_version(void);
const char *bc_last_error(void);
int bc_device_count(void);

/* One-shot count from host CSR buffers: H2D, preprocessing, count, D2H.
 * Replaces count_bicliques (engine.py:419-500) incl. prepare_structures. */
int bc_count(const int64_t *u_off, const int32_t *u_idx, int64_t n_u,
             const int64_t *v_off, const int32_t *v_idx, int64_t n_v,
             int32_t p, int32_t q, const bc_config *cfg, bc_report *out);

/* Device-resident graph: upload once, count many times. */
int bc_graph_create(const int64_t *u_off, const int32_t *u_idx, int64_t n_u,
                    const int64_t *v_off, const int32_t *v_idx, int64_t n_v,
                    int32_t device, bc_graph **out);
/* Same, from CSR arrays already resident on `device` (e.g. a graph generated on the
 * GPU): device-to-device copy, no host round trip.  Not in the reference (its graphs
 * are host lists); used for the FR-scale config, whose 1e8-edge CSR is built on device. */
int bc_graph_create_device(const int64_t *u_off, const int32_t *u_idx, int64_t n_u,
                           const int64_t *v_off, const int32_t *v_idx, int64_t n_v,
                           int32_t device, bc_graph **out);
int bc_graph_count(bc_graph *g, int32_t p, int32_t q, const bc_config *cfg, bc_report *out);
void bc_graph_destroy(bc_graph *g);

/* Enumeration mode (EngineConfig.enumerate_results, engine.py:271-304, 480-483): every
 * (p,q)-biclique as a leaf record [L: p_eff anchor-layer ids, c = |C_R|, C_R: c ids], one
 * record per search leaf with c >= q_eff (it stands for combinations(C_R, q_eff)).  The
 * records are written to `records` when `*words_needed` <= cap_words; otherwise call again
 * with a buffer of *words_needed int32 words.  order_mode must be 0. */
int bc_graph_enumerate(bc_graph *g, int32_t p, int32_t q, const bc_config *cfg,
                       int32_t *records, int64_t cap_words, int64_t *words_needed,
                       bc_report *out);

/* Border column reordering (reorder.py:146-179 border_reorder): greedy 1-block
 * reduction of `layer` (0 = U, 1 = V) by column swaps, on the device.  Writes the
 * permutation (perm[old id] = new id, n_layer entries) and the 1-block history
 * (at most iterations + 1 entries, count in *n_history).  Bit-identical to the
 * reference's choice rules.  iterations < 0 -> BC_EINVAL. */
int bc_graph_border(bc_graph *g, int32_t layer, int64_t iterations, int64_t *perm,
                    int64_t *history, int64_t *n_history);

/* Kernel launches of the last bc_graph_border call on this thread. */
int64_t bc_last_launch_count(void);

/* Sharded preprocessing (multi-GPU, one process per GPU).  bc_graph_twohop_slice builds
 * the upper 2-hop lists ({w > u : |N(u) & N(w)| >= q_eff}, graph.py:192-215 restricted to
 * the upper triangle) of the anchors shard `shard` of `nshards` owns (snake order over the
 * LPT order; the union over shards is every anchor); export them with BC_X_SLICE_LENS /
 * BC_X_SLICE_IDS.  After the ranks exchange them (all-gather), bc_graph_count_upper counts
 * with the whole upper CSR given in device memory (upper_off int64[n+1], upper_ids
 * int32[n_pairs], borrowed) and skips the 2-hop construction; results are identical to
 * bc_graph_count.  order_mode must be 0. */
int bc_graph_twohop_slice(bc_graph *g, int32_t p, int32_t q, const bc_config *cfg, int32_t shard,
                          int32_t nshards, bc_structs **out);
int bc_graph_count_upper(bc_graph *g, int32_t p, int32_t q, const bc_config *cfg,
                         const int64_t *upper_off, const int32_t *upper_ids, int64_t n_pairs,
                         bc_report *out);
/* Whole upper CSR from `world` gathered slices, all device pointers: lens_all int32[world*n]
 * (rank r's BC_X_SLICE_LENS at r*n), ids_all (rank r's BC_X_SLICE_IDS at r*ids_stride);
 * writes upper_off int64[n+1] and upper_ids (capacity ids_cap), *n_pairs = pair count. */
int bc_assemble_upper(int32_t device, int32_t world, int64_t n, const int32_t *lens_all,
                      const int32_t *ids_all, int64_t ids_stride, int64_t *upper_off,
                      int32_t *upper_ids, int64_t ids_cap, int64_t *n_pairs);
/* Like bc_export, into device memory (cudaMemcpy device to device). */
int bc_export_device(const bc_structs *s, int32_t what, void *device_dst);

/* Prepared structures on device (prepare_structures, engine.py:115-144),
 * exported for bit-exact comparison against the reference's. */
int bc_prepare(bc_graph *g, int32_t p, int32_t q, const bc_config *cfg, bc_structs **out);
int64_t bc_export_len(const bc_structs *s, int32_t what);
int bc_export(const bc_structs *s, int32_t what, void *host_dst);
void bc_structs_destroy(bc_structs *s);

/* Hand the cached scratch of the library's per-device memory pools back to the device
   (live graphs and structures keep their allocations). */
void bc_shutdown(void);

/* Development builds compiled with -DBC_PHASE_PROF: per-phase SM-cycle tallies of
 * the enumeration since the last read (reset on read); returns the number of
 * phases written, 0 in normal builds (out is zero-filled). */
int bc_debug_phase_cycles(uint64_t *out, int32_t n);

#ifdef __cplusplus
}
#endif
#endif
