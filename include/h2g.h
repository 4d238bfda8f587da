/*
 * h2g.h — C ABI of the B200-native H2* / (H2+H)* matrix-vector product.
 *
 * This is the drop-in boundary for the reference's operator object.  The
 * reference (pkg/src/h2weak, pure Python) has no FFI; its operator interface
 * is duck-typed Python:
 *
 *   HierRep.matvec(q) -> phi            engine.py:250-269   -> h2g_matvec / h2g_matvec_host
 *   compute_potential(rep, q)           engine.py:321-322   -> h2g_matvec_host
 *   BlockLowRankRep.matvec(q)           blr.py:32-33        -> (BLR leg inside the plan)
 *   build_variant(...) -> HierRep       engine.py:325-373   -> h2g_plan_create (from the
 *                                                              packed export of that rep)
 *   rep.mem_scalars                     engine.py:184-186   -> h2g_plan_stats.mem_scalars
 *
 * The Python host (paper_2309_14085_b200/gpu_rep.py) binds these with ctypes
 * and exposes GpuHierRep.matvec with the reference's contract (same
 * ValueError("vector length mismatch"), fp64 promotion, fresh output).
 *
 * Conventions
 *  - All arrays in h2g_export_desc are HOST pointers owned by the caller;
 *    h2g_plan_create copies what it needs to the device, so they may be freed
 *    after it returns.  The plan owns all device memory it allocates.
 *  - Vectors are in ORIGINAL point order (the plan applies the tree
 *    permutation itself).  nrhs right-hand sides are stored point-major:
 *    element (i, j) at q[i * ld + j] (a C-contiguous N x nrhs array).
 *  - Return codes: 0 = OK, otherwise an H2G_ERR_* code; h2g_error_string()
 *    gives a static message and h2g_last_error_detail() a per-thread detail.
 *  - Threading: one plan = one CUDA stream of work; matvec calls on the same
 *    plan must not run concurrently (the coefficient workspace is shared).
 */
#ifndef H2G_H
#define H2G_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define H2G_ABI_VERSION 3

enum {
  H2G_OK = 0,
  H2G_ERR_LENGTH_MISMATCH = 1, /* -> ValueError("vector length mismatch") (engine.py:253-254) */
  H2G_ERR_BAD_EXPORT = 2,      /* inconsistent packed export */
  H2G_ERR_CUDA = 3,            /* CUDA runtime error (detail has the CUDA message) */
  H2G_ERR_NO_DEVICE = 4,       /* no usable sm_100 device */
  H2G_ERR_INVALID_ARG = 5,
  H2G_ERR_OOM = 6
};

/* One nested channel (reference NestedOperatorSet, engine.py:117-130).
 * Offsets index the fp64 blob (in doubles); -1 = operator absent.
 * All matrices column-major. */
typedef struct h2g_channel_desc {
  const int32_t* r_in;        /* [n_clusters] incoming rank (PivotQuad.rank_in, lowrank.py:53-55) */
  const int32_t* r_out;       /* [n_clusters] outgoing rank (lowrank.py:57-59) */
  const int64_t* p2m_off;     /* [n_clusters] r_out x n_X            ops.p2m[X]        */
  const int64_t* l2p_off;     /* [n_clusters] n_X x r_in             ops.l2p[X]        */
  const int64_t* m2m_off;     /* [n_clusters] r_out(P) x r_out(c)    ops.m2m[(P, c)]   keyed by child c */
  const int64_t* l2l_off;     /* [n_clusters] r_in(c) x r_in(P)      ops.l2l[(c, P)]   keyed by child c */
  const int64_t* m2l_rowptr;  /* [n_clusters + 1] CSR by target X                      */
  const int32_t* m2l_src;     /* [nnz] source Y, lists_fn order (partition.py:133-136) */
  const int64_t* m2l_off;     /* [nnz] r_in(X) x r_out(Y)            ops.m2l[(X, Y)]
                                 -1 = not stored: evaluated on the device as
                                 K[t_i(X), s_o(Y)] (engine.py:176-179) */
  /* NCA pivots (PivotQuad.t_i / s_o, lowrank.py:45-59) as TREE POSITIONS, CSR
   * by cluster (piv_in: r_in entries, piv_out: r_out entries).  Needed only
   * for M2L recompute; NULL otherwise. */
  const int64_t* piv_in_ptr;  /* [n_clusters + 1] */
  const int64_t* piv_in;      /* t_i(X) */
  const int64_t* piv_out_ptr; /* [n_clusters + 1] */
  const int64_t* piv_out;     /* s_o(X) */
} h2g_channel_desc;

/* The packed export (paper_2309_14085_b200/packed.py, SURVEY.md §8(a')). */
typedef struct h2g_export_desc {
  int32_t abi_version;        /* H2G_ABI_VERSION */
  int32_t dim;                /* 1..3 */
  int32_t kappa;              /* tree depth (tree.py:140-143) */
  int32_t n_channels;         /* 0..2 nested channels (h2star-bt: 2, h2plusH-star: 1) */
  int64_t n_points;           /* N */
  int64_t n_clusters;         /* level_offset[kappa + 1] */
  int64_t mem_scalars;        /* reference tally (engine.py:184-186, 315; blr.py:59) */
  const int64_t* perm;        /* [N] tree position -> original index (tree.py:152-165) */
  const int64_t* level_offset;/* [kappa + 2] (tree.py:72-75) */
  const int64_t* cl_start;    /* [n_clusters] tree-order slice of every cluster */
  const int64_t* cl_end;
  h2g_channel_desc channels[2];
  /* BLR leg of (H2+H)* (blr.py:72-83): CSR by target over rank>0 factors */
  const int64_t* blr_rowptr;  /* [n_clusters + 1] */
  const int32_t* blr_src;     /* [nnz] */
  const int32_t* blr_rank;    /* [nnz] p */
  const int64_t* blr_u_off;   /* [nnz] U: n_X x p LEAF-BLOCKED: the rows of leaf L in X
                                 form an n_L x p column-major block at
                                 blr_u_off + (cl_start[L] - cl_start[X]) * p */
  const int64_t* blr_v_off;   /* [nnz] V: n_Y x p row-major (= V^T column-major) */
  /* near field (engine.py:260-268): CSR by target leaf */
  const int64_t* near_rowptr; /* [n_clusters + 1] */
  const int32_t* near_src;    /* [nnz] */
  const int64_t* near_off;    /* [nnz] n_X x n_Y column-major; -1 = not stored
                                 (reference store_near=False, engine.py:260-268:
                                 kernel.block(t^X, t^Y) evaluated on the device) */
  int64_t blob_len;           /* doubles */
  const double* blob;         /* all operator matrices */
  /* ---- kernel-evaluation ("recompute", P2P-style) path, ABI 3 ----
   * The M2L blocks are raw kernel blocks K[t_i(X), s_o(Y)] and the near
   * blocks K[t^X, t^Y] (engine.py:176-179, 309-318), so the device can
   * evaluate them from point coordinates instead of streaming them.
   * Kernel rules follow Kernel.block (kernels.py:36-57). */
  const double* points_tree;  /* [N x dim] coordinates in tree order (NULL: no recompute) */
  int32_t kernel_type;        /* H2G_KERNEL_* (-1: unknown -> no recompute) */
  int32_t has_diag;           /* Kernel.diag is not None */
  double zero_value;          /* value at r == 0, i != j */
  double diag;                /* value at i == j (if has_diag) */
  double shift;               /* added at i == j */
  double sigma;               /* Gaussian width */
  int32_t recompute;          /* H2G_RECOMPUTE_* mask: evaluate these blocks even where stored */
  int32_t pad0;
  double m2l_recompute_share; /* (0, 1]: with H2G_RECOMPUTE_M2L, the share of each level's
                                 stored M2L entries evaluated; the rest of every target's
                                 blocks stream through the same P2P task (fp64 pipe and HBM
                                 busy at once); 0 or 1 = all of them */
} h2g_export_desc;

enum { H2G_KERNEL_LOG2D = 0, H2G_KERNEL_LAP3D = 1, H2G_KERNEL_GAUSSIAN = 2 };
enum { H2G_RECOMPUTE_NEAR = 1, H2G_RECOMPUTE_M2L = 2 };

typedef struct h2g_plan h2g_plan;

typedef struct h2g_plan_stats {
  int64_t n_points;
  int64_t mem_scalars;         /* reference tally */
  int64_t alg_bytes;           /* 8 * mem_scalars + 16 * N */
  int64_t blob_bytes;          /* device bytes of the operator blob (incl. alignment) */
  int64_t workspace_bytes;     /* coefficient arena + task tables */
  int32_t n_phases;            /* device phases per matvec */
  int32_t n_launches;          /* kernel launches per single-RHS matvec */
  int64_t n_tasks;
  int64_t n_terms;
  int32_t device;
  int32_t graph;               /* 1 if the fixed phases run as one CUDA graph */
} h2g_plan_stats;

/* Build a plan (upload + schedule) for one operator on CUDA device `device`. */
int h2g_plan_create(const h2g_export_desc* desc, int device, h2g_plan** out);
int h2g_plan_destroy(h2g_plan* plan);
int h2g_plan_get_stats(const h2g_plan* plan, h2g_plan_stats* out);

/* phi = K q for nrhs right-hand sides, DEVICE pointers, stream-ordered on
 * `stream` (a cudaStream_t used as given: NULL = the legacy default stream,
 * as everywhere in CUDA); no host sync. */
int h2g_matvec(h2g_plan* plan, const double* q_dev, double* phi_dev, int64_t n,
               int64_t nrhs, int64_t ld, void* stream);

/* Same with HOST pointers: H2D copy, matvec, D2H copy, synchronous
 * (the reference's call shape, engine.py:250-269). */
int h2g_matvec_host(h2g_plan* plan, const double* q_host, double* phi_host, int64_t n,
                    int64_t nrhs, int64_t ld);

/* Per-phase device timing: runs `iters` matvecs phase by phase with CUDA events
 * on the plan's stream.  ms[i] = mean duration of phase i, bytes[i] = its
 * algorithmic bytes, names[i] = static name.  Up to `cap` phases are written;
 * returns the number of phases through *n_out. */
int h2g_profile_phases(h2g_plan* plan, const double* q_dev, double* phi_dev, int iters,
                       double* ms, int64_t* bytes, const char** names, int cap, int* n_out);

/* Diagnostics: per-phase timing of one pass of the batched-RHS engine
 * (kb = 8 or 16 right-hand sides; reduce + DMMA launches per phase).  Same
 * output convention as h2g_profile_phases (bytes = stored operator bytes). */
int h2g_profile_phases_batched(h2g_plan* plan, int kb, int iters, double* ms, int64_t* bytes,
                               const char** names, int cap, int* n_out);

/* Host-only: compile the schedule for `desc` as if for a device with n_sm
 * SMs (no CUDA calls) and write a JSON summary per phase into buf. */
int h2g_schedule_info(const h2g_export_desc* desc, int n_sm, char* buf, int64_t buflen);

/* ---- multi-GPU (one process per GPU) ----
 * Subtrees at level L_s are split into nranks contiguous Morton ranges; rank
 * r computes the clusters of its subtrees (and the replicated coarse levels)
 * and the phi rows [row_begin, row_end) of tree order.  q is replicated.
 * One matvec:  h2g_matvec_begin(q)  ->  h2g_shard_pack(send)  ->
 * all-gather of send (max_send_slots doubles per rank, rank-major, e.g. NCCL
 * ncclAllGather) into recv  ->  h2g_shard_unpack(recv)  ->  h2g_matvec_end(phi)
 * (phi receives this rank's rows only).  A rank uploads only the operator
 * blocks its tasks read. */
typedef struct h2g_shard_info {
  int32_t rank, nranks;
  int32_t level;               /* L_s */
  int32_t pad;
  int64_t row_begin, row_end;  /* owned tree-order rows */
  int64_t send_slots;          /* doubles this rank contributes to the exchange */
  int64_t max_send_slots;      /* per-rank stride of the all-gather buffer */
  int64_t blob_bytes;          /* operator bytes resident on this rank */
  int64_t halo_slots;          /* x-halo doubles this rank contributes (distributed q) */
  int64_t max_halo_slots;      /* per-rank stride of the x-halo all-gather buffer */
} h2g_shard_info;

int h2g_plan_create_sharded(const h2g_export_desc* desc, int device, int rank, int nranks,
                            h2g_plan** out);
int h2g_shard_get_info(const h2g_plan* plan, h2g_shard_info* out);
int h2g_matvec_begin(h2g_plan* plan, const double* q_dev, int64_t n, void* stream);
int h2g_shard_pack(h2g_plan* plan, double* send_dev, void* stream);
int h2g_shard_unpack(h2g_plan* plan, const double* recv_dev, void* stream);
/* The owned near field (it reads only q) as its own step: call it between
 * h2g_shard_pack and h2g_shard_unpack, after starting the all-gather, and it
 * runs while the exchange is in flight; the leaf tasks add its partial sums
 * (fixed order).  h2g_matvec_end / h2g_shard_store_phi run it themselves if
 * the caller did not.  H2G_SHARD_OVERLAP=0 at plan creation keeps the near
 * field inside the leaf phase. */
int h2g_shard_overlap(h2g_plan* plan, void* stream);
int h2g_matvec_end(h2g_plan* plan, double* phi_dev, int64_t n, void* stream);

/* Distributed vectors: q and phi live as each rank's OWN tree-order rows
 * [row_begin, row_end) (points perm[row_begin .. row_end)), no replicated q.
 * One matvec:  h2g_shard_load_q(q_own)  ->  h2g_halo_pack(hsend)  ->
 * all-gather (max_halo_slots doubles per rank, rank-major) into hrecv  ->
 * h2g_halo_unpack(hrecv)  ->  h2g_shard_part0  ->  h2g_shard_pack / all-gather
 * / h2g_shard_unpack (as above)  ->  h2g_shard_store_phi(phi_own).  The x
 * halo is the q rows other ranks read: near-field sources and the BLR V^T
 * sources of owned targets across subtree boundaries. */
int h2g_shard_load_q(h2g_plan* plan, const double* q_own_dev, void* stream);
int h2g_halo_pack(h2g_plan* plan, double* send_dev, void* stream);
int h2g_halo_unpack(h2g_plan* plan, const double* recv_dev, void* stream);
int h2g_shard_part0(h2g_plan* plan, void* stream);
int h2g_shard_store_phi(h2g_plan* plan, double* phi_own_dev, void* stream);

/* Host-only view of rank `rank`'s schedule (no CUDA; emulation and tests):
 * named int64 arrays "tasks" [n x 5: y_off, m, t_begin, t_end, row_rec],
 * "terms" [n x 6: a_off, x_off, lda, ncols, a_space, self], "phases" [n x 4:
 * task_begin, task_end, part, alg_bytes], "pack" / "unpack" [n x 3: src, dst,
 * len], "halo" [n x 3: sending rank, tree row, len] (the x-halo ranges of
 * every rank), "meta" [n_slots, q_tree, phi_tree, ones_off, n_ones, row_begin,
 * row_end, send_slots, max_send_slots, level], the compacted f64 "blob"
 * (empty when nranks == 1 and no block was re-laid out: terms index the
 * export's blob) and the f64 point records "recs" [n x 4] of kernel-evaluated
 * terms.  a_space: 0 blob, 1 arena, 2 evaluated = K[records row_rec .. + m,
 * records a_off .. + ncols] (self = 1: rows and columns are the same records,
 * the i == j rule applies). */
typedef struct h2g_sched h2g_sched;
int h2g_schedule_build(const h2g_export_desc* desc, int rank, int nranks, h2g_sched** out);
int h2g_schedule_get(const h2g_sched* sched, const char* name, const void** ptr, int64_t* len,
                     int32_t* is_f64);
void h2g_schedule_free(h2g_sched* sched);

/* Number of kernels a single-RHS matvec launches (for bench gpu_launches). */
int h2g_launches_per_matvec(const h2g_plan* plan, int64_t nrhs);

const char* h2g_error_string(int code);
const char* h2g_last_error_detail(void);
int h2g_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* H2G_H */
