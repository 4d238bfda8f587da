/*
 * h2b.h — C ABI of the native (C++/OpenMP) operator builder.
 *
 * Restates the reference's construction of the H2* / (H2+H)* operators so
 * that operators at the benchmark sizes can be built on the GPU box itself
 * (the reference's Python build takes ~20-30 min at N=1M and cannot run
 * there).  Output is the packed export consumed by h2g_plan_create
 * (include/h2g.h).  Reference interfaces restated:
 *
 *   build_tree(particles, n_max)              tree.py:111-185
 *   build_partition(tree, WeakVertex())       partition.py:77-137
 *   Kernel.block(rows, cols) (+ Log2D,        kernels.py:36-57, 63-81
 *     InverseR, Gaussian via the _f hook)
 *   aca / aca_pivots / aca_factor             lowrank.py:69-159
 *   solve_square / rsolve (LU, singular test) lowrank.py:162-180
 *   _pivot_pair (retry at eps/10)             engine.py:39-51
 *   select_pivots_b2t / select_pivots_t2b     engine.py:54-114
 *   build_operators                           engine.py:133-187
 *   build_blr(lists="ver", include_near=0)    blr.py:46-69
 *   _attach_near(store_near=True)             engine.py:309-318
 *   build_variant("h2star-bt"|"h2plusH-star") engine.py:325-373
 */
#ifndef H2B_H
#define H2B_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define H2B_ABI_VERSION 1

enum { H2B_VARIANT_H2STAR_BT = 0, H2B_VARIANT_H2PLUSH_STAR = 1 };
enum { H2B_KERNEL_LOG2D = 0, H2B_KERNEL_LAP3D = 1, H2B_KERNEL_GAUSSIAN = 2 };
enum { H2B_SKIP_NEAR = 1, H2B_SKIP_M2L = 2 };
enum { H2B_OK = 0, H2B_ERR_INVALID_ARG = 1, H2B_ERR_SINGULAR = 2, H2B_ERR_OOM = 3 };

typedef struct h2b_params {
  int32_t abi_version;   /* H2B_ABI_VERSION */
  int32_t dim;           /* 1..3 */
  int64_t n_points;
  const double* points;  /* n_points x dim, row-major, original order */
  int32_t n_max;         /* leaf size (tree.py:111) */
  int32_t variant;       /* H2B_VARIANT_* */
  int32_t kernel;        /* H2B_KERNEL_* */
  int32_t has_diag;      /* Kernel.diag is not None */
  double zero_value;     /* Kernel.zero_value (r == 0, i != j) */
  double diag;           /* Kernel.diag */
  double shift;          /* Kernel.shift (added on i == j) */
  double sigma;          /* Gaussian width */
  double eps_far;        /* NCA tolerance of the far channel */
  double eps_ver;        /* NCA / ACA tolerance of the vertex leg */
  int32_t n_threads;     /* 0 = OpenMP default */
  int32_t skip_blocks;   /* H2B_SKIP_* mask: blocks NOT stored (offset -1 in the export,
                            evaluated on the device: h2g.h recompute path); they still
                            count in mem_scalars (engine.py:315 counts lazy near blocks) */
} h2b_params;

typedef struct h2b_result h2b_result;

/* dtype codes for h2b_get_array */
enum { H2B_I32 = 0, H2B_I64 = 1, H2B_F64 = 2 };

int h2b_build(const h2b_params* params, h2b_result** out);
/* Named arrays of the packed export (packed.py field names, channel fields
 * prefixed "ch0_"/"ch1_", incl. the NCA pivots "chK_piv_in_ptr/_piv_in/
 * _piv_out_ptr/_piv_out" as tree positions).  The pointer stays valid until h2b_free. */
int h2b_get_array(const h2b_result* r, const char* name, const void** ptr, int64_t* len,
                  int32_t* dtype);
/* Scalars: "kappa", "n_channels", "mem_scalars", "n_clusters". */
int64_t h2b_get_scalar(const h2b_result* r, const char* name);
/* Wall-clock seconds of the build stages: "tree", "partition", "pivots",
 * "operators", "blr", "near", "total". */
double h2b_get_timing(const h2b_result* r, const char* name);
void h2b_free(h2b_result* r);
const char* h2b_last_error(void);
int h2b_abi_version(void);

/* Materialise the raw kernel blocks of a packed export (the blocks a build
 * with skip_blocks left out): every M2L block (X, Y) with m2l_off >= 0 is
 * K[t_i(X), s_o(Y)] (engine.py:176-179, r_in(X) x r_out(Y), column-major)
 * and every near block with near_off >= 0 is K[t^X, t^Y] (engine.py:309-318,
 * n_X x n_Y); rows / columns are tree positions into points_tree, entries
 * follow Kernel.block (kernels.py:36-57) exactly as h2b_build fills them
 * (bitwise).  Parallel over target clusters (OpenMP). */
typedef struct h2b_fill_channel {
  const int32_t* r_in;          /* [n_clusters] */
  const int32_t* r_out;         /* [n_clusters] */
  const int64_t* m2l_rowptr;    /* [n_clusters + 1] */
  const int32_t* m2l_src;       /* [nnz] */
  const int64_t* m2l_off;       /* [nnz]: blob offset to fill, -1 = skip */
  const int64_t* piv_in_ptr;    /* [n_clusters + 1] t_i as tree positions */
  const int64_t* piv_in;
  const int64_t* piv_out_ptr;   /* [n_clusters + 1] s_o as tree positions */
  const int64_t* piv_out;
} h2b_fill_channel;

typedef struct h2b_fill_desc {
  int32_t dim;
  int32_t kernel;               /* H2B_KERNEL_* */
  int32_t has_diag;
  int32_t n_channels;
  int64_t n_points;
  int64_t n_clusters;
  const double* points_tree;    /* n_points x dim, tree order */
  double zero_value, diag, shift, sigma;
  const int64_t* cl_start;      /* [n_clusters] */
  const int64_t* cl_end;
  const int64_t* near_rowptr;   /* [n_clusters + 1] */
  const int32_t* near_src;
  const int64_t* near_off;      /* blob offset to fill, -1 = skip */
  h2b_fill_channel channels[2];
  int32_t n_threads;            /* 0 = OpenMP default */
  int32_t pad;
} h2b_fill_desc;

int h2b_fill_kernel_blocks(const h2b_fill_desc* desc, double* blob, int64_t blob_len);

#ifdef __cplusplus
}
#endif
#endif /* H2B_H */
