// h2b_build.cpp — native (C++/OpenMP) restatement of the reference's
// H2* / (H2+H)* operator construction; emits the packed export that
// h2g_plan_create consumes.  See include/h2b.h for the reference map.
//
// Parallelism: clusters of one tree level are independent in every stage
// (pivot selection, operator assembly, BLR factors, near blocks), so each
// stage is an OpenMP loop over a level with a barrier between levels --
// the "parallelize per-cluster within a level" of the reference SPEC.
//
// Arithmetic follows the reference step by step (same candidate orders,
// same ACA pivoting and stopping rule, LU with partial pivoting and the
// same singularity test) so that pivots and ranks match it; BLAS-internal
// summation orders (norms, dots, LU updates) are plain sequential loops
// here, so the resulting matrices agree with the reference to roundoff
// amplified by the cross-matrix conditioning (~eps * cond).
#include <omp.h>

#include <algorithm>
#include <array>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/h2b.h"

namespace {

thread_local std::string g_err;

using Idx = std::vector<int64_t>;

struct SingularCross : std::runtime_error {
  explicit SingularCross(const std::string& m) : std::runtime_error(m) {}
};

// ------------------------------------------------------------------ kernel
// kernels.py:36-57: r = cdist (sequential sum of squared differences), f(r),
// r == 0 -> zero_value, i == j -> diag (if set) + shift.
struct Kernel {
  int type = 0;
  int d = 2;
  const double* pts = nullptr;
  double zero_value = 0, diag = 0, shift = 0, sigma = 0.1;
  bool has_diag = false;

  inline double f(double r) const {
    switch (type) {
      case H2B_KERNEL_LOG2D: return std::log(r);                          // kernels.py:70-71
      case H2B_KERNEL_LAP3D: return 1.0 / r;                              // kernels.py:80-81
      default: return std::exp(-(r * r) / (2.0 * sigma * sigma));         // Gaussian (cfg 4)
    }
  }
  inline double entry(int64_t i, int64_t j) const {
    const double* a = pts + i * d;
    const double* b = pts + j * d;
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      const double t = a[k] - b[k];
      s += t * t;
    }
    const double r = std::sqrt(s);
    if (r == 0.0) {
      double v = zero_value;
      if (i == j) {
        if (has_diag) v = diag;
        v += shift;
      }
      return v;
    }
    double v = f(r);
    if (shift != 0.0 && i == j) v += shift;
    return v;
  }
  // column-major rows x cols block into out (leading dim ld)
  void block_cm(const int64_t* rows, int64_t nr, const int64_t* cols, int64_t nc, double* out,
                int64_t ld) const {
    for (int64_t c = 0; c < nc; ++c)
      for (int64_t r = 0; r < nr; ++r) out[c * ld + r] = entry(rows[r], cols[c]);
  }
};

// ------------------------------------------------------------------ LU
// Partial-pivoting LU (LAPACK dgetrf semantics, first max |a| as pivot),
// matrix column-major n x n in place.
struct LU {
  int n = 0;
  std::vector<double> a;  // column-major
  std::vector<int> piv;
};

void lu_factor(LU& L) {
  const int n = L.n;
  double* A = L.a.data();
  L.piv.resize(n);
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::fabs(A[k * n + k]);
    for (int i = k + 1; i < n; ++i) {
      const double v = std::fabs(A[k * n + i]);
      if (v > best) {
        best = v;
        p = i;
      }
    }
    L.piv[k] = p;
    if (p != k)
      for (int c = 0; c < n; ++c) std::swap(A[c * n + k], A[c * n + p]);
    const double d = A[k * n + k];
    if (d != 0.0) {
      for (int i = k + 1; i < n; ++i) A[k * n + i] /= d;
    }
    for (int c = k + 1; c < n; ++c) {
      const double akc = A[c * n + k];
      if (akc == 0.0) continue;
      double* colc = A + (size_t)c * n;
      const double* colk = A + (size_t)k * n;
      for (int i = k + 1; i < n; ++i) colc[i] -= colk[i] * akc;
    }
  }
}

// lowrank.py:169-174: singular when min|U_ii| <= 0.5 * eps_mach * max(max|U_ii|, 1e-300)
bool lu_singular(const LU& L) {
  double mn = INFINITY, mx = 0.0;
  for (int i = 0; i < L.n; ++i) {
    const double v = std::fabs(L.a[(size_t)i * L.n + i]);
    mn = std::min(mn, v);
    mx = std::max(mx, v);
  }
  return mn <= 0.5 * DBL_EPSILON * std::max(mx, 1e-300);
}

// solve A X = B in place for k right-hand sides (B column-major n x k)
void lu_solve(const LU& L, double* B, int64_t k) {
  const int n = L.n;
  const double* A = L.a.data();
  for (int64_t j = 0; j < k; ++j) {
    double* b = B + j * n;
    for (int i = 0; i < n; ++i)
      if (L.piv[i] != i) std::swap(b[i], b[L.piv[i]]);
    for (int c = 0; c < n; ++c) {  // L unit lower
      const double bc = b[c];
      if (bc != 0.0)
        for (int i = c + 1; i < n; ++i) b[i] -= A[(size_t)c * n + i] * bc;
    }
    for (int c = n - 1; c >= 0; --c) {  // U
      b[c] /= A[(size_t)c * n + c];
      const double bc = b[c];
      if (bc != 0.0)
        for (int i = 0; i < c; ++i) b[i] -= A[(size_t)c * n + i] * bc;
    }
  }
}

// ------------------------------------------------------------------ ACA
// lowrank.py:69-147 (partially pivoted ACA, incremental Frobenius rule).
struct AcaOut {
  std::vector<std::vector<double>> us, vs;  // u: length m, v: length n
  Idx tau, sigma;
};

int first_row(const Kernel& K, const Idx& rows, const Idx& cols) {  // lowrank.py:69-74
  if (cols.empty()) return 0;
  const int d = K.d;
  double cen[3] = {0, 0, 0};
  for (int64_t c : cols)
    for (int k = 0; k < d; ++k) cen[k] += K.pts[c * d + k];
  for (int k = 0; k < d; ++k) cen[k] /= (double)cols.size();
  int best = 0;
  double bd = INFINITY;
  for (size_t a = 0; a < rows.size(); ++a) {
    double s = 0;
    for (int k = 0; k < d; ++k) {
      const double t = K.pts[rows[a] * d + k] - cen[k];
      s += t * t;
    }
    if (s < bd) {
      bd = s;
      best = (int)a;
    }
  }
  return best;
}

// ACA work is O(r^2 (m + n)); at the coarse tree levels a single ACA spans
// 10^5..10^6 candidates, so its loops run in parallel over fixed blocks of
// kBlk entries.  Reductions (dots, argmax) combine per-block partials in block
// order, so results do not depend on the thread count; for m, n <= kBlk the
// arithmetic is exactly the sequential loop's.
constexpr int64_t kBlk = 2048;

template <class F>
void for_blocks(int64_t n, bool par, F f) {
  const int64_t nb = (n + kBlk - 1) / kBlk;
  if (par && nb > 1) {
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < nb; ++b) f(b, b * kBlk, std::min(n, (b + 1) * kBlk));
  } else {
    for (int64_t b = 0; b < nb; ++b) f(b, b * kBlk, std::min(n, (b + 1) * kBlk));
  }
}

// sum_i a[i] * b[i] over [0, n) with 8 interleaved partial sums (vectorised;
// fixed order, so independent of the thread count).  The reference's
// np.vdot / np.linalg.norm are BLAS reductions with their own blocking, so
// these only enter the Frobenius stopping estimate, never a pivot choice.
inline double dot8(const double* a, const double* b, int64_t n) {
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int64_t i = 0;
  for (; i + 8 <= n; i += 8)
    for (int l = 0; l < 8; ++l) acc[l] += a[i + l] * b[i + l];
  for (int l = 0; i < n; ++i, ++l) acc[l] += a[i] * b[i];
  return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

// sum_i a[i] * b[i] with fixed block partials
double dot_blocked(const double* a, const double* b, int64_t n, bool par) {
  const int64_t nb = (n + kBlk - 1) / kBlk;
  std::vector<double> part(std::max<int64_t>(nb, 1), 0.0);
  for_blocks(n, par, [&](int64_t blk, int64_t b0, int64_t b1) {
    part[blk] = dot8(a + b0, b + b0, b1 - b0);
  });
  double s = 0;
  for (int64_t k = 0; k < nb; ++k) s += part[k];
  return s;
}

// Kernel row K[ri, cols[b0 .. b1)] into out, columns' coordinates gathered
// contiguously in cp (n x d).  1/r runs as a vector loop (sqrt and division
// are correctly rounded, so every entry is bitwise the scalar Kernel::entry);
// r == 0 entries (coincident points, i == j) are fixed up by entry().
void row_entries(const Kernel& K, int64_t ri, const int64_t* cols, const double* cp, int64_t b0,
                 int64_t b1, double* out) {
  const int d = K.d;
  const double* a = K.pts + ri * d;
  if (K.type == H2B_KERNEL_LAP3D) {
    const double a0 = a[0], a1 = d > 1 ? a[1] : 0.0, a2 = d > 2 ? a[2] : 0.0;
    if (d == 3) {
      for (int64_t j = b0; j < b1; ++j) {
        const double t0 = a0 - cp[3 * j], t1 = a1 - cp[3 * j + 1], t2 = a2 - cp[3 * j + 2];
        double s2 = 0.0;
        s2 += t0 * t0;
        s2 += t1 * t1;
        s2 += t2 * t2;
        out[j] = 1.0 / std::sqrt(s2);
      }
    } else {
      for (int64_t j = b0; j < b1; ++j) {
        double s2 = 0.0;
        for (int k = 0; k < d; ++k) {
          const double t = a[k] - cp[d * j + k];
          s2 += t * t;
        }
        out[j] = 1.0 / std::sqrt(s2);
      }
    }
    for (int64_t j = b0; j < b1; ++j)
      if (std::isinf(out[j])) out[j] = K.entry(ri, cols[j]);  // r == 0
    return;
  }
  for (int64_t j = b0; j < b1; ++j) out[j] = K.entry(ri, cols[j]);
}

// first index of max(mask ? 0 : |v|) (numpy argmax semantics); returns (idx, max)
std::pair<int64_t, double> argmax_masked(const double* v, const char* used, int64_t n, bool par) {
  const int64_t nb = (n + kBlk - 1) / kBlk;
  std::vector<std::pair<int64_t, double>> part(std::max<int64_t>(nb, 1), {0, -1.0});
  for_blocks(n, par, [&](int64_t blk, int64_t b0, int64_t b1) {
    int64_t jb = b0;
    double mb = -1.0;
    for (int64_t j = b0; j < b1; ++j) {
      const double mv = used[j] ? 0.0 : std::fabs(v[j]);
      if (mv > mb) {
        mb = mv;
        jb = j;
      }
    }
    part[blk] = {jb, mb};
  });
  std::pair<int64_t, double> best = part[0];
  for (int64_t k = 1; k < nb; ++k)
    if (part[k].second > best.second) best = part[k];
  return best;
}

AcaOut aca(const Kernel& K, const Idx& rows, const Idx& cols, double eps, bool keep_factors,
           bool par = false) {
  AcaOut out;
  const int64_t m = (int64_t)rows.size(), n = (int64_t)cols.size();
  const int64_t max_rank = std::min(m, n);
  if (m == 0 || n == 0 || max_rank == 0) return out;
  std::vector<char> used_rows(m, 0), used_cols(n, 0);
  double fro2 = 0.0;
  int64_t i = first_row(K, rows, cols);
  std::vector<double> row(n), col(m);
  auto& us = out.us;
  auto& vs = out.vs;
  std::vector<double> cp((size_t)n * K.d);  // column coordinates, contiguous
  for (int64_t j = 0; j < n; ++j)
    for (int k = 0; k < K.d; ++k) cp[(size_t)j * K.d + k] = K.pts[cols[j] * K.d + k];
  const int64_t nblk = (n + kBlk - 1) / kBlk;
  // per block: <row, row> and <row, v_k> partials, computed while the block's
  // v_k are still in cache (fused with the residual row)
  std::vector<double> p_vv(std::max<int64_t>(nblk, 1)), p_cross;
  while (true) {
    // residual row i: K[rows[i], cols] - sum_k u_k[i] v_k (k in order, per entry)
    const size_t nk = us.size();
    p_cross.assign((size_t)std::max<int64_t>(nblk, 1) * (nk + 1), 0.0);
    for_blocks(n, par, [&](int64_t blk, int64_t b0, int64_t b1) {
      const int64_t ri = rows[i];
      row_entries(K, ri, cols.data(), cp.data(), b0, b1, row.data());
      for (size_t k = 0; k < nk; ++k) {
        const double ui = us[k][i];
        const double* v = vs[k].data();
        for (int64_t j = b0; j < b1; ++j) row[j] = row[j] - ui * v[j];
      }
      p_vv[blk] = dot8(row.data() + b0, row.data() + b0, b1 - b0);
      for (size_t k = 0; k < nk; ++k)
        p_cross[(size_t)blk * nk + k] = dot8(row.data() + b0, vs[k].data() + b0, b1 - b0);
    });
    used_rows[i] = 1;
    const auto [jb, mb] = argmax_masked(row.data(), used_cols.data(), n, par);
    const double piv = row[jb];
    if (mb <= 1e-14 * std::max(1.0, std::sqrt(fro2))) {
      int64_t un = -1;
      for (int64_t a = 0; a < m; ++a)
        if (!used_rows[a]) {
          un = a;
          break;
        }
      if (un < 0) break;  // exhausted
      i = un;
      continue;
    }
    std::vector<double> u(m);
    for_blocks(m, par, [&](int64_t, int64_t b0, int64_t b1) {
      const int64_t cj = cols[jb];
      for (int64_t a = b0; a < b1; ++a) col[a] = K.entry(rows[a], cj);
      for (size_t k = 0; k < us.size(); ++k) {
        const double vj = vs[k][jb];
        const double* uk = us[k].data();
        for (int64_t a = b0; a < b1; ++a) col[a] = col[a] - vj * uk[a];
      }
      for (int64_t a = b0; a < b1; ++a) u[a] = col[a] / piv;
    });
    used_cols[jb] = 1;
    const double nu = std::sqrt(dot_blocked(u.data(), u.data(), m, par));
    double vv = 0.0;
    for (int64_t b = 0; b < nblk; ++b) vv += p_vv[b];
    const double nv = std::sqrt(vv);
    double cross = 0.0;
    for (size_t k = 0; k < nk; ++k) {
      double rv = 0.0;
      for (int64_t b = 0; b < nblk; ++b) rv += p_cross[(size_t)b * nk + k];
      cross += dot_blocked(us[k].data(), u.data(), m, par) * rv;
    }
    fro2 += 2.0 * cross + (nu * nv) * (nu * nv);
    us.push_back(std::move(u));
    vs.push_back(row);
    out.tau.push_back(rows[i]);
    out.sigma.push_back(cols[jb]);
    if (nu * nv <= eps * std::sqrt(fro2) || (int64_t)us.size() >= max_rank) break;
    const auto [ib, mu] = argmax_masked(us.back().data(), used_rows.data(), m, par);
    if (mu <= 0.0) {  // masked.max() == 0
      int64_t un = -1;
      for (int64_t a = 0; a < m; ++a)
        if (!used_rows[a]) {
          un = a;
          break;
        }
      if (un < 0) break;
      i = un;
    } else {
      i = ib;
    }
  }
  if (!keep_factors) {
    us.clear();
    vs.clear();
  }
  return out;
}

LU make_lu(const Kernel& K, const Idx& r, const Idx& c, bool transpose) {
  LU L;
  L.n = (int)r.size();
  L.a.resize((size_t)L.n * L.n);
  if (!transpose)
    K.block_cm(r.data(), L.n, c.data(), L.n, L.a.data(), L.n);
  else  // A^T column-major == A row-major
    for (int a = 0; a < L.n; ++a)
      for (int b = 0; b < L.n; ++b) L.a[(size_t)a * L.n + b] = K.entry(r[a], c[b]);
  lu_factor(L);
  return L;
}

// engine.py:39-51
void pivot_pair(const Kernel& K, const Idx& rows, const Idx& cols, double eps, int64_t cid,
                Idx& tau, Idx& sigma, bool par = false) {
  for (double te : {eps, eps / 10.0}) {
    AcaOut a = aca(K, rows, cols, te, false, par);
    if (a.tau.empty()) {
      tau.clear();
      sigma.clear();
      return;
    }
    LU L = make_lu(K, a.tau, a.sigma, false);
    if (!lu_singular(L)) {
      tau = std::move(a.tau);
      sigma = std::move(a.sigma);
      return;
    }
  }
  throw SingularCross("singular cross matrix after retry (cluster " + std::to_string(cid) + ")");
}

Idx sorted_union(std::vector<const Idx*> parts) {
  Idx u;
  size_t tot = 0;
  for (auto* p : parts) tot += p->size();
  u.reserve(tot);
  for (auto* p : parts) u.insert(u.end(), p->begin(), p->end());
  std::sort(u.begin(), u.end());
  u.erase(std::unique(u.begin(), u.end()), u.end());
  return u;
}

struct Quad {
  Idx t_i, s_i, t_o, s_o;
  bool empty() const { return t_i.empty() && t_o.empty(); }
};

// ------------------------------------------------------------------ tree
struct Tree {
  int d = 2, kappa = 1;
  int64_t N = 0;
  std::vector<int64_t> lo;       // level offsets (kappa + 2)
  std::vector<int64_t> perm;     // tree position -> original index
  std::vector<int64_t> st, en;   // slices
  int64_t nc() const { return lo.back(); }
  int level_of(int64_t c) const {
    int l = 0;
    while (c >= lo[l + 1]) ++l;
    return l;
  }
  int64_t parent(int64_t c, int l) const { return lo[l - 1] + ((c - lo[l]) >> d); }
  int64_t child0(int64_t c, int l) const { return lo[l + 1] + ((c - lo[l]) << d); }
  Idx index_set(int64_t c) const { return Idx(perm.begin() + st[c], perm.begin() + en[c]); }
  int64_t size(int64_t c) const { return en[c] - st[c]; }
};

int64_t morton(const int64_t* cell, int d, int level) {  // tree.py:93-100
  int64_t out = 0;
  for (int bit = 0; bit < level; ++bit)
    for (int ax = 0; ax < d; ++ax) out |= ((cell[ax] >> bit) & 1LL) << (bit * d + ax);
  return out;
}

void demorton(int64_t m, int d, int level, int64_t* coord) {  // tree.py:103-108
  for (int ax = 0; ax < d; ++ax) coord[ax] = 0;
  for (int bit = 0; bit < level; ++bit)
    for (int ax = 0; ax < d; ++ax) coord[ax] |= ((m >> (bit * d + ax)) & 1LL) << bit;
}

Tree build_tree(const double* pts, int64_t N, int d, int n_max) {  // tree.py:111-185
  Tree T;
  T.d = d;
  T.N = N;
  double lo[3], hi[3];
  for (int k = 0; k < d; ++k) lo[k] = hi[k] = pts[k];
  for (int64_t i = 0; i < N; ++i)
    for (int k = 0; k < d; ++k) {
      lo[k] = std::min(lo[k], pts[i * d + k]);
      hi[k] = std::max(hi[k], pts[i * d + k]);
    }
  double side = 0;
  for (int k = 0; k < d; ++k) side = std::max(side, hi[k] - lo[k]);
  if (side == 0.0) side = 1.0;
  double root_low[3];
  for (int k = 0; k < d; ++k) root_low[k] = 0.5 * (lo[k] + hi[k]) - 0.5 * side;
  int kappa = 1;
  if (N > n_max) {
    kappa = (int)std::ceil(std::log((double)N / (double)n_max) / std::log((double)(1 << d)));
    kappa = std::max(1, kappa);
  }
  T.kappa = kappa;
  const int64_t ncell = 1LL << kappa;
  const int64_t nleaf = 1LL << (d * kappa);
  std::vector<int64_t> leaf_m(N);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    int64_t cell[3];
    for (int k = 0; k < d; ++k) {
      int64_t c = (int64_t)std::floor((pts[i * d + k] - root_low[k]) / side * (double)ncell);
      cell[k] = std::min<int64_t>(std::max<int64_t>(c, 0), ncell - 1);
    }
    leaf_m[i] = morton(cell, d, kappa);
  }
  // stable counting sort by leaf code (== lexsort((arange, leaf_m)))
  std::vector<int64_t> cnt(nleaf + 1, 0);
  for (int64_t i = 0; i < N; ++i) cnt[leaf_m[i] + 1]++;
  for (int64_t m = 0; m < nleaf; ++m) cnt[m + 1] += cnt[m];
  T.perm.resize(N);
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
  for (int64_t i = 0; i < N; ++i) T.perm[pos[leaf_m[i]]++] = i;
  T.lo.assign(1, 0);
  for (int l = 0; l <= kappa; ++l) T.lo.push_back(T.lo.back() + (1LL << (d * l)));
  const int64_t nc = T.lo.back();
  T.st.assign(nc, 0);
  T.en.assign(nc, 0);
  for (int64_t m = 0; m < nleaf; ++m) {
    T.st[T.lo[kappa] + m] = cnt[m];
    T.en[T.lo[kappa] + m] = cnt[m + 1];
  }
  for (int l = kappa - 1; l >= 0; --l)
    for (int64_t c = T.lo[l]; c < T.lo[l + 1]; ++c) {
      const int64_t c0 = T.child0(c, l);
      T.st[c] = T.st[c0];
      T.en[c] = T.en[c0 + (1 << d) - 1];
    }
  return T;
}

// ------------------------------------------------------------------ partition
// partition.py:77-137 (weak / vertex-sharing admissibility)
struct Lists {
  std::vector<std::vector<int64_t>> far, ver, near;
};

int relation(const int64_t* a, const int64_t* b, int d) {  // partition.py:67-74; -1 SELF, -2 FAR
  int64_t mx = 0;
  int zeros = 0;
  for (int k = 0; k < d; ++k) {
    const int64_t df = std::llabs(a[k] - b[k]);
    mx = std::max(mx, df);
    zeros += df == 0;
  }
  if (mx == 0) return -1;
  if (mx <= 1) return zeros;
  return -2;
}

Lists build_partition(const Tree& T) {
  const int d = T.d;
  Lists P;
  const int64_t nc = T.nc();
  P.far.resize(nc);
  P.ver.resize(nc);
  P.near.resize(nc);
  P.near[0] = {0};
  // itertools.product((-1, 0, 1), repeat=d) / ((0, 1), repeat=d): last axis fastest
  std::vector<std::array<int64_t, 3>> offs, kids;
  {
    int n3 = 1;
    for (int k = 0; k < d; ++k) n3 *= 3;
    for (int t = 0; t < n3; ++t) {
      std::array<int64_t, 3> o{0, 0, 0};
      int v = t;
      for (int k = d - 1; k >= 0; --k) {
        o[k] = v % 3 - 1;
        v /= 3;
      }
      offs.push_back(o);
    }
    for (int t = 0; t < (1 << d); ++t) {
      std::array<int64_t, 3> o{0, 0, 0};
      for (int k = d - 1, v = t; k >= 0; --k, v >>= 1) o[k] = v & 1;
      kids.push_back(o);
    }
  }
  for (int l = 1; l <= T.kappa; ++l) {
    const int64_t side = 1LL << l, pside = side >> 1;
    const int64_t base = T.lo[l];
#pragma omp parallel for schedule(static)
    for (int64_t c = T.lo[l]; c < T.lo[l + 1]; ++c) {
      int64_t cx[3], cy[3], px[3], py[3];
      demorton(c - base, d, l, cx);
      auto& nr = P.near[c];
      auto& fr = P.far[c];
      auto& vr = P.ver[c];
      for (auto& o : offs) {
        bool ok = true;
        for (int k = 0; k < d; ++k) {
          cy[k] = cx[k] + o[k];
          ok &= cy[k] >= 0 && cy[k] < side;
        }
        if (!ok) continue;
        const int rel = relation(cx, cy, d);
        if (rel == -1)
          nr.push_back(c);
        else if (rel != 0)
          nr.push_back(base + morton(cy, d, l));
      }
      for (int k = 0; k < d; ++k) px[k] = cx[k] >> 1;
      for (auto& o : offs) {
        bool ok = true;
        for (int k = 0; k < d; ++k) {
          py[k] = px[k] + o[k];
          ok &= py[k] >= 0 && py[k] < pside;
        }
        if (!ok) continue;
        if (relation(px, py, d) == 0) continue;  // vertex-only parents
        for (auto& ch : kids) {
          for (int k = 0; k < d; ++k) cy[k] = 2 * py[k] + ch[k];
          const int rel = relation(cx, cy, d);
          if (rel == -2)
            fr.push_back(base + morton(cy, d, l));
          else if (rel == 0)
            vr.push_back(base + morton(cy, d, l));
        }
      }
      std::sort(nr.begin(), nr.end());
      std::sort(fr.begin(), fr.end());
      std::sort(vr.begin(), vr.end());
    }
  }
  return P;
}

// ------------------------------------------------------------------ channels
struct Channel {
  std::vector<Quad> quads;
  const std::vector<std::vector<int64_t>>* lists = nullptr;
  std::vector<int32_t> r_in, r_out;
  std::vector<int64_t> p2m_off, l2p_off, m2m_off, l2l_off;
  std::vector<int64_t> m2l_rowptr, m2l_off;
  std::vector<int32_t> m2l_src;
};

void finish_ranks(Channel& ch, int64_t nc) {
  ch.r_in.assign(nc, 0);
  ch.r_out.assign(nc, 0);
  for (int64_t c = 0; c < nc; ++c) {
    ch.r_in[c] = (int32_t)ch.quads[c].t_i.size();
    ch.r_out[c] = (int32_t)ch.quads[c].t_o.size();
  }
}

double now();

// Run body(x, par) for x in [lo, hi): clusters in parallel when the level has
// enough of them, otherwise one cluster at a time with the ACA loops inside
// running in parallel (the coarse levels' few, huge candidate sets).
template <class F>
void level_loop(int64_t lo, int64_t hi, F body) {
  const int64_t cnt = hi - lo;
  int64_t par_below = 2 * (int64_t)omp_get_max_threads();
  if (const char* e = getenv("H2B_PAR_BELOW")) par_below = atoll(e);
  if (cnt < par_below) {
    for (int64_t x = lo; x < hi; ++x) body(x, true);
  } else {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t x = lo; x < hi; ++x) body(x, false);
  }
}

// engine.py:54-86
void select_b2t(const Tree& T, const Kernel& K, Channel& ch, double eps) {
  const int64_t nc = T.nc();
  ch.quads.assign(nc, Quad());
  const auto& L = *ch.lists;
  for (int l = T.kappa; l >= 1; --l) {
    const bool leaf = l == T.kappa;
    std::string err;
    const double tl0 = now();
    level_loop(T.lo[l], T.lo[l + 1], [&](int64_t x, bool par) {
      try {
        if (L[x].empty()) return;
        Quad q;
        Idx ti_c, so_c, si_c, to_c;
        if (leaf) {
          ti_c = T.index_set(x);
          so_c = ti_c;
          std::vector<Idx> mem;
          for (int64_t y : L[x]) mem.push_back(T.index_set(y));
          std::vector<const Idx*> ptrs;
          for (auto& v : mem) ptrs.push_back(&v);
          si_c = sorted_union(ptrs);
          to_c = si_c;
        } else {
          std::vector<const Idx*> a, b, c2, d2;
          const int64_t c0 = T.child0(x, l);
          for (int64_t c = c0; c < c0 + (1 << T.d); ++c) {
            a.push_back(&ch.quads[c].t_i);
            b.push_back(&ch.quads[c].s_o);
          }
          for (int64_t y : L[x]) {
            const int64_t y0 = T.child0(y, l);
            for (int64_t yc = y0; yc < y0 + (1 << T.d); ++yc) {
              c2.push_back(&ch.quads[yc].s_o);
              d2.push_back(&ch.quads[yc].t_i);
            }
          }
          ti_c = sorted_union(a);
          so_c = sorted_union(b);
          si_c = sorted_union(c2);
          to_c = sorted_union(d2);
        }
        pivot_pair(K, ti_c, si_c, eps, x, q.t_i, q.s_i, par);
        pivot_pair(K, to_c, so_c, eps, x, q.t_o, q.s_o, par);
        ch.quads[x] = std::move(q);
      } catch (const std::exception& e) {
#pragma omp critical
        err = e.what();
      }
    });
    if (getenv("H2B_VERBOSE")) fprintf(stderr, "b2t level %d: %.2f s\n", l, now() - tl0);
    if (!err.empty()) throw SingularCross(err);
  }
  finish_ranks(ch, nc);
}

// engine.py:89-114
void select_t2b(const Tree& T, const Kernel& K, Channel& ch, double eps) {
  const int64_t nc = T.nc();
  ch.quads.assign(nc, Quad());
  const auto& L = *ch.lists;
  for (int l = 1; l <= T.kappa; ++l) {
    std::string err;
    const double tl0 = now();
    level_loop(T.lo[l], T.lo[l + 1], [&](int64_t x, bool par) {
      try {
        const Quad* pq = nullptr;
        if (l >= 2) {
          const Quad& p = ch.quads[T.parent(x, l)];
          if (!p.empty()) pq = &p;
        }
        if (L[x].empty() && !pq) return;
        std::vector<Idx> mem;
        for (int64_t y : L[x]) mem.push_back(T.index_set(y));
        std::vector<const Idx*> a, b;
        for (auto& v : mem) {
          a.push_back(&v);
          b.push_back(&v);
        }
        if (pq) {
          a.push_back(&pq->s_i);
          b.push_back(&pq->t_o);
        }
        const Idx si_c = sorted_union(a);
        const Idx to_c = sorted_union(b);
        const Idx xs = T.index_set(x);
        Quad q;
        pivot_pair(K, xs, si_c, eps, x, q.t_i, q.s_i, par);
        pivot_pair(K, to_c, xs, eps, x, q.t_o, q.s_o, par);
        ch.quads[x] = std::move(q);
      } catch (const std::exception& e) {
#pragma omp critical
        err = e.what();
      }
    });
    if (getenv("H2B_VERBOSE")) fprintf(stderr, "t2b level %d: %.2f s\n", l, now() - tl0);
    if (!err.empty()) throw SingularCross(err);
  }
  finish_ranks(ch, nc);
}

// ------------------------------------------------------------------ blob
struct Blob {
  int64_t len = 0;
  std::vector<double> data;
  int64_t take(int64_t n) {
    const int64_t o = len;
    len += n;
    return o;
  }
};

// engine.py:133-187: sizes first (offsets in the exporter's order), then fill
// store_m2l = false: M2L blocks are not stored (offset -1, evaluated on the
// device from the pivots); their scalars still count in mem_scalars.
int64_t layout_channel(const Tree& T, Channel& ch, Blob& B, bool store_m2l = true) {
  int64_t unstored = 0;
  const int64_t nc = T.nc();
  const int k = T.kappa;
  ch.p2m_off.assign(nc, -1);
  ch.l2p_off.assign(nc, -1);
  ch.m2m_off.assign(nc, -1);
  ch.l2l_off.assign(nc, -1);
  const auto& Q = ch.quads;
  for (int64_t x = T.lo[k]; x < T.lo[k + 1]; ++x)
    if (Q[x].t_o.size() && T.size(x)) ch.p2m_off[x] = B.take((int64_t)Q[x].t_o.size() * T.size(x));
  for (int64_t x = T.lo[k]; x < T.lo[k + 1]; ++x)
    if (Q[x].t_i.size() && T.size(x)) ch.l2p_off[x] = B.take((int64_t)Q[x].t_i.size() * T.size(x));
  for (int l = 1; l < k; ++l)
    for (int64_t x = T.lo[l]; x < T.lo[l + 1]; ++x) {
      if (Q[x].t_o.empty()) continue;
      const int64_t c0 = T.child0(x, l);
      for (int64_t c = c0; c < c0 + (1 << T.d); ++c)
        if (Q[c].t_o.size()) ch.m2m_off[c] = B.take((int64_t)Q[x].t_o.size() * Q[c].t_o.size());
    }
  for (int l = 1; l < k; ++l)
    for (int64_t x = T.lo[l]; x < T.lo[l + 1]; ++x) {
      if (Q[x].t_i.empty()) continue;
      const int64_t c0 = T.child0(x, l);
      for (int64_t c = c0; c < c0 + (1 << T.d); ++c)
        if (Q[c].t_i.size()) ch.l2l_off[c] = B.take((int64_t)Q[c].t_i.size() * Q[x].t_i.size());
    }
  ch.m2l_rowptr.assign(nc + 1, 0);
  ch.m2l_src.clear();
  ch.m2l_off.clear();
  const auto& L = *ch.lists;
  for (int64_t x = 0; x < nc; ++x) {
    if (Q[x].t_i.size())
      for (int64_t y : L[x])
        if (Q[y].t_o.size()) {
          const int64_t n = (int64_t)Q[x].t_i.size() * Q[y].t_o.size();
          ch.m2l_src.push_back((int32_t)y);
          ch.m2l_off.push_back(store_m2l ? B.take(n) : -1);
          if (!store_m2l) unstored += n;
        }
    ch.m2l_rowptr[x + 1] = (int64_t)ch.m2l_src.size();
  }
  return unstored;
}

void fill_channel(const Tree& T, const Kernel& K, const Channel& ch, double* blob) {
  const int k = T.kappa;
  const auto& Q = ch.quads;
  const auto& L = *ch.lists;
  for (int l = 1; l <= k; ++l) {
    const bool leaf = l == k;
    std::string err;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t x = T.lo[l]; x < T.lo[l + 1]; ++x) {
      try {
        const Quad& q = Q[x];
        if (q.empty()) continue;
        const int64_t ri = (int64_t)q.t_i.size(), ro = (int64_t)q.t_o.size();
        if (ri) {
          // rsolve(B, A_i) = solve_square(A_i^T, B^T)^T  (lowrank.py:178-180)
          LU Lt = make_lu(K, q.t_i, q.s_i, true);
          if (lu_singular(Lt))
            throw SingularCross("singular cross matrix (cluster " + std::to_string(x) + ")");
          auto rsolve_into = [&](const Idx& rows, double* out) {
            // out (nr x ri, column-major) = K[rows, s_i] A_i^{-1}
            const int64_t nr = (int64_t)rows.size();
            std::vector<double> bt((size_t)ri * nr);  // B^T column-major: ri x nr
            for (int64_t r = 0; r < nr; ++r)
              for (int64_t c = 0; c < ri; ++c) bt[(size_t)r * ri + c] = K.entry(rows[r], q.s_i[c]);
            lu_solve(Lt, bt.data(), nr);
            for (int64_t r = 0; r < nr; ++r)
              for (int64_t c = 0; c < ri; ++c) out[c * nr + r] = bt[(size_t)r * ri + c];
          };
          if (leaf) {
            if (ch.l2p_off[x] >= 0) rsolve_into(T.index_set(x), blob + ch.l2p_off[x]);
          } else {
            const int64_t c0 = T.child0(x, l);
            for (int64_t c = c0; c < c0 + (1 << T.d); ++c)
              if (ch.l2l_off[c] >= 0) rsolve_into(Q[c].t_i, blob + ch.l2l_off[c]);
          }
        }
        if (ro) {
          LU Lo = make_lu(K, q.t_o, q.s_o, false);
          if (lu_singular(Lo))
            throw SingularCross("singular cross matrix (cluster " + std::to_string(x) + ")");
          auto solve_into = [&](const Idx& cols, double* out) {
            // out (ro x nc, column-major) = A_o^{-1} K[t_o, cols]
            K.block_cm(q.t_o.data(), ro, cols.data(), (int64_t)cols.size(), out, ro);
            lu_solve(Lo, out, (int64_t)cols.size());
          };
          if (leaf) {
            if (ch.p2m_off[x] >= 0) solve_into(T.index_set(x), blob + ch.p2m_off[x]);
          } else {
            const int64_t c0 = T.child0(x, l);
            for (int64_t c = c0; c < c0 + (1 << T.d); ++c)
              if (ch.m2m_off[c] >= 0) solve_into(Q[c].s_o, blob + ch.m2m_off[c]);
          }
        }
        // M2L is the raw kernel block K[t_i(X), s_o(Y)] (engine.py:176-179)
        for (int64_t kk = ch.m2l_rowptr[x]; kk < ch.m2l_rowptr[x + 1]; ++kk) {
          if (ch.m2l_off[kk] < 0) continue;  // evaluated on the device
          const Quad& yq = Q[ch.m2l_src[kk]];
          K.block_cm(q.t_i.data(), ri, yq.s_o.data(), (int64_t)yq.s_o.size(),
                     blob + ch.m2l_off[kk], ri);
        }
        (void)L;
      } catch (const std::exception& e) {
#pragma omp critical
        err = e.what();
      }
    }
    if (!err.empty()) throw SingularCross(err);
  }
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

struct h2b_result {
  std::map<std::string, std::vector<int64_t>> i64;
  std::map<std::string, std::vector<int32_t>> i32;
  std::map<std::string, std::vector<double>> f64;
  std::map<std::string, int64_t> scalars;
  std::map<std::string, double> timing;
};

namespace {

int build_impl(const h2b_params* P, h2b_result** out) {
  if (!P || !out) {
    g_err = "null argument";
    return H2B_ERR_INVALID_ARG;
  }
  if (P->abi_version != H2B_ABI_VERSION || P->dim < 1 || P->dim > 3 || P->n_points < 1 ||
      !P->points || P->n_max < 1 || (P->variant != 0 && P->variant != 1) || P->kernel < 0 ||
      P->kernel > 2) {
    g_err = "invalid parameters";
    return H2B_ERR_INVALID_ARG;
  }
  if (P->n_threads > 0) omp_set_num_threads(P->n_threads);
  auto R = new h2b_result();
  const double t_start = now();
  const int d = P->dim;
  Kernel K;
  K.type = P->kernel;
  K.d = d;
  K.pts = P->points;
  K.zero_value = P->zero_value;
  K.diag = P->diag;
  K.has_diag = P->has_diag != 0;
  K.shift = P->shift;
  K.sigma = P->sigma;

  double t0 = now();
  Tree T = build_tree(P->points, P->n_points, d, P->n_max);
  R->timing["tree"] = now() - t0;
  t0 = now();
  Lists PL = build_partition(T);
  R->timing["partition"] = now() - t0;
  const int64_t nc = T.nc();

  // channels (engine.py:351-358)
  std::vector<Channel> chans;
  t0 = now();
  {
    Channel far;
    far.lists = &PL.far;
    select_b2t(T, K, far, P->eps_far);
    chans.push_back(std::move(far));
    if (P->variant == H2B_VARIANT_H2STAR_BT) {
      Channel ver;
      ver.lists = &PL.ver;
      select_t2b(T, K, ver, P->eps_ver);
      chans.push_back(std::move(ver));
    }
  }
  R->timing["pivots"] = now() - t0;

  Blob B;
  const bool store_near = (P->skip_blocks & H2B_SKIP_NEAR) == 0;
  const bool store_m2l = (P->skip_blocks & H2B_SKIP_M2L) == 0;
  int64_t unstored = 0;
  for (auto& ch : chans) unstored += layout_channel(T, ch, B, store_m2l);
  int64_t mem = B.len + unstored;  // channel operators (non-symmetric: no shared views)

  // BLR leg (blr.py:46-69, lists="ver", include_near=False)
  t0 = now();
  std::vector<int64_t> blr_x, blr_y;
  for (int l = 1; l <= T.kappa; ++l)
    for (int64_t x = T.lo[l]; x < T.lo[l + 1]; ++x)
      for (int64_t y : PL.ver[x])
        if (P->variant == H2B_VARIANT_H2PLUSH_STAR) {
          blr_x.push_back(x);
          blr_y.push_back(y);
        }
  std::vector<AcaOut> fac(blr_x.size());
  {
    // factors with huge candidate sets (coarse levels): one at a time, ACA
    // loops in parallel; the rest: factors in parallel
    const int64_t big = 1 << 16;
    for (int64_t f = 0; f < (int64_t)blr_x.size(); ++f)
      if (T.size(blr_x[f]) + T.size(blr_y[f]) > big)
        fac[f] = aca(K, T.index_set(blr_x[f]), T.index_set(blr_y[f]), P->eps_ver, true, true);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t f = 0; f < (int64_t)blr_x.size(); ++f)
      if (T.size(blr_x[f]) + T.size(blr_y[f]) <= big)
        fac[f] = aca(K, T.index_set(blr_x[f]), T.index_set(blr_y[f]), P->eps_ver, true);
  }
  R->timing["blr"] = now() - t0;
  std::vector<int64_t> blr_rowptr(nc + 1, 0), blr_u, blr_v;
  std::vector<int32_t> blr_src, blr_rank;
  {
    size_t f = 0;
    for (int64_t x = 0; x < nc; ++x) {
      // factors are grouped by x (level-major, x ascending, y ascending)
      while (f < blr_x.size() && blr_x[f] == x) {
        const int64_t p = (int64_t)fac[f].us.size();
        mem += p * (T.size(x) + T.size(blr_y[f]));
        if (p > 0) {
          blr_src.push_back((int32_t)blr_y[f]);
          blr_rank.push_back((int32_t)p);
          blr_u.push_back(B.take(p * T.size(x)));
          blr_v.push_back(B.take(p * T.size(blr_y[f])));
        } else {
          blr_u.push_back(-1);  // placeholder removed below
          blr_v.push_back(-1);
          blr_src.push_back(-1);
          blr_rank.push_back(0);
        }
        ++f;
      }
      blr_rowptr[x + 1] = (int64_t)blr_src.size();
    }
  }

  // near field (engine.py:309-318)
  std::vector<int64_t> near_rowptr(nc + 1, 0), near_off;
  std::vector<int32_t> near_src;
  for (int64_t x = 0; x < nc; ++x) {
    if (T.level_of(x) == T.kappa)
      for (int64_t y : PL.near[x]) {
        mem += T.size(x) * T.size(y);
        if (T.size(x) && T.size(y)) {
          near_src.push_back((int32_t)y);
          near_off.push_back(store_near ? B.take(T.size(x) * T.size(y)) : -1);
        }
      }
    near_rowptr[x + 1] = (int64_t)near_src.size();
  }

  // allocate + fill the blob
  std::vector<double>& blob = R->f64["blob"];
  try {
    blob.assign((size_t)B.len + 16, 0.0);
  } catch (const std::bad_alloc&) {
    g_err = "host out of memory for the operator blob";
    delete R;
    return H2B_ERR_OOM;
  }
  t0 = now();
  try {
    for (auto& ch : chans) fill_channel(T, K, ch, blob.data());
  } catch (const SingularCross& e) {
    g_err = e.what();
    delete R;
    return H2B_ERR_SINGULAR;
  }
  R->timing["operators"] = now() - t0;
  t0 = now();
  {
    // copy BLR factors: U (n_X x p) column-major, V (n_Y x p) row-major
    std::vector<int64_t> fidx(blr_src.size());
    for (size_t k = 0; k < fidx.size(); ++k) fidx[k] = (int64_t)k;  // k-th entry <-> fac[k]
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t kk = 0; kk < (int64_t)blr_src.size(); ++kk) {
      const AcaOut& a = fac[kk];
      const int64_t p = (int64_t)a.us.size();
      if (!p) continue;
      const int64_t nx = (int64_t)a.us[0].size(), ny = (int64_t)a.vs[0].size();
      double* U = blob.data() + blr_u[kk];
      double* V = blob.data() + blr_v[kk];
      // leaf-blocked U (h2g.h): rows of each leaf L of X form one n_L x p
      // column-major block at (cl_start[L] - cl_start[X]) * p
      const int64_t x = blr_x[kk];
      const int lx = T.level_of(x);
      const int shift = T.d * (T.kappa - lx);
      const int64_t first = T.lo[T.kappa] + ((x - T.lo[lx]) << shift);
      for (int64_t L = first; L < first + (1LL << shift); ++L) {
        const int64_t r0 = T.st[L] - T.st[x], nl = T.size(L);
        double* B = U + r0 * p;
        for (int64_t c = 0; c < p; ++c)
          std::memcpy(B + c * nl, a.us[c].data() + r0, nl * sizeof(double));
      }
      (void)nx;
      for (int64_t r = 0; r < ny; ++r)
        for (int64_t c = 0; c < p; ++c) V[r * p + c] = a.vs[c][r];
    }
    fac.clear();
    fac.shrink_to_fit();
    // drop rank-0 placeholders (mvp_blr skips rank-0 factors, blr.py:79-80)
    std::vector<int64_t> rp(nc + 1, 0), u2, v2;
    std::vector<int32_t> s2, k2;
    for (int64_t x = 0; x < nc; ++x) {
      for (int64_t kk = blr_rowptr[x]; kk < blr_rowptr[x + 1]; ++kk)
        if (blr_rank[kk] > 0) {
          s2.push_back(blr_src[kk]);
          k2.push_back(blr_rank[kk]);
          u2.push_back(blr_u[kk]);
          v2.push_back(blr_v[kk]);
        }
      rp[x + 1] = (int64_t)s2.size();
    }
    blr_rowptr.swap(rp);
    blr_src.swap(s2);
    blr_rank.swap(k2);
    blr_u.swap(u2);
    blr_v.swap(v2);
  }
  R->timing["blr"] += now() - t0;
  t0 = now();
  {
    std::vector<int64_t> nx_of(near_src.size());
    for (int64_t x = 0; x < nc; ++x)
      for (int64_t kk = near_rowptr[x]; kk < near_rowptr[x + 1]; ++kk) nx_of[kk] = x;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t kk = 0; kk < (int64_t)near_src.size(); ++kk) {
      if (near_off[kk] < 0) continue;  // evaluated on the device (store_near=False)
      const int64_t x = nx_of[kk], y = near_src[kk];
      K.block_cm(T.perm.data() + T.st[x], T.size(x), T.perm.data() + T.st[y], T.size(y),
                 blob.data() + near_off[kk], T.size(x));
    }
  }
  R->timing["near"] = now() - t0;

  // ---- outputs (packed.py field names)
  std::vector<int64_t> inv_perm(T.N);
  for (int64_t i = 0; i < T.N; ++i) inv_perm[T.perm[i]] = i;
  R->i64["perm"] = T.perm;
  R->i64["level_offset"] = T.lo;
  R->i64["cl_start"] = T.st;
  R->i64["cl_end"] = T.en;
  for (size_t c = 0; c < chans.size(); ++c) {
    const std::string p = "ch" + std::to_string(c) + "_";
    Channel& ch = chans[c];
    R->i32[p + "r_in"] = ch.r_in;
    R->i32[p + "r_out"] = ch.r_out;
    R->i64[p + "p2m_off"] = ch.p2m_off;
    R->i64[p + "l2p_off"] = ch.l2p_off;
    R->i64[p + "m2m_off"] = ch.m2m_off;
    R->i64[p + "l2l_off"] = ch.l2l_off;
    R->i64[p + "m2l_rowptr"] = ch.m2l_rowptr;
    R->i32[p + "m2l_src"] = ch.m2l_src;
    R->i64[p + "m2l_off"] = ch.m2l_off;
    // NCA pivots t_i / s_o as tree positions (M2L evaluation on the device)
    std::vector<int64_t> ip(nc + 1, 0), op(nc + 1, 0), iv, ov;
    for (int64_t x = 0; x < nc; ++x) {
      for (int64_t g : ch.quads[x].t_i) iv.push_back(inv_perm[g]);
      for (int64_t g : ch.quads[x].s_o) ov.push_back(inv_perm[g]);
      ip[x + 1] = (int64_t)iv.size();
      op[x + 1] = (int64_t)ov.size();
    }
    R->i64[p + "piv_in_ptr"] = std::move(ip);
    R->i64[p + "piv_in"] = std::move(iv);
    R->i64[p + "piv_out_ptr"] = std::move(op);
    R->i64[p + "piv_out"] = std::move(ov);
  }
  R->i64["blr_rowptr"] = blr_rowptr;
  R->i32["blr_src"] = blr_src;
  R->i32["blr_rank"] = blr_rank;
  R->i64["blr_u_off"] = blr_u;
  R->i64["blr_v_off"] = blr_v;
  R->i64["near_rowptr"] = near_rowptr;
  R->i32["near_src"] = near_src;
  R->i64["near_off"] = near_off;
  {
    std::vector<double>& pt = R->f64["points_tree"];
    pt.resize((size_t)T.N * d);
    for (int64_t i = 0; i < T.N; ++i)
      for (int k = 0; k < d; ++k) pt[(size_t)i * d + k] = P->points[T.perm[i] * d + k];
  }
  R->scalars["kappa"] = T.kappa;
  R->scalars["n_channels"] = (int64_t)chans.size();
  R->scalars["mem_scalars"] = mem;
  R->scalars["n_clusters"] = nc;
  R->timing["total"] = now() - t_start;
  *out = R;
  return H2B_OK;
}

}  // namespace

extern "C" {

int h2b_abi_version(void) { return H2B_ABI_VERSION; }

int h2b_fill_kernel_blocks(const h2b_fill_desc* f, double* blob, int64_t blob_len) {
  if (!f || !blob || !f->points_tree || f->dim < 1 || f->dim > 3 || f->n_channels < 0 ||
      f->n_channels > 2 || !f->cl_start || !f->cl_end || !f->near_rowptr) {
    g_err = "h2b_fill_kernel_blocks: bad descriptor";
    return H2B_ERR_INVALID_ARG;
  }
  Kernel K;  // Kernel::entry on tree positions == on original indices (same points)
  K.type = f->kernel;
  K.d = f->dim;
  K.pts = f->points_tree;
  K.zero_value = f->zero_value;
  K.diag = f->diag;
  K.shift = f->shift;
  K.sigma = f->sigma;
  K.has_diag = f->has_diag != 0;
  if (f->n_threads > 0) omp_set_num_threads(f->n_threads);
  const int64_t nc = f->n_clusters;
  std::string err;
  for (int ch = 0; ch < f->n_channels; ++ch) {
    const h2b_fill_channel& c = f->channels[ch];
    if (!c.r_in || !c.r_out || !c.m2l_rowptr || (c.m2l_rowptr[nc] > 0 && (!c.piv_in || !c.piv_out))) {
      g_err = "h2b_fill_kernel_blocks: channel arrays missing";
      return H2B_ERR_INVALID_ARG;
    }
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t x = 0; x < nc; ++x) {
      const int64_t ri = c.r_in[x];
      for (int64_t k = c.m2l_rowptr[x]; k < c.m2l_rowptr[x + 1]; ++k) {
        if (c.m2l_off[k] < 0) continue;
        const int64_t y = c.m2l_src[k];
        const int64_t ro = c.r_out[y];
        if (c.m2l_off[k] + ri * ro > blob_len) {
#pragma omp critical
          err = "m2l block out of blob";
          continue;
        }
        K.block_cm(c.piv_in + c.piv_in_ptr[x], ri, c.piv_out + c.piv_out_ptr[y], ro,
                   blob + c.m2l_off[k], ri);
      }
    }
  }
  std::vector<int64_t> pos(f->n_points);
  for (int64_t i = 0; i < f->n_points; ++i) pos[i] = i;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t x = 0; x < nc; ++x) {
    const int64_t nx = f->cl_end[x] - f->cl_start[x];
    for (int64_t k = f->near_rowptr[x]; k < f->near_rowptr[x + 1]; ++k) {
      if (!f->near_off || f->near_off[k] < 0) continue;
      const int64_t y = f->near_src[k];
      const int64_t ny = f->cl_end[y] - f->cl_start[y];
      if (f->near_off[k] + nx * ny > blob_len) {
#pragma omp critical
        err = "near block out of blob";
        continue;
      }
      K.block_cm(pos.data() + f->cl_start[x], nx, pos.data() + f->cl_start[y], ny,
                 blob + f->near_off[k], nx);
    }
  }
  if (!err.empty()) {
    g_err = err;
    return H2B_ERR_INVALID_ARG;
  }
  return H2B_OK;
}
const char* h2b_last_error(void) { return g_err.c_str(); }

int h2b_build(const h2b_params* params, h2b_result** out) {
  try {
    return build_impl(params, out);
  } catch (const std::bad_alloc&) {
    g_err = "host out of memory";
    return H2B_ERR_OOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return H2B_ERR_SINGULAR;
  }
}

int h2b_get_array(const h2b_result* r, const char* name, const void** ptr, int64_t* len,
                  int32_t* dtype) {
  if (!r || !name) return H2B_ERR_INVALID_ARG;
  const std::string n(name);
  if (auto it = r->i64.find(n); it != r->i64.end()) {
    *ptr = it->second.data();
    *len = (int64_t)it->second.size();
    *dtype = H2B_I64;
    return H2B_OK;
  }
  if (auto it = r->i32.find(n); it != r->i32.end()) {
    *ptr = it->second.data();
    *len = (int64_t)it->second.size();
    *dtype = H2B_I32;
    return H2B_OK;
  }
  if (auto it = r->f64.find(n); it != r->f64.end()) {
    *ptr = it->second.data();
    *len = (int64_t)it->second.size();
    *dtype = H2B_F64;
    return H2B_OK;
  }
  g_err = "no array named " + n;
  return H2B_ERR_INVALID_ARG;
}

int64_t h2b_get_scalar(const h2b_result* r, const char* name) {
  if (!r || !name) return -1;
  auto it = r->scalars.find(name);
  return it == r->scalars.end() ? -1 : it->second;
}

double h2b_get_timing(const h2b_result* r, const char* name) {
  if (!r || !name) return -1;
  auto it = r->timing.find(name);
  return it == r->timing.end() ? -1.0 : it->second;
}

void h2b_free(h2b_result* r) { delete r; }

}  // extern "C"
