/* TEST INFRASTRUCTURE ONLY — see pb_oracle.h.  Plain-C restatement of the
 * reference's hot path; each function cites the reference file:line it
 * restates (paths relative to /root/reference/proj/include/panelblas/).
 * Compiled with -ffp-contract=off: every a*b+c below is a rounded multiply
 * followed by a rounded add, exactly like the reference's x86-64 build. */
#include "pb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define NR 4 /* KernelConfig::nr (micro_kernel.hpp:26-33) */
#define MR 8 /* KernelConfig::mr */
#define PS 4 /* KernelConfig::ps */

static int imax(int a, int b) { return a > b ? a : b; }
static int imin(int a, int b) { return a < b ? a : b; }

/* netlib flag parsing, mat_view.hpp:26-58 ('C' is Trans). */
static int p_trans(char c) {
  switch (c) { case 'n': case 'N': return 0; case 't': case 'T': case 'c': case 'C': return 1; }
  return -1;
}
static int p_uplo(char c) { /* 1 = Lower, 0 = Upper */
  switch (c) { case 'l': case 'L': return 1; case 'u': case 'U': return 0; }
  return -1;
}
static int p_side(char c) { /* 1 = Left, 0 = Right */
  switch (c) { case 'l': case 'L': return 1; case 'r': case 'R': return 0; }
  return -1;
}
static int p_diag(char c) { /* 1 = Unit, 0 = NonUnit */
  switch (c) { case 'n': case 'N': return 0; case 'u': case 'U': return 1; }
  return -1;
}

#define CM(p, ld, i, j) ((p)[(long long)(i) + (long long)(j) * (ld)])
static long long poff(int i, int j, int ps, int cn) { /* panel_mat.hpp:39-42 */
  return (long long)(i / ps) * ps * cn + (long long)j * ps + i % ps;
}
#define PM(d, i, j) ((d).data[poff((i), (j), (d).ps, (d).cn)])

/* scale_ab (micro_kernel.hpp:263-273): beta == 0 never reads c. */
static double scale_ab(double alpha, double beta, double t, const double* c) {
  if (beta == 0.0) return t * alpha;
  return alpha * t + beta * (*c);
}

/* ------------------------------------------------------------------ dgemm */
/* blas.hpp:73-102 (validation + quick returns) -> gemm.hpp:427-459.  All five
 * variants share one accumulation order (micro_kernel.hpp:8-11): t = 0, then
 * t += op(a)(i,l) * op(b)(l,j) for l ascending, then scale_ab.  The
 * alpha == 0 || k == 0 path is scale_only (gemm.hpp:404-419): scale_ab with
 * alpha = 0 over an empty accumulation. */
int orc_dgemm(char transa, char transb, int m, int n, int k, double alpha, const double* a, int lda,
              const double* b, int ldb, double beta, double* c, int ldc) {
  int ta = p_trans(transa), tb = p_trans(transb);
  if (ta < 0) return 1;
  if (tb < 0) return 2;
  if (m < 0) return 3;
  if (n < 0) return 4;
  if (k < 0) return 5;
  if (lda < imax(1, ta ? k : m)) return 8;
  if (ldb < imax(1, tb ? n : k)) return 10;
  if (ldc < imax(1, m)) return 13;
  if (m == 0 || n == 0) return 0;
  if ((alpha == 0.0 || k == 0) && beta == 1.0) return 0;
  int scale_only = alpha == 0.0 || k == 0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) {
      double t = 0.0;
      if (!scale_only)
        for (int l = 0; l < k; ++l) {
          double av = ta ? CM(a, lda, l, i) : CM(a, lda, i, l);
          double bv = tb ? CM(b, ldb, j, l) : CM(b, ldb, l, j);
          t += av * bv;
        }
      CM(c, ldc, i, j) = scale_ab(scale_only ? 0.0 : alpha, beta, t, &CM(c, ldc, i, j));
    }
  return 0;
}

/* ------------------------------------------------------------------ dsyrk */
/* blas.hpp:104-128 -> level3.hpp:220-246 (syrk_path_b/c, scale_tri).  Only
 * the uplo triangle is read from c or written. */
int orc_dsyrk(char uplo, char trans, int n, int k, double alpha, const double* a, int lda,
              double beta, double* c, int ldc) {
  int lo = p_uplo(uplo), tr = p_trans(trans);
  if (lo < 0) return 1;
  if (tr < 0) return 2;
  if (n < 0) return 3;
  if (k < 0) return 4;
  if (lda < imax(1, tr ? k : n)) return 7;
  if (ldc < imax(1, n)) return 10;
  if (n == 0) return 0;
  if ((alpha == 0.0 || k == 0) && beta == 1.0) return 0;
  int scale_only = alpha == 0.0 || k == 0;
  for (int j = 0; j < n; ++j)
    for (int i = lo ? j : 0; i < (lo ? n : j + 1); ++i) {
      /* Upper runs the lower schedule on transposed windows: element (i, j)
       * is the transposed tile's (j, i), products commute exactly. */
      int r = lo ? i : j, s = lo ? j : i;
      double t = 0.0;
      if (!scale_only)
        for (int l = 0; l < k; ++l) {
          double x = tr ? CM(a, lda, l, r) : CM(a, lda, r, l);
          double y = tr ? CM(a, lda, l, s) : CM(a, lda, s, l);
          t += x * y;
        }
      CM(c, ldc, i, j) = scale_ab(scale_only ? 0.0 : alpha, beta, t, &CM(c, ldc, i, j));
    }
  return 0;
}

/* ------------------------------------------------------------------ dtrsm */
/* Right-side solve core, level3.hpp:174-214 + kernel_trsm_right
 * micro_kernel.hpp:522-543 + edge_trsm_right 330-356.  x(r, c) addresses
 * the effective (possibly transposed) right-hand side; opa(l, c) the
 * effective op(A).  Rows are independent; column tiles of NR run in
 * dependency order. */
typedef struct {
  double* b; int ldb; int twin;       /* x(r,c) = twin ? B(c,r) : B(r,c) */
  const double* a; int lda; int trans; /* opa(l,c) = trans ? A(c,l) : A(l,c) */
} trsm_ctx;
static double* tx(const trsm_ctx* s, int r, int c) {
  return s->twin ? &CM(s->b, s->ldb, c, r) : &CM(s->b, s->ldb, r, c);
}
static double topa(const trsm_ctx* s, int l, int c) {
  return s->trans ? CM(s->a, s->lda, c, l) : CM(s->a, s->lda, l, c);
}
static void trsm_right_rows(const trsm_ctx* s, int lower, int unit, int mm, int nn, double alpha) {
  int eff_lower = lower == !s->trans;
  int ntiles = (nn + NR - 1) / NR;
  double t[NR];
  for (int r = 0; r < mm; ++r) {
    for (int ti = 0; ti < ntiles; ++ti) {
      int j0 = (eff_lower ? ntiles - 1 - ti : ti) * NR;
      int na = imin(NR, nn - j0);
      int l0 = eff_lower ? j0 + na : 0, l1 = eff_lower ? nn : j0;
      for (int c = 0; c < na; ++c) {
        double acc = 0.0;
        for (int l = l0; l < l1; ++l) acc += *tx(s, r, l) * topa(s, l, j0 + c);
        t[c] = -1.0 * acc + alpha * *tx(s, r, j0 + c); /* scale_ab(-1, alpha) */
      }
      for (int step = 0; step < na; ++step) {
        int c = eff_lower ? na - 1 - step : step;
        if (eff_lower) {
          for (int l = c + 1; l < na; ++l) t[c] -= t[l] * topa(s, j0 + l, j0 + c);
        } else {
          for (int l = 0; l < c; ++l) t[c] -= t[l] * topa(s, j0 + l, j0 + c);
        }
        if (!unit) t[c] *= 1.0 / topa(s, j0 + c, j0 + c);
      }
      for (int c = 0; c < na; ++c) *tx(s, r, j0 + c) = t[c];
    }
  }
}

/* blas.hpp:178-188 (trimul_adapter 133-162) -> level3.hpp:280-314. */
int orc_dtrsm(char side, char uplo, char transa, char diag, int m, int n, double alpha,
              const double* a, int lda, double* b, int ldb) {
  int sd = p_side(side), lo = p_uplo(uplo), tr = p_trans(transa), un = p_diag(diag);
  if (sd < 0) return 1;
  if (lo < 0) return 2;
  if (tr < 0) return 3;
  if (un < 0) return 4;
  if (m < 0) return 5;
  if (n < 0) return 6;
  int t = sd ? m : n;
  if (lda < imax(1, t)) return 9;
  if (ldb < imax(1, m)) return 11;
  if (m == 0 || n == 0) return 0;
  if (alpha == 0.0) { /* scale_only(beta = 0): zeros, a never read */
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < m; ++i) CM(b, ldb, i, j) = 0.0 * 0.0;
    return 0;
  }
  if (!un)
    for (int i = 0; i < t; ++i)
      if (CM(a, lda, i, i) == 0.0) return i + 1; /* before any write */
  trsm_ctx s = {b, ldb, sd, a, lda, sd ? !tr : tr};
  trsm_right_rows(&s, lo, un, sd ? n : m, sd ? m : n, alpha);
  return 0;
}

/* ------------------------------------------------------------------ dtrmm */
/* Right-side multiply core, level3.hpp:132-170 (trmm_right_core) +
 * kernel_trmm_right micro_kernel.hpp:566-586 + edge_trmm_right 357-378.
 * For each NR-column tile of the effective problem: t = 0; t += X(r,l) *
 * opA(l, j0+c) over the rectangular range (l ascending: [j0+na, nn) when
 * op(A) is effectively lower, [0, j0) when upper); then the triangular edge
 * l in [j0+c, j0+na) (eff. lower) or [j0, j0+c] (eff. upper), unit diagonals
 * counted as 1 and never read; then scale_ab(alpha, 0) = t * alpha.  The
 * row band of X is packed before any tile of that band is stored, so b may
 * be the destination. */
static void trmm_right_rows(const trsm_ctx* s, int lower, int unit, int mm, int nn, double alpha,
                            double* xrow) {
  int eff_lower = lower == !s->trans;
  double t[NR];
  for (int r = 0; r < mm; ++r) {
    for (int l = 0; l < nn; ++l) xrow[l] = *tx(s, r, l); /* pack_row_block */
    for (int j0 = 0; j0 < nn; j0 += NR) {
      int na = imin(NR, nn - j0);
      int l0 = eff_lower ? j0 + na : 0, l1 = eff_lower ? nn : j0;
      for (int c = 0; c < na; ++c) {
        double acc = 0.0;
        for (int l = l0; l < l1; ++l) acc += xrow[l] * topa(s, l, j0 + c);
        int lo = eff_lower ? c : 0, hi = eff_lower ? na : c + 1;
        for (int l = lo; l < hi; ++l) {
          double f = (l == c && unit) ? 1.0 : topa(s, j0 + l, j0 + c);
          acc += xrow[j0 + l] * f;
        }
        t[c] = acc * alpha;
      }
      for (int c = 0; c < na; ++c) *tx(s, r, j0 + c) = t[c];
    }
  }
}

/* blas.hpp:166-176 (trimul_adapter 133-162, same validation as dtrsm) ->
 * level3.hpp:250-275. */
int orc_dtrmm(char side, char uplo, char transa, char diag, int m, int n, double alpha,
              const double* a, int lda, double* b, int ldb) {
  int sd = p_side(side), lo = p_uplo(uplo), tr = p_trans(transa), un = p_diag(diag);
  if (sd < 0) return 1;
  if (lo < 0) return 2;
  if (tr < 0) return 3;
  if (un < 0) return 4;
  if (m < 0) return 5;
  if (n < 0) return 6;
  int t = sd ? m : n;
  if (lda < imax(1, t)) return 9;
  if (ldb < imax(1, m)) return 11;
  if (m == 0 || n == 0) return 0;
  if (alpha == 0.0) { /* scale_only(beta = 0): zeros, a never read */
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < m; ++i) CM(b, ldb, i, j) = 0.0 * 0.0;
    return 0;
  }
  trsm_ctx s = {b, ldb, sd, a, lda, sd ? !tr : tr};
  double* xrow = (double*)malloc(sizeof(double) * (size_t)imax(1, t));
  trmm_right_rows(&s, lo, un, sd ? n : m, sd ? m : n, alpha, xrow);
  free(xrow);
  return 0;
}

/* ----------------------------------------------------------------- dpotrf */
/* blas.hpp:190-202 -> factor.hpp:45-99 (potrf_core) with
 * kernel_potrf_sub/_diag (micro_kernel.hpp:607-636), edge_potrf 309-325 and
 * edge_trsm_right 330-356.  Left-looking over MR-row bands x NR-column
 * tiles; element (i, j) of the factor is
 *   t = a(i,j) - sum_{l < j0} L(i,l) L(j,l)       (j0 = NR*floor(j/NR))
 *   t -= L(i,l) L(j,l)  for l = j0 .. j-1        (edge, after column l is final)
 *   L(j,j) = sqrt(t);  L(i,j) = t * (1 / L(j,j))
 * Tiles are stored in schedule order, so a failure leaves exactly the tiles
 * the reference stored (test_factor.cpp:251-277). Upper = twin windows. */
typedef struct { double* a; int lda; int upper; } pot_ctx;
static double* pa(const pot_ctx* s, int i, int j) { /* lower-triangle coordinates */
  return s->upper ? &CM(s->a, s->lda, j, i) : &CM(s->a, s->lda, i, j);
}

static int potrf_lower_sched(const pot_ctx* s, int n) {
  /* L holds the echo image of stored tiles (the reference's BandPack). */
  double* L = (double*)calloc((size_t)n * n, sizeof(double));
  double t[MR][NR];
  int info = 0;
  for (int i0 = 0; i0 < n && !info; i0 += MR) {
    int ma = imin(MR, n - i0);
    for (int j0 = 0; j0 < i0 + ma; j0 += NR) {
      int na = imin(NR, n - j0);
      int diag = j0 + na > i0, d = j0 - i0;
      for (int r = 0; r < ma; ++r)
        for (int c = 0; c < na; ++c) {
          double acc = 0.0;
          for (int l = 0; l < j0; ++l) acc += L[(i0 + r) + (size_t)l * n] * L[(j0 + c) + (size_t)l * n];
          /* crossing tiles read dead lanes above the diagonal; never stored */
          double src = (i0 + r >= j0 + c) ? *pa(s, i0 + r, j0 + c) : 0.0;
          t[r][c] = src - acc;
        }
      if (!diag) {
        for (int c = 0; c < na; ++c) {
          for (int l = 0; l < c; ++l) {
            double f = L[(j0 + c) + (size_t)(j0 + l) * n];
            for (int r = 0; r < ma; ++r) t[r][c] -= t[r][l] * f;
          }
          double inv = 1.0 / L[(j0 + c) + (size_t)(j0 + c) * n];
          for (int r = 0; r < ma; ++r) t[r][c] *= inv;
        }
        for (int r = 0; r < ma; ++r)
          for (int c = 0; c < na; ++c) {
            *pa(s, i0 + r, j0 + c) = t[r][c];
            L[(i0 + r) + (size_t)(j0 + c) * n] = t[r][c];
          }
      } else {
        int fail = 0;
        for (int c = 0; c < na && !fail; ++c) {
          int pr = d + c;
          double piv = t[pr][c];
          if (piv <= 0.0) { fail = c + 1; break; }
          double sq = sqrt(piv);
          t[pr][c] = sq;
          double inv = 1.0 / sq;
          for (int r = pr + 1; r < ma; ++r) t[r][c] *= inv;
          for (int c2 = c + 1; c2 < na; ++c2) {
            double f = t[d + c2][c];
            for (int r = d + c2; r < ma; ++r) t[r][c2] -= t[r][c] * f;
          }
        }
        if (fail) { info = j0 + fail; break; }
        for (int r = 0; r < ma; ++r)
          for (int c = 0; c < na; ++c) {
            if (r - c >= d) *pa(s, i0 + r, j0 + c) = t[r][c];
            L[(i0 + r) + (size_t)(j0 + c) * n] = (r - c >= d) ? t[r][c] : 0.0;
          }
      }
    }
  }
  free(L);
  return info;
}

int orc_dpotrf(char uplo, int n, double* a, int lda) {
  int lo = p_uplo(uplo);
  if (lo < 0) return -1;
  if (n < 0) return -2;
  if (lda < imax(1, n)) return -4;
  if (n == 0) return 0;
  pot_ctx s = {a, lda, !lo};
  return potrf_lower_sched(&s, n);
}

/* ----------------------------------------------------------------- dgetrf */
/* blas.hpp:204-215 -> factor.hpp:105-230: right-looking, NR-wide blocks.
 * Pivot: strict '>' over |v| from the diagonal down (ties -> lowest row);
 * zero pivot: no swap, no scale, first one recorded, continue; rank-1 skips
 * zero multipliers; swaps outside the panel in pivot order; U12 by the
 * unit-lower solve (ascending, unfused); trailing update
 * c <- (-1 * sum_l L21(i,l) U12(l,q)) + 1 * c  with the sum l-ascending. */
int orc_dgetrf(int m, int n, double* a, int lda, int* ipiv) {
  if (m < 0) return -1;
  if (n < 0) return -2;
  if (lda < imax(1, m)) return -4;
  int minmn = imin(m, n);
  if (minmn == 0) return 0;
  int first_zero = 0;
  for (int j0 = 0; j0 < minmn; j0 += NR) {
    int jb = imin(NR, minmn - j0);
    for (int c = 0; c < jb; ++c) {
      int col = j0 + c;
      int piv = col;
      double best = fabs(CM(a, lda, col, col));
      for (int i = col + 1; i < m; ++i) {
        double v = fabs(CM(a, lda, i, col));
        if (v > best) { best = v; piv = i; }
      }
      ipiv[col] = piv + 1;
      if (CM(a, lda, piv, col) != 0.0) {
        if (piv != col)
          for (int l = j0; l < j0 + jb; ++l) {
            double x = CM(a, lda, col, l);
            CM(a, lda, col, l) = CM(a, lda, piv, l);
            CM(a, lda, piv, l) = x;
          }
        double inv = 1.0 / CM(a, lda, col, col);
        for (int i = col + 1; i < m; ++i) CM(a, lda, i, col) *= inv;
      } else if (first_zero == 0) {
        first_zero = col + 1;
      }
      for (int i = col + 1; i < m; ++i) {
        double f = CM(a, lda, i, col);
        if (f != 0.0)
          for (int c2 = c + 1; c2 < jb; ++c2) CM(a, lda, i, j0 + c2) -= f * CM(a, lda, col, j0 + c2);
      }
    }
    for (int c = 0; c < jb; ++c) {
      int p = ipiv[j0 + c] - 1, row = j0 + c;
      if (p == row) continue;
      for (int l = 0; l < n; ++l) {
        if (l >= j0 && l < j0 + jb) continue;
        double x = CM(a, lda, row, l);
        CM(a, lda, row, l) = CM(a, lda, p, l);
        CM(a, lda, p, l) = x;
      }
    }
    int nw = n - j0 - jb;
    if (nw == 0) continue;
    for (int q = j0 + jb; q < n; ++q) { /* U12 = L11^{-1} A12, per column */
      double u[NR];
      for (int c = 0; c < jb; ++c) u[c] = -1.0 * 0.0 + 1.0 * CM(a, lda, j0 + c, q);
      for (int c = 0; c < jb; ++c)
        for (int l = 0; l < c; ++l) u[c] -= u[l] * CM(a, lda, j0 + c, j0 + l);
      for (int c = 0; c < jb; ++c) CM(a, lda, j0 + c, q) = u[c];
    }
    for (int q = j0 + jb; q < n; ++q)
      for (int i = j0 + jb; i < m; ++i) {
        double t = 0.0;
        for (int l = 0; l < jb; ++l) t += CM(a, lda, i, j0 + l) * CM(a, lda, j0 + l, q);
        CM(a, lda, i, q) = -1.0 * t + 1.0 * CM(a, lda, i, q);
      }
  }
  return first_zero;
}

/* --------------------------------------------------------- panel routines */
static int panel_ok(orc_dmat r, int m, int n) { /* level3.hpp:327-333 */
  return r.data != NULL && r.ps == PS && r.m == m && r.n == n;
}

/* level3.hpp:360-403 (+ scale_tiles_nd 342-353). */
int orc_gemm_nd(char transa, char transb, int m, int n, int k, double alpha, orc_dmat a, orc_dmat b,
                double beta, orc_dmat c, orc_dmat d) {
  if (p_trans(transa) != 0) return -1000;
  int tb = p_trans(transb);
  if (m < 0) return -4;
  if (n < 0) return -5;
  if (k < 0) return -6;
  if (!panel_ok(a, m, k)) return -8;
  if (!panel_ok(b, tb ? n : k, tb ? k : n)) return -9;
  if (!panel_ok(c, m, n)) return -11;
  if (!panel_ok(d, m, n)) return -12;
  if (m == 0 || n == 0) return 0;
  int scale_only = alpha == 0.0 || k == 0;
  /* c may alias d exactly: each element reads its own c before writing. */
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) {
      double t = 0.0;
      if (!scale_only)
        for (int l = 0; l < k; ++l) t += PM(a, i, l) * (tb ? PM(b, j, l) : PM(b, l, j));
      PM(d, i, j) = scale_ab(scale_only ? 0.0 : alpha, beta, t, &PM(c, i, j));
    }
  return 0;
}

/* level3.hpp:407-441: lower triangle only, strictly-upper d untouched. */
int orc_syrk_nd(int n, int k, double alpha, orc_dmat a, double beta, orc_dmat c, orc_dmat d) {
  if (n < 0) return -2;
  if (k < 0) return -3;
  if (!panel_ok(a, n, k)) return -5;
  if (!panel_ok(c, n, n)) return -7;
  if (!panel_ok(d, n, n)) return -8;
  if (n == 0) return 0;
  int scale_only = alpha == 0.0 || k == 0;
  for (int j = 0; j < n; ++j)
    for (int i = j; i < n; ++i) {
      double t = 0.0;
      if (!scale_only)
        for (int l = 0; l < k; ++l) t += PM(a, i, l) * PM(a, j, l);
      PM(d, i, j) = scale_ab(scale_only ? 0.0 : alpha, beta, t, &PM(c, i, j));
    }
  return 0;
}

/* level3.hpp:484-526 + kernel_trsm_right_ppp micro_kernel.hpp:549-564:
 * X * A^T = alpha * B, A lower non-unit; solved columns read back from d. */
int orc_trsm_rltn_nd(int m, int n, double alpha, orc_dmat a, orc_dmat b, orc_dmat d) {
  if (m < 0) return -2;
  if (n < 0) return -3;
  if (!panel_ok(a, n, n)) return -5;
  if (!panel_ok(b, m, n)) return -6;
  if (!panel_ok(d, m, n)) return -7;
  if (m == 0 || n == 0) return 0;
  for (int i = 0; i < n; ++i)
    if (PM(a, i, i) == 0.0) return i + 1;
  if (alpha == 0.0) {
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < m; ++i) PM(d, i, j) = 0.0 * 0.0;
    return 0;
  }
  double t[NR];
  for (int r = 0; r < m; ++r)
    for (int j0 = 0; j0 < n; j0 += NR) {
      int na = imin(NR, n - j0);
      for (int c = 0; c < na; ++c) {
        double acc = 0.0;
        for (int l = 0; l < j0; ++l) acc += PM(d, r, l) * PM(a, j0 + c, l);
        t[c] = -1.0 * acc + alpha * PM(b, r, j0 + c);
      }
      for (int c = 0; c < na; ++c) {
        for (int l = 0; l < c; ++l) t[c] -= t[l] * PM(a, j0 + c, j0 + l);
        t[c] *= 1.0 / PM(a, j0 + c, j0 + c);
      }
      for (int c = 0; c < na; ++c) PM(d, r, j0 + c) = t[c];
    }
  return 0;
}

/* level3.hpp:446-479 + kernel_trmm_right_p micro_kernel.hpp:588-601:
 * d <- alpha * b * a, a lower non-unit, untransposed (effectively lower):
 * per NR-column tile, the rectangular part l in [j0+na, n) (inner_gemm_nn_pp,
 * l ascending), then the edge l in [j0+c, j0+na), then t * alpha.  b may
 * alias d: each tile reads columns at or right of its own and the sweep
 * stores left to right, so rows are staged before they are overwritten. */
int orc_trmm_rlnn_nd(int m, int n, double alpha, orc_dmat a, orc_dmat b, orc_dmat d) {
  if (m < 0) return -2;
  if (n < 0) return -3;
  if (!panel_ok(a, n, n)) return -5;
  if (!panel_ok(b, m, n)) return -6;
  if (!panel_ok(d, m, n)) return -7;
  if (m == 0 || n == 0) return 0;
  if (alpha == 0.0) {
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < m; ++i) PM(d, i, j) = 0.0 * 0.0;
    return 0;
  }
  double* xrow = (double*)malloc(sizeof(double) * (size_t)n);
  double t[NR];
  for (int r = 0; r < m; ++r) {
    for (int l = 0; l < n; ++l) xrow[l] = PM(b, r, l);
    for (int j0 = 0; j0 < n; j0 += NR) {
      int na = imin(NR, n - j0);
      for (int c = 0; c < na; ++c) {
        double acc = 0.0;
        for (int l = j0 + na; l < n; ++l) acc += xrow[l] * PM(a, l, j0 + c);
        for (int l = c; l < na; ++l) acc += xrow[j0 + l] * PM(a, j0 + l, j0 + c);
        t[c] = acc * alpha;
      }
      for (int c = 0; c < na; ++c) PM(d, r, j0 + c) = t[c];
    }
  }
  free(xrow);
  return 0;
}

/* level3.hpp:533-575 + kernel_syrk_potrf_sub/_diag micro_kernel.hpp:640-673:
 * lower d <- chol(c + a b^T), left-looking; tile value before the edge is
 * (c(i,j) - sum_{l<j0} D(i,l) D(j,l)) + a(i,0) b(j,0) + ... (l ascending);
 * diagonal tiles are stored LowerZero, sub tiles Full. */
int orc_syrk_potrf_nd(int n, int k, orc_dmat a, orc_dmat b, orc_dmat c, orc_dmat d) {
  if (n < 0) return -2;
  if (k < 0) return -3;
  if (!panel_ok(a, n, k)) return -4;
  if (!panel_ok(b, n, k)) return -5;
  if (!panel_ok(c, n, n)) return -6;
  if (!panel_ok(d, n, n)) return -7;
  if (n == 0) return 0;
  double t[MR][NR];
  for (int i0 = 0; i0 < n; i0 += MR) {
    int ma = imin(MR, n - i0);
    for (int j0 = 0; j0 < i0 + ma; j0 += NR) {
      int na = imin(NR, n - j0);
      int diag = j0 + na > i0, dd = j0 - i0;
      for (int r = 0; r < ma; ++r)
        for (int q = 0; q < na; ++q) {
          int i = i0 + r, j = j0 + q;
          double acc = 0.0;
          for (int l = 0; l < j0; ++l) acc += PM(d, i, l) * PM(d, j, l);
          double v = PM(c, i, j) - acc;
          for (int l = 0; l < k; ++l) v += PM(a, i, l) * PM(b, j, l);
          t[r][q] = v;
        }
      if (!diag) {
        for (int q = 0; q < na; ++q) {
          for (int l = 0; l < q; ++l) {
            double f = PM(d, j0 + q, j0 + l);
            for (int r = 0; r < ma; ++r) t[r][q] -= t[r][l] * f;
          }
          double inv = 1.0 / PM(d, j0 + q, j0 + q);
          for (int r = 0; r < ma; ++r) t[r][q] *= inv;
        }
        for (int r = 0; r < ma; ++r)
          for (int q = 0; q < na; ++q) PM(d, i0 + r, j0 + q) = t[r][q];
      } else {
        for (int q = 0; q < na; ++q) {
          int pr = dd + q;
          double piv = t[pr][q];
          if (piv <= 0.0) return j0 + q + 1;
          double sq = sqrt(piv);
          t[pr][q] = sq;
          double inv = 1.0 / sq;
          for (int r = pr + 1; r < ma; ++r) t[r][q] *= inv;
          for (int q2 = q + 1; q2 < na; ++q2) {
            double f = t[dd + q2][q];
            for (int r = dd + q2; r < ma; ++r) t[r][q2] -= t[r][q] * f;
          }
        }
        for (int r = 0; r < ma; ++r)
          for (int q = 0; q < na; ++q) PM(d, i0 + r, j0 + q) = (r - q >= dd) ? t[r][q] : 0.0;
      }
    }
  }
  return 0;
}

/* ----------------------------------------------------------- batch loops */
typedef struct { long long lo, hi; void* arg; void (*fn)(long long, void*); } slice_t;
static void* run_slice(void* p) {
  slice_t* s = (slice_t*)p;
  for (long long i = s->lo; i < s->hi; ++i) s->fn(i, s->arg);
  return NULL;
}
static void par_for(long long batch, int threads, void (*fn)(long long, void*), void* arg) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  slice_t sl[256];
  long long per = (batch + threads - 1) / threads;
  int used = 0;
  for (int t = 0; t < threads; ++t) {
    long long lo = t * per, hi = lo + per < batch ? lo + per : batch;
    if (lo >= hi) break;
    sl[t].lo = lo; sl[t].hi = hi; sl[t].arg = arg; sl[t].fn = fn;
    pthread_create(&th[t], NULL, run_slice, &sl[t]);
    ++used;
  }
  for (int t = 0; t < used; ++t) pthread_join(th[t], NULL);
}

typedef struct {
  char ta, tb; int m, n, k; double alpha, beta;
  const double *a, *b; double* c; int lda, ldb, ldc; long long sa, sb, sc;
} gemm_args;
static void gemm_one(long long p, void* v) {
  gemm_args* g = (gemm_args*)v;
  orc_dgemm(g->ta, g->tb, g->m, g->n, g->k, g->alpha, g->a + p * g->sa, g->lda, g->b + p * g->sb,
            g->ldb, g->beta, g->c + p * g->sc, g->ldc);
}
void orc_dgemm_batch(char ta, char tb, int m, int n, int k, double alpha, const double* a, int lda,
                     long long sa, const double* b, int ldb, long long sb, double beta, double* c,
                     int ldc, long long sc, long long batch, int threads) {
  gemm_args g = {ta, tb, m, n, k, alpha, beta, a, b, c, lda, ldb, ldc, sa, sb, sc};
  par_for(batch, threads, gemm_one, &g);
}

typedef struct { char uplo; int m, n, lda; double* a; long long sa; int* ipiv; long long sp; int* info; } fac_args;
static void potrf_one(long long p, void* v) {
  fac_args* f = (fac_args*)v;
  f->info[p] = orc_dpotrf(f->uplo, f->n, f->a + p * f->sa, f->lda);
}
void orc_dpotrf_batch(char uplo, int n, double* a, int lda, long long sa, int* info,
                      long long batch, int threads) {
  fac_args f = {uplo, n, n, lda, a, sa, NULL, 0, info};
  par_for(batch, threads, potrf_one, &f);
}
static void getrf_one(long long p, void* v) {
  fac_args* f = (fac_args*)v;
  f->info[p] = orc_dgetrf(f->m, f->n, f->a + p * f->sa, f->lda, f->ipiv + p * f->sp);
}
void orc_dgetrf_batch(int m, int n, double* a, int lda, long long sa, int* ipiv, long long sipiv,
                      int* info, long long batch, int threads) {
  fac_args f = {'l', m, n, lda, a, sa, ipiv, sipiv, info};
  par_for(batch, threads, getrf_one, &f);
}

typedef struct {
  char ta, tb; int m, n, k; double alpha, beta;
  orc_dmat a, b, c, d; long long sa, sb, sc, sd;
} gemm_nd_args;
static void gemm_nd_one(long long p, void* v) {
  gemm_nd_args* g = (gemm_nd_args*)v;
  orc_dmat a = g->a, b = g->b, c = g->c, d = g->d;
  a.data += p * g->sa; b.data += p * g->sb; c.data += p * g->sc; d.data += p * g->sd;
  orc_gemm_nd(g->ta, g->tb, g->m, g->n, g->k, g->alpha, a, b, g->beta, c, d);
}
void orc_gemm_nd_batch(char ta, char tb, int m, int n, int k, double alpha, orc_dmat a, long long sa,
                       orc_dmat b, long long sb, double beta, orc_dmat c, long long sc, orc_dmat d,
                       long long sd, long long batch, int threads) {
  gemm_nd_args g = {ta, tb, m, n, k, alpha, beta, a, b, c, d, sa, sb, sc, sd};
  par_for(batch, threads, gemm_nd_one, &g);
}

/* Config-5 chain per problem (the reference's own
 * calls, as ref_shim.cpp's ref_chain_*_batch):
 *   cm: dsyrk('l','n') C += A A^T; dpotrf('l') C; dtrsm('r','l','t','n') X L^T = B
 *   pm: syrk_potrf_nd(n, n, A, A, C, C); trsm_rltn_nd(n, n, 1, C, B, B) */
typedef struct { const int* nv; const long long* off; double *A, *C, *B; int* info; int pm; } chain_args;
static orc_dmat pmat(double* p, int n) { orc_dmat d = {p, PS, n, n, (n + PS - 1) / PS * PS, (n + PS - 1) / PS * PS}; return d; }
static void chain_one(long long p, void* v) {
  chain_args* c = (chain_args*)v;
  int n = c->nv[p];
  double *a = c->A + c->off[p], *cc = c->C + c->off[p], *b = c->B + c->off[p];
  int inf;
  if (!c->pm) {
    orc_dsyrk('l', 'n', n, n, 1.0, a, n, 1.0, cc, n);
    inf = orc_dpotrf('l', n, cc, n);
    if (inf == 0) inf = orc_dtrsm('r', 'l', 't', 'n', n, n, 1.0, cc, n, b, n);
  } else {
    orc_dmat A = pmat(a, n), C = pmat(cc, n), B = pmat(b, n);
    inf = orc_syrk_potrf_nd(n, n, A, A, C, C);
    if (inf == 0) inf = orc_trsm_rltn_nd(n, n, 1.0, C, B, B);
  }
  c->info[p] = inf;
}
void orc_chain_batch(int pm, const int* nvec, const long long* off, double* A, double* C, double* B,
                     int* info, long long batch, int threads) {
  chain_args c = {nvec, off, A, C, B, info, pm};
  par_for(batch, threads, chain_one, &c);
}
