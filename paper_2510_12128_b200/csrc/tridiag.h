// tridiag.h — symmetric tridiagonal eigen-solver used by the SLQ log-det (row A6) and the
// Lanczos lambda_0 solve (row A1/A2).  Host+device so tests can call it on the CPU.
//
// tql_first(): implicit-shift QL iteration (Wilkinson shift) on a symmetric tridiagonal T
// (diag d[0..k-1], off-diagonal e[0..k-2] coupling i and i+1).  On return d holds the
// eigenvalues (unordered) and z the FIRST component of each normalised eigenvector — the
// only part of the eigenvectors Gauss quadrature needs (tau_l in SURVEY §8(a) row A6).
// Each Givens rotation G acting on rows (i, i+1) of the eigenvector matrix only needs to
// be applied to row 0, so the cost is O(k^2) instead of O(k^3).
// Attribution: this is the textbook implicit-shift QL algorithm for symmetric tridiagonal
// matrices (EISPACK tql1/tql2, Bowdler, Martin, Reinsch & Wilkinson 1968; the same iteration as
// "tqli" in Numerical Recipes), restated here with the eigenvector update reduced to row 0.
#pragma once
#include <cmath>

#if defined(__CUDACC__)
#define NUGPR_HD __host__ __device__
#else
#define NUGPR_HD
#endif

namespace nugpr {

NUGPR_HD inline double hypot_safe(double a, double b) {
  double aa = fabs(a), bb = fabs(b);
  if (aa > bb) { double r = bb / aa; return aa * sqrt(1.0 + r * r); }
  if (bb == 0.0) return 0.0;
  double r = aa / bb;
  return bb * sqrt(1.0 + r * r);
}

// Returns 0 on success, -1 if an eigenvalue failed to converge in 60 sweeps.
// e must have room for k entries (e[k-1] is used as scratch and set to 0).
NUGPR_HD inline int tql_first(int k, double* d, double* e, double* z) {
  for (int i = 0; i < k; ++i) z[i] = (i == 0) ? 1.0 : 0.0;
  if (k <= 0) return 0;
  e[k - 1] = 0.0;
  const double eps = 2.220446049250313e-16;
  for (int l = 0; l < k; ++l) {
    int iter = 0;
    int m;
    do {
      for (m = l; m < k - 1; ++m) {
        double dd = fabs(d[m]) + fabs(d[m + 1]);
        if (fabs(e[m]) <= eps * dd) break;
      }
      if (m != l) {
        if (iter++ == 60) return -1;
        // Wilkinson-type shift from the leading 2x2 of the unreduced part.
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot_safe(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? fabs(r) : -fabs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool deflated = false;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          double b = c * e[i];
          r = hypot_safe(f, g);
          e[i + 1] = r;
          if (r == 0.0) {          // underflow: split here and restart
            d[i + 1] -= p;
            e[m] = 0.0;
            deflated = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          // rotate the first row of the eigenvector matrix
          double zf = z[i + 1];
          z[i + 1] = s * z[i] + c * zf;
          z[i] = c * z[i] - s * zf;
        }
        if (deflated) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  return 0;
}

// Number of eigenvalues of T (diag a, off b) strictly less than x (Sturm count via LDL^T).
NUGPR_HD inline int sturm_count(int k, const double* a, const double* b, double x) {
  int cnt = 0;
  double q = a[0] - x;
  if (q < 0.0) ++cnt;
  for (int i = 1; i < k; ++i) {
    double qq = (q == 0.0) ? 1e-300 : q;
    q = a[i] - x - b[i - 1] * b[i - 1] / qq;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

// Smallest eigenvalue of T by bisection to (near) full precision.
NUGPR_HD inline double tridiag_min_eig(int k, const double* a, const double* b) {
  double lo = a[0], hi = a[0];
  for (int i = 0; i < k; ++i) {
    double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i < k - 1 ? fabs(b[i]) : 0.0);
    lo = fmin(lo, a[i] - r);
    hi = fmax(hi, a[i] + r);
  }
  for (int it = 0; it < 200; ++it) {
    double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (sturm_count(k, a, b, mid) >= 1) hi = mid; else lo = mid;
  }
  return 0.5 * (lo + hi);
}

// Eigenvector of T for eigenvalue th by two steps of inverse iteration (Thomas algorithm
// on T - th I with tiny-pivot guard).  Writes the normalised vector into s (length k);
// w is scratch of length 2k.
NUGPR_HD inline void tridiag_eigvec(int k, const double* a, const double* b, double th,
                                    double* s, double* w) {
  double scale = 0.0;
  for (int i = 0; i < k; ++i) scale = fmax(scale, fabs(a[i]) + (i < k - 1 ? fabs(b[i]) : 0.0));
  double tiny = 1e-300 + 1e-15 * scale;
  for (int i = 0; i < k; ++i) s[i] = 1.0;
  double* cp = w;       // modified super-diagonal
  double* dp = w + k;   // modified rhs
  for (int step = 0; step < 3; ++step) {
    double den = a[0] - th;
    if (fabs(den) < tiny) den = (den >= 0 ? tiny : -tiny);
    cp[0] = (k > 1 ? b[0] : 0.0) / den;
    dp[0] = s[0] / den;
    for (int i = 1; i < k; ++i) {
      den = (a[i] - th) - b[i - 1] * cp[i - 1];
      if (fabs(den) < tiny) den = (den >= 0 ? tiny : -tiny);
      cp[i] = (i < k - 1 ? b[i] : 0.0) / den;
      dp[i] = (s[i] - b[i - 1] * dp[i - 1]) / den;
    }
    s[k - 1] = dp[k - 1];
    for (int i = k - 2; i >= 0; --i) s[i] = dp[i] - cp[i] * s[i + 1];
    double nrm = 0.0;
    for (int i = 0; i < k; ++i) nrm += s[i] * s[i];
    nrm = sqrt(nrm);
    if (!(nrm > 0.0)) { for (int i = 0; i < k; ++i) s[i] = (i == 0); return; }
    for (int i = 0; i < k; ++i) s[i] /= nrm;
  }
}

}  // namespace nugpr
