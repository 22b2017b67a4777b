/*
 * oracle/direct.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct direct O(m^2)/O(m^3) convolution sums that
 * define what the implicitly dealiased convolutions of Bowman & Roberts
 * (arXiv 1008.1366, /root/reference/PAPER.md = "P:") must compute.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  It shares no code with the CUDA
 * path (paper_1008_1366_b200/csrc) and includes none of its headers.
 *
 * Definitions:
 *   D1 cconv1d  h_k = sum_{p=0}^{k} f_p g_{k-p},          k = 0..m-1
 *   D2 hconv1d  h_k = sum_{p=k-m+1}^{m-1} f_p g_{k-p},    k = 0..m-1
 *               with f_{-p} := conj(f_p) and f_0 := Re f_0 (AMB-7)
 *   D3 tconv1d  t_k = sum_{p+q+r=k, |p|,|q|,|r|<=m-1} f_p g_q h_r
 *   D4 cconv2d, D6 cconv3d: the 2D/3D analogues of D1
 *   D5 hconv2d, D7 hconv3d: centered x (and y), Hermitian last axis
 *
 * Accuracy: every product is split exactly with TwoProd (fma) and all terms
 * are accumulated with Neumaier compensated summation (AMB-20).
 * Complex numbers are interleaved (re, im) doubles.  Compile with
 * -ffp-contract=off so that the error-free transforms stay error free.
 *
 * Every entry point returns 0 on success, -1 if the number of multiply-adds
 * would exceed the work cap (orc_set_work_cap, default 2^36), -2 on bad args.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double s, c; } acc_t;          /* Neumaier accumulator */

static inline void acc_add(acc_t *a, double x) {
  double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
  else                       a->c += (x - t) + a->s;
  a->s = t;
}
static inline double acc_val(const acc_t *a) { return a->s + a->c; }

/* exact product x*y = p + e, added to the accumulator */
static inline void acc_addprod(acc_t *a, double x, double y) {
  double p = x * y;
  double e = fma(x, y, -p);
  acc_add(a, p);
  acc_add(a, e);
}

typedef struct { acc_t re, im; } cacc_t;

/* (ar + i ai)(br + i bi) = (ar br - ai bi) + i (ar bi + ai br) */
static inline void cacc_addmul(cacc_t *a, double ar, double ai, double br, double bi) {
  acc_addprod(&a->re, ar, br);
  acc_addprod(&a->re, -ai, bi);
  acc_addprod(&a->im, ar, bi);
  acc_addprod(&a->im, ai, br);
}

static double g_work_cap = 68719476736.0; /* 2^36 complex MACs */
void orc_set_work_cap(double macs) { g_work_cap = macs; }
static int over_cap(double macs) { return macs > g_work_cap; }

/* ------------------------------------------------------------------ D1 -- */
int orc_cconv1d(const double *f, const double *g, double *h, int64_t m, int64_t batch) {
  if (m < 1 || batch < 1) return -2;
  if (over_cap(0.5 * (double)m * (double)(m + 1) * (double)batch)) return -1;
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t k = 0; k < m; ++k) {
      const double *F = f + 2 * b * m, *G = g + 2 * b * m;
      cacc_t a = {{0, 0}, {0, 0}};
      for (int64_t p = 0; p <= k; ++p)
        cacc_addmul(&a, F[2 * p], F[2 * p + 1], G[2 * (k - p)], G[2 * (k - p) + 1]);
      h[2 * (b * m + k)] = acc_val(&a.re);
      h[2 * (b * m + k) + 1] = acc_val(&a.im);
    }
  return 0;
}

/* centered Hermitian extension of a length-m half spectrum:
 * E[p + (m-1)] = U_p for p = -(m-1)..(m-1), U_{-p} = conj(U_p), U_0 := Re U_0 */
static void hermitian_extend1d(const double *U, double *E, int64_t m) {
  for (int64_t p = 0; p < m; ++p) {
    E[2 * (m - 1 + p)] = U[2 * p];
    E[2 * (m - 1 + p) + 1] = U[2 * p + 1];
    E[2 * (m - 1 - p)] = U[2 * p];
    E[2 * (m - 1 - p) + 1] = -U[2 * p + 1];
  }
  E[2 * (m - 1) + 1] = 0.0;
}

/* ------------------------------------------------------------------ D2 -- */
int orc_hconv1d(const double *f, const double *g, double *h, int64_t m, int64_t batch) {
  if (m < 1 || batch < 1) return -2;
  if (over_cap((double)m * (double)(2 * m) * (double)batch)) return -1;
  int64_t n = 2 * m - 1;
  double *E = (double *)malloc(sizeof(double) * 4 * n * batch);
  if (!E) return -2;
  for (int64_t b = 0; b < batch; ++b) {
    hermitian_extend1d(f + 2 * b * m, E + 4 * b * n, m);
    hermitian_extend1d(g + 2 * b * m, E + 4 * b * n + 2 * n, m);
  }
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t k = 0; k < m; ++k) {
      const double *F = E + 4 * b * n, *G = E + 4 * b * n + 2 * n;
      cacc_t a = {{0, 0}, {0, 0}};
      for (int64_t p = k - m + 1; p <= m - 1; ++p) {
        int64_t q = k - p; /* |q| <= m-1 holds for p in this range */
        cacc_addmul(&a, F[2 * (p + m - 1)], F[2 * (p + m - 1) + 1],
                    G[2 * (q + m - 1)], G[2 * (q + m - 1) + 1]);
      }
      h[2 * (b * m + k)] = acc_val(&a.re);
      h[2 * (b * m + k) + 1] = acc_val(&a.im);
    }
  free(E);
  return 0;
}

/* ------------------------------------------------------------------ D3 -- */
/* Two-stage exact form: e_s = sum_p f_p g_{s-p} (|p|,|s-p| <= m-1), kept as a
 * double-double (hi + lo); then t_k = sum_s e_s h_{k-s} over |k-s| <= m-1. */
int orc_tconv1d(const double *f, const double *g, const double *hh, double *t, int64_t m, int64_t batch) {
  if (m < 1 || batch < 1) return -2;
  if (over_cap(((double)(4 * m) * (double)(2 * m) + (double)m * (double)(2 * m)) * (double)batch)) return -1;
  int64_t n = 2 * m - 1, ne = 4 * m - 3;
  double *E = (double *)malloc(sizeof(double) * 2 * n * 3 * batch);
  double *ehi = (double *)malloc(sizeof(double) * 2 * ne * batch);
  double *elo = (double *)malloc(sizeof(double) * 2 * ne * batch);
  if (!E || !ehi || !elo) { free(E); free(ehi); free(elo); return -2; }
  for (int64_t b = 0; b < batch; ++b) {
    hermitian_extend1d(f + 2 * b * m, E + 2 * n * (3 * b + 0), m);
    hermitian_extend1d(g + 2 * b * m, E + 2 * n * (3 * b + 1), m);
    hermitian_extend1d(hh + 2 * b * m, E + 2 * n * (3 * b + 2), m);
  }
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t si = 0; si < ne; ++si) {
      int64_t s = si - (2 * m - 2);
      const double *F = E + 2 * n * (3 * b), *G = E + 2 * n * (3 * b + 1);
      int64_t plo = s - (m - 1) > -(m - 1) ? s - (m - 1) : -(m - 1);
      int64_t phi = s + (m - 1) < (m - 1) ? s + (m - 1) : (m - 1);
      cacc_t a = {{0, 0}, {0, 0}};
      for (int64_t p = plo; p <= phi; ++p)
        cacc_addmul(&a, F[2 * (p + m - 1)], F[2 * (p + m - 1) + 1],
                    G[2 * (s - p + m - 1)], G[2 * (s - p + m - 1) + 1]);
      double hr = acc_val(&a.re), hi = acc_val(&a.im);
      ehi[2 * (b * ne + si)] = hr;
      ehi[2 * (b * ne + si) + 1] = hi;
      elo[2 * (b * ne + si)] = (a.re.s - hr) + a.re.c;
      elo[2 * (b * ne + si) + 1] = (a.im.s - hi) + a.im.c;
    }
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t k = 0; k < m; ++k) {
      const double *H = E + 2 * n * (3 * b + 2);
      cacc_t a = {{0, 0}, {0, 0}};
      for (int64_t s = k - (m - 1); s <= k + (m - 1); ++s) {
        if (s < -(2 * m - 2) || s > 2 * m - 2) continue;
        int64_t si = s + 2 * m - 2, r = k - s;
        double hr = H[2 * (r + m - 1)], hi = H[2 * (r + m - 1) + 1];
        cacc_addmul(&a, ehi[2 * (b * ne + si)], ehi[2 * (b * ne + si) + 1], hr, hi);
        cacc_addmul(&a, elo[2 * (b * ne + si)], elo[2 * (b * ne + si) + 1], hr, hi);
      }
      t[2 * (b * m + k)] = acc_val(&a.re);
      t[2 * (b * m + k) + 1] = acc_val(&a.im);
    }
  free(E); free(ehi); free(elo);
  return 0;
}

/* brute-force triple sum (small m only), the literal definition P:963-964.
 * Accumulated in x86 long double (64-bit mantissa): for m <= 32 the at most
 * (2m-1)^2 terms leave an error far below double rounding. */
int orc_tconv1d_brute(const double *f, const double *g, const double *hh, double *t, int64_t m) {
  if (m < 1) return -2;
  if (over_cap((double)m * (double)(2 * m) * (double)(2 * m))) return -1;
  int64_t n = 2 * m - 1;
  double *E = (double *)malloc(sizeof(double) * 6 * n);
  if (!E) return -2;
  hermitian_extend1d(f, E, m);
  hermitian_extend1d(g, E + 2 * n, m);
  hermitian_extend1d(hh, E + 4 * n, m);
  for (int64_t k = 0; k < m; ++k) {
    long double sr = 0.0L, si = 0.0L;
    for (int64_t p = -(m - 1); p <= m - 1; ++p)
      for (int64_t q = -(m - 1); q <= m - 1; ++q) {
        int64_t r = k - p - q;
        if (r < -(m - 1) || r > m - 1) continue;
        const double *F = E + 2 * (p + m - 1), *G = E + 2 * n + 2 * (q + m - 1), *H = E + 4 * n + 2 * (r + m - 1);
        long double ar = (long double)F[0] * G[0] - (long double)F[1] * G[1];
        long double ai = (long double)F[0] * G[1] + (long double)F[1] * G[0];
        sr += ar * H[0] - ai * H[1];
        si += ar * H[1] + ai * H[0];
      }
    t[2 * k] = (double)sr;
    t[2 * k + 1] = (double)si;
  }
  free(E);
  return 0;
}

/* ------------------------------------------------------------ D4 / D6 -- */
/* Complex d-dimensional (d = 2, 3) truncated linear convolution at a list of
 * output points.  Arrays are row-major (n0, n1, n2) with n2 = 1 for 2D.
 * out_idx holds nout linear indices i*(n1*n2) + j*n2 + l. */
int orc_cconv3d_at(const double *f, const double *g, int64_t n0, int64_t n1, int64_t n2,
                   const int64_t *out_idx, int64_t nout, double *out) {
  if (n0 < 1 || n1 < 1 || n2 < 1 || nout < 0) return -2;
  double per = (double)n0 * (double)n1 * (double)n2; /* upper bound per point */
  if (over_cap(per * (double)nout)) return -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t o = 0; o < nout; ++o) {
    int64_t lin = out_idx[o];
    int64_t i = lin / (n1 * n2), j = (lin / n2) % n1, l = lin % n2;
    cacc_t a = {{0, 0}, {0, 0}};
    for (int64_t p = 0; p <= i; ++p)
      for (int64_t q = 0; q <= j; ++q)
        for (int64_t r = 0; r <= l; ++r) {
          const double *F = f + 2 * ((p * n1 + q) * n2 + r);
          const double *G = g + 2 * (((i - p) * n1 + (j - q)) * n2 + (l - r));
          cacc_addmul(&a, F[0], F[1], G[0], G[1]);
        }
    out[2 * o] = acc_val(&a.re);
    out[2 * o + 1] = acc_val(&a.im);
  }
  return 0;
}

/* ------------------------------------------------------------ D5 / D7 -- */
/* Centered-Hermitian 3D (2D when my == 1 is passed as a centered length-1 axis):
 * storage A[i][j][l], i in [0, 2mx-1), j in [0, 2my-1), l in [0, mz),
 * A[i][j][l] = U_{i-(mx-1), j-(my-1), l}.  Extension U_{kx,ky,-kz} :=
 * conj(U_{-kx,-ky,kz}); the kz = 0 plane is projected
 * U_{kx,ky,0} := (U_{kx,ky,0} + conj(U_{-kx,-ky,0}))/2  (AMB-7).
 * The full centered array X[(2mx-1)][(2my-1)][(2mz-1)] is built first, then
 * h_{k} = sum_p X_p X'_{k-p} over the centered box, at the requested output
 * points (linear indices into the (2mx-1, 2my-1, mz) storage). */
static void hermitian_extend3d(const double *A, double *X, int64_t mx, int64_t my, int64_t mz) {
  int64_t nx = 2 * mx - 1, ny = 2 * my - 1, nz = 2 * mz - 1;
  for (int64_t i = 0; i < nx; ++i)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t l = 0; l < mz; ++l) {
        const double *a = A + 2 * ((i * ny + j) * mz + l);
        const double *b = A + 2 * (((nx - 1 - i) * ny + (ny - 1 - j)) * mz + l); /* mirror (-kx,-ky) */
        double *x = X + 2 * ((i * ny + j) * nz + (mz - 1 + l));
        double *xm = X + 2 * (((nx - 1 - i) * ny + (ny - 1 - j)) * nz + (mz - 1 - l));
        if (l == 0) {
          x[0] = 0.5 * (a[0] + b[0]);
          x[1] = 0.5 * (a[1] - b[1]);
        } else {
          x[0] = a[0];
          x[1] = a[1];
          xm[0] = a[0];
          xm[1] = -a[1];
        }
      }
}

int orc_hconv3d_at(const double *f, const double *g, int64_t mx, int64_t my, int64_t mz,
                   const int64_t *out_idx, int64_t nout, double *out) {
  if (mx < 1 || my < 1 || mz < 1 || nout < 0) return -2;
  int64_t nx = 2 * mx - 1, ny = 2 * my - 1, nz = 2 * mz - 1;
  if (over_cap((double)nx * (double)ny * (double)nz * (double)nout)) return -1;
  double *F = (double *)malloc(sizeof(double) * 2 * nx * ny * nz);
  double *G = (double *)malloc(sizeof(double) * 2 * nx * ny * nz);
  if (!F || !G) { free(F); free(G); return -2; }
  hermitian_extend3d(f, F, mx, my, mz);
  hermitian_extend3d(g, G, mx, my, mz);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t o = 0; o < nout; ++o) {
    int64_t lin = out_idx[o];
    int64_t i = lin / (ny * mz), j = (lin / mz) % ny, l = lin % mz;
    int64_t kx = i - (mx - 1), ky = j - (my - 1), kz = l;
    cacc_t a = {{0, 0}, {0, 0}};
    for (int64_t px = -(mx - 1); px <= mx - 1; ++px) {
      int64_t qx = kx - px;
      if (qx < -(mx - 1) || qx > mx - 1) continue;
      for (int64_t py = -(my - 1); py <= my - 1; ++py) {
        int64_t qy = ky - py;
        if (qy < -(my - 1) || qy > my - 1) continue;
        for (int64_t pz = -(mz - 1); pz <= mz - 1; ++pz) {
          int64_t qz = kz - pz;
          if (qz < -(mz - 1) || qz > mz - 1) continue;
          const double *x = F + 2 * (((px + mx - 1) * ny + (py + my - 1)) * nz + (pz + mz - 1));
          const double *y = G + 2 * (((qx + mx - 1) * ny + (qy + my - 1)) * nz + (qz + mz - 1));
          cacc_addmul(&a, x[0], x[1], y[0], y[1]);
        }
      }
    }
    out[2 * o] = acc_val(&a.re);
    out[2 * o + 1] = acc_val(&a.im);
  }
  free(F); free(G);
  return 0;
}

/* 2D centered Hermitian (D5): storage (2mx-1, my); it is the my-axis-Hermitian
 * special case of the above with a centered y axis of length 1 removed.
 * Extension U_{kx,-ky} := conj(U_{-kx,ky}); ky = 0 line projected. */
int orc_hconv2d_at(const double *f, const double *g, int64_t mx, int64_t my,
                   const int64_t *out_idx, int64_t nout, double *out) {
  /* (2mx-1, my) == (2mx-1, 2*1-1, my): reuse the 3D routine with my_c = 1 */
  return orc_hconv3d_at(f, g, mx, 1, my, out_idx, nout, out);
}

/* D7 at sampled outputs without materialising the extended array (for the
 * full-size config 5b, where the extension would take 17 GB): the mirror
 * U_{-p} = conj(U_p) and the kz = 0 projection are evaluated on the fly. */
static inline void herm_val(const double *A, int64_t mx, int64_t my, int64_t mz, int64_t px, int64_t py,
                            int64_t pz, double *re, double *im) {
  const int64_t ny = 2 * my - 1;
  if (pz > 0) {
    const double *a = A + 2 * (((px + mx - 1) * ny + (py + my - 1)) * mz + pz);
    *re = a[0]; *im = a[1];
  } else if (pz < 0) {
    const double *a = A + 2 * (((-px + mx - 1) * ny + (-py + my - 1)) * mz - pz);
    *re = a[0]; *im = -a[1];
  } else {
    const double *a = A + 2 * (((px + mx - 1) * ny + (py + my - 1)) * mz);
    const double *b = A + 2 * (((-px + mx - 1) * ny + (-py + my - 1)) * mz);
    *re = 0.5 * (a[0] + b[0]); *im = 0.5 * (a[1] - b[1]);
  }
}

int orc_hconv3d_at_mirror(const double *f, const double *g, int64_t mx, int64_t my, int64_t mz,
                          const int64_t *out_idx, int64_t nout, double *out) {
  if (mx < 1 || my < 1 || mz < 1 || nout < 0) return -2;
  int64_t ny = 2 * my - 1;
  if (over_cap((double)(2 * mx - 1) * (double)ny * (double)(2 * mz - 1) * (double)nout)) return -1;
  for (int64_t o = 0; o < nout; ++o) {
    int64_t lin = out_idx[o];
    int64_t i = lin / (ny * mz), j = (lin / mz) % ny, l = lin % mz;
    int64_t kx = i - (mx - 1), ky = j - (my - 1), kz = l;
    double sre = 0, sim = 0, cre = 0, cim = 0;
    /* parallel over px; per-thread compensated partial sums, combined exactly-ish below */
    int64_t nth = 2 * mx - 1;
    double *part = (double *)calloc((size_t)nth * 4, sizeof(double));
    if (!part) return -2;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t pxi = 0; pxi < nth; ++pxi) {
      int64_t px = pxi - (mx - 1), qx = kx - px;
      if (qx < -(mx - 1) || qx > mx - 1) continue;
      cacc_t a = {{0, 0}, {0, 0}};
      for (int64_t py = -(my - 1); py <= my - 1; ++py) {
        int64_t qy = ky - py;
        if (qy < -(my - 1) || qy > my - 1) continue;
        int64_t pz0 = kz - (mz - 1) > -(mz - 1) ? kz - (mz - 1) : -(mz - 1);
        for (int64_t pz = pz0; pz <= mz - 1; ++pz) {
          double xr, xi, yr, yi;
          herm_val(f, mx, my, mz, px, py, pz, &xr, &xi);
          herm_val(g, mx, my, mz, qx, qy, kz - pz, &yr, &yi);
          cacc_addmul(&a, xr, xi, yr, yi);
        }
      }
      part[4 * pxi] = a.re.s; part[4 * pxi + 1] = a.re.c;
      part[4 * pxi + 2] = a.im.s; part[4 * pxi + 3] = a.im.c;
    }
    acc_t R = {0, 0}, I = {0, 0};
    for (int64_t t = 0; t < nth; ++t) {
      acc_add(&R, part[4 * t]); acc_add(&R, part[4 * t + 1]);
      acc_add(&I, part[4 * t + 2]); acc_add(&I, part[4 * t + 3]);
    }
    free(part);
    (void)sre; (void)sim; (void)cre; (void)cim;
    out[2 * o] = acc_val(&R);
    out[2 * o + 1] = acc_val(&I);
  }
  return 0;
}

/* D6 at sampled outputs, parallel inside each point (for the 512^3 config). */
int orc_cconv3d_at_par(const double *f, const double *g, int64_t n0, int64_t n1, int64_t n2,
                       const int64_t *out_idx, int64_t nout, double *out) {
  if (n0 < 1 || n1 < 1 || n2 < 1 || nout < 0) return -2;
  if (over_cap((double)n0 * (double)n1 * (double)n2 * (double)nout)) return -1;
  for (int64_t o = 0; o < nout; ++o) {
    int64_t lin = out_idx[o];
    int64_t i = lin / (n1 * n2), j = (lin / n2) % n1, l = lin % n2;
    double *part = (double *)calloc((size_t)(i + 1) * 4, sizeof(double));
    if (!part) return -2;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t p = 0; p <= i; ++p) {
      cacc_t a = {{0, 0}, {0, 0}};
      for (int64_t q = 0; q <= j; ++q)
        for (int64_t r = 0; r <= l; ++r) {
          const double *F = f + 2 * ((p * n1 + q) * n2 + r);
          const double *G = g + 2 * (((i - p) * n1 + (j - q)) * n2 + (l - r));
          cacc_addmul(&a, F[0], F[1], G[0], G[1]);
        }
      part[4 * p] = a.re.s; part[4 * p + 1] = a.re.c; part[4 * p + 2] = a.im.s; part[4 * p + 3] = a.im.c;
    }
    acc_t R = {0, 0}, I = {0, 0};
    for (int64_t t = 0; t <= i; ++t) {
      acc_add(&R, part[4 * t]); acc_add(&R, part[4 * t + 1]);
      acc_add(&I, part[4 * t + 2]); acc_add(&I, part[4 * t + 3]);
    }
    free(part);
    out[2 * o] = acc_val(&R);
    out[2 * o + 1] = acc_val(&I);
  }
  return 0;
}

/* ------------------------------------------------ D7 sampled, line form -- */
/* D7 at sampled outputs of a large array (config 5b, O5): the same terms as
 * orc_hconv3d_at / orc_hconv3d_at_mirror, organised for speed without
 * changing what is summed.  For each output k and each (px, py) with
 * (qx, qy) = (kx - px, ky - py) in range, the z sum
 *   sum_{pz} U^f_{px,py,pz} U^g_{qx,qy,kz-pz},   |pz|, |kz-pz| <= mz-1,
 * with U_{.,.,-z} = conj U_{-px,-py,z} and the z = 0 entries projected
 * (AMB-7), is cut where pz or kz - pz changes sign into runs of stored
 * entries read in place (a = U^f_{px,py,.}, b = U^f_{-px,-py,.},
 * c = U^g_{qx,qy,.}, d = U^g_{-qx,-qy,.}):
 *   pz = -u < 0 (u = 1..mz-1-kz):  conj(b[u]) * c[kz+u]
 *   pz = 0:                         P(a,b)[0] * (kz > 0 ? c[kz] : P(c,d)[0])
 *   0 < pz < kz:                    a[pz] * c[kz-pz]
 *   pz = kz > 0:                    a[kz] * P(c,d)[0]
 *   kz < pz <= mz-1:                a[pz] * conj(d[pz-kz])
 * (P(a,b)[0] = (a[0] + conj b[0])/2).  Accumulation: Ogita-Rump-Oishi Dot2
 * (TwoProd + TwoSum: the result as if computed in twice the working
 * precision) in 8 independent lanes, combined with Neumaier summation
 * (AMB-20). */
typedef struct { double p[8], s[8]; } dot8_t;

#define DOT2_LANE(D, l, x, y)                                  \
  do {                                                         \
    double h_ = (x) * (y), r_ = fma((x), (y), -h_);            \
    double t_ = (D)->p[l] + h_, z_ = t_ - (D)->p[l];           \
    double q_ = ((D)->p[l] - (t_ - z_)) + (h_ - z_);           \
    (D)->p[l] = t_;                                            \
    (D)->s[l] += q_ + r_;                                      \
  } while (0)

static inline void cmac2(dot8_t *re, dot8_t *im, double xr, double xi, double yr, double yi) {
  DOT2_LANE(re, 0, xr, yr);
  DOT2_LANE(re, 0, -xi, yi);
  DOT2_LANE(im, 0, xr, yi);
  DOT2_LANE(im, 0, xi, yr);
}

/* sum_{j<n} (x_j^cx) (y_{SY j}^cy), x ascending, y ascending (SY = 1) or
 * descending (SY = -1); cx, cy = +1 (as stored) or -1 (conjugate) */
#define CDOT2_BODY(SY)                                                                   \
  double rp[8], rs[8], ip[8], is[8];                                                     \
  for (int l = 0; l < 8; ++l) { rp[l] = re->p[l]; rs[l] = re->s[l]; ip[l] = im->p[l]; is[l] = im->s[l]; } \
  int64_t j = 0;                                                                         \
  for (; j + 8 <= n; j += 8) {                                                           \
    _Pragma("omp simd")                                                                  \
    for (int l = 0; l < 8; ++l) {                                                        \
      const double xr = x[2 * (j + l)], xi = cx * x[2 * (j + l) + 1];                    \
      const double yr = y[2 * (SY) * (j + l)], yi = cy * y[2 * (SY) * (j + l) + 1];      \
      double h, r, t, z, q;                                                              \
      D2(rp[l], rs[l], xr, yr) D2(rp[l], rs[l], -xi, yi)                                 \
      D2(ip[l], is[l], xr, yi) D2(ip[l], is[l], xi, yr)                                  \
    }                                                                                    \
  }                                                                                      \
  for (int l = 0; l < 8; ++l) { re->p[l] = rp[l]; re->s[l] = rs[l]; im->p[l] = ip[l]; im->s[l] = is[l]; } \
  for (; j < n; ++j)                                                                     \
    cmac2(re, im, x[2 * j], cx * x[2 * j + 1], y[2 * (SY) * j], cy * y[2 * (SY) * j + 1]);
#define D2(P, S, a, b) h = (a) * (b); r = fma((a), (b), -h); t = P + h; z = t - P; q = (P - (t - z)) + (h - z); P = t; S += q + r;
static void cdot2_fwd(const double *restrict x, double cx, const double *restrict y, double cy, int64_t n,
                      dot8_t *re, dot8_t *im) {
  CDOT2_BODY(1)
}
static void cdot2_rev(const double *restrict x, double cx, const double *restrict y, double cy, int64_t n,
                      dot8_t *re, dot8_t *im) {
  CDOT2_BODY(-1)
}
#undef D2

/* the z sum above for one (px, py) pair and output kz, added to (re, im) */
static void zsum(const double *a, const double *b, const double *c, const double *d, int64_t mz, int64_t kz,
                 dot8_t *re, dot8_t *im) {
  const double a0r = 0.5 * (a[0] + b[0]), a0i = 0.5 * (a[1] - b[1]);   /* projected z = 0 */
  const double c0r = 0.5 * (c[0] + d[0]), c0i = 0.5 * (c[1] - d[1]);
  if (mz - 1 - kz > 0) cdot2_fwd(b + 2, -1.0, c + 2 * (kz + 1), 1.0, mz - 1 - kz, re, im);   /* pz < 0 */
  if (kz > 0) {
    cmac2(re, im, a0r, a0i, c[2 * kz], c[2 * kz + 1]);                                     /* pz = 0 */
    if (kz > 1) cdot2_rev(a + 2, 1.0, c + 2 * (kz - 1), 1.0, kz - 1, re, im);             /* 0 < pz < kz */
    cmac2(re, im, a[2 * kz], a[2 * kz + 1], c0r, c0i);                                     /* pz = kz */
  } else {
    cmac2(re, im, a0r, a0i, c0r, c0i);                                                      /* pz = kz = 0 */
  }
  if (mz - 1 - kz > 0) cdot2_fwd(a + 2 * (kz + 1), 1.0, d + 2, -1.0, mz - 1 - kz, re, im);   /* pz > kz */
}

/* D7 at the outputs (kx, ky, kz[t]), t < nkz, of one (kx, ky) line: the
 * x-y loop is shared by all kz (each pair of z lines is read once for all
 * of them -- the sampled config-5b check is memory-bound otherwise). */
int orc_hconv3d_at_zlist(const double *f, const double *g, int64_t mx, int64_t my, int64_t mz, int64_t kx,
                         int64_t ky, const int64_t *kz, int64_t nkz, double *out) {
  if (mx < 1 || my < 1 || mz < 1 || nkz < 0 || kx < -(mx - 1) || kx > mx - 1 || ky < -(my - 1) || ky > my - 1)
    return -2;
  for (int64_t t = 0; t < nkz; ++t)
    if (kz[t] < 0 || kz[t] > mz - 1) return -2;
  const int64_t ny = 2 * my - 1, nth = 2 * mx - 1;
  if (over_cap((double)nth * (double)ny * (double)(2 * mz - 1) * (double)nkz)) return -1;
  double *part = (double *)calloc((size_t)nth * nkz * 4, sizeof(double));
  if (!part) return -2;
#pragma omp parallel
  {
    dot8_t *re = (dot8_t *)malloc(sizeof(dot8_t) * (nkz ? nkz : 1));
    dot8_t *im = (dot8_t *)malloc(sizeof(dot8_t) * (nkz ? nkz : 1));
#pragma omp for schedule(dynamic, 1)
    for (int64_t pxi = 0; pxi < nth; ++pxi) {
      const int64_t px = pxi - (mx - 1), qx = kx - px;
      if (qx < -(mx - 1) || qx > mx - 1) continue;
      memset(re, 0, sizeof(dot8_t) * nkz);
      memset(im, 0, sizeof(dot8_t) * nkz);
      for (int64_t py = -(my - 1); py <= my - 1; ++py) {
        const int64_t qy = ky - py;
        if (qy < -(my - 1) || qy > my - 1) continue;
        const double *a = f + 2 * (((px + mx - 1) * ny + (py + my - 1)) * mz);
        const double *b = f + 2 * (((-px + mx - 1) * ny + (-py + my - 1)) * mz);
        const double *c = g + 2 * (((qx + mx - 1) * ny + (qy + my - 1)) * mz);
        const double *d = g + 2 * (((-qx + mx - 1) * ny + (-qy + my - 1)) * mz);
        for (int64_t t = 0; t < nkz; ++t) zsum(a, b, c, d, mz, kz[t], &re[t], &im[t]);
      }
      for (int64_t t = 0; t < nkz; ++t) {
        acc_t R = {0, 0}, I = {0, 0};
        for (int l = 0; l < 8; ++l) {
          acc_add(&R, re[t].p[l]); acc_add(&R, re[t].s[l]);
          acc_add(&I, im[t].p[l]); acc_add(&I, im[t].s[l]);
        }
        double *q = part + 4 * (pxi * nkz + t);
        q[0] = R.s; q[1] = R.c; q[2] = I.s; q[3] = I.c;
      }
    }
    free(re); free(im);
  }
  for (int64_t t = 0; t < nkz; ++t) {
    acc_t R = {0, 0}, I = {0, 0};
    for (int64_t p = 0; p < nth; ++p) {
      const double *q = part + 4 * (p * nkz + t);
      acc_add(&R, q[0]); acc_add(&R, q[1]);
      acc_add(&I, q[2]); acc_add(&I, q[3]);
    }
    out[2 * t] = acc_val(&R);
    out[2 * t + 1] = acc_val(&I);
  }
  free(part);
  return 0;
}
