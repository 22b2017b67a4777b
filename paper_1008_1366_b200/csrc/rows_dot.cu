// rows_dot.cu -- multivector dot-product centered Hermitian convolutions
// and the small elementwise helpers of the 2D
// pseudospectral application.
//
// "we allow the convolution inputs to be arrays of vectors, f_i
// and g_i (i = 1..M), interpreting in Functions cconv, conv and tconv the
// product f * g as the element-by-element dot product sum_i f_i * g_i".
// K3d below is K3 (centered Hermitian, three residues) with the
// product stage summed over the M pairs before the forward transforms: per
// residue r the M packed streams w^{f_i}_r + i w^{g_i}_r are backward
// transformed (two c2r each) and their real products summed,
// p_r = sum_i (Re * Im); the forward transforms and the recombination
// 3m h_k = P_0 + zeta_{3m}^{k} P_{-1} + zeta_{3m}^{-k} P_1 (Eq. fft0forwardB)
// run once.  For M = 2 that is the paper's "five Fourier transforms" per
// input-pair set at the 1D level: 4 c2r + 1 r2c per residue.
//
// Layout: pair i's rows start at f + i * istride (g likewise); row j of pair
// i is f + i * istride + j * m.  The result goes to pair 0's rows (f).
#define IDC_ROW_UNIT 1   // row kernels: coherent pass-twiddle loads at E >= 16 (fft_dev.cuh)
#include "fft_dev.cuh"
#include "launch.cuh"
#include "kernels.cuh"
#include "tables.cuh"
#include "tma.cuh"

namespace idc {

namespace {

template <int M>
struct DCfg {
  static constexpr int E = M < 8 ? M : (M <= 512 ? 8 : 16);
  static constexpr int T = M / E;
  static constexpr int G = T >= 256 ? 1 : 256 / T;          // rows per CTA
  static constexpr int THREADS = G * T;
  static constexpr int XB = xbuf_elems<M, E>() > M ? xbuf_elems<M, E>() : M;
  static constexpr bool NAMED = (T % 32 == 0) && G > 1;
};

template <bool NAMED>
struct DSync;
template <>
struct DSync<true> {
  int id, n;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
};
template <>
struct DSync<false> {
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync 0;" ::: "memory"); }
};

template <int M>
__device__ __forceinline__ DSync<DCfg<M>::NAMED> dsync(int grp) {
  if constexpr (DCfg<M>::NAMED) return DSync<true>{1 + grp, DCfg<M>::T};
  else return DSync<false>{};
}

}  // namespace

// ===================================================================== K3d ==
template <int M>
__global__ void __launch_bounds__(DCfg<M>::THREADS, 1)
k_hconv_dot_rows(double2* __restrict__ f, const double2* __restrict__ g, int npairs, long istride, long nrows,
                 const double2* __restrict__ twM, const double2* __restrict__ tw3M) {
  pdl_entry();
  using C = DCfg<M>;
  constexpr int E = C::E, T = C::T, G = C::G;
  extern __shared__ __align__(16) double2 smem[];
  const int grp = threadIdx.x / T, t = threadIdx.x - grp * T;
  double2* xb = smem + grp * C::XB;
  const auto sync = dsync<M>(grp);
  const double inv = 1.0 / (3.0 * M);
  const double s3 = 0.86602540378443864676372317075294;  // sqrt(3)/2
  for (long row0 = (long)blockIdx.x * G; row0 < nrows; row0 += (long)gridDim.x * G) {
    const long row = row0 + grp;
    if constexpr (C::NAMED) {
      if (row >= nrows) break;
    }
    const bool ok = row < nrows;
    const long roff = (ok ? row : 0) * (long)M;
    double2 v[E], Q[E];
    double p[E];
#pragma unroll 1
    for (int rr = 0; rr < 3; ++rr) {
      const int r = rr == 0 ? 0 : (rr == 1 ? 1 : -1);
      const double2 c = make_double2(r == 0 ? 1.0 : -0.5, r == 0 ? 0.0 : (r < 0 ? s3 : -s3));  // zeta_3^{-r}
#pragma unroll
      for (int i = 0; i < E; ++i) p[i] = 0.0;
#pragma unroll 1
      for (int q = 0; q < npairs; ++q) {                       // p_r = sum_i Re * Im (the dot product)
        const double2* fr = f + q * istride + roff;
        const double2* gr = g + q * istride + roff;
        const double2 zt = ldtw(&tw3M[t]);
        auto split = [&](int i, double2 zr) {
          const int k = t + T * i;
          if (i == 0 && t == 0) {
            v[i] = make_double2(ldv(&fr[0]).x, ldv(&gr[0]).x);   // w_{0,r} = Re U_0 (AMB-7)
          } else {
            const double2 fk = ldv(&fr[k]), gk = ldv(&gr[k]), fm = ldv(&fr[M - k]), gm = ldv(&gr[M - k]);
            const double2 P = make_double2(fk.x - gk.y, fk.y + gk.x);
            const double2 R = make_double2(fm.x + gm.y, gm.x - fm.y);
            v[i] = cmul(zr, cadd(P, cmul(c, R)));
          }
        };
        if (r == 0) {
#pragma unroll
          for (int i = 0; i < E; ++i) split(i, make_double2(1.0, 0.0));
        } else if (r > 0) {
          for_roots<3 * E, 1, +1, E>(zt, split);
        } else {
          for_roots<3 * E, 1, -1, E>(cconj(zt), split);
        }
        fft<M, E, +1>(v, t, xb, twM, sync);                    // two c2r in one complex FFT
#pragma unroll
        for (int i = 0; i < E; ++i) p[i] = fma(v[i].x, v[i].y, p[i]);
      }
      if (r == 0) {
#pragma unroll
        for (int i = 0; i < E; ++i) Q[i].x = p[i];
      } else if (r == 1) {
#pragma unroll
        for (int i = 0; i < E; ++i) Q[i].y = p[i];
        fft<M, E, -1>(Q, t, xb, twM, sync);                    // Q = fft(p_0 + i p_1)
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = make_double2(p[i], 0.0);
        fft<M, E, -1>(v, t, xb, twM, sync);                    // P_{-1}
      }
    }
    // P_0, P_1 from Q through Q_{m-k}; recombination (Eq. fft0forwardB)
#pragma unroll
    for (int i = 0; i < E; ++i) xb[t + T * i] = Q[i];
    sync();
    if (ok) {
      double2* fw = f + roff;
      for_roots<3 * E, 1, +1, E>(ldtw(&tw3M[t]), [&](int i, double2 tz) {
        const int k = t + T * i;
        const double2 a = Q[i], b = cconj(xb[(M - k) & (M - 1)]);
        const double2 pp0 = cscale(cadd(a, b), 0.5);
        const double2 d = csub(a, b);
        const double2 pp1 = make_double2(0.5 * d.y, -0.5 * d.x);
        fw[k] = cscale(cadd(cadd(pp0, cmul(v[i], tz)), cmulc(pp1, tz)), inv);
      });
    }
    sync();
  }
}

// ===================================================================== K2d ==
// Function cconv with the dot product: for each residue r the
// products of all pairs are accumulated, acc_r = sum_i fft^{-1}(f_i^r) *
// fft^{-1}(g_i^r), and each accumulator is forward transformed once:
// f_0 <- (fft(acc_0) + zeta_{2m}^{-k} fft(acc_1)) / (2m).  E = 8 so that the
// two accumulators and the pair being transformed fit in registers; the two
// transforms of a pair (and the two forward transforms) run in lockstep.
template <int M>
struct D2Cfg {
  static constexpr int E = M < 8 ? M : 8;
  static constexpr int T = M / E;
  static constexpr int G = T >= 256 ? 1 : 256 / T;
  static constexpr int THREADS = G * T;
  static constexpr int XB = xbuf_elems<M, E>() > M ? xbuf_elems<M, E>() : M;
  static constexpr bool NAMED = (T % 32 == 0) && G > 1;
};

template <int M>
__device__ __forceinline__ DSync<D2Cfg<M>::NAMED> d2sync(int grp) {
  if constexpr (D2Cfg<M>::NAMED) return DSync<true>{1 + grp, D2Cfg<M>::T};
  else return DSync<false>{};
}

template <int M>
__global__ void __launch_bounds__(D2Cfg<M>::THREADS, 1)
k_cconv_dot_rows(double2* __restrict__ f, const double2* __restrict__ g, int npairs, long istride, long nrows,
                 const double2* __restrict__ twM, const double2* __restrict__ tw2M) {
  pdl_entry();
  using C = D2Cfg<M>;
  constexpr int E = C::E, T = C::T, G = C::G;
  extern __shared__ __align__(16) double2 smem[];
  const int grp = threadIdx.x / T, t = threadIdx.x - grp * T;
  double2* xb = smem + grp * 2 * C::XB;
  double2* xb2 = xb + C::XB;
  const auto sync = d2sync<M>(grp);
  const double inv = 1.0 / (2.0 * M);
  for (long row0 = (long)blockIdx.x * G; row0 < nrows; row0 += (long)gridDim.x * G) {
    const long row = row0 + grp;
    if constexpr (C::NAMED) {
      if (row >= nrows) break;
    }
    const bool ok = row < nrows;
    const long roff = (ok ? row : 0) * (long)M;
    double2 a0[E], a1[E], x[E], y[E];
#pragma unroll
    for (int i = 0; i < E; ++i) a0[i] = a1[i] = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int q = 0; q < npairs; ++q) {
      const double2* fr = f + q * istride + roff;
      const double2* gr = g + q * istride + roff;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        x[i] = ldv(&fr[t + T * i]);
        y[i] = ldv(&gr[t + T * i]);
      }
      fft2<M, E, +1>(x, y, t, xb, xb2, twM, sync);                         // r = 0
#pragma unroll
      for (int i = 0; i < E; ++i) a0[i] = cadd(a0[i], cmul(x[i], y[i]));
      const double2 zt = ldtw(&tw2M[t]);                                   // zeta_{2m}^k = zeta_{2m}^t zeta_{2E}^i
      for_roots<2 * E, 1, +1, E>(zt, [&](int i, double2 w) {
        x[i] = cmul(ldv(&fr[t + T * i]), w);
        y[i] = cmul(ldv(&gr[t + T * i]), w);
      });
      fft2<M, E, +1>(x, y, t, xb, xb2, twM, sync);                         // r = 1
#pragma unroll
      for (int i = 0; i < E; ++i) a1[i] = cadd(a1[i], cmul(x[i], y[i]));
    }
    fft2<M, E, -1>(a0, a1, t, xb, xb2, twM, sync);                         // forward
    if (ok) {
      double2* fw = f + roff;
      for_roots<2 * E, 1, -1, E>(cconj(ldtw(&tw2M[t])), [&](int i, double2 w) {
        fw[t + T * i] = cscale(cadd(a0[i], cmul(a1[i], w)), inv);
      });
    }
  }
}

// ===================================================================== K4d ==
// Centered Hermitian ternary dot product sum_i f_i * g_i * h_i (P:859-867
// applied to Function tconv): per residue pair (r0, r0 + 1) of the four-
// residue form every triple's
// products u^f u^g u^h are accumulated before the one forward transform of
// the pair; the first pair's recombined contribution is kept in shared
// memory (ACC) until the second pair adds to it.
template <int M>
__global__ void __launch_bounds__(D2Cfg<M>::THREADS, 1)
k_tconv_dot_rows(double2* __restrict__ f, const double2* __restrict__ g, const double2* __restrict__ h, int npairs,
                 long istride, long nrows, const double2* __restrict__ twM, const double2* __restrict__ tw4M) {
  pdl_entry();
  using C = D2Cfg<M>;
  constexpr int E = C::E, T = C::T, G = C::G;
  extern __shared__ __align__(16) double2 smem[];
  const int grp = threadIdx.x / T, t = threadIdx.x - grp * T;
  double2* xb = smem + grp * (C::XB + M);
  double2* ACC = xb + C::XB;
  const auto sync = d2sync<M>(grp);
  const double inv = 1.0 / (4.0 * M);
  for (long row0 = (long)blockIdx.x * G; row0 < nrows; row0 += (long)gridDim.x * G) {
    const long row = row0 + grp;
    if constexpr (C::NAMED) {
      if (row >= nrows) break;
    }
    const bool ok = row < nrows;
    const long roff = (ok ? row : 0) * (long)M;
    auto pair = [&](auto R0) {
      constexpr int r0 = decltype(R0)::value;
      const double2 ca = r0 == 0 ? make_double2(1, 0) : make_double2(-1, 0);   // (-i)^{r0}
      const double2 cb = r0 == 0 ? make_double2(0, -1) : make_double2(0, 1);   // (-i)^{r0+1}
      double2 acc[E], v[E];
      double a0[E], a1[E];
#pragma unroll
      for (int i = 0; i < E; ++i) acc[i] = make_double2(0.0, 0.0);
#pragma unroll 1
      for (int q = 0; q < npairs; ++q) {
        const double2* fr = f + q * istride + roff;
        const double2* gr = g + q * istride + roff;
        const double2* hr = h + q * istride + roff;
        // f/g streams r0, r0 + 1 (two c2r each), then h packed across the pair
        const double2 za = ldtw(&tw4M[r0 * t]), zb = ldtw(&tw4M[(r0 + 1) * t]);
        static_for<E>([&](auto I) {
          constexpr int i = decltype(I)::value;
          const int k = t + T * i;
          if (i == 0 && t == 0) {
            v[i] = make_double2(ldv(&fr[0]).x, ldv(&gr[0]).x);
          } else {
            const double2 fk = ldv(&fr[k]), gk = ldv(&gr[k]), fm = ldv(&fr[M - k]), gm = ldv(&gr[M - k]);
            const double2 P = make_double2(fk.x - gk.y, fk.y + gk.x);
            const double2 R = make_double2(fm.x + gm.y, gm.x - fm.y);
            v[i] = cmul(twc<r0 * i, 4 * E, +1>(za), cadd(P, cmul(ca, R)));
          }
        });
        fft<M, E, +1>(v, t, xb, twM, sync);
#pragma unroll
        for (int i = 0; i < E; ++i) a0[i] = v[i].x * v[i].y;
        const double2 zb2 = ldtw(&tw4M[(r0 + 1) * t]);
        static_for<E>([&](auto I) {
          constexpr int i = decltype(I)::value;
          const int k = t + T * i;
          if (i == 0 && t == 0) {
            v[i] = make_double2(ldv(&fr[0]).x, ldv(&gr[0]).x);
          } else {
            const double2 fk = ldv(&fr[k]), gk = ldv(&gr[k]), fm = ldv(&fr[M - k]), gm = ldv(&gr[M - k]);
            const double2 P = make_double2(fk.x - gk.y, fk.y + gk.x);
            const double2 R = make_double2(fm.x + gm.y, gm.x - fm.y);
            v[i] = cmul(twc<(r0 + 1) * i, 4 * E, +1>(zb2), cadd(P, cmul(cb, R)));
          }
        });
        fft<M, E, +1>(v, t, xb, twM, sync);
#pragma unroll
        for (int i = 0; i < E; ++i) a1[i] = v[i].x * v[i].y;
        const double2 za3 = ldtw(&tw4M[r0 * t]), zb3 = ldtw(&tw4M[(r0 + 1) * t]);
        static_for<E>([&](auto I) {
          constexpr int i = decltype(I)::value;
          const int k = t + T * i;
          if (i == 0 && t == 0) {
            const double h0 = ldv(&hr[0]).x;
            v[i] = make_double2(h0, h0);
          } else {
            const double2 hk = ldv(&hr[k]), hm = cconj(ldv(&hr[M - k]));
            const double2 w0 = cmul(twc<r0 * i, 4 * E, +1>(za3), cadd(hk, cmul(ca, hm)));
            const double2 w1 = cmul(twc<(r0 + 1) * i, 4 * E, +1>(zb3), cadd(hk, cmul(cb, hm)));
            v[i] = make_double2(w0.x - w1.y, w0.y + w1.x);
          }
        });
        fft<M, E, +1>(v, t, xb, twM, sync);
#pragma unroll
        for (int i = 0; i < E; ++i) acc[i] = make_double2(fma(a0[i], v[i].x, acc[i].x), fma(a1[i], v[i].y, acc[i].y));
      }
      fft<M, E, -1>(acc, t, xb, twM, sync);
      // separate the pair's two real-data spectra through acc_{m-k}, recombine
#pragma unroll
      for (int i = 0; i < E; ++i) xb[t + T * i] = acc[i];
      sync();
      const double2 za4 = ldtw(&tw4M[r0 * t]), zb4 = ldtw(&tw4M[(r0 + 1) * t]);
      static_for<E>([&](auto I) {
        constexpr int i = decltype(I)::value;
        const int k = t + T * i;
        const double2 a = acc[i], b = cconj(xb[(M - k) & (M - 1)]);
        const double2 pp0 = cscale(cadd(a, b), 0.5);
        const double2 d = csub(a, b);
        const double2 pp1 = make_double2(0.5 * d.y, -0.5 * d.x);
        const double2 ct = cadd(cmulc(pp0, twc<r0 * i, 4 * E, +1>(za4)), cmulc(pp1, twc<(r0 + 1) * i, 4 * E, +1>(zb4)));
        if constexpr (r0 == 0) ACC[k] = ct;
        else if (ok) f[roff + k] = cscale(cadd(ACC[k], ct), inv);
      });
      sync();
    };
    pair(std::integral_constant<int, 0>{});
    pair(std::integral_constant<int, 2>{});
  }
}

// ===================================================================== K2pq ==
// General p/q implicit padding: rows of
// L = pm complex modes, implicitly zero padded to N = qm (q >= 2p: the linear
// convolution of the first pm terms is alias free).  j = q l + r, k = t m + s:
//   u_{ql+r} = sum_s zeta_m^{ls} sum_{t<p} zeta_{qm}^{r(tm+s)} U_{tm+s}
// -- q transforms of size m per input -- and the forward
//   qm U_k = sum_{r<q} zeta_{qm}^{-rk} sum_l zeta_m^{-kl} u_{ql+r},  k < pm.
// Per residue r the two inputs' streams are transformed in lockstep, their
// product forward transformed, and its contribution zeta_{qm}^{-rk} F_r(k mod
// m) added to the p output accumulators (registers) of the row.
template <int M, int P>
__global__ void __launch_bounds__(D2Cfg<M>::THREADS, 1)
k_cconv_pq_rows(double2* __restrict__ f, const double2* __restrict__ g, int q, long nrows,
                const double2* __restrict__ twM, const double2* __restrict__ twqM) {
  pdl_entry();
  using C = D2Cfg<M>;
  constexpr int E = C::E, T = C::T, G = C::G;
  extern __shared__ __align__(16) double2 smem[];
  const int grp = threadIdx.x / T, t = threadIdx.x - grp * T;
  double2* xb = smem + grp * 2 * C::XB;
  double2* xb2 = xb + C::XB;
  const auto sync = d2sync<M>(grp);
  const long L = (long)P * M;
  const double inv = 1.0 / ((double)q * M);
  for (long row0 = (long)blockIdx.x * G; row0 < nrows; row0 += (long)gridDim.x * G) {
    const long row = row0 + grp;
    if constexpr (C::NAMED) {
      if (row >= nrows) break;
    }
    const bool ok = row < nrows;
    const double2* fr = f + (ok ? row : 0) * L;
    const double2* gr = g + (ok ? row : 0) * L;
    double2 acc[P][E], x[E], y[E];
#pragma unroll
    for (int tt = 0; tt < P; ++tt)
#pragma unroll
      for (int i = 0; i < E; ++i) acc[tt][i] = make_double2(0.0, 0.0);
    const int qm = q * M;
    // index of zeta_{qm}^{r(tm+s)} in the qm-entry table: (rt mod q) m + rs < 2qm
    auto zidx = [&](int r, int tt, int s) {
      const int j = ((r * tt) % q) * M + r * s;
      return j >= qm ? j - qm : j;
    };
#pragma unroll 1
    for (int r = 0; r < q; ++r) {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int s = t + T * i;
        double2 xs = make_double2(0.0, 0.0), ys = make_double2(0.0, 0.0);
#pragma unroll
        for (int tt = 0; tt < P; ++tt) {
          const int k = tt * M + s;
          const double2 z = ldtw(&twqM[zidx(r, tt, s)]);              // zeta_{qm}^{r(tm+s)}
          xs = cadd(xs, cmul(z, ldv(&fr[k])));
          ys = cadd(ys, cmul(z, ldv(&gr[k])));
        }
        x[i] = xs;
        y[i] = ys;
      }
      fft2<M, E, +1>(x, y, t, xb, xb2, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] = cmul(x[i], y[i]);
      fft<M, E, -1>(x, t, xb, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int s = t + T * i;
#pragma unroll
        for (int tt = 0; tt < P; ++tt)
          acc[tt][i] = cadd(acc[tt][i], cmulc(x[i], ldtw(&twqM[zidx(r, tt, s)])));   // zeta_{qm}^{-rk}
      }
    }
    if (ok) {
      double2* fw = f + row * L;
#pragma unroll
      for (int tt = 0; tt < P; ++tt)
#pragma unroll
        for (int i = 0; i < E; ++i) fw[(long)tt * M + t + T * i] = cscale(acc[tt][i], inv);
    }
  }
}

// ------------------------------------------------------- 2D helpers ------
// Hermitian projection of the stored ky = 0 line of a (2mx-1) x my centered
// array (AMB-7; "automatically enforce Hermitian symmetry"):
// U_{kx,0} <- (U_{kx,0} + conj U_{-kx,0}) / 2, U_{0,0} real.
__global__ void k_enforce_symmetry_2d(double2* __restrict__ a, int mx, int my, long batch) {
  pdl_entry();
  const long n = (long)mx * batch;                   // kx = 0..mx-1 for every item
  for (long id = (long)blockIdx.x * blockDim.x + threadIdx.x; id < n; id += (long)gridDim.x * blockDim.x) {
    const long b = id / mx;
    const int kx = (int)(id - b * mx);
    double2* A = a + b * (long)(2 * mx - 1) * my;
    double2* P = A + (long)(mx - 1 + kx) * my;       // (kx, 0)
    double2* N = A + (long)(mx - 1 - kx) * my;       // (-kx, 0)
    const double2 u = *P, w = *N;
    const double2 s = make_double2(0.5 * (u.x + w.x), 0.5 * (u.y - w.y));
    *P = s;
    *N = cconj(s);
  }
}

// Inputs of the 2D Euler advective term: from the vorticity
// spectrum w (centered kx, Hermitian ky >= 0), the M = 2 dot-product pairs
//   f_1 = i kx w,  f_2 = i ky w,  g_1 = i ky w / k^2,  g_2 = -i kx w / k^2
// (1/k^2 := 0 at k = 0: no mean flow).  f, g: 2 x (2mx-1) x my each.
__global__ void k_advection2d_inputs(const double2* __restrict__ w, double2* __restrict__ f, double2* __restrict__ g,
                                     int mx, int my) {
  pdl_entry();
  const long n = (long)(2 * mx - 1) * my;
  for (long id = (long)blockIdx.x * blockDim.x + threadIdx.x; id < n; id += (long)gridDim.x * blockDim.x) {
    const long i = id / my;
    const double kx = (double)(i - (mx - 1)), ky = (double)(id - i * my);
    const double2 a = w[id];
    const double k2 = kx * kx + ky * ky;
    const double ik2 = k2 > 0.0 ? 1.0 / k2 : 0.0;
    f[id] = make_double2(-kx * a.y, kx * a.x);                    // i kx w
    f[n + id] = make_double2(-ky * a.y, ky * a.x);                // i ky w
    g[id] = make_double2(-ky * a.y * ik2, ky * a.x * ik2);        // i ky w / k^2
    g[n + id] = make_double2(kx * a.y * ik2, -kx * a.x * ik2);    // -i kx w / k^2
  }
}

// ================================================================ launchers ==
template <int M>
cudaError_t hconv_dot_rows(double2* f, const double2* g, int npairs, long istride, long nrows, cudaStream_t s) {
  using C = DCfg<M>;
  const double2* twM = pass_table(M, C::E);
  const double2* tw3M = zeta_table(3 * M);
  if (!twM || !tw3M) return cudaErrorMemoryAllocation;
  const size_t smem = (size_t)C::G * C::XB * 16;
  cudaError_t e = cudaFuncSetAttribute(k_hconv_dot_rows<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  long need = (nrows + C::G - 1) / C::G;
  long grid = num_sms();
  if (need < grid) grid = need;
  if (grid < 1) grid = 1;
  void* args[] = {&f, &g, &npairs, &istride, &nrows, &twM, &tw3M};
  return launch_kernel((const void*)k_hconv_dot_rows<M>, dim3((unsigned)grid), dim3(C::THREADS), args, smem, s,
                       {"K3d", M, nrows * npairs});
}

cudaError_t launch_hconv_dot_rows(double2* f, const double2* g, int npairs, long istride, int m, long nrows,
                                  cudaStream_t s) {
  switch (m) {
    case 2: return hconv_dot_rows<2>(f, g, npairs, istride, nrows, s);
    case 4: return hconv_dot_rows<4>(f, g, npairs, istride, nrows, s);
    case 8: return hconv_dot_rows<8>(f, g, npairs, istride, nrows, s);
    case 16: return hconv_dot_rows<16>(f, g, npairs, istride, nrows, s);
    case 32: return hconv_dot_rows<32>(f, g, npairs, istride, nrows, s);
    case 64: return hconv_dot_rows<64>(f, g, npairs, istride, nrows, s);
    case 128: return hconv_dot_rows<128>(f, g, npairs, istride, nrows, s);
    case 256: return hconv_dot_rows<256>(f, g, npairs, istride, nrows, s);
    case 512: return hconv_dot_rows<512>(f, g, npairs, istride, nrows, s);
    case 1024: return hconv_dot_rows<1024>(f, g, npairs, istride, nrows, s);
    case 2048: return hconv_dot_rows<2048>(f, g, npairs, istride, nrows, s);
    case 4096: return hconv_dot_rows<4096>(f, g, npairs, istride, nrows, s);
  }
  return cudaErrorInvalidValue;
}

template <int M>
cudaError_t cconv_dot_rows(double2* f, const double2* g, int npairs, long istride, long nrows, cudaStream_t s) {
  using C = D2Cfg<M>;
  const double2* twM = pass_table(M, C::E);
  const double2* tw2M = zeta_table(2 * M);
  if (!twM || !tw2M) return cudaErrorMemoryAllocation;
  const size_t smem = (size_t)C::G * 2 * C::XB * 16;
  cudaError_t e = cudaFuncSetAttribute(k_cconv_dot_rows<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  long need = (nrows + C::G - 1) / C::G, grid = num_sms();
  if (need < grid) grid = need;
  if (grid < 1) grid = 1;
  void* args[] = {&f, &g, &npairs, &istride, &nrows, &twM, &tw2M};
  return launch_kernel((const void*)k_cconv_dot_rows<M>, dim3((unsigned)grid), dim3(C::THREADS), args, smem, s,
                       {"K2d", M, nrows * npairs});
}

template <int M>
cudaError_t tconv_dot_rows(double2* f, const double2* g, const double2* h, int npairs, long istride, long nrows,
                           cudaStream_t s) {
  using C = D2Cfg<M>;
  const double2* twM = pass_table(M, C::E);
  const double2* tw4M = zeta_table(4 * M);
  if (!twM || !tw4M) return cudaErrorMemoryAllocation;
  const size_t smem = (size_t)C::G * (C::XB + M) * 16;
  cudaError_t e = cudaFuncSetAttribute(k_tconv_dot_rows<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  long need = (nrows + C::G - 1) / C::G, grid = num_sms();
  if (need < grid) grid = need;
  if (grid < 1) grid = 1;
  void* args[] = {&f, &g, &h, &npairs, &istride, &nrows, &twM, &tw4M};
  return launch_kernel((const void*)k_tconv_dot_rows<M>, dim3((unsigned)grid), dim3(C::THREADS), args, smem, s,
                       {"K4d", M, nrows * npairs});
}

cudaError_t launch_cconv_dot_rows(double2* f, const double2* g, int npairs, long istride, int m, long nrows,
                                  cudaStream_t s) {
#define IDC_CALL(MM) cconv_dot_rows<MM>(f, g, npairs, istride, nrows, s)
  switch (m) {
    case 1: return IDC_CALL(1);
    case 2: return IDC_CALL(2);
    case 4: return IDC_CALL(4);
    case 8: return IDC_CALL(8);
    case 16: return IDC_CALL(16);
    case 32: return IDC_CALL(32);
    case 64: return IDC_CALL(64);
    case 128: return IDC_CALL(128);
    case 256: return IDC_CALL(256);
    case 512: return IDC_CALL(512);
    case 1024: return IDC_CALL(1024);
    case 2048: return IDC_CALL(2048);
    case 4096: return IDC_CALL(4096);
  }
#undef IDC_CALL
  return cudaErrorInvalidValue;
}

cudaError_t launch_tconv_dot_rows(double2* f, const double2* g, const double2* h, int npairs, long istride, int m,
                                  long nrows, cudaStream_t s) {
#define IDC_CALL(MM) tconv_dot_rows<MM>(f, g, h, npairs, istride, nrows, s)
  switch (m) {
    case 2: return IDC_CALL(2);
    case 4: return IDC_CALL(4);
    case 8: return IDC_CALL(8);
    case 16: return IDC_CALL(16);
    case 32: return IDC_CALL(32);
    case 64: return IDC_CALL(64);
    case 128: return IDC_CALL(128);
    case 256: return IDC_CALL(256);
    case 512: return IDC_CALL(512);
    case 1024: return IDC_CALL(1024);
    case 2048: return IDC_CALL(2048);
    case 4096: return IDC_CALL(4096);
  }
#undef IDC_CALL
  return cudaErrorInvalidValue;
}

template <int M, int P>
cudaError_t cconv_pq_rows(double2* f, const double2* g, int q, long nrows, cudaStream_t s) {
  using C = D2Cfg<M>;
  const double2* twM = pass_table(M, C::E);
  const double2* twqM = zeta_table(q * M);
  if (!twM || !twqM) return cudaErrorMemoryAllocation;
  const size_t smem = (size_t)C::G * 2 * C::XB * 16;
  cudaError_t e = cudaFuncSetAttribute(k_cconv_pq_rows<M, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  long need = (nrows + C::G - 1) / C::G, grid = num_sms();
  if (need < grid) grid = need;
  if (grid < 1) grid = 1;
  void* args[] = {&f, &g, &q, &nrows, &twM, &twqM};
  return launch_kernel((const void*)k_cconv_pq_rows<M, P>, dim3((unsigned)grid), dim3(C::THREADS), args, smem, s,
                       {"K2pq", M, nrows});
}

template <int P>
cudaError_t cconv_pq_dispatch(double2* f, const double2* g, int q, int m, long nrows, cudaStream_t s) {
  switch (m) {
    case 8: return cconv_pq_rows<8, P>(f, g, q, nrows, s);
    case 16: return cconv_pq_rows<16, P>(f, g, q, nrows, s);
    case 32: return cconv_pq_rows<32, P>(f, g, q, nrows, s);
    case 64: return cconv_pq_rows<64, P>(f, g, q, nrows, s);
    case 128: return cconv_pq_rows<128, P>(f, g, q, nrows, s);
    case 256: return cconv_pq_rows<256, P>(f, g, q, nrows, s);
    case 512: return cconv_pq_rows<512, P>(f, g, q, nrows, s);
    case 1024: return cconv_pq_rows<1024, P>(f, g, q, nrows, s);
    case 2048: return cconv_pq_rows<2048, P>(f, g, q, nrows, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_cconv_pq_rows(double2* f, const double2* g, int p, int q, int m, long nrows, cudaStream_t s) {
  switch (p) {
    case 1: return cconv_pq_dispatch<1>(f, g, q, m, nrows, s);
    case 2: return cconv_pq_dispatch<2>(f, g, q, m, nrows, s);
    case 3: return cconv_pq_dispatch<3>(f, g, q, m, nrows, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_enforce_symmetry_2d(double2* a, int mx, int my, long batch, cudaStream_t s) {
  const long n = (long)mx * batch;
  const int threads = 256;
  long blocks = (n + threads - 1) / threads;
  if (blocks > 4L * num_sms() * 8) blocks = 4L * num_sms() * 8;
  if (blocks < 1) blocks = 1;
  void* args[] = {&a, &mx, &my, &batch};
  return launch_kernel((const void*)k_enforce_symmetry_2d, dim3((unsigned)blocks), dim3(threads), args, 0, s,
                       {"Ksym", my, (long)(2 * mx - 1) * batch});
}

cudaError_t launch_advection2d_inputs(const double2* w, double2* f, double2* g, int mx, int my, cudaStream_t s) {
  const long n = (long)(2 * mx - 1) * my;
  const int threads = 256;
  long blocks = (n + threads - 1) / threads;
  if (blocks > 16L * num_sms()) blocks = 16L * num_sms();
  if (blocks < 1) blocks = 1;
  void* args[] = {&w, &f, &g, &mx, &my};
  return launch_kernel((const void*)k_advection2d_inputs, dim3((unsigned)blocks), dim3(threads), args, 0, s,
                       {"Kadv", my, (long)(2 * mx - 1)});
}

}  // namespace idc
