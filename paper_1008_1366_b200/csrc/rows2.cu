// rows2.cu -- fused 1D row convolutions, register-resident variant (m <= 4096).
//
// Same method and equations as conv1d.cu (K2/K3/K4, Functions cconv / conv /
// tconv of the paper), organised for occupancy:
//   * E = 8 elements per thread (radix-8 Stockham passes), T = m/8 threads
//     per row, rows of a CTA synchronise with their own named barrier;
//   * the per-row intermediates that must survive a transform (the r = 0
//     product of cconv, the (p0, p1) spectrum of hconv, the output
//     accumulator of tconv) stay in registers; shared memory holds only the
//     Stockham exchange buffer (plus, for tconv, the f*g stream products), so
//     the row's inputs stay L1-resident for the mirrored (U_{m-k}) loads.
#define IDC_ROW_UNIT 1   // row kernels: coherent pass-twiddle loads at E >= 16 (fft_dev.cuh)
#include "config.cuh"
#include "fft_dev.cuh"
#include "launch.cuh"
#include "kernels.cuh"
#include "tables.cuh"
#include "tma.cuh"

#ifndef IDC_FFT2_STAGGER
#define IDC_FFT2_STAGGER 1
#endif
#if IDC_FFT2_STAGGER
#define IDC_FFT2 fft2s
#else
#define IDC_FFT2 fft2
#endif

namespace idc {

namespace {

template <int M, int E, int G>
struct Cfg2 {
  static constexpr int T = M / E;
  static constexpr int THREADS = G * T;
  static constexpr int XB = xbuf_elems<M, E>() > M ? xbuf_elems<M, E>() : M;
  static constexpr bool NAMED = (T % 32 == 0) && G > 1;
  // cap registers at 128 per thread: 16 warps per SM for 512-thread CTAs,
  // two 256-thread CTAs per SM otherwise
// K2 up to this m: f and g rows staged in shared memory by bulk copies
// (mbarrier), the next row's copies issued as soon as the current row's last
// split has read the stage; above it the rows are read from global memory
// after an L2 prefetch.  Measured: m = 512 0.66 -> 0.63 ms (cconv3d 512^3
// 22.0 -> 21.55 ms), m = 64 -3%, m = 1024 +2-5% (so kept off there).
// K2 with E = 16 from this m up: park the r = 0 result in shared memory
// instead of keeping it in registers across the r = 1 transforms (removes
// the spills: m = 4096 1.064 -> 0.983 ms; m = 1024 neutral, m = 2048 +2.5%)
  static constexpr int MINB = (65536 / (THREADS * IDC_ROWS_REGS)) < 1 ? 1 : 65536 / (THREADS * IDC_ROWS_REGS);
};

// K2 shared-memory layout per row group, used by the kernel and its launcher:
// staged f, g rows (m <= IDC_ROWS2_TMA_MAX), one exchange buffer per vector
// transformed at once (two for the pairs at E = 8; pairs at E = 16 measured
// slower: cconv1d 1024 0.704 -> 0.784 ms, profiles/r02/ab/k2_pairs_e16.log),
// and the parked r = 0 result (single transforms from IDC_K2_PARK_MIN up).
template <int M, int E>
struct K2Layout {
  static constexpr bool FFT2 = E <= 8;
  static constexpr bool ST = M <= IDC_ROWS2_TMA_MAX;
  static constexpr bool PARK = !FFT2 && M >= IDC_K2_PARK_MIN;
  static constexpr int XB = xbuf_elems<M, E>() > M ? xbuf_elems<M, E>() : M;
  static constexpr int PER = (ST ? 2 * M : 0) + (FFT2 ? 2 : 1) * XB + (PARK ? M : 0);
};

template <bool NAMED>
struct RowSync;
template <>
struct RowSync<true> {
  int id, n;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
};
template <>
struct RowSync<false> {
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync 0;" ::: "memory"); }
};

template <int M, int E, int G>
__device__ __forceinline__ RowSync<Cfg2<M, E, G>::NAMED> row_sync(int grp) {
  if constexpr (Cfg2<M, E, G>::NAMED) return RowSync<true>{1 + grp, Cfg2<M, E, G>::T};
  else return RowSync<false>{};
}

// Z_k = w^f_{k,r} + i w^g_{k,r}, w_{k,r} = zr (U_k + c conj U_{m-k}), k >= 1
__device__ __forceinline__ double2 herm_pair2(double2 fk, double2 gk, double2 fm, double2 gm, double2 zr, double2 c) {
  const double2 P = make_double2(fk.x - gk.y, fk.y + gk.x);
  const double2 R = make_double2(fm.x + gm.y, gm.x - fm.y);
  return cmul(zr, cadd(P, cmul(c, R)));
}

// K2 row reads: the shared-memory stage (plain loads; the FFT barriers'
// memory clobbers already force the re-reads) or global memory (ldv)
template <bool ST>
__device__ __forceinline__ double2 ldrow(const double2* p) {
  if constexpr (ST) return *p;
  else return ldv(p);
}

}  // namespace

// ====================================================================== K2 ==
// Function cconv, see conv1d.cu for the step-by-step mapping.
template <int M, int E, int G>
__global__ void __launch_bounds__(Cfg2<M, E, G>::THREADS, Cfg2<M, E, G>::MINB)
k_cconv_rows2(double2* __restrict__ f, double2* __restrict__ g, long nrows, const double2* __restrict__ twM,
              const double2* __restrict__ tw2M, RowSets rs) {
  pdl_entry();
  using C = Cfg2<M, E, G>;
  constexpr int T = C::T;
  extern __shared__ __align__(16) double2 smem[];
  const int grp = threadIdx.x / T, t = threadIdx.x - grp * T;
  constexpr bool FFT2 = K2Layout<M, E>::FFT2;   // transforms in (staggered) pairs, two exchange buffers
  // ST: per group the staged f and g rows, then the exchange buffer(s); the
  // groups' mbarriers after all groups.  Otherwise exchange buffers only.
  constexpr bool ST = M <= IDC_ROWS2_TMA_MAX;
  constexpr bool PARK = K2Layout<M, E>::PARK;   // r = 0 result parked in shared memory
  constexpr int PER = K2Layout<M, E>::PER;
  double2* Fs = smem + grp * PER;
  double2* Gs = Fs + M;
  double2* xb = ST ? Gs + M : Fs;
  double2* pk = xb + C::XB;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + G * PER) + grp;
  const long step = (long)gridDim.x * G;
  auto issue = [&](long r) {   // bulk copies of row r's f and g into the stage
    mbar_arrive_expect_tx(bar, 2u * M * 16u);
    tma_load_1d(Fs, row_ptr(f, rs.f1, rs.n0, r, M), M * 16u, bar);
    tma_load_1d(Gs, row_ptr(g, rs.g1, rs.n0, r, M), M * 16u, bar);
  };
  if constexpr (ST) {
    if (t == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (t == 0 && (long)blockIdx.x * G + grp < nrows) issue((long)blockIdx.x * G + grp);
  }
  uint32_t phase = 0;
  double2* xb2 = xb + C::XB;
  const auto sync = row_sync<M, E, G>(grp);
  const double inv = 1.0 / (2.0 * M);
  for (long row0 = (long)blockIdx.x * G; row0 < nrows; row0 += (long)gridDim.x * G) {
    const long row = row0 + grp;
    if constexpr (C::NAMED) {
      if (row >= nrows) break;
    }
    const bool ok = row < nrows;
    double2* fo = row_ptr(f, rs.f1, rs.n0, ok ? row : 0, M);   // output row
    const double2* fr = ST ? Fs : fo;                             // row reads: stage or global
    const double2* gr = ST ? Gs : row_ptr(g, rs.g1, rs.n0, ok ? row : 0, M);
    if constexpr (ST) {
      if (ok) {
        mbar_wait(bar, phase);
        phase ^= 1;
      }
    } else if (IDC_ROWS_PREFETCH && t == 0 && row + step < nrows) {
      // the next rows of this group: bulk prefetch into L2 (hides the HBM
      // latency of the first loads of the next iteration)
      prefetch_l2(row_ptr(f, rs.f1, rs.n0, row + step, M), M * 16u);
      prefetch_l2(row_ptr(g, rs.g1, rs.n0, row + step, M), M * 16u);
    }
    // after the last read of the staged rows (the r = 1 split): next row's copies
    auto refill = [&]() {
      if constexpr (ST) {
        sync();
        if (t == 0 && row + step < nrows) issue(row + step);
      }
    };
    // Every intermediate in registers (at most three E-vectors live): no
    // shared-memory stash traffic, only the FFT exchanges.  With E = 8 the
    // independent transforms run pairwise in lockstep (fft2: one barrier pair
    // per pass; 2-7% faster at m <= 512); with E = 16 the second vector's
    // codelet registers spill, so the transforms run one at a time.
    double2 x[E], y[E], z[E];
    double2 zt;   // zeta_{2m}^t; zeta_{2m}^k = zeta_{2m}^t zeta_{2E}^i (immediate), k = t + T i
    if constexpr (FFT2 && ST && IDC_K2_ONE_READ) {
      // both residues' streams from one read of the staged rows (the r = 1
      // pair held in registers, E = 8): the stage is refilled before the
      // first transform and its reads halve
      double2 y1[E];
      zt = ldtw(&tw2M[t]);
      for_roots<2 * E, 1, +1, E>(zt, [&](int i, double2 w) {
        const double2 a = fr[t + T * i], b = gr[t + T * i];
        x[i] = a;
        y[i] = b;
        y1[i] = cmul(a, w);                                                 // r = 1
        z[i] = cmul(b, w);
      });
      refill();
      IDC_FFT2<M, E, +1>(x, y, t, xb, xb2, twM, sync);                        // r = 0
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] = cmul(x[i], y[i]);
      IDC_FFT2<M, E, +1>(y1, z, t, xb, xb2, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) y[i] = cmul(y1[i], z[i]);
      IDC_FFT2<M, E, -1>(x, y, t, xb, xb2, twM, sync);                        // forward
    } else if constexpr (FFT2) {
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] = ldrow<ST>(&fr[t + T * i]);
#pragma unroll
      for (int i = 0; i < E; ++i) y[i] = ldrow<ST>(&gr[t + T * i]);
      IDC_FFT2<M, E, +1>(x, y, t, xb, xb2, twM, sync);                        // r = 0
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] = cmul(x[i], y[i]);
      // r = 1: zeta_{2m}^k-shifted streams
      zt = ldtw(&tw2M[t]);
      for_roots<2 * E, 1, +1, E>(zt, [&](int i, double2 w) { y[i] = cmul(ldrow<ST>(&fr[t + T * i]), w); });
      for_roots<2 * E, 1, +1, E>(zt, [&](int i, double2 w) { z[i] = cmul(ldrow<ST>(&gr[t + T * i]), w); });
      refill();
      IDC_FFT2<M, E, +1>(y, z, t, xb, xb2, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) y[i] = cmul(y[i], z[i]);
      IDC_FFT2<M, E, -1>(x, y, t, xb, xb2, twM, sync);                        // forward
    } else if constexpr (PARK) {
      // r = 0 stream all the way back first, parked in this thread's own
      // shared-memory slots while the r = 1 stream is transformed: two
      // E-vectors live instead of three
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] = ldrow<ST>(&fr[t + T * i]);
      fft<M, E, +1>(x, t, xb, twM, sync);                                 // r = 0
#pragma unroll
      for (int i = 0; i < E; ++i) y[i] = ldrow<ST>(&gr[t + T * i]);
      fft<M, E, +1>(y, t, xb, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] = cmul(x[i], y[i]);
      fft<M, E, -1>(x, t, xb, twM, sync);                                 // forward
#pragma unroll
      for (int i = 0; i < E; ++i) pk[t + T * i] = x[i];
      zt = ldtw(&tw2M[t]);
      for_roots<2 * E, 1, +1, E>(zt, [&](int i, double2 w) { y[i] = cmul(ldrow<ST>(&fr[t + T * i]), w); });
      fft<M, E, +1>(y, t, xb, twM, sync);                                 // r = 1
      for_roots<2 * E, 1, +1, E>(zt, [&](int i, double2 w) { x[i] = cmul(ldrow<ST>(&gr[t + T * i]), w); });
      refill();
      fft<M, E, +1>(x, t, xb, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) y[i] = cmul(y[i], x[i]);
      fft<M, E, -1>(y, t, xb, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] = pk[t + T * i];
    } else {
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] = ldrow<ST>(&fr[t + T * i]);
      fft<M, E, +1>(x, t, xb, twM, sync);                                 // r = 0
#pragma unroll
      for (int i = 0; i < E; ++i) y[i] = ldrow<ST>(&gr[t + T * i]);
      fft<M, E, +1>(y, t, xb, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] = cmul(x[i], y[i]);
      zt = ldtw(&tw2M[t]);
      for_roots<2 * E, 1, +1, E>(zt, [&](int i, double2 w) { y[i] = cmul(ldrow<ST>(&fr[t + T * i]), w); });
      fft<M, E, +1>(y, t, xb, twM, sync);                                 // r = 1
      for_roots<2 * E, 1, +1, E>(zt, [&](int i, double2 w) { z[i] = cmul(ldrow<ST>(&gr[t + T * i]), w); });
      refill();
      fft<M, E, +1>(z, t, xb, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) y[i] = cmul(y[i], z[i]);
      fft<M, E, -1>(y, t, xb, twM, sync);                                 // forward
      fft<M, E, -1>(x, t, xb, twM, sync);
    }
    // recombination and 1/(2m)
    if (ok) {
      double2* fw = fo;
      for_roots<2 * E, 1, -1, E>(cconj(zt), [&](int i, double2 w) {       // zeta_{2m}^{-k}
        fw[t + T * i] = cscale(cadd(x[i], cmul(y[i], w)), inv);
      });
    }
  }
}

// ====================================================================== K3 ==
// Centered Hermitian convolution, N = 3m; see conv1d.cu.
// Order: r = 0 (p0 kept), r = 1 -> FFT(p0 + i p1) = Q kept in registers,
// r = -1 -> FFT(p_{-1}); then Q_{m-k} through shared memory and the
// recombination 3m h_k = P_0 + zeta_{3m}^{k} P_{-1} + zeta_{3m}^{-k} P_1.
template <int M, int E, int G>
__global__ void __launch_bounds__(Cfg2<M, E, G>::THREADS, Cfg2<M, E, G>::MINB)
k_hconv_rows2(double2* __restrict__ f, double2* __restrict__ g, long nrows, const double2* __restrict__ twM,
              const double2* __restrict__ tw3M) {
  pdl_entry();
  using C = Cfg2<M, E, G>;
  constexpr int T = C::T;
  extern __shared__ __align__(16) double2 smem[];
  const int grp = threadIdx.x / T, t = threadIdx.x - grp * T;
  double2* xb = smem + grp * (C::XB + M + (M + 1) / 2);
  double2* QS = xb + C::XB;
  double* P0S = reinterpret_cast<double*>(QS + M);
  const auto sync = row_sync<M, E, G>(grp);
  const double inv = 1.0 / (3.0 * M);
  const double s3 = 0.86602540378443864676372317075294;  // sqrt(3)/2
  for (long row0 = (long)blockIdx.x * G; row0 < nrows; row0 += (long)gridDim.x * G) {
    const long row = row0 + grp;
    if constexpr (C::NAMED) {
      if (row >= nrows) break;
    }
    const bool ok = row < nrows;
    const double2* fr = f + (ok ? row : 0) * (long)M;
    const double2* gr = g + (ok ? row : 0) * (long)M;
    double2 v[E];
#pragma unroll
    for (int rr = 0; rr < 3; ++rr) {
      const int r = rr == 0 ? 0 : (rr == 1 ? 1 : -1);
      const double2 c = make_double2(r == 0 ? 1.0 : -0.5, r == 0 ? 0.0 : (r < 0 ? s3 : -s3));  // zeta_3^{-r}
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int k = t + T * i;
        if (k == 0) {
          v[i] = make_double2(ldv(&fr[0]).x, ldv(&gr[0]).x);                 // w_{0,r} = Re U_0 (AMB-7)
        } else {
          const double2 tz = ldtw(&tw3M[k]);
          const double2 zr = r == 0 ? make_double2(1.0, 0.0) : (r > 0 ? tz : cconj(tz));
          v[i] = herm_pair2(ldv(&fr[k]), ldv(&gr[k]), ldv(&fr[M - k]), ldv(&gr[M - k]), zr, c);
        }
      }
      fft<M, E, +1>(v, t, xb, twM, sync);                      // two c2r in one complex FFT
      if (r == 0) {
#pragma unroll
        for (int i = 0; i < E; ++i) P0S[t + T * i] = v[i].x * v[i].y;
      } else if (r == 1) {
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = make_double2(P0S[t + T * i], v[i].x * v[i].y);
        fft<M, E, -1>(v, t, xb, twM, sync);
#pragma unroll
        for (int i = 0; i < E; ++i) QS[t + T * i] = v[i];
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = make_double2(v[i].x * v[i].y, 0.0);
        fft<M, E, -1>(v, t, xb, twM, sync);
      }
    }
    // separate P_0, P_1 from Q via Q_{m-k}; recombine (Eq. fft0forwardB)
    sync();   // every thread's Q is in QS
    if (ok) {
      double2* fw = f + row * (long)M;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int k = t + T * i;
        const double2 a = QS[k], b = cconj(QS[(M - k) & (M - 1)]);
        const double2 tz = ldtw(&tw3M[k]);
        const double2 pp0 = cscale(cadd(a, b), 0.5);
        const double2 d = csub(a, b);
        const double2 pp1 = make_double2(0.5 * d.y, -0.5 * d.x);
        const double2 h = cadd(cadd(pp0, cmul(v[i], tz)), cmulc(pp1, tz));
        fw[k] = cscale(h, inv);
      }
    }
    sync();
  }
}

// ====================================================================== K4 ==
// Centered Hermitian ternary convolution, N = 4m, four residues of size m
// (see conv1d.cu and DESIGN.md "tconv with four residues").
template <int M, int E, int G>
__global__ void __launch_bounds__(Cfg2<M, E, G>::THREADS, Cfg2<M, E, G>::MINB)
k_tconv_rows2(double2* __restrict__ f, double2* __restrict__ g, double2* __restrict__ h, long nrows,
              const double2* __restrict__ twM, const double2* __restrict__ tw4M) {
  pdl_entry();
  using C = Cfg2<M, E, G>;
  constexpr int T = C::T;
  extern __shared__ __align__(16) double2 smem[];
  const int grp = threadIdx.x / T, t = threadIdx.x - grp * T;
  double2* xb = smem + grp * (C::XB + 2 * M);
  double2* AP = xb + C::XB;
  double2* ACC = AP + M;
  const auto sync = row_sync<M, E, G>(grp);
  const double inv = 1.0 / (4.0 * M);
  for (long row0 = (long)blockIdx.x * G; row0 < nrows; row0 += (long)gridDim.x * G) {
    const long row = row0 + grp;
    if constexpr (C::NAMED) {
      if (row >= nrows) break;
    }
    const bool ok = row < nrows;
    const double2* fr = f + (ok ? row : 0) * (long)M;
    const double2* gr = g + (ok ? row : 0) * (long)M;
    const double2* hr = h + (ok ? row : 0) * (long)M;
    double2 v[E];
#pragma unroll
    for (int r0 = 0; r0 < 4; r0 += 2) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int r = r0 + s;
        const double2 c = r == 0 ? make_double2(1, 0) : r == 1 ? make_double2(0, -1) : r == 2 ? make_double2(-1, 0)
                                                                                    : make_double2(0, 1);  // (-i)^r
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int k = t + T * i;
          if (k == 0) v[i] = make_double2(ldv(&fr[0]).x, ldv(&gr[0]).x);
          else v[i] = herm_pair2(ldv(&fr[k]), ldv(&gr[k]), ldv(&fr[M - k]), ldv(&gr[M - k]), ldtw(&tw4M[r * k]), c);
        }
        fft<M, E, +1>(v, t, xb, twM, sync);
#pragma unroll
        for (int i = 0; i < E; ++i) {
          if (s == 0) AP[t + T * i].x = v[i].x * v[i].y;
          else AP[t + T * i].y = v[i].x * v[i].y;
        }
      }
      {  // h packed across the residue pair: w^h_r + i w^h_{r+1}
        const double2 c0 = r0 == 0 ? make_double2(1, 0) : make_double2(-1, 0);
        const double2 c1 = r0 == 0 ? make_double2(0, -1) : make_double2(0, 1);
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int k = t + T * i;
          if (k == 0) {
            v[i] = make_double2(ldv(&hr[0]).x, ldv(&hr[0]).x);
          } else {
            const double2 hk = ldv(&hr[k]), hm = cconj(ldv(&hr[M - k]));
            const double2 w0 = cmul(ldtw(&tw4M[r0 * k]), cadd(hk, cmul(c0, hm)));
            const double2 w1 = cmul(ldtw(&tw4M[(r0 + 1) * k]), cadd(hk, cmul(c1, hm)));
            v[i] = make_double2(w0.x - w1.y, w0.y + w1.x);
          }
        }
      }
      fft<M, E, +1>(v, t, xb, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const double2 a = AP[t + T * i];
        v[i] = make_double2(a.x * v[i].x, a.y * v[i].y);
      }
      fft<M, E, -1>(v, t, xb, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) xb[t + T * i] = v[i];
      sync();
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int k = t + T * i;
        const double2 a = v[i], b = cconj(xb[(M - k) & (M - 1)]);
        const double2 pp0 = cscale(cadd(a, b), 0.5);
        const double2 d = csub(a, b);
        const double2 pp1 = make_double2(0.5 * d.y, -0.5 * d.x);
        const double2 ct = cadd(cmulc(pp0, ldtw(&tw4M[r0 * k])), cmulc(pp1, ldtw(&tw4M[(r0 + 1) * k])));
        ACC[k] = r0 == 0 ? ct : cadd(ACC[k], ct);
      }
      sync();
    }
    if (ok) {
      double2* fw = f + row * (long)M;
#pragma unroll
      for (int i = 0; i < E; ++i) fw[t + T * i] = cscale(ACC[t + T * i], inv);
    }
  }
}

// ================================================================ launchers ==
namespace {

template <class K>
cudaError_t launch2(K kernel, int threads, size_t smem, long nrows, int groups, cudaStream_t s, void** args,
                    const char* tag, int m) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  long need = (nrows + groups - 1) / groups;
  long grid = (long)num_sms() * per_sm;
  if (need < grid) grid = need;
  if (grid < 1) grid = 1;
  return launch_kernel((const void*)kernel, dim3((unsigned)grid), dim3(threads), args, smem, s, {tag, m, nrows});
}

// elements per thread and rows per CTA of the v2 kernels
// E = 8 for m <= 512 (three radix-8 passes at 512; 5-9% faster there),
// 16 from 1024 up (three passes instead of four)
template <int M>
struct Tune {
  static constexpr int E = M < IDC_ROWS_E ? M : (M <= 512 ? 8 : IDC_ROWS_E);
  static constexpr int T = M / E;
  static constexpr int G = M == 512 ? IDC_K2_G512 : (T >= IDC_ROWS_CTA_THREADS ? 1 : IDC_ROWS_CTA_THREADS / T);
};

}  // namespace

template <int M>
cudaError_t cconv_rows2(double2* f, double2* g, long nrows, cudaStream_t s, RowSets rs) {
  constexpr int E = Tune<M>::E, G = Tune<M>::G;
  using C = Cfg2<M, E, G>;
  const double2* twM = pass_table(M, Tune<M>::E);
  const double2* tw2M = zeta_table(2 * M);
  if (!twM || !tw2M) return cudaErrorMemoryAllocation;
  void* args[] = {&f, &g, &nrows, &twM, &tw2M, &rs};
  // staged f, g rows (m <= IDC_ROWS2_TMA_MAX) + exchange buffer(s) + mbarriers
  constexpr size_t per = K2Layout<M, E>::PER;
  static_assert((size_t)G * per * 16 + (size_t)G * 8 <= 227 * 1024, "K2 configuration exceeds shared memory");
  return launch2(k_cconv_rows2<M, E, G>, C::THREADS, (size_t)G * per * 16 + (size_t)G * 8, nrows, G, s, args, "K2", M);
}

template <int M>
cudaError_t hconv_rows2(double2* f, double2* g, long nrows, cudaStream_t s) {
  constexpr int E = Tune<M>::E, G = Tune<M>::G;
  using C = Cfg2<M, E, G>;
  const double2* twM = pass_table(M, Tune<M>::E);
  const double2* tw3M = zeta_table(3 * M);
  if (!twM || !tw3M) return cudaErrorMemoryAllocation;
  void* args[] = {&f, &g, &nrows, &twM, &tw3M};
  return launch2(k_hconv_rows2<M, E, G>, C::THREADS, (size_t)G * (C::XB + M + (M + 1) / 2) * 16, nrows, G, s,
                 args, "K3", M);
}

template <int M>
cudaError_t tconv_rows2(double2* f, double2* g, double2* h, long nrows, cudaStream_t s) {
  constexpr int E = Tune<M>::E, G = Tune<M>::G;
  using C = Cfg2<M, E, G>;
  const double2* twM = pass_table(M, Tune<M>::E);
  const double2* tw4M = zeta_table(4 * M);
  if (!twM || !tw4M) return cudaErrorMemoryAllocation;
  void* args[] = {&f, &g, &h, &nrows, &twM, &tw4M};
  return launch2(k_tconv_rows2<M, E, G>, C::THREADS, (size_t)G * (C::XB + 2 * M) * 16, nrows, G, s, args, "K4", M);
}

#define IDC_INST2(M)                                                                        \
  template cudaError_t cconv_rows2<M>(double2*, double2*, long, cudaStream_t, RowSets);     \
  template cudaError_t hconv_rows2<M>(double2*, double2*, long, cudaStream_t);              \
  template cudaError_t tconv_rows2<M>(double2*, double2*, double2*, long, cudaStream_t);
IDC_INST2(1)
IDC_INST2(2)
IDC_INST2(4)
IDC_INST2(8)
IDC_INST2(16)
IDC_INST2(32)
IDC_INST2(64)
IDC_INST2(128)
IDC_INST2(256)
IDC_INST2(512)
IDC_INST2(1024)
IDC_INST2(2048)
IDC_INST2(4096)

}  // namespace idc
