// rows3.cu -- Hermitian / ternary 1D row convolutions with TMA-staged rows.
//
// Same equations as conv1d.cu / rows2.cu (K3: centered Hermitian with three
// residues; K4: ternary with four residues, P:1007-1034 and
// DESIGN.md "tconv with four residues").  What changes is the data flow:
//
//   * each row group stages its f and g rows in shared memory with one TMA
//     bulk copy per row (cp.async.bulk + mbarrier), so the residue split
//     w_{k,r} = zeta^{rk}(U_k + c_r conj U_{m-k}) reads U_k and the mirror
//     U_{m-k} from shared memory instead of re-reading L2 once per residue;
//   * as soon as the last residue split of a row has read the staged row the
//     group issues the bulk copy of its NEXT row, which then lands while the
//     remaining transforms of the current row run;
//   * the cross-transform state (p0 and the packed (p0, p1) spectrum Q of
//     hconv; the f*g stream products of tconv) lives in registers; tconv
//     parks the first residue pair's partial sum in the (already staged)
//     global f row and finishes it with the second pair.
#define IDC_ROW_UNIT 1   // row kernels: coherent pass-twiddle loads at E >= 16 (fft_dev.cuh)
#include "config.cuh"
#include "fft_dev.cuh"
#include "launch.cuh"
#include "kernels.cuh"
#include "tables.cuh"
#include "tma.cuh"

// K3: elements per thread up to which all three residue streams come from one
// read of the staged row (the r = -1 stream held in registers)

namespace idc {

namespace {

// H: K3 (true) or K4 (false); they differ only in the row groups per CTA at m <= 512
template <int M, bool H = true>
struct Cfg3 {
  static constexpr int E = M <= IDC_ROWS3_E8_MAX ? 8 : 16;   // 8 at m = 512 (measured 8% faster there)
  static constexpr int T = M / E;
  // row groups per CTA: at m <= 512 K3 runs 6 (12 warps per SM at 168
  // registers: hconv1d 512 0.569 -> 0.537 ms, hconv3d 55.5 -> 54.4 ms), K4
  // keeps 4 (6 groups spill 88 bytes: tconv1d 512 +5%; profiles/r02/ab/rows3_groups_512.log)
  static constexpr int G = M <= 512 ? (H ? IDC_K3_G512 : IDC_K4_G512) : (T >= 256 ? 1 : 256 / T);
  static constexpr int THREADS = G * T;
  static constexpr int XB = xbuf_elems<M, E>() > M ? xbuf_elems<M, E>() : M;
  // K3 pairs independent transforms with staggered exchanges (fft2s) where a
  // second exchange buffer fits: m <= IDC_K3_STAGGER_MAX_M
  static constexpr bool STAG = M <= IDC_K3_STAGGER_MAX_M;
  static constexpr int PER = 2 * M + (STAG ? 2 : 1) * XB;   // staged f, g + exchange buffer(s) (double2)
  static constexpr size_t SMEM = (size_t)G * PER * 16 + (size_t)G * 16;  // + one mbarrier per group
  static constexpr bool NAMED = G > 1;
  static constexpr int MINB = M <= 512 ? IDC_ROWS3_MINB_SMALL : 1;   // CTAs per SM (register cap)
};

template <bool NAMED>
struct Sync3;
template <>
struct Sync3<true> {
  int id, n;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
};
template <>
struct Sync3<false> {
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync 0;" ::: "memory"); }
};

template <int M, bool H = true>
__device__ __forceinline__ Sync3<Cfg3<M, H>::NAMED> sync3(int grp) {
  if constexpr (Cfg3<M, H>::NAMED) return Sync3<true>{1 + grp, Cfg3<M, H>::T};
  else return Sync3<false>{};
}

// packed residue stream of the staged pair (f, g) at k >= 1:
// Z = zr (P_k + c R_{m-k}),  P = f_k + i g_k,  R = conj f_{m-k} + i conj g_{m-k}
__device__ __forceinline__ double2 zpair(const double2* F, const double2* Gs, int k, int mk, double2 zr, double2 c) {
  const double2 fk = F[k], gk = Gs[k], fm = F[mk], gm = Gs[mk];
  const double2 P = make_double2(fk.x - gk.y, fk.y + gk.x);
  const double2 R = make_double2(fm.x + gm.y, gm.x - fm.y);
  return cmul(zr, cadd(P, cmul(c, R)));
}

}  // namespace

// ====================================================================== K3 ==
template <int M>
__global__ void __launch_bounds__(Cfg3<M>::THREADS, Cfg3<M>::MINB)
k_hconv_rows3(double2* __restrict__ f, double2* __restrict__ g, long nrows, const double2* __restrict__ twM,
              const double2* __restrict__ tw3M, RowSets rs) {
  pdl_entry();
  using C = Cfg3<M>;
  constexpr int E = C::E, T = C::T, G = C::G;
  extern __shared__ __align__(128) double2 smem[];
  const int grp = threadIdx.x / T, t = threadIdx.x - grp * T;
  double2* F = smem + grp * C::PER;
  double2* Gs = F + M;
  double2* xb = Gs + M;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + G * C::PER) + grp;
  const auto sync = sync3<M>(grp);
  const long stride = (long)gridDim.x * G;
  long row = (long)blockIdx.x * G + grp;
  if (t == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (t == 0 && row < nrows) {
    mbar_arrive_expect_tx(bar, 2u * M * 16u);
    tma_load_1d(F, row_ptr(f, rs.f1, rs.n0, row, M), M * 16u, bar);
    tma_load_1d(Gs, row_ptr(g, rs.g1, rs.n0, row, M), M * 16u, bar);
  }
  const double inv = 1.0 / (3.0 * M);
  const double s3 = 0.86602540378443864676372317075294;  // sqrt(3)/2
  uint32_t phase = 0;
  for (; row < nrows; row += stride) {
    mbar_wait(bar, phase);
    phase ^= 1;
    double2 v[E], Q[E];
    double p0[E];
    // ONE: all three residue streams from one read of the staged pair, the
    // r = -1 stream kept in registers (at E = 16 spill-free since the E = 16
    // rows reload pass twiddles per pass: hconv1d 4096 0.437 -> 0.419 ms,
    // hconv2d 4095 x 2048 0.600 -> 0.584 ms, profiles/r02/ab/k3_one_split_e16.log);
    // halves the split's shared-memory wavefronts and frees the stage for
    // the next row's bulk copy before the first transform
    constexpr bool ONE = E <= IDC_K3_ONE_SPLIT_MAXE;
    double2 Vm[ONE ? E : 1];
    // residues r = 0 and r = 1 (and r = -1) from ONE read of the staged pair
    // (P:531-537): P_k = f_k + i g_k, R_k = conj f_{m-k} + i conj g_{m-k};
    // v = P + R (r = 0), Q = zeta_{3m}^{k} (P + zeta_3^{-1} R) (r = 1),
    // Vm = zeta_{3m}^{-k} (P + zeta_3 R) (r = -1); with A = P - R/2 and
    // B = i (sqrt 3 / 2) R: P + zeta_3^{-1} R = A - B, P + zeta_3 R = A + B
    for_roots<3 * E, 1, +1, E>(ldtw(&tw3M[t]), [&](int i, double2 zr) {
      const int k = t + T * i;
      if (i == 0 && t == 0) {
        v[i] = Q[i] = make_double2(F[0].x, Gs[0].x);              // w_{0,r} = Re U_0 (AMB-7)
        if constexpr (ONE) Vm[i] = v[i];
      } else {
        const double2 fk = F[k], gk = Gs[k], fm = F[M - k], gm = Gs[M - k];
        const double2 P = make_double2(fk.x - gk.y, fk.y + gk.x);
        const double2 R = make_double2(fm.x + gm.y, gm.x - fm.y);
        v[i] = cadd(P, R);
        const double2 A = make_double2(fma(-0.5, R.x, P.x), fma(-0.5, R.y, P.y));
        const double2 B = make_double2(-s3 * R.y, s3 * R.x);
        Q[i] = cmul(zr, csub(A, B));
        if constexpr (ONE) Vm[i] = cmulc(cadd(A, B), zr);          // conj(zeta^k) (A + B)
      }
    });
    // STAGF (no room for a second exchange buffer): the first pair of
    // transforms runs staggered with the just-consumed stage as its second
    // buffer, and the next row's copies are issued after that pair
    // (m >= IDC_K3_STAGE_AS_XB: hconv1d 4096 0.428 -> 0.415 ms, hconv2d
    // 4095 x 2048 0.558 -> 0.554 ms; m = 1024 within noise, off;
    // profiles/r02/ab/k3_stage_as_xb.log)
    constexpr bool STAGF = ONE && !C::STAG && IDC_K3_STAGE_AS_XB > 0 && M >= IDC_K3_STAGE_AS_XB && 2 * M >= C::XB;
    auto refill_next = [&]() {
      sync();
      if (t == 0 && row + stride < nrows) {
        mbar_arrive_expect_tx(bar, 2u * M * 16u);
        tma_load_1d(F, row_ptr(f, rs.f1, rs.n0, row + stride, M), M * 16u, bar);
        tma_load_1d(Gs, row_ptr(g, rs.g1, rs.n0, row + stride, M), M * 16u, bar);
      }
    };
    if constexpr (ONE && !STAGF) refill_next();
    if constexpr (STAGF) {
      sync();                                                   // every thread's split read of the stage done
      fft2s<M, E, +1>(v, Q, t, xb, F, twM, sync);               // two c2r pairs, residues 0 and 1
#pragma unroll
      for (int i = 0; i < E; ++i) Q[i] = make_double2(v[i].x * v[i].y, Q[i].x * Q[i].y);
      fence_proxy_async_smem();                                 // generic writes to the stage before the TMA refill
      refill_next();                                            // the stage's last use as a buffer is over
      fft<M, E, -1>(Q, t, xb, twM, sync);                       // Q = fft(p_0 + i p_1)
      fft<M, E, +1>(Vm, t, xb, twM, sync);                      // r = -1 pair
#pragma unroll
      for (int i = 0; i < E; ++i) v[i] = make_double2(Vm[i].x * Vm[i].y, 0.0);
    } else if constexpr (C::STAG && ONE) {
      // five transforms as two staggered pairs and one single: (v, Q)
      // backward; (Q forward, r = -1 stream backward); P_{-1} forward
      double2* xb2 = xb + C::XB;
      fft2s<M, E, +1>(v, Q, t, xb, xb2, twM, sync);             // two c2r pairs, residues 0 and 1
#pragma unroll
      for (int i = 0; i < E; ++i) Q[i] = make_double2(v[i].x * v[i].y, Q[i].x * Q[i].y);
      fft2s<M, E, -1, +1>(Q, Vm, t, xb, xb2, twM, sync);         // Q = fft(p_0 + i p_1); r = -1 pair
#pragma unroll
      for (int i = 0; i < E; ++i) v[i] = make_double2(Vm[i].x * Vm[i].y, 0.0);
    } else {
    fft<M, E, +1>(v, t, xb, twM, sync);                         // two c2r in one complex FFT
#pragma unroll
    for (int i = 0; i < E; ++i) p0[i] = v[i].x * v[i].y;
    fft<M, E, +1>(Q, t, xb, twM, sync);
#pragma unroll
    for (int i = 0; i < E; ++i) Q[i] = make_double2(p0[i], Q[i].x * Q[i].y);
    fft<M, E, -1>(Q, t, xb, twM, sync);                         // Q = fft(p_0 + i p_1)
    if constexpr (ONE) {
#pragma unroll
      for (int i = 0; i < E; ++i) v[i] = Vm[i];
    } else {
      // r = -1: the last read of the staged row, then the next row's bulk copy
      const double2 cm = make_double2(-0.5, s3);                // zeta_3^{+1}
      for_roots<3 * E, 1, -1, E>(cconj(ldtw(&tw3M[t])), [&](int i, double2 zr) {
        if (i == 0 && t == 0) v[i] = make_double2(F[0].x, Gs[0].x);
        else v[i] = zpair(F, Gs, t + T * i, M - t - T * i, zr, cm);
      });
      sync();
      if (t == 0 && row + stride < nrows) {
        mbar_arrive_expect_tx(bar, 2u * M * 16u);
        tma_load_1d(F, row_ptr(f, rs.f1, rs.n0, row + stride, M), M * 16u, bar);
        tma_load_1d(Gs, row_ptr(g, rs.g1, rs.n0, row + stride, M), M * 16u, bar);
      }
    }
    fft<M, E, +1>(v, t, xb, twM, sync);
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = make_double2(v[i].x * v[i].y, 0.0);
    }
    fft<M, E, -1>(v, t, xb, twM, sync);                         // P_{-1}
    // P_0, P_1 from Q via Q_{m-k}; 3m h_k = P_0 + zeta^{k} P_{-1} + zeta^{-k} P_1 (Eq. fft0forwardB)
#pragma unroll
    for (int i = 0; i < E; ++i) xb[t + T * i] = Q[i];
    sync();
    double2* fw = row_ptr(f, rs.f1, rs.n0, row, M);
    auto recombine = [&](int i, double2 tz) {
      const int k = t + T * i;
      const double2 a = Q[i], b = cconj(xb[(M - k) & (M - 1)]);
      const double2 pp0 = cscale(cadd(a, b), 0.5);
      const double2 d = csub(a, b);
      const double2 pp1 = make_double2(0.5 * d.y, -0.5 * d.x);
      fw[k] = cscale(cadd(cadd(pp0, cmul(v[i], tz)), cmulc(pp1, tz)), inv);
    };
    for_roots<3 * E, 1, +1, E>(ldtw(&tw3M[t]), recombine);
    sync();
  }
}

// ====================================================================== K4 ==
template <int M>
__global__ void __launch_bounds__(Cfg3<M, false>::THREADS, Cfg3<M, false>::MINB)
k_tconv_rows3(double2* __restrict__ f, const double2* __restrict__ g, const double2* __restrict__ h, long nrows,
              const double2* __restrict__ twM, const double2* __restrict__ tw4M) {
  pdl_entry();
  using C = Cfg3<M, false>;
  constexpr int E = C::E, T = C::T, G = C::G;
  extern __shared__ __align__(128) double2 smem[];
  const int grp = threadIdx.x / T, t = threadIdx.x - grp * T;
  double2* F = smem + grp * C::PER;
  double2* Gs = F + M;
  double2* xb = Gs + M;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + G * C::PER) + grp;
  const auto sync = sync3<M, false>(grp);
  const long stride = (long)gridDim.x * G;
  long row = (long)blockIdx.x * G + grp;
  if (t == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (t == 0 && row < nrows) {
    mbar_arrive_expect_tx(bar, 2u * M * 16u);
    tma_load_1d(F, f + row * (long)M, M * 16u, bar);
    tma_load_1d(Gs, g + row * (long)M, M * 16u, bar);
  }
  const double inv = 1.0 / (4.0 * M);
  uint32_t phase = 0;
  for (; row < nrows; row += stride) {
    mbar_wait(bar, phase);
    phase ^= 1;
    const double2* hr = h + row * (long)M;
    double2* fw = f + row * (long)M;   // staged: free to serve as the partial-sum scratch
    if (t == 0 && row + stride < nrows) prefetch_l2(h + (row + stride) * (long)M, M * 16u);
    double a0[E], a1[E];
    // Residue pairs (r0, r0 + 1), r0 = 0, 2, in a runtime loop so that the
    // four transforms of a pair are instantiated once (instruction-cache
    // footprint); only the small split / pack / recombine stages are
    // specialised on r0 for their compile-time roots
    // zeta_{4m}^{rk} = zeta_{4m}^{rt} x zeta_{4E}^{ri}, c_r = (-i)^r.
    // (za, zb are re-loaded per stage -- volatile loads -- so that the derived
    // per-element roots are recomputed, not kept live across transforms.)
    double2 v[E], w[E];
    // c_r = (-i)^r = i^{-r} is applied by sign flips / swaps (mul_i); residue
    // r = 0 has no root at all.
    auto split = [&](auto R0) {   // both f/g residue streams of the pair, one read of the staged row
      constexpr int r0 = decltype(R0)::value;
      const double2 za = r0 == 0 ? make_double2(1, 0) : ldtw(&tw4M[r0 * t]);
      const double2 zb = ldtw(&tw4M[(r0 + 1) * t]);
      static_for<E>([&](auto I) {
        constexpr int i = decltype(I)::value;
        const int k = t + T * i;
        if (i == 0 && t == 0) {
          v[i] = w[i] = make_double2(F[0].x, Gs[0].x);            // w_{0,r} = Re U_0 (AMB-7)
        } else {
          const double2 fk = F[k], gk = Gs[k], fm = F[M - k], gm = Gs[M - k];
          const double2 P = make_double2(fk.x - gk.y, fk.y + gk.x);
          const double2 R = make_double2(fm.x + gm.y, gm.x - fm.y);
          const double2 sa = cadd(P, mul_i<-r0>(R));
          if constexpr (r0 == 0) v[i] = sa;
          else v[i] = cmul(twc<r0 * i, 4 * E, +1>(za), sa);
          w[i] = cmul(twc<(r0 + 1) * i, 4 * E, +1>(zb), cadd(P, mul_i<-(r0 + 1)>(R)));
        }
      });
    };
    auto hpack = [&](auto R0) {   // h packed across the pair: w^h_{r0} + i w^h_{r0+1}
      constexpr int r0 = decltype(R0)::value;
      const double2 za = r0 == 0 ? make_double2(1, 0) : ldtw(&tw4M[r0 * t]);
      const double2 zb = ldtw(&tw4M[(r0 + 1) * t]);
      static_for<E>([&](auto I) {
        constexpr int i = decltype(I)::value;
        const int k = t + T * i;
        if (i == 0 && t == 0) {
          const double h0 = ldv(&hr[0]).x;
          v[i] = make_double2(h0, h0);
        } else {
          const double2 hk = ldv(&hr[k]), hm = cconj(ldv(&hr[M - k]));
          double2 w0 = cadd(hk, mul_i<-r0>(hm));
          if constexpr (r0 != 0) w0 = cmul(twc<r0 * i, 4 * E, +1>(za), w0);
          const double2 w1 = cmul(twc<(r0 + 1) * i, 4 * E, +1>(zb), cadd(hk, mul_i<-(r0 + 1)>(hm)));
          v[i] = make_double2(w0.x - w1.y, w0.y + w1.x);
        }
      });
    };
    auto recombine = [&](auto R0) {   // separate the pair's real-data spectra via v_{m-k}
      constexpr int r0 = decltype(R0)::value;
      const double2 za = r0 == 0 ? make_double2(1, 0) : ldtw(&tw4M[r0 * t]);
      const double2 zb = ldtw(&tw4M[(r0 + 1) * t]);
      static_for<E>([&](auto I) {
        constexpr int i = decltype(I)::value;
        const int k = t + T * i;
        const double2 a = v[i], b = cconj(xb[(M - k) & (M - 1)]);
        const double2 pp0 = cscale(cadd(a, b), 0.5);
        const double2 d = csub(a, b);
        const double2 pp1 = make_double2(0.5 * d.y, -0.5 * d.x);
        double2 c0 = pp0;
        if constexpr (r0 != 0) c0 = cmulc(pp0, twc<r0 * i, 4 * E, +1>(za));
        const double2 ct = cadd(c0, cmulc(pp1, twc<(r0 + 1) * i, 4 * E, +1>(zb)));
        if constexpr (r0 == 0) fw[k] = ct;                         // partial sum of residues 0, 1
        else fw[k] = cscale(cadd(ldv(&fw[k]), ct), inv);           // + residues 2, 3, then 1/(4m)
      });
    };
#pragma unroll 1
    for (int r0 = 0; r0 < 4; r0 += 2) {
      if (r0 == 0) split(std::integral_constant<int, 0>{});
      else split(std::integral_constant<int, 2>{});
      if (r0 == 2) {  // last read of the staged row: prefetch the next one
        sync();
        if (t == 0 && row + stride < nrows) {
          mbar_arrive_expect_tx(bar, 2u * M * 16u);
          tma_load_1d(F, f + (row + stride) * (long)M, M * 16u, bar);
          tma_load_1d(Gs, g + (row + stride) * (long)M, M * 16u, bar);
        }
      }
      fft<M, E, +1>(v, t, xb, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) a0[i] = v[i].x * v[i].y;
      fft<M, E, +1>(w, t, xb, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) a1[i] = w[i].x * w[i].y;
      if (r0 == 0) hpack(std::integral_constant<int, 0>{});
      else hpack(std::integral_constant<int, 2>{});
      fft<M, E, +1>(v, t, xb, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) v[i] = make_double2(a0[i] * v[i].x, a1[i] * v[i].y);
      fft<M, E, -1>(v, t, xb, twM, sync);
#pragma unroll
      for (int i = 0; i < E; ++i) xb[t + T * i] = v[i];
      sync();
      if (r0 == 0) recombine(std::integral_constant<int, 0>{});
      else recombine(std::integral_constant<int, 2>{});
      sync();
    }
  }
}

// ================================================================ launchers ==
namespace {
template <class K>
cudaError_t launch3(K kernel, int threads, size_t smem, long nrows, int groups, cudaStream_t s, void** args,
                    const char* tag, int m) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  long need = (nrows + groups - 1) / groups;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  if (per_sm < 1) per_sm = 1;
  long grid = (long)num_sms() * per_sm;
  if (need < grid) grid = need;
  if (grid < 1) grid = 1;
  return launch_kernel((const void*)kernel, dim3((unsigned)grid), dim3(threads), args, smem, s, {tag, m, nrows});
}
}  // namespace

template <int M>
cudaError_t hconv_rows3(double2* f, double2* g, long nrows, cudaStream_t s, RowSets rs) {
  using C = Cfg3<M>;
  const double2* twM = pass_table(M, Cfg3<M>::E);
  const double2* tw3M = zeta_table(3 * M);
  if (!twM || !tw3M) return cudaErrorMemoryAllocation;
  void* args[] = {&f, &g, &nrows, &twM, &tw3M, &rs};
  return launch3(k_hconv_rows3<M>, C::THREADS, C::SMEM, nrows, C::G, s, args, "K3", M);
}

template <int M>
cudaError_t tconv_rows3(double2* f, double2* g, double2* h, long nrows, cudaStream_t s) {
  using C = Cfg3<M, false>;
  const double2* twM = pass_table(M, C::E);
  const double2* tw4M = zeta_table(4 * M);
  if (!twM || !tw4M) return cudaErrorMemoryAllocation;
  void* args[] = {&f, &g, &h, &nrows, &twM, &tw4M};
  return launch3(k_tconv_rows3<M>, C::THREADS, C::SMEM, nrows, C::G, s, args, "K4", M);
}

#define IDC_INST3(M)                                                                        \
  template cudaError_t hconv_rows3<M>(double2*, double2*, long, cudaStream_t, RowSets);     \
  template cudaError_t tconv_rows3<M>(double2*, double2*, double2*, long, cudaStream_t);
IDC_INST3(512)
IDC_INST3(1024)
IDC_INST3(2048)
IDC_INST3(4096)

}  // namespace idc
