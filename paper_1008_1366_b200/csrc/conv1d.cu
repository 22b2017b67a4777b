// conv1d.cu -- fused 1D implicitly dealiased row convolutions (K2, K3, K4).
//
// One thread group (T = m/E threads) owns one row (one convolution) at a
// time and carries it through the whole method on chip: twiddle-shift into
// residue streams, backward FFTs, pointwise product, forward FFTs,
// recombination and 1/N scaling.  The user's f and g are read from HBM once
// and f is written once: one HBM round trip per convolution (SURVEY §8(a)
// a2-a6).  The 1D work vectors u, v (w) of the paper (P:374-377, P:644-647,
// P:1079-1083) live in registers / shared memory ("stash"), never in HBM,
// except for m = 8192 where the stash spills to the caller's workspace
// (L2-resident).
#define IDC_ROW_UNIT 1   // row kernels: coherent pass-twiddle loads at E >= 16 (fft_dev.cuh)
#include "config.cuh"
#include <atomic>

#include "fft_dev.cuh"
#include "launch.cuh"
#include "kernels.cuh"
#include "tables.cuh"

namespace idc {

namespace {

template <int M>
struct RowCfg {
  static constexpr int E = M < 16 ? M : 16;                 // elements per thread
  static constexpr int T = M / E;                           // threads per row
  static constexpr int G = T >= 256 ? 1 : 256 / T;          // rows (groups) per CTA
  static constexpr int THREADS = G * T;
  static constexpr int XB = xbuf_elems<M, E>() > M ? xbuf_elems<M, E>() : M;  // exchange + mirror buffer
};

// double2 elements of stash per group, and whether it lives in global memory.
template <int M, int STASH>
struct StashCfg {
  static constexpr bool GLOBAL = (RowCfg<M>::XB + STASH) * 16 * RowCfg<M>::G > 200 * 1024;
  static constexpr int SMEM_PER_GROUP = RowCfg<M>::XB + (GLOBAL ? 0 : STASH);
  static constexpr size_t SMEM_BYTES = (size_t)SMEM_PER_GROUP * 16 * RowCfg<M>::G;
};

// Stash sizes (double2 elements per row in flight).
template <int M> constexpr int kCconvStash = 2 * M;  // p0 = u0*v0, zeta^{-k} F1
template <int M> constexpr int kHconvStash = M + M / 2 + (M < 2 ? 1 : 0);  // acc (M) + p0 (M doubles)
template <int M> constexpr int kTconvStash = 2 * M;  // acc (M) + (a_r, a_r') pairs (M)

int g_sms = 0;

}  // namespace

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

int num_sms() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

// ====================================================================== K2 ==
// Function cconv:
//   r = 0: u = fft^{-1}(f), v = fft^{-1}(g), u <- u*v
//   r = 1: f_k, g_k <- zeta_{2m}^k f_k, g_k; v = fft^{-1}(f),
//          f = fft^{-1}(g), v <- v*f
//   f = fft(u), u = fft(v); f_k <- (f_k + zeta_{2m}^{-k} u_k)/(2m)
template <int M, bool GSTASH>
__global__ void __launch_bounds__(RowCfg<M>::THREADS, 1)
k_cconv_rows(double2* __restrict__ f, double2* __restrict__ g, long nrows,
             const double2* __restrict__ twM, const double2* __restrict__ tw2M,
             double2* __restrict__ gwork) {
  pdl_entry();
  using C = RowCfg<M>;
  constexpr int E = C::E, T = C::T, G = C::G;
  extern __shared__ __align__(16) double2 smem[];
  const int grp = threadIdx.x / T, t = threadIdx.x - grp * T;
  constexpr int PER = StashCfg<M, kCconvStash<M>>::SMEM_PER_GROUP;
  double2* xb = smem + grp * PER;
  double2* S1 = GSTASH ? gwork + ((size_t)blockIdx.x * G + grp) * kCconvStash<M> : xb + C::XB;
  double2* S2 = S1 + M;
  CtaSync sync;
  const double inv = 1.0 / (2.0 * M);
  for (long row0 = (long)blockIdx.x * G; row0 < nrows; row0 += (long)gridDim.x * G) {
    const long row = row0 + grp;
    const bool ok = row < nrows;
    const double2* fr = f + (ok ? row : 0) * (long)M;
    const double2* gr = g + (ok ? row : 0) * (long)M;
    double2 v[E];
    // ---- r = 0
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = fr[t + T * i];
    fft<M, E, +1>(v, t, xb, twM, sync);
#pragma unroll
    for (int i = 0; i < E; ++i) S1[t + T * i] = v[i];
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = gr[t + T * i];
    fft<M, E, +1>(v, t, xb, twM, sync);
#pragma unroll
    for (int i = 0; i < E; ++i) S1[t + T * i] = cmul(S1[t + T * i], v[i]);
    // ---- r = 1 (zeta_{2m}^k shift)
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = cmul(fr[t + T * i], ldtw(&tw2M[t + T * i]));
    fft<M, E, +1>(v, t, xb, twM, sync);
#pragma unroll
    for (int i = 0; i < E; ++i) S2[t + T * i] = v[i];
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = cmul(gr[t + T * i], ldtw(&tw2M[t + T * i]));
    fft<M, E, +1>(v, t, xb, twM, sync);
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = cmul(S2[t + T * i], v[i]);
    // ---- forward transforms + recombination
    fft<M, E, -1>(v, t, xb, twM, sync);
#pragma unroll
    for (int i = 0; i < E; ++i) S2[t + T * i] = cmulc(v[i], ldtw(&tw2M[t + T * i]));
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = S1[t + T * i];
    fft<M, E, -1>(v, t, xb, twM, sync);
    if (ok) {
      double2* fw = f + row * (long)M;
#pragma unroll
      for (int i = 0; i < E; ++i) fw[t + T * i] = cscale(cadd(v[i], S2[t + T * i]), inv);
    }
  }
}

// Residue stream of a Hermitian pair packed in one complex vector:
//   Z_k = w^f_{k,r} + i w^g_{k,r},
//   w_{k,r} = zeta_{qm}^{rk} (U_k + zeta_q^{-r} conj U_{m-k})  (k >= 1),  w_{0,r} = Re U_0
// (P:531-537 for q = 3; the same derivation with q = 4 for the ternary case,
// DESIGN.md "tconv with four residues").  `zr` = zeta_{qm}^{rk}, `c` = zeta_q^{-r}.
__device__ __forceinline__ double2 herm_pair(double2 fk, double2 gk, double2 fm, double2 gm, double2 zr, double2 c) {
  // P = f_k + i g_k ; R = conj f_{m-k} + i conj g_{m-k}
  const double2 P = make_double2(fk.x - gk.y, fk.y + gk.x);
  const double2 R = make_double2(fm.x + gm.y, gm.x - fm.y);
  return cmul(zr, cadd(P, cmul(c, R)));
}

// ====================================================================== K3 ==
// Centered Hermitian convolution with N = 3m: for r in {-1,0,1}
// the packed stream w^f_r + i w^g_r is inverse transformed (two c2r in one
// complex FFT, SURVEY a.11), the real product Re*Im is formed, and the
// forward transforms are Eq. fft0forwardB:
//   3m h_k = sum_r zeta_{3m}^{-rk} sum_l zeta_m^{-lk} u_{3l+r},  k = 0..m-1.
// p_{-1} is transformed alone; (p_0, p_1) share one complex FFT and are
// separated with the Hermitian symmetry of real-data spectra.
template <int M, bool GSTASH>
__global__ void __launch_bounds__(RowCfg<M>::THREADS, 1)
k_hconv_rows(double2* __restrict__ f, double2* __restrict__ g, long nrows,
             const double2* __restrict__ twM, const double2* __restrict__ tw3M,
             double2* __restrict__ gwork) {
  pdl_entry();
  using C = RowCfg<M>;
  constexpr int E = C::E, T = C::T, G = C::G;
  extern __shared__ __align__(16) double2 smem[];
  const int grp = threadIdx.x / T, t = threadIdx.x - grp * T;
  constexpr int PER = StashCfg<M, kHconvStash<M>>::SMEM_PER_GROUP;
  double2* xb = smem + grp * PER;
  double2* ACC = GSTASH ? gwork + ((size_t)blockIdx.x * G + grp) * kHconvStash<M> : xb + C::XB;
  double* P0 = reinterpret_cast<double*>(ACC + M);
  CtaSync sync;
  const double inv = 1.0 / (3.0 * M);
  const double s3 = 0.86602540378443864676372317075294;  // sqrt(3)/2
  for (long row0 = (long)blockIdx.x * G; row0 < nrows; row0 += (long)gridDim.x * G) {
    const long row = row0 + grp;
    const bool ok = row < nrows;
    const double2* fr = f + (ok ? row : 0) * (long)M;
    const double2* gr = g + (ok ? row : 0) * (long)M;
    double2 v[E];
#pragma unroll
    for (int rr = 0; rr < 3; ++rr) {
      const int r = rr == 0 ? -1 : (rr == 1 ? 0 : 1);
      const double2 c = make_double2(r == 0 ? 1.0 : -0.5, r == 0 ? 0.0 : (r < 0 ? s3 : -s3));  // zeta_3^{-r}
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int k = t + T * i;
        if (k == 0) {
          v[i] = make_double2(fr[0].x, gr[0].x);
        } else {
          const double2 tz = ldtw(&tw3M[k]);
          const double2 zr = r == 0 ? make_double2(1.0, 0.0) : (r > 0 ? tz : cconj(tz));
          v[i] = herm_pair(fr[k], gr[k], fr[M - k], gr[M - k], zr, c);
        }
      }
      fft<M, E, +1>(v, t, xb, twM, sync);
      if (r == -1) {
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = make_double2(v[i].x * v[i].y, 0.0);
        fft<M, E, -1>(v, t, xb, twM, sync);
#pragma unroll
        for (int i = 0; i < E; ++i) ACC[t + T * i] = cmul(v[i], ldtw(&tw3M[t + T * i]));  // zeta_{3m}^{+k} P_{-1}
      } else if (r == 0) {
#pragma unroll
        for (int i = 0; i < E; ++i) P0[t + T * i] = v[i].x * v[i].y;
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = make_double2(P0[t + T * i], v[i].x * v[i].y);
        fft<M, E, -1>(v, t, xb, twM, sync);
        // separate the two real-data spectra: P0 = (Q_k + conj Q_{m-k})/2, P1 = (Q_k - conj Q_{m-k})/(2i)
#pragma unroll
        for (int i = 0; i < E; ++i) xb[t + T * i] = v[i];
        sync();
        double2 q[E];
#pragma unroll
        for (int i = 0; i < E; ++i) q[i] = xb[(M - (t + T * i)) & (M - 1)];
        sync();
        if (ok) {
          double2* fw = f + row * (long)M;
#pragma unroll
          for (int i = 0; i < E; ++i) {
            const int k = t + T * i;
            const double2 a = v[i], b = cconj(q[i]);
            const double2 p0 = cscale(cadd(a, b), 0.5);
            const double2 d = csub(a, b);
            const double2 p1 = make_double2(0.5 * d.y, -0.5 * d.x);
            const double2 h = cadd(cadd(ACC[k], p0), cmulc(p1, ldtw(&tw3M[k])));
            fw[k] = cscale(h, inv);
          }
        }
      }
    }
  }
}

// ====================================================================== K4 ==
// Centered Hermitian ternary convolution with N = 4m.  The 4m
// padded transform is split at the outermost level into q = 4 residue
// streams of size m, j = 4l + r (the general-padding construction of
// P:693-716 applied to the centered Hermitian data of P:1012-1020; DESIGN.md
// "tconv with four residues"):
//   u_{4l+r} = sum_{k=0}^{m-1} zeta_m^{lk} w_{k,r},
//   w_{k,r} = zeta_{4m}^{rk} (U_k + (-i)^r conj U_{m-k}),  w_{0,r} = Re U_0,
//   4m t_k = sum_{r=0}^{3} zeta_{4m}^{-rk} sum_l zeta_m^{-lk} (u^f u^g u^h)_{4l+r}.
// Residues are processed in pairs (r, r+1): (f,g) packed per residue, h
// packed across the pair, the two real triple products share one forward FFT.
template <int M, bool GSTASH>
__global__ void __launch_bounds__(RowCfg<M>::THREADS, 1)
k_tconv_rows(double2* __restrict__ f, double2* __restrict__ g, double2* __restrict__ h, long nrows,
             const double2* __restrict__ twM, const double2* __restrict__ tw4M,
             double2* __restrict__ gwork) {
  pdl_entry();
  using C = RowCfg<M>;
  constexpr int E = C::E, T = C::T, G = C::G;
  extern __shared__ __align__(16) double2 smem[];
  const int grp = threadIdx.x / T, t = threadIdx.x - grp * T;
  constexpr int PER = StashCfg<M, kTconvStash<M>>::SMEM_PER_GROUP;
  double2* xb = smem + grp * PER;
  double2* ACC = GSTASH ? gwork + ((size_t)blockIdx.x * G + grp) * kTconvStash<M> : xb + C::XB;
  double2* AP = ACC + M;  // (a_r, a_{r+1}) products of the f and g streams
  CtaSync sync;
  const double inv = 1.0 / (4.0 * M);
  for (long row0 = (long)blockIdx.x * G; row0 < nrows; row0 += (long)gridDim.x * G) {
    const long row = row0 + grp;
    const bool ok = row < nrows;
    const double2* fr = f + (ok ? row : 0) * (long)M;
    const double2* gr = g + (ok ? row : 0) * (long)M;
    const double2* hr = h + (ok ? row : 0) * (long)M;
    double2 v[E];
#pragma unroll 1
    for (int r0 = 0; r0 < 4; r0 += 2) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int r = r0 + s;
        // (-i)^r
        const double2 c = r == 0 ? make_double2(1, 0) : r == 1 ? make_double2(0, -1) : r == 2 ? make_double2(-1, 0)
                                                                                    : make_double2(0, 1);
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int k = t + T * i;
          if (k == 0) v[i] = make_double2(fr[0].x, gr[0].x);
          else v[i] = herm_pair(fr[k], gr[k], fr[M - k], gr[M - k], ldtw(&tw4M[r * k]), c);
        }
        fft<M, E, +1>(v, t, xb, twM, sync);
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const double a = v[i].x * v[i].y;
          if (s == 0) AP[t + T * i].x = a;
          else AP[t + T * i].y = a;
        }
      }
      // h: w^h_r + i w^h_{r+1}
      {
        const int r = r0;
        const double2 c0 = r == 0 ? make_double2(1, 0) : make_double2(-1, 0);   // (-i)^r, r in {0, 2}
        const double2 c1 = r == 0 ? make_double2(0, -1) : make_double2(0, 1);   // (-i)^{r+1}
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int k = t + T * i;
          if (k == 0) {
            v[i] = make_double2(hr[0].x, hr[0].x);
          } else {
            const double2 hk = hr[k], hm = cconj(hr[M - k]);
            const double2 w0 = cmul(ldtw(&tw4M[r * k]), cadd(hk, cmul(c0, hm)));
            const double2 w1 = cmul(ldtw(&tw4M[(r + 1) * k]), cadd(hk, cmul(c1, hm)));
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
      double2 q[E];
#pragma unroll
      for (int i = 0; i < E; ++i) q[i] = xb[(M - (t + T * i)) & (M - 1)];
      sync();
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int k = t + T * i;
        const double2 a = v[i], b = cconj(q[i]);
        const double2 p0 = cscale(cadd(a, b), 0.5);
        const double2 d = csub(a, b);
        const double2 p1 = make_double2(0.5 * d.y, -0.5 * d.x);
        const double2 contrib = cadd(cmulc(p0, ldtw(&tw4M[r0 * k])), cmulc(p1, ldtw(&tw4M[(r0 + 1) * k])));
        ACC[k] = r0 == 0 ? contrib : cadd(ACC[k], contrib);
      }
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
cudaError_t launch_persistent(K kernel, int threads, size_t smem, long nrows, int groups, cudaStream_t s,
                              void** args, const char* tag, int m) {
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

template <int M>
size_t grid_cap() {
  return (size_t)num_sms();  // global-stash variants run with one CTA per SM
}

template <int M>
cudaError_t cconv_m(double2* f, double2* g, long nrows, double2* work, cudaStream_t s) {
  using C = RowCfg<M>;
  using SC = StashCfg<M, kCconvStash<M>>;
  const double2* twM = pass_table(M, RowCfg<M>::E);
  const double2* tw2M = zeta_table(2 * M);
  if (!twM || !tw2M) return cudaErrorMemoryAllocation;
  void* args[] = {&f, &g, &nrows, &twM, &tw2M, &work};
  return launch_persistent(k_cconv_rows<M, SC::GLOBAL>, C::THREADS, SC::SMEM_BYTES, nrows, C::G, s, args, "K2v1", M);
}

template <int M>
cudaError_t hconv_m(double2* f, double2* g, long nrows, double2* work, cudaStream_t s) {
  using C = RowCfg<M>;
  using SC = StashCfg<M, kHconvStash<M>>;
  const double2* twM = pass_table(M, RowCfg<M>::E);
  const double2* tw3M = zeta_table(3 * M);
  if (!twM || !tw3M) return cudaErrorMemoryAllocation;
  void* args[] = {&f, &g, &nrows, &twM, &tw3M, &work};
  return launch_persistent(k_hconv_rows<M, SC::GLOBAL>, C::THREADS, SC::SMEM_BYTES, nrows, C::G, s, args, "K3v1", M);
}

template <int M>
cudaError_t tconv_m(double2* f, double2* g, double2* h, long nrows, double2* work, cudaStream_t s) {
  using C = RowCfg<M>;
  using SC = StashCfg<M, kTconvStash<M>>;
  const double2* twM = pass_table(M, RowCfg<M>::E);
  const double2* tw4M = zeta_table(4 * M);
  if (!twM || !tw4M) return cudaErrorMemoryAllocation;
  void* args[] = {&f, &g, &h, &nrows, &twM, &tw4M, &work};
  return launch_persistent(k_tconv_rows<M, SC::GLOBAL>, C::THREADS, SC::SMEM_BYTES, nrows, C::G, s, args, "K4v1", M);
}

template <int M, int STASH>
size_t stash_bytes() {
  using SC = StashCfg<M, STASH>;
  return SC::GLOBAL ? (size_t)num_sms() * RowCfg<M>::G * STASH * sizeof(double2) : 0;
}

}  // namespace

#define IDC_DISPATCH_M(m, ...)           \
  switch (m) {                           \
    case 1: { constexpr int MM = 1; __VA_ARGS__; } \
    case 2: { constexpr int MM = 2; __VA_ARGS__; } \
    case 4: { constexpr int MM = 4; __VA_ARGS__; } \
    case 8: { constexpr int MM = 8; __VA_ARGS__; } \
    case 16: { constexpr int MM = 16; __VA_ARGS__; } \
    case 32: { constexpr int MM = 32; __VA_ARGS__; } \
    case 64: { constexpr int MM = 64; __VA_ARGS__; } \
    case 128: { constexpr int MM = 128; __VA_ARGS__; } \
    case 256: { constexpr int MM = 256; __VA_ARGS__; } \
    case 512: { constexpr int MM = 512; __VA_ARGS__; } \
    case 1024: { constexpr int MM = 1024; __VA_ARGS__; } \
    case 2048: { constexpr int MM = 2048; __VA_ARGS__; } \
    case 4096: { constexpr int MM = 4096; __VA_ARGS__; } \
    case 8192: { constexpr int MM = 8192; __VA_ARGS__; } \
    default: break;                      \
  }


// The v1 kernels of this file (global-memory stash) serve m = 8192 only: up to
// 4096 the register-resident rows2.cu / TMA-staged rows3.cu kernels run.
constexpr int kV1M = 8192;
size_t cconv_rows_work_bytes(int m) { return m == kV1M ? stash_bytes<kV1M, kCconvStash<kV1M>>() : 0; }
size_t hconv_rows_work_bytes(int m) { return m == kV1M ? stash_bytes<kV1M, kHconvStash<kV1M>>() : 0; }
size_t tconv_rows_work_bytes(int m) { return m == kV1M ? stash_bytes<kV1M, kTconvStash<kV1M>>() : 0; }

cudaError_t launch_cconv_rows(double2* f, double2* g, int m, long nrows, double2* work, cudaStream_t s) {
  if (m <= IDC_V2_MAX_M) { IDC_DISPATCH_M(m, return cconv_rows2<MM>(f, g, nrows, s)); }
  if (m == kV1M) return cconv_m<kV1M>(f, g, nrows, work, s);
  return cudaErrorInvalidValue;
}
cudaError_t launch_hconv_rows(double2* f, double2* g, int m, long nrows, double2* work, cudaStream_t s) {
  if (m >= IDC_V3_MIN_M && m <= 4096) {
    switch (m) {
      case 512: return hconv_rows3<512>(f, g, nrows, s);
      case 1024: return hconv_rows3<1024>(f, g, nrows, s);
      case 2048: return hconv_rows3<2048>(f, g, nrows, s);
      case 4096: return hconv_rows3<4096>(f, g, nrows, s);
    }
  }
  if (m <= IDC_V2_MAX_M) { IDC_DISPATCH_M(m, return hconv_rows2<MM>(f, g, nrows, s)); }
  if (m == kV1M) return hconv_m<kV1M>(f, g, nrows, work, s);
  return cudaErrorInvalidValue;
}
cudaError_t launch_tconv_rows(double2* f, double2* g, double2* h, int m, long nrows, double2* work,
                              cudaStream_t s) {
  if (m >= IDC_V3_MIN_M && m <= 4096) {
    switch (m) {
      case 512: return tconv_rows3<512>(f, g, h, nrows, s);
      case 1024: return tconv_rows3<1024>(f, g, h, nrows, s);
      case 2048: return tconv_rows3<2048>(f, g, h, nrows, s);
      case 4096: return tconv_rows3<4096>(f, g, h, nrows, s);
    }
  }
  if (m <= IDC_V2_MAX_M) { IDC_DISPATCH_M(m, return tconv_rows2<MM>(f, g, h, nrows, s)); }
  if (m == kV1M) return tconv_m<kV1M>(f, g, h, nrows, work, s);
  return cudaErrorInvalidValue;
}

// Both residue-stream row sets of an outer transform in one launch where the
// kernel supports it (K2 rows2, K3 rows3), two launches otherwise.
cudaError_t launch_cconv_rows_sets(double2* f, double2* g, long n0, double2* f1, double2* g1, long n1, int m,
                                   double2* work, cudaStream_t s) {
  RowSets rs{f1, g1, n0};
  if (m <= IDC_V2_MAX_M) { IDC_DISPATCH_M(m, return cconv_rows2<MM>(f, g, n0 + n1, s, rs)); }
  cudaError_t e = launch_cconv_rows(f, g, m, n0, work, s);
  return e != cudaSuccess ? e : launch_cconv_rows(f1, g1, m, n1, work, s);
}
cudaError_t launch_hconv_rows_sets(double2* f, double2* g, long n0, double2* f1, double2* g1, long n1, int m,
                                   double2* work, cudaStream_t s) {
  RowSets rs{f1, g1, n0};
  if (m >= IDC_V3_MIN_M && m <= 4096) {
    switch (m) {
      case 512: return hconv_rows3<512>(f, g, n0 + n1, s, rs);
      case 1024: return hconv_rows3<1024>(f, g, n0 + n1, s, rs);
      case 2048: return hconv_rows3<2048>(f, g, n0 + n1, s, rs);
      case 4096: return hconv_rows3<4096>(f, g, n0 + n1, s, rs);
    }
  }
  cudaError_t e = launch_hconv_rows(f, g, m, n0, work, s);
  return e != cudaSuccess ? e : launch_hconv_rows(f1, g1, m, n1, work, s);
}

}  // namespace idc
