// pencils.cu -- outer-dimension ("multivector") implicit padded
// transforms on strided pencils (K5-K8 of SURVEY §2.4).
//
// A pencil is one column x[0..n) of a row-major (rows x ncols) array with
// row stride `ncols` (the x direction of a 2D array, or of a 3D array viewed
// as rows x (my*mz) columns, or the y direction inside one 3D slab).  A CTA
// owns W adjacent columns and all rows: thread (t, c) = threadIdx.x = c + W*t
// holds elements t + T*i (i < E) of column c, so every global access is a run
// of W*16 contiguous bytes per row, and the shared exchange buffer is
// interleaved by column (slot = pos*W + c): eight lanes of a quarter warp
// touch eight consecutive 16-byte slots.
//
//   K5 pad_bwd   Procedure fftpadBackward: even stream in place,
//                odd stream (zeta_{2m}^k shifted) to the work array U.
//   K6 pad_fwd   Procedure fftpadForward: f_k <- (F_k + zeta_{2m}^{-k} U_k)/(2m).
//   K7 pad0_bwd  Eqs. fft0backwardA/B, centered 2m-1 -> 3 streams;
//                listing P:466-487 is garbled (AMB-1), the equations are used.
//   K8 pad0_fwd  Eq. fft0forward: 3m U_k = sum_r zeta_{3m}^{-rk} S_r(k mod m).
// Stream storage of K7/K8 (the paper's layout, AMB-1/AMB-10):
//   r = +1: rows m-1..2m-2 of f;  r = 0: rows 0..m-2 of f and row m of U;
//   r = -1: rows 0..m-1 of U.  (U has m+1 rows.)
#include "config.cuh"
#include "fft_dev.cuh"
#include "launch.cuh"
#include "kernels.cuh"
#include "nd_internal.cuh"
#include "tables.cuh"

namespace idc {

namespace {

template <int N, int E, int W>
struct PCfg {
  static constexpr int T = N / E;
  static constexpr int THREADS = T * W;
  static constexpr int XB = (xbuf_elems<N, E>() > 0 ? xbuf_elems<N, E>() : 1) * W;
};

template <int W>
struct ColSlot {
  int c;
  __device__ __forceinline__ int operator()(int i) const { return i * W + c; }
};

struct Pencil {
  long ncols;        // columns per batch item (row stride of the pencil array)
  long bstride;      // elements between batch items of the input array
  long ustride;      // elements between batch items of the work array U
};

}  // namespace

// ------------------------------------------------------------------- K5 --
template <int N, int E, int W>
__global__ void __launch_bounds__(PCfg<N, E, W>::THREADS)
k_pad_bwd(double2* __restrict__ f, double2* __restrict__ g, double2* __restrict__ U, double2* __restrict__ V,
          Pencil pc, const double2* __restrict__ twN, const double2* __restrict__ tw2N, double2 ophase) {
  pdl_entry();
  using C = PCfg<N, E, W>;
  constexpr int T = C::T;
  extern __shared__ __align__(16) double2 smem[];
  const int c = threadIdx.x % W, t = threadIdx.x / W;
  const long col = (long)blockIdx.x * W + c;
  const bool ok = col < pc.ncols;
  double2* a = (blockIdx.z == 0 ? f : g) + blockIdx.y * pc.bstride + (ok ? col : 0);
  double2* u = (blockIdx.z == 0 ? U : V) + blockIdx.y * pc.ustride + (ok ? col : 0);
  const ColSlot<W> xs{c};
  double2 v[E], x0[E];
#pragma unroll
  for (int i = 0; i < E; ++i) x0[i] = ok ? a[(long)(t + T * i) * pc.ncols] : make_double2(0, 0);
  // odd stream u_{2l+1} = sum_k zeta_m^{lk} zeta_{2m}^k U_k  (Eq. cconv1backward)
#pragma unroll
  for (int i = 0; i < E; ++i) v[i] = cmul(x0[i], cmul(ldtw(&tw2N[t + T * i]), ophase));
  fft<N, E, +1>(v, t, smem, twN, CtaSync{}, xs);
  if (ok) {
#pragma unroll
    for (int i = 0; i < E; ++i) u[(long)(t + T * i) * pc.ncols] = v[i];
  }
  // even stream u_{2l} = sum_k zeta_m^{lk} U_k, in place
  fft<N, E, +1>(x0, t, smem, twN, CtaSync{}, xs);
  if (ok) {
#pragma unroll
    for (int i = 0; i < E; ++i) a[(long)(t + T * i) * pc.ncols] = x0[i];
  }
}

// ------------------------------------------------------------------- K6 --
template <int N, int E, int W>
__global__ void __launch_bounds__(PCfg<N, E, W>::THREADS)
k_pad_fwd(double2* __restrict__ f, const double2* __restrict__ U, Pencil pc, const double2* __restrict__ twN,
          const double2* __restrict__ tw2N, double2 ophase) {
  pdl_entry();
  using C = PCfg<N, E, W>;
  constexpr int T = C::T;
  extern __shared__ __align__(16) double2 smem[];
  const int c = threadIdx.x % W, t = threadIdx.x / W;
  const long col = (long)blockIdx.x * W + c;
  const bool ok = col < pc.ncols;
  double2* a = f + blockIdx.y * pc.bstride + (ok ? col : 0);
  const double2* u = U + blockIdx.y * pc.ustride + (ok ? col : 0);
  const ColSlot<W> xs{c};
  double2 v[E], s[E];
#pragma unroll
  for (int i = 0; i < E; ++i) v[i] = ok ? u[(long)(t + T * i) * pc.ncols] : make_double2(0, 0);
  fft<N, E, -1>(v, t, smem, twN, CtaSync{}, xs);
#pragma unroll
  for (int i = 0; i < E; ++i) s[i] = cmul(cmulc(v[i], ldtw(&tw2N[t + T * i])), ophase);  // c zeta_{2m}^{-k} U_k
#pragma unroll
  for (int i = 0; i < E; ++i) v[i] = ok ? a[(long)(t + T * i) * pc.ncols] : make_double2(0, 0);
  fft<N, E, -1>(v, t, smem, twN, CtaSync{}, xs);
  const double inv = 1.0 / (2.0 * N);
  if (ok) {
#pragma unroll
    for (int i = 0; i < E; ++i) a[(long)(t + T * i) * pc.ncols] = cscale(cadd(v[i], s[i]), inv);
  }
}

// ------------------------------------------------------------------- K7 --
// Centered column of 2N-1 entries (row i holds k = i - (N-1)); N = m.
template <int N, int E, int W>
__global__ void __launch_bounds__(PCfg<N, E, W>::THREADS)
k_pad0_bwd(double2* __restrict__ f, double2* __restrict__ g, double2* __restrict__ U, double2* __restrict__ V,
           Pencil pc, const double2* __restrict__ twN, const double2* __restrict__ tw3N) {
  pdl_entry();
  using C = PCfg<N, E, W>;
  constexpr int T = C::T;
  extern __shared__ __align__(16) double2 smem[];
  const int c = threadIdx.x % W, t = threadIdx.x / W;
  const long col = (long)blockIdx.x * W + c;
  const bool ok = col < pc.ncols;
  double2* a = (blockIdx.z == 0 ? f : g) + blockIdx.y * pc.bstride + (ok ? col : 0);
  double2* u = (blockIdx.z == 0 ? U : V) + blockIdx.y * pc.ustride + (ok ? col : 0);
  const ColSlot<W> xs{c};
  const long S = pc.ncols;
  double2 up[E], un[E], v[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int k = t + T * i;
    up[i] = ok ? a[(long)(N - 1 + k) * S] : make_double2(0, 0);           // U_k
    un[i] = (ok && k > 0) ? a[(long)(k - 1) * S] : make_double2(0, 0);    // U_{k-m}
  }
  const double s3 = 0.86602540378443864676372317075294;
#pragma unroll 1
  for (int rr = 0; rr < 3; ++rr) {
    const int r = rr - 1;  // -1, 0, 1
    const double2 z3 = make_double2(r == 0 ? 1.0 : -0.5, r == 0 ? 0.0 : (r < 0 ? s3 : -s3));  // zeta_3^{-r}
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int k = t + T * i;
      if (k == 0) {
        v[i] = up[i];                                                      // w_{0,r} = U_0
      } else {
        const double2 tz = ldtw(&tw3N[k]);
        const double2 zr = r == 0 ? make_double2(1, 0) : (r > 0 ? tz : cconj(tz));
        v[i] = cmul(zr, cadd(up[i], cmul(z3, un[i])));
      }
    }
    fft<N, E, +1>(v, t, smem, twN, CtaSync{}, xs);
    if (ok) {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int l = t + T * i;
        double2* dst = r == 1 ? a + (long)(N - 1 + l) * S
                     : r == -1 ? u + (long)l * S
                               : (l < N - 1 ? a + (long)l * S : u + (long)N * S);
        *dst = v[i];
      }
    }
  }
}

// ------------------------------------------------------------------- K8 --
template <int N, int E, int W>
__global__ void __launch_bounds__(PCfg<N, E, W>::THREADS)
k_pad0_fwd(double2* __restrict__ f, const double2* __restrict__ U, Pencil pc, const double2* __restrict__ twN,
           const double2* __restrict__ tw3N) {
  pdl_entry();
  using C = PCfg<N, E, W>;
  constexpr int T = C::T;
  extern __shared__ __align__(16) double2 smem[];
  const int c = threadIdx.x % W, t = threadIdx.x / W;
  const long col = (long)blockIdx.x * W + c;
  const bool ok = col < pc.ncols;
  double2* a = f + blockIdx.y * pc.bstride + (ok ? col : 0);
  const double2* u = U + blockIdx.y * pc.ustride + (ok ? col : 0);
  const ColSlot<W> xs{c};
  const long S = pc.ncols;
  const double s3 = 0.86602540378443864676372317075294;
  double2 v[E], ap[E], an[E];
#pragma unroll 1
  for (int rr = 0; rr < 3; ++rr) {
    const int r = rr - 1;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int l = t + T * i;
      const double2* src = r == 1 ? a + (long)(N - 1 + l) * S
                         : r == -1 ? u + (long)l * S
                                   : (l < N - 1 ? a + (long)l * S : u + (long)N * S);
      v[i] = ok ? *src : make_double2(0, 0);
    }
    fft<N, E, -1>(v, t, smem, twN, CtaSync{}, xs);
    // 3m U_k   = sum_r zeta_{3m}^{-rk} S_r(k)            (k = 0..m-1)
    // 3m U_{k-m} = sum_r zeta_{3m}^{-rk} zeta_3^{r} S_r(k) (k = 1..m-1)
    const double2 z3 = make_double2(r == 0 ? 1.0 : -0.5, r == 0 ? 0.0 : (r > 0 ? s3 : -s3));  // zeta_3^{r}
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int k = t + T * i;
      const double2 tz = ldtw(&tw3N[k]);
      const double2 zr = r == 0 ? make_double2(1, 0) : (r > 0 ? cconj(tz) : tz);  // zeta_{3m}^{-rk}
      const double2 p = cmul(zr, v[i]);
      if (rr == 0) {
        ap[i] = p;
        an[i] = cmul(z3, p);
      } else {
        ap[i] = cadd(ap[i], p);
        an[i] = cadd(an[i], cmul(z3, p));
      }
    }
  }
  const double inv = 1.0 / (3.0 * N);
  // all stream reads of this column are done before any output write (barriers inside fft)
  __syncthreads();
  if (ok) {
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int k = t + T * i;
      a[(long)(N - 1 + k) * S] = cscale(ap[i], inv);
      if (k > 0) a[(long)(k - 1) * S] = cscale(an[i], inv);
    }
  }
}

// ================================================================ launchers ==
namespace {

template <int N>
struct PTune {
  static constexpr int E = N < 8 ? N : (N >= 8192 ? 16 : 8);
  static constexpr int T = N / E;
  // W columns per CTA: aim for 512 threads, at least 1, at most 16
  static constexpr int W0 = 512 / T < 1 ? 1 : (512 / T > 16 ? 16 : 512 / T);
  static constexpr int W = W0;
};

template <class K>
cudaError_t launchp(K kernel, int threads, size_t smem, dim3 grid, cudaStream_t s, void** args, const LaunchTag& tag) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_kernel((const void*)kernel, grid, dim3(threads), args, smem, s, tag);
}

template <int N>
cudaError_t pad_bwd_n(double2* f, double2* g, double2* U, double2* V, long ncols, long batch, long bstride,
                      long ustride, cudaStream_t s, double2 ophase) {
  constexpr int E = PTune<N>::E, W = PTune<N>::W;
  using C = PCfg<N, E, W>;
  const double2* twN = pass_table(N, PTune<N>::E);
  const double2* tw2N = zeta_table(2 * N);
  if (!twN || !tw2N) return cudaErrorMemoryAllocation;
  Pencil pc{ncols, bstride, ustride};
  void* args[] = {&f, &g, &U, &V, &pc, &twN, &tw2N, &ophase};
  dim3 grid((unsigned)((ncols + W - 1) / W), (unsigned)batch, g ? 2 : 1);
  return launchp(k_pad_bwd<N, E, W>, C::THREADS, (size_t)C::XB * 16, grid, s, args, {"K5s", N, ncols * batch * (g ? 2 : 1)});
}

template <int N>
cudaError_t pad_fwd_n(double2* f, const double2* U, long ncols, long batch, long bstride, long ustride,
                      cudaStream_t s, double2 ophase) {
  constexpr int E = PTune<N>::E, W = PTune<N>::W;
  using C = PCfg<N, E, W>;
  const double2* twN = pass_table(N, PTune<N>::E);
  const double2* tw2N = zeta_table(2 * N);
  if (!twN || !tw2N) return cudaErrorMemoryAllocation;
  Pencil pc{ncols, bstride, ustride};
  void* args[] = {&f, &U, &pc, &twN, &tw2N, &ophase};
  dim3 grid((unsigned)((ncols + W - 1) / W), (unsigned)batch, 1);
  return launchp(k_pad_fwd<N, E, W>, C::THREADS, (size_t)C::XB * 16, grid, s, args, {"K6s", N, ncols * batch});
}

template <int N>
cudaError_t pad0_bwd_n(double2* f, double2* g, double2* U, double2* V, long ncols, long batch, long bstride,
                       long ustride, cudaStream_t s) {
  constexpr int E = PTune<N>::E, W = PTune<N>::W;
  using C = PCfg<N, E, W>;
  const double2* twN = pass_table(N, PTune<N>::E);
  const double2* tw3N = zeta_table(3 * N);
  if (!twN || !tw3N) return cudaErrorMemoryAllocation;
  Pencil pc{ncols, bstride, ustride};
  void* args[] = {&f, &g, &U, &V, &pc, &twN, &tw3N};
  dim3 grid((unsigned)((ncols + W - 1) / W), (unsigned)batch, g ? 2 : 1);
  return launchp(k_pad0_bwd<N, E, W>, C::THREADS, (size_t)C::XB * 16, grid, s, args, {"K7s", N, ncols * batch * (g ? 2 : 1)});
}

template <int N>
cudaError_t pad0_fwd_n(double2* f, const double2* U, long ncols, long batch, long bstride, long ustride,
                       cudaStream_t s) {
  constexpr int E = PTune<N>::E, W = PTune<N>::W;
  using C = PCfg<N, E, W>;
  const double2* twN = pass_table(N, PTune<N>::E);
  const double2* tw3N = zeta_table(3 * N);
  if (!twN || !tw3N) return cudaErrorMemoryAllocation;
  Pencil pc{ncols, bstride, ustride};
  void* args[] = {&f, &U, &pc, &twN, &tw3N};
  dim3 grid((unsigned)((ncols + W - 1) / W), (unsigned)batch, 1);
  return launchp(k_pad0_fwd<N, E, W>, C::THREADS, (size_t)C::XB * 16, grid, s, args, {"K8s", N, ncols * batch});
}

}  // namespace

#define IDC_PDISPATCH(m, ...)                               \
  switch (m) {                                              \
    case 1: { constexpr int NN = 1; __VA_ARGS__; }          \
    case 2: { constexpr int NN = 2; __VA_ARGS__; }          \
    case 4: { constexpr int NN = 4; __VA_ARGS__; }          \
    case 8: { constexpr int NN = 8; __VA_ARGS__; }          \
    case 16: { constexpr int NN = 16; __VA_ARGS__; }        \
    case 32: { constexpr int NN = 32; __VA_ARGS__; }        \
    case 64: { constexpr int NN = 64; __VA_ARGS__; }        \
    case 128: { constexpr int NN = 128; __VA_ARGS__; }      \
    case 256: { constexpr int NN = 256; __VA_ARGS__; }      \
    case 512: { constexpr int NN = 512; __VA_ARGS__; }      \
    case 1024: { constexpr int NN = 1024; __VA_ARGS__; }    \
    case 2048: { constexpr int NN = 2048; __VA_ARGS__; }    \
    case 4096: { constexpr int NN = 4096; __VA_ARGS__; }    \
    case 8192: { constexpr int NN = 8192; __VA_ARGS__; }    \
    default: break;                                         \
  }

#define IDC_TDISPATCH(m, ...)                                       \
  if (IDC_PENCIL_TMA) switch (m) {                                  \
      case 64: { constexpr int NN = 64; __VA_ARGS__; }              \
      case 128: { constexpr int NN = 128; __VA_ARGS__; }            \
      case 256: { constexpr int NN = 256; __VA_ARGS__; }            \
      case 512: { constexpr int NN = 512; __VA_ARGS__; }            \
      case 1024: { constexpr int NN = 1024; __VA_ARGS__; }          \
      case 2048: { constexpr int NN = 2048; __VA_ARGS__; }          \
      case 4096: { constexpr int NN = 4096; __VA_ARGS__; }          \
      default: break;                                               \
    }

// dl (distributed blocked stream layout, dist.cu): the TMA pencils only; the
// other sizes return cudaErrorNotSupported and dist.cu packs instead
cudaError_t launch_pad_bwd(double2* f, double2* g, double2* U, double2* V, int m, long ncols, long batch,
                           long bstride, long ustride, cudaStream_t s, double2 odd_phase, const DistLayout* dl) {
  IDC_TDISPATCH(m, return pad_bwd_tma<NN>(f, g, U, V, ncols, batch, bstride, ustride, s, odd_phase, dl));
  if (dl) return cudaErrorNotSupported;
  IDC_PDISPATCH(m, return pad_bwd_n<NN>(f, g, U, V, ncols, batch, bstride, ustride, s, odd_phase));
  return cudaErrorInvalidValue;
}
cudaError_t launch_pad_fwd(double2* f, const double2* U, int m, long ncols, long batch, long bstride, long ustride,
                           cudaStream_t s, double2 odd_phase, const DistLayout* dl) {
  IDC_TDISPATCH(m, return pad_fwd_tma<NN>(f, U, ncols, batch, bstride, ustride, s, odd_phase, dl));
  if (dl) return cudaErrorNotSupported;
  IDC_PDISPATCH(m, return pad_fwd_n<NN>(f, U, ncols, batch, bstride, ustride, s, odd_phase));
  return cudaErrorInvalidValue;
}
cudaError_t launch_pad0_bwd(double2* f, double2* g, double2* U, double2* V, int m, long ncols, long batch,
                            long bstride, long ustride, cudaStream_t s, const DistLayout* dl) {
  IDC_TDISPATCH(m, return pad0_bwd_tma<NN>(f, g, U, V, ncols, batch, bstride, ustride, s, dl));
  if (dl) return cudaErrorNotSupported;
  IDC_PDISPATCH(m, return pad0_bwd_n<NN>(f, g, U, V, ncols, batch, bstride, ustride, s));
  return cudaErrorInvalidValue;
}
cudaError_t launch_pad0_fwd(double2* f, const double2* U, int m, long ncols, long batch, long bstride, long ustride,
                            cudaStream_t s, const DistLayout* dl) {
  IDC_TDISPATCH(m, return pad0_fwd_tma<NN>(f, U, ncols, batch, bstride, ustride, s, dl));
  if (dl) return cudaErrorNotSupported;
  IDC_PDISPATCH(m, return pad0_fwd_n<NN>(f, U, ncols, batch, bstride, ustride, s));
  return cudaErrorInvalidValue;
}

}  // namespace idc
