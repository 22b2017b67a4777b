// fft_dev.cuh -- fp64 complex FFT codelets for sm_100a (device functions).
//
// The implicit method reduces every padded transform to size-m complex FFTs
// (P:204-205).  This engine computes one such
// FFT per thread group, with the data in registers:
//
//   * a group of T = N/E threads holds one N-point vector; thread t owns
//     elements x[t + T*i], i = 0..E-1 (the "natural strided" distribution);
//   * each pass is a Stockham radix-R step (R = E, the last pass may use a
//     smaller radix): twiddle by exp(+-2 pi i r (j mod Ns)/(Ns R)), an
//     in-register DFT_R, and a permutation through shared memory;
//   * the input of the first pass and the output of the last pass are both
//     in the natural strided distribution, so a backward FFT, a pointwise
//     product ("the scrambled Fourier subtransforms of the two
//     input vectors can be multiplied together as they are produced") and a
//     forward FFT chain in registers with no reordering pass at all;
//   * the exchange buffer is padded (phys = pos + Ns*(pos >> log2(Ns R)))
//     so that both the strided Stockham writes and the unit-stride reads hit
//     eight distinct 16-byte bank groups per quarter warp (conflict-free
//     128-bit shared accesses).
//
// Twiddles come from a per-size table tw[k] = exp(+2 pi i k/N), k < N,
// built on the host in long double (no fp64 sincos on the hot path); the
// forward direction multiplies by the conjugate.  Constant twiddles inside a
// DFT_R (R <= 32) are compile-time immediates; trivial ones (1, +-i, -1) cost
// no arithmetic.
#pragma once
#include <cuda_runtime.h>
#include <utility>

namespace idc {

// ------------------------------------------------------------ complex ops --
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
// Twiddle-table load.  Volatile so the compiler cannot hoist the (loop
// invariant) table reads of every pass of every transform to the top of the
// row loop and keep them all live -- that costs ~90 registers per thread.
// Per-element table loads (zeta_{qm}^{rk} of the residue split / recombination):
// coherent loads, so ptxas cannot hoist these loop-invariant reads out of a
// row loop and hold E x (#residues) complex values live (~200 registers).
__device__ __forceinline__ double2 ldtw(const double2* p) {
  double2 r;
  asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
// Stockham pass twiddles: read-only path (few per pass; ptxas keeps them in
// registers across the row loop) unless a unit defines IDC_PASS_TW_COHERENT
// (reloaded per pass from L1: fewer registers, more L1 traffic).
#ifdef IDC_PASS_TW_COHERENT
__device__ __forceinline__ double2 ldtw_pass(const double2* p) { return ldtw(p); }
#else
__device__ __forceinline__ double2 ldtw_pass(const double2* p) { return __ldg(p); }
#endif
// Data load that the compiler may not merge with an earlier load of the same
// address (the residue loops re-read the row; keeping the first read live
// across transforms would cost 4 registers per element).  L1-cached.
__device__ __forceinline__ double2 ldv(const double2* p) {
  double2 r;
  asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// multiply by w (SIGN > 0) or conj(w) (SIGN < 0)
template <int SIGN>
__device__ __forceinline__ double2 cmul_dir(double2 a, double2 w) {
  if constexpr (SIGN > 0) return cmul(a, w);
  else return cmulc(a, w);
}

// ------------------------------------------------- compile-time twiddles --
// cos(pi j / 16), j = 0..8
__host__ __device__ constexpr double cos16tab(int j) {
  return j == 0 ? 1.0
       : j == 1 ? 0.98078528040323044912618223613424
       : j == 2 ? 0.92387953251128675612818318939679
       : j == 3 ? 0.83146961230254523707878837761791
       : j == 4 ? 0.70710678118654752440084436210485
       : j == 5 ? 0.55557023301960222474283081394853
       : j == 6 ? 0.38268343236508977172845998403040
       : j == 7 ? 0.19509032201612826784828486847702
       : 0.0;
}
// cos(2 pi j / 32) for any integer j
__host__ __device__ constexpr double cos32(int j) {
  return ((j & 31) <= 8)  ? cos16tab(j & 31)
       : ((j & 31) <= 16) ? -cos16tab(16 - (j & 31))
       : ((j & 31) <= 24) ? -cos16tab((j & 31) - 16)
                          : cos16tab(32 - (j & 31));
}
__host__ __device__ constexpr double sin32(int j) { return cos32(j - 8); }

// a * exp(SIGN * 2 pi i K / L), L | 32, resolved at compile time
template <int K, int L, int SIGN>
__device__ __forceinline__ double2 twc(double2 a) {
  constexpr int j = ((K * (32 / L)) % 32 + 32) % 32;
  if constexpr (j == 0) {
    return a;
  } else if constexpr (j == 8) {            // * (SIGN i)
    if constexpr (SIGN > 0) return make_double2(-a.y, a.x);
    else return make_double2(a.y, -a.x);
  } else if constexpr (j == 16) {
    return make_double2(-a.x, -a.y);
  } else if constexpr (j == 24) {           // * (-SIGN i)
    if constexpr (SIGN > 0) return make_double2(a.y, -a.x);
    else return make_double2(-a.y, a.x);
  } else {
    constexpr double c = cos32(j);
    constexpr double s = SIGN > 0 ? sin32(j) : -sin32(j);
    return make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
  }
}

// ----------------------------------------------- in-register DFT_R (R<=32) --
// Radix-2 decimation in frequency over v[O + S*i], i < L, compile-time
// indices; leaves the sub-block in bit-reversed order.
template <int J, int H, int O, int S, int L, int SIGN, int E>
__device__ __forceinline__ void dif_bfly(double2 (&v)[E]) {
  double2 a = v[O + S * J], b = v[O + S * (J + H)];
  v[O + S * J] = cadd(a, b);
  v[O + S * (J + H)] = twc<J, L, SIGN>(csub(a, b));
}
template <int H, int O, int S, int L, int SIGN, int E, int... J>
__device__ __forceinline__ void dif_level(double2 (&v)[E], std::integer_sequence<int, J...>) {
  (dif_bfly<J, H, O, S, L, SIGN, E>(v), ...);
}
template <int L, int O, int S, int SIGN, int E>
__device__ __forceinline__ void dif_rec(double2 (&v)[E]) {
  if constexpr (L > 1) {
    constexpr int H = L / 2;
    dif_level<H, O, S, L, SIGN, E>(v, std::make_integer_sequence<int, H>{});
    dif_rec<H, O, S, SIGN, E>(v);
    dif_rec<H, O + S * H, S, SIGN, E>(v);
  }
}
__host__ __device__ constexpr int brev(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
  return r;
}
__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }

// X[k] = sum_n x[n] exp(SIGN 2 pi i n k / R), natural order in and out.
template <int R, int SIGN>
__device__ __forceinline__ void dft(double2 (&x)[R]) {
  if constexpr (R > 1) {
    dif_rec<R, 0, 1, SIGN, R>(x);
    double2 t[R];
#pragma unroll
    for (int k = 0; k < R; ++k) t[k] = x[brev(k, ilog2(R))];
#pragma unroll
    for (int k = 0; k < R; ++k) x[k] = t[k];
  }
}

// ------------------------------------------------------- Stockham passes --
// Exchange-buffer index of Stockham output position `pos` written by a pass
// with stride NS and radix R (see file header).
template <int NS, int R>
__device__ __forceinline__ int xpad(int pos) {
  return pos + NS * (pos >> ilog2(NS * R));
}
// Elements of padded exchange buffer needed by an N-point FFT with E per thread.
template <int N, int E>
__host__ __device__ constexpr int xbuf_elems() { return N <= E ? 0 : N + N / E; }

// One Stockham radix-R pass; twiddles then DFT_R, data stays in registers.
template <int N, int E, int R, int NS, int SIGN>
__device__ __forceinline__ void pass_compute(double2 (&v)[E], int t, const double2* __restrict__ tw) {
  constexpr int T = N / E, B = E / R;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    double2 x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = v[b + r * B];
    if constexpr (NS > 1) {
      // w^r, w = exp(2 pi i jm/(NS R)), r = Q a + c: load w^c (c < Q) and
      // w^{Qa} (a < R/Q), one complex product for the mixed terms
      const int jm = (t + T * b) & (NS - 1);
      constexpr int STEP = N / (NS * R);
      constexpr int Q = R >= 16 ? 4 : (R >= 4 ? 2 : 1);
      double2 lo[Q], hi[R / Q];
#pragma unroll
      for (int c = 1; c < Q; ++c) lo[c] = ldtw_pass(&tw[c * jm * STEP]);
#pragma unroll
      for (int a = 1; a < R / Q; ++a) hi[a] = ldtw_pass(&tw[Q * a * jm * STEP]);
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const int a = r / Q, c = r % Q;
        const double2 w = a == 0 ? lo[c] : (c == 0 ? hi[a] : cmul(hi[a], lo[c]));
        x[r] = cmul_dir<SIGN>(x[r], w);
      }
    }
    dft<R, SIGN>(x);
#pragma unroll
    for (int r = 0; r < R; ++r) v[b + r * B] = x[r];
  }
}

// Permute the pass output through shared memory back into the natural
// strided distribution.  SYNC is the group barrier.  XS(i) maps a padded
// element index to the shared-memory slot (lets pencil kernels interleave
// several columns).
template <int N, int E, int R, int NS, class Sync, class XS>
__device__ __forceinline__ void pass_exchange(double2 (&v)[E], int t, double2* __restrict__ xb, Sync sync, XS xs) {
  constexpr int T = N / E, B = E / R;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = t + T * b;
    const int base = (j / NS) * NS * R + (j & (NS - 1));
#pragma unroll
    for (int r = 0; r < R; ++r) xb[xs(xpad<NS, R>(base + r * NS))] = v[b + r * B];
  }
  sync();
#pragma unroll
  for (int i = 0; i < E; ++i) v[i] = xb[xs(xpad<NS, R>(t + T * i))];
  sync();
}

template <int N, int E, int NS, int SIGN, class Sync, class XS>
__device__ __forceinline__ void fft_passes(double2 (&v)[E], int t, double2* __restrict__ xb,
                                           const double2* __restrict__ tw, Sync sync, XS xs) {
  if constexpr (NS < N) {
    constexpr int R = (NS * E <= N) ? E : N / NS;
    pass_compute<N, E, R, NS, SIGN>(v, t, tw);
    if constexpr (NS * R < N) {
      pass_exchange<N, E, R, NS>(v, t, xb, sync, xs);
      fft_passes<N, E, NS * R, SIGN>(v, t, xb, tw, sync, xs);
    }
  }
}

struct IdentitySlot {
  __device__ __forceinline__ int operator()(int i) const { return i; }
};

// Unnormalised N-point FFT of the group's vector, sign SIGN (+1 = backward,
// P:185-186; -1 = forward).  All threads of the group (and, with a CTA-wide
// barrier, of the CTA) must call it together.
template <int N, int E, int SIGN, class Sync, class XS = IdentitySlot>
__device__ __forceinline__ void fft(double2 (&v)[E], int t, double2* __restrict__ xb,
                                    const double2* __restrict__ tw, Sync sync, XS xs = XS{}) {
  static_assert(N % E == 0 && (E & (E - 1)) == 0 && (N & (N - 1)) == 0, "power-of-two sizes");
  // Launder the thread index so that the (thread-invariant) exchange and
  // twiddle addresses are recomputed per transform instead of being hoisted
  // out of the caller's row loop and held live in registers across it.
  int tl;
  asm volatile("mov.b32 %0, %1;" : "=r"(tl) : "r"(t));
  fft_passes<N, E, 1, SIGN>(v, tl, xb, tw, sync, xs);
}

// CTA barrier as volatile asm: it keeps its order relative to the volatile
// table loads (ldtw), so the next pass's twiddles are not hoisted above it.
struct CtaSync {
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync 0;" ::: "memory"); }
};

// Barrier over one thread group (named barrier `id`, `n` threads, n % 32 == 0)
// so that the row groups of a CTA progress independently.
struct GroupSync {
  int id, n;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
  }
};

}  // namespace idc
