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

#include "config.cuh"
#include "pdl.cuh"
#include <type_traits>
#include <utility>

namespace idc {

// ------------------------------------------------- transform counter (debug) --
// Instrumentation for the transform-count invariant (6 / 9 /
// 8 transforms per 1D convolution), compiled
// only into the debug library libidconv_count.so (-DIDC_COUNT_FFT=1, built by
// _build.py next to the product library): while idc_fft_count_begin() ..
// idc_fft_count_end() is active, every transform executed adds 1 (per thread
// group) to counter[log2 N] in device memory.  The pointer lives in a
// __constant__ of each translation unit (device code is not relocatable), set
// through setters the units register at load time.  The product library has
// no counter code in its kernels (the check cost registers in the row kernels).
#ifndef IDC_COUNT_FFT
#define IDC_COUNT_FFT 0
#endif
using FftCounterSetter = cudaError_t (*)(unsigned long long*);
void register_fft_counter_setter(FftCounterSetter);   // launch.cu
#if IDC_COUNT_FFT
namespace {
__constant__ unsigned long long* g_fft_counter;
cudaError_t set_fft_counter(unsigned long long* p) { return cudaMemcpyToSymbol(g_fft_counter, &p, sizeof(p)); }
struct FftCounterRegistration {
  FftCounterRegistration() { register_fft_counter_setter(&set_fft_counter); }
};
FftCounterRegistration g_fft_counter_registration;
}  // namespace
#endif
__device__ __forceinline__ void count_fft(int log2n, int t, unsigned n) {
#if IDC_COUNT_FFT
  unsigned long long* p = g_fft_counter;
  if (p != nullptr && t == 0) atomicAdd(p + log2n, (unsigned long long)n);
#endif
}

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
// Stockham pass twiddles: read-only path (ptxas may keep them in registers
// across the row loop) or coherent loads (reloaded per pass from L1: fewer
// registers, more L1 traffic).  Coherent in the row kernels with E >= 16
// (IDC_ROWS_TW_COH_MIN_E; units defining IDC_ROW_UNIT): there the hoisted
// twiddles pushed the 255-register kernels into local-memory spills (K2<1024>
// 264 -> 16 bytes of stack, K4<4096> 232 -> 8; cconv1d 1024 0.740 -> 0.716 ms,
// tconv1d 4096 0.868 -> 0.844 ms), while at E = 8 and in the pencil kernels
// the reloads cost more than they save (hconv1d 512 0.592 -> 0.616 ms,
// hconv3d 56.1 -> 57.5 ms; profiles/r02/ab/pass_tw_coherent.log).
// IDC_PASS_TW_COHERENT makes every unit coherent (experiments).
#ifndef IDC_ROW_UNIT
#define IDC_ROW_UNIT 0
#endif
template <int E>
__host__ __device__ constexpr bool pass_tw_coherent() {
#ifdef IDC_PASS_TW_COHERENT
  return true;
#else
  return IDC_ROW_UNIT && E >= IDC_ROWS_TW_COH_MIN_E;
#endif
}
template <int E>
__device__ __forceinline__ double2 ldtw_pass(const double2* p) {
  if constexpr (pass_tw_coherent<E>()) return ldtw(p);
  else return __ldg(p);
}
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
// cos(2 pi j / 192), j = 0..48 (first quadrant; 192 = lcm of the 32-, 48-
// and 64-point roots the kernels need as immediates), 35 significant digits
__host__ __device__ constexpr double cos192tab(int j) {
  return j == 0  ? 1.00000000000000000000000000000000000
       : j == 1  ? 0.99946458747636564442983644624285995
       : j == 2  ? 0.99785892323860350673806979127277760
       : j == 3  ? 0.99518472667219688624483695310947992
       : j == 4  ? 0.99144486137381041114455752692856287
       : j == 5  ? 0.98664333208487900474692393298420604
       : j == 6  ? 0.98078528040323044912618223613423904
       : j == 7  ? 0.97387697927733364814968997013355039
       : j == 8  ? 0.96592582628906828674974319972889737
       : j == 9  ? 0.95694033573220886493579788698026997
       : j == 10 ? 0.94693012949510566425580427485398368
       : j == 11 ? 0.93590592675732570029170724946673536
       : j == 12 ? 0.92387953251128675612818318939678829
       : j == 13 ? 0.91086382492117581857329170716055065
       : j == 14 ? 0.89687274153268830389410393639308120
       : j == 15 ? 0.88192126434835502971275686366038835
       : j == 16 ? 0.86602540378443864676372317075293618
       : j == 17 ? 0.84920218152657888764909693734310022
       : j == 18 ? 0.83146961230254523707878837761790576
       : j == 19 ? 0.81284668459161521657909614327190880
       : j == 20 ? 0.79335334029123516457977696150129928
       : j == 21 ? 0.77301045336273696081090660975846980
       : j == 22 ? 0.75183980747897739640751940637696144
       : j == 23 ? 0.72986407269783565735010119440318188
       : j == 24 ? 0.70710678118654752440084436210484904
       : j == 25 ? 0.68359230202287128051349759431615512
       : j == 26 ? 0.65934581510006886842512461205533745
       : j == 27 ? 0.63439328416364549821517161322549337
       : j == 28 ? 0.60876142900872063941609754289816400
       : j == 29 ? 0.58247769686780214919713476703611245
       : j == 30 ? 0.55557023301960222474283081394853287
       : j == 31 ? 0.52806785065036799587344882033760557
       : j == 32 ? 0.50000000000000000000000000000000000
       : j == 33 ? 0.47139673682599764855638762590525438
       : j == 34 ? 0.44228869021900128199523897732424473
       : j == 35 ? 0.41270702980439473704770218607336747
       : j == 36 ? 0.38268343236508977172845998403039887
       : j == 37 ? 0.35225004792123350653175231975871267
       : j == 38 ? 0.32143946530316158070105762407890159
       : j == 39 ? 0.29028467725446236763619237581739527
       : j == 40 ? 0.25881904510252076234889883762404833
       : j == 41 ? 0.22707626303437320758569669257708809
       : j == 42 ? 0.19509032201612826784828486847702224
       : j == 43 ? 0.16289547339458873948080063970826556
       : j == 44 ? 0.13052619222005159154840622789548901
       : j == 45 ? 0.09801714032956060199419556388864185
       : j == 46 ? 0.06540312923014306681531555877517544
       : j == 47 ? 0.03271908282177614206365992631728813
       : 0.0;
}
// cos(2 pi j / 192) for any integer j
__host__ __device__ constexpr int mod192(int j) { return (j % 192 + 192) % 192; }
__host__ __device__ constexpr double cos192(int j) {
  return (mod192(j) <= 48)  ? cos192tab(mod192(j))
       : (mod192(j) <= 96)  ? -cos192tab(96 - mod192(j))
       : (mod192(j) <= 144) ? -cos192tab(mod192(j) - 96)
                            : cos192tab(192 - mod192(j));
}
__host__ __device__ constexpr double sin192(int j) { return cos192(j - 48); }

// a * exp(SIGN * 2 pi i K / L), L | 192, resolved at compile time; the
// trivial roots (1, +-i, -1) cost no arithmetic
template <int K, int L, int SIGN>
__device__ __forceinline__ double2 twc(double2 a) {
  static_assert(192 % L == 0, "compile-time roots need L | 192");
  constexpr int j = mod192(K * (192 / L));
  if constexpr (j == 0) {
    return a;
  } else if constexpr (j == 48) {           // * (SIGN i)
    if constexpr (SIGN > 0) return make_double2(-a.y, a.x);
    else return make_double2(a.y, -a.x);
  } else if constexpr (j == 96) {
    return make_double2(-a.x, -a.y);
  } else if constexpr (j == 144) {          // * (-SIGN i)
    if constexpr (SIGN > 0) return make_double2(a.y, -a.x);
    else return make_double2(-a.y, a.x);
  } else if constexpr (j % 48 == 24) {     // odd multiples of pi/4: |cos| = |sin|, 3 instructions
    constexpr double c = cos192(j);
    constexpr double s = SIGN > 0 ? sin192(j) : -sin192(j);
    constexpr double h = 0.70710678118654752440084436210484904;   // sqrt(1/2)
    // a (c + i s) with c = sc h, s = ss h: re = a.x c - ss (a.y h), im = a.x s + sc (a.y h)
    constexpr double sc = c > 0 ? 1.0 : -1.0, ss = s > 0 ? 1.0 : -1.0;
    const double ty = a.y * h;
    return make_double2(fma(a.x, sc * h, -ss * ty), fma(a.x, ss * h, sc * ty));
  } else {
    constexpr double c = cos192(j);
    constexpr double s = SIGN > 0 ? sin192(j) : -sin192(j);
    return make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
  }
}

// x * i^Q (Q mod 4): sign flips and swaps only (a generic cmul by the
// constant (0, 1) would still cost four fp64 instructions under IEEE rules)
template <int Q>
__device__ __forceinline__ double2 mul_i(double2 x) {
  constexpr int q = ((Q % 4) + 4) % 4;
  if constexpr (q == 0) return x;
  else if constexpr (q == 1) return make_double2(-x.y, x.x);
  else if constexpr (q == 2) return make_double2(-x.x, -x.y);
  else return make_double2(x.y, -x.x);
}

// Per-element roots of the residue split / recombination: element i of a
// lane (k = t + T i, T = M / E) needs zeta_{QM}^{R k} = zeta_{QM}^{R t} *
// zeta_{QE}^{R i}.  The lane loads zt = zeta_{QM}^{R t} once; the second
// factor is a compile-time root.  f(i, w_i) is called for i = 0..E-1 with
// w_i = zt * zeta_{QE}^{SIGN R i} (4 fp64 instructions instead of one
// 16-byte table load per element).
template <int QE, int R, int SIGN, class F, int... I>
__device__ __forceinline__ void roots_apply(double2 zt, F& f, std::integer_sequence<int, I...>) {
  (f(I, twc<R * I, QE, SIGN>(zt)), ...);
}
template <int QE, int R, int SIGN, int E, class F>
__device__ __forceinline__ void for_roots(double2 zt, F&& f) {
  roots_apply<QE, R, SIGN>(zt, f, std::make_integer_sequence<int, E>{});
}

// f(std::integral_constant<int, I>{}) for I = 0..N-1 (compile-time element index)
template <class F, int... I>
__device__ __forceinline__ void static_for_impl(F& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
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

// Pass twiddle tables (one per (N, E), built on the host by pass_table()):
// for every pass with NS > 1 (radix R, Q = 4, 2 or 1 as below), a block of
// (Q - 1 + R/Q - 1) rows of NS entries: row c - 1 (c = 1..Q-1) holds
// w^c and row Q - 2 + a (a = 1..R/Q-1) holds w^{Qa}, w = zeta_N^{j N/(NS R)},
// at column j.  Lanes read consecutive j: contiguous 16-byte loads (a gather
// from the full zeta_N table touched up to 32 cache lines per warp load).
// (storing every w^r instead -- one multiply per element, R - 1 loads per
// butterfly -- measured 6-12% slower: more L1 wavefronts)
__host__ __device__ constexpr int pass_q(int R) { return R >= 16 ? 4 : (R >= 4 ? 2 : 1); }
__host__ __device__ constexpr int pass_radix(int N, int E, int NS) { return (NS * E <= N) ? E : N / NS; }
// Table rows per pass of radix R: folded (IDC_FOLD_TW, below) w^{2^l}, l < log2 R;
// otherwise w^c (c < Q) and w^{Qa} (a < R/Q).
__host__ __device__ constexpr int pass_rows(int R) {
  return IDC_FOLD_TW ? ilog2(R) : (pass_q(R) - 1 + R / pass_q(R) - 1);
}
template <int N, int E>
__host__ __device__ constexpr int pass_tab_offset(int ns_target) {
  int off = 0;
  for (int NS = 1; NS < N;) {
    const int R = pass_radix(N, E, NS);
    if (NS == ns_target) return off;
    if (NS > 1) off += pass_rows(R) * NS;
    NS *= R;
  }
  return off;
}

// One Stockham radix-R pass; twiddles then DFT_R, data stays in registers.
// Twiddles of one Stockham pass for this thread: for each of its B = E/R
// butterflies, w^c (c < Q) and w^{Qa} (a < R/Q), w = exp(2 pi i jm/(NS R)),
// from the pass table.  Loaded ahead of the exchange that precedes the pass,
// so the load latency is hidden behind the barriers.
template <int N, int E, int R, int NS>
struct PassTw {
  static constexpr int B = E / R, Q = pass_q(R), LR = ilog2(R) > 0 ? ilog2(R) : 1;
#if IDC_FOLD_TW
  double2 p[B][LR];      // w^{2^l}
#else
  double2 lo[B][Q], hi[B][R / Q];
#endif
};
template <int N, int E, int R, int NS>
__device__ __forceinline__ PassTw<N, E, R, NS> load_pass_tw(int t, const double2* __restrict__ tw) {
  PassTw<N, E, R, NS> p{};
  if constexpr (NS > 1) {
    constexpr int T = N / E, B = E / R;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int jm = (t + T * b) & (NS - 1);
      const double2* tp = tw + pass_tab_offset<N, E>(NS) + jm;
#if IDC_FOLD_TW
#pragma unroll
      for (int l = 0; l < ilog2(R); ++l) p.p[b][l] = ldtw_pass<E>(&tp[l * NS]);
#else
      constexpr int Q = pass_q(R);
#pragma unroll
      for (int c = 1; c < Q; ++c) p.lo[b][c] = ldtw_pass<E>(&tp[(c - 1) * NS]);
#pragma unroll
      for (int a = 1; a < R / Q; ++a) p.hi[b][a] = ldtw_pass<E>(&tp[(Q - 2 + a) * NS]);
#endif
    }
  }
  return p;
}

// ------------------------------------- twiddled DFT_R with folded twiddles --
// X_k = sum_r x_r w^r omega_R^{rk} (omega_R = exp(SIGN 2 pi i / R)) as an
// in-register radix-2 decimation in time whose butterflies absorb the pass
// twiddle: with E_k, O_k the same problem over the even / odd r with base
// w^2, X_k = E_k + (w omega_R^k) O_k and X_{k+R/2} = E_k - (w omega_R^k) O_k.
// Level L (sub-DFTs of size L) has base u_L = w^{R/L}; its butterflies
// a +- t b (t = u_L omega_L^k) cost 6 fp64 instructions in FMA form
// (y0 = a + t b by two FMAs per component, y1 = 2a - y0 by one), against 8
// for a separate complex multiply and two complex adds.  Per 16 points of a
// radix-16 pass: 32 butterflies (192) + 14 for the t_k = u omega^k, against
// 24 twiddle multiplies (96) + 168 in DFT16 with the table scheme below.
// wp[l] = w^{2^l} from the pass table (direction +1; conjugated for SIGN < 0).
__device__ __forceinline__ void bfly_fma(double2& a, double2& b, double2 t) {
  const double2 y0 = make_double2(fma(t.x, b.x, fma(-t.y, b.y, a.x)), fma(t.x, b.y, fma(t.y, b.x, a.y)));
  b = make_double2(fma(2.0, a.x, -y0.x), fma(2.0, a.y, -y0.y));
  a = y0;
}
template <int R, int L, int SIGN>
__device__ __forceinline__ void dit_level(double2 (&y)[R], double2 u) {
  // t_k = u omega_L^k for k < L/2, t_{k + L/4} = (SIGN i) t_k; one t live at a time
  static_for<(L >= 4 ? L / 4 : 1)>([&](auto K) {
    constexpr int k = decltype(K)::value;
    const double2 t = twc<k, L, SIGN>(u);
    static_for<R / L>([&](auto Gi) {
      constexpr int g = decltype(Gi)::value;
      bfly_fma(y[g * L + k], y[g * L + k + L / 2], t);
    });
    if constexpr (L >= 4) {
      const double2 ti = twc<1, 4, SIGN>(t);
      static_for<R / L>([&](auto Gi) {
        constexpr int g = decltype(Gi)::value;
        bfly_fma(y[g * L + k + L / 4], y[g * L + k + L / 4 + L / 2], ti);
      });
    }
  });
}
template <int R, int SIGN, int L = 2>
__device__ __forceinline__ void dit_levels(double2 (&y)[R], const double2* wp) {
  if constexpr (L <= R) {
    double2 u = wp[ilog2(R / L)];                   // w^{R/L}
    if constexpr (SIGN < 0) u.y = -u.y;
    dit_level<R, L, SIGN>(y, u);
    dit_levels<R, SIGN, 2 * L>(y, wp);
  }
}
template <int R, int SIGN>
__device__ __forceinline__ void dft_tw(double2 (&x)[R], const double2* wp) {
  double2 y[R];
#pragma unroll
  for (int k = 0; k < R; ++k) y[k] = x[brev(k, ilog2(R))];
  dit_levels<R, SIGN>(y, wp);
#pragma unroll
  for (int k = 0; k < R; ++k) x[k] = y[k];
}

// One Stockham radix-R pass with preloaded twiddles; data stays in registers.
template <int N, int E, int R, int NS, int SIGN>
__device__ __forceinline__ void pass_compute(double2 (&v)[E], const PassTw<N, E, R, NS>& pt) {
  constexpr int B = E / R;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    double2 x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = v[b + r * B];
#if IDC_FOLD_TW
    if constexpr (NS > 1) {
      dft_tw<R, SIGN>(x, pt.p[b]);
    } else {
      dft<R, SIGN>(x);
    }
#else
    if constexpr (NS > 1) {
      // x[Qa + c] * w^c * w^{Qa}: two multiplies per element instead of
      // forming every w^r = w^{Qa} w^c first (same multiply count, but no
      // R-element twiddle set live in registers: -7% time at m = 4096)
      constexpr int Q = pass_q(R);
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const int a = r / Q, c = r % Q;
        if (c != 0) x[r] = cmul_dir<SIGN>(x[r], pt.lo[b][c]);
        if (a != 0) x[r] = cmul_dir<SIGN>(x[r], pt.hi[b][a]);
      }
    }
    dft<R, SIGN>(x);
#endif
#pragma unroll
    for (int r = 0; r < R; ++r) v[b + r * B] = x[r];
  }
}

template <int N, int E, int R, int NS, int SIGN>
__device__ __forceinline__ void pass_compute(double2 (&v)[E], int t, const double2* __restrict__ tw) {
  pass_compute<N, E, R, NS, SIGN>(v, load_pass_tw<N, E, R, NS>(t, tw));
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

struct NoPre {
  __device__ __forceinline__ void operator()() const {}
};

// `pre` runs once, after the first pass's arithmetic and before the first
// write to xb: a caller whose earlier TMA store still reads xb waits there,
// so the wait overlaps the first radix pass instead of preceding the FFT.
template <int N, int E, int NS, int SIGN, class Sync, class XS, class Pre = NoPre>
__device__ __forceinline__ void fft_passes(double2 (&v)[E], int t, double2* __restrict__ xb,
                                           const double2* __restrict__ tw, Sync sync, XS xs,
                                           const PassTw<N, E, pass_radix(N, E, NS), NS>& pt, Pre pre = Pre{}) {
  if constexpr (NS < N) {
    constexpr int R = pass_radix(N, E, NS);
    pass_compute<N, E, R, NS, SIGN>(v, pt);
    if constexpr (NS == 1) pre();
    if constexpr (NS * R < N) {
      const auto next = load_pass_tw<N, E, pass_radix(N, E, NS * R), NS * R>(t, tw);   // ahead of the exchange
      pass_exchange<N, E, R, NS>(v, t, xb, sync, xs);
      fft_passes<N, E, NS * R, SIGN>(v, t, xb, tw, sync, xs, next);
    }
  } else {
    pre();
  }
}

struct IdentitySlot {
  __device__ __forceinline__ int operator()(int i) const { return i; }
};

// Unnormalised N-point FFT of the group's vector, sign SIGN (+1 = backward,
// P:185-186; -1 = forward).  All threads of the group (and, with a CTA-wide
// barrier, of the CTA) must call it together.
template <int N, int E, int SIGN, class Sync, class XS = IdentitySlot, class Pre = NoPre>
__device__ __forceinline__ void fft(double2 (&v)[E], int t, double2* __restrict__ xb,
                                    const double2* __restrict__ tw, Sync sync, XS xs = XS{}, Pre pre = Pre{}) {
  static_assert(N % E == 0 && (E & (E - 1)) == 0 && (N & (N - 1)) == 0, "power-of-two sizes");
  // Launder the thread index so that the (thread-invariant) exchange and
  // twiddle addresses are recomputed per transform instead of being hoisted
  // out of the caller's row loop and held live in registers across it.
  int tl;
  asm volatile("mov.b32 %0, %1;" : "=r"(tl) : "r"(t));
  count_fft(ilog2(N), tl, 1);
  fft_passes<N, E, 1, SIGN>(v, tl, xb, tw, sync, xs, PassTw<N, E, pass_radix(N, E, 1), 1>{}, pre);
}

// Two independent N-point FFTs (same sign) in lockstep: each pass computes
// both vectors' butterflies, then both are exchanged (v through xb, w through
// xb2) under one pair of barriers -- half the barriers of two fft() calls and
// twice the independent work between them.
template <int N, int E, int NS, int SIGN, class Sync, class XS>
__device__ __forceinline__ void fft2_passes(double2 (&v)[E], double2 (&w)[E], int t, double2* __restrict__ xb,
                                            double2* __restrict__ xb2, const double2* __restrict__ tw, Sync sync,
                                            XS xs, const PassTw<N, E, pass_radix(N, E, NS), NS>& pt) {
  if constexpr (NS < N) {
    constexpr int R = pass_radix(N, E, NS);
    pass_compute<N, E, R, NS, SIGN>(v, pt);
    pass_compute<N, E, R, NS, SIGN>(w, pt);
    if constexpr (NS * R < N) {
      const auto next = load_pass_tw<N, E, pass_radix(N, E, NS * R), NS * R>(t, tw);
      constexpr int T = N / E, B = E / R;
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int j = t + T * b;
        const int base = (j / NS) * NS * R + (j & (NS - 1));
#pragma unroll
        for (int r = 0; r < R; ++r) {
          xb[xs(xpad<NS, R>(base + r * NS))] = v[b + r * B];
          xb2[xs(xpad<NS, R>(base + r * NS))] = w[b + r * B];
        }
      }
      sync();
#pragma unroll
      for (int i = 0; i < E; ++i) {
        v[i] = xb[xs(xpad<NS, R>(t + T * i))];
        w[i] = xb2[xs(xpad<NS, R>(t + T * i))];
      }
      sync();
      fft2_passes<N, E, NS * R, SIGN>(v, w, t, xb, xb2, tw, sync, xs, next);
    }
  }
}

template <int N, int E, int SIGN, class Sync, class XS = IdentitySlot>
__device__ __forceinline__ void fft2(double2 (&v)[E], double2 (&w)[E], int t, double2* __restrict__ xb,
                                     double2* __restrict__ xb2, const double2* __restrict__ tw, Sync sync,
                                     XS xs = XS{}) {
  int tl;
  asm volatile("mov.b32 %0, %1;" : "=r"(tl) : "r"(t));
  count_fft(ilog2(N), tl, 2);
  fft2_passes<N, E, 1, SIGN>(v, w, tl, xb, xb2, tw, sync, xs, PassTw<N, E, pass_radix(N, E, 1), 1>{});
}

// Two independent N-point FFTs with their exchanges staggered by half a pass
// (IDC_FFT2_STAGGER): while one vector's pass output goes through shared
// memory, the other vector's butterflies run, so the shared-memory pipe and
// the fp64 pipe work at the same time (tools/pipe_overlap.cu: on B200 a mix
// of independent DFMA and STS/LDS.128 streams takes max(F, S), not F + S).
// Per pass with an exchange after it (v computed, w ready):
//   store v -> xb ; compute w ; barrier ; load v ; store w -> xb2 ;
//   compute v (next pass) ; barrier ; load w
// -- the same two barriers per pass as fft2, both buffers as in fft2.
template <int N, int E, int R, int NS, class XS>
__device__ __forceinline__ void pass_store(const double2 (&v)[E], int t, double2* __restrict__ xb, XS xs) {
  constexpr int T = N / E, B = E / R;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = t + T * b;
    const int base = (j / NS) * NS * R + (j & (NS - 1));
#pragma unroll
    for (int r = 0; r < R; ++r) xb[xs(xpad<NS, R>(base + r * NS))] = v[b + r * B];
  }
}
template <int N, int E, int R, int NS, class XS>
__device__ __forceinline__ void pass_load(double2 (&v)[E], int t, const double2* __restrict__ xb, XS xs) {
  constexpr int T = N / E;
#pragma unroll
  for (int i = 0; i < E; ++i) v[i] = xb[xs(xpad<NS, R>(t + T * i))];
}
template <int N, int E, int NS, int SIGN, int SIGN2, class Sync, class XS>
__device__ __forceinline__ void fft2s_step(double2 (&v)[E], double2 (&w)[E], int t, double2* __restrict__ xb,
                                           double2* __restrict__ xb2, const double2* __restrict__ tw, Sync sync,
                                           XS xs) {
  constexpr int R = pass_radix(N, E, NS), NR = NS * R;
  if constexpr (NR < N) {
    pass_store<N, E, R, NS>(v, t, xb, xs);
    pass_compute<N, E, R, NS, SIGN2>(w, t, tw);
    sync();
    pass_load<N, E, R, NS>(v, t, xb, xs);
    pass_store<N, E, R, NS>(w, t, xb2, xs);
    pass_compute<N, E, pass_radix(N, E, NR), NR, SIGN>(v, t, tw);
    sync();
    pass_load<N, E, R, NS>(w, t, xb2, xs);
    fft2s_step<N, E, NR, SIGN, SIGN2>(v, w, t, xb, xb2, tw, sync, xs);
  } else {
    pass_compute<N, E, R, NS, SIGN2>(w, t, tw);
  }
}
// v transformed with sign SIGN, w with SIGN2 (default the same)
template <int N, int E, int SIGN, int SIGN2 = SIGN, class Sync, class XS = IdentitySlot>
__device__ __forceinline__ void fft2s(double2 (&v)[E], double2 (&w)[E], int t, double2* __restrict__ xb,
                                      double2* __restrict__ xb2, const double2* __restrict__ tw, Sync sync,
                                      XS xs = XS{}) {
  int tl;
  asm volatile("mov.b32 %0, %1;" : "=r"(tl) : "r"(t));
  count_fft(ilog2(N), tl, 2);
  pass_compute<N, E, pass_radix(N, E, 1), 1, SIGN>(v, tl, tw);
  fft2s_step<N, E, 1, SIGN, SIGN2>(v, w, tl, xb, xb2, tw, sync, xs);
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
