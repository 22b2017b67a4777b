// pencils2.cu -- TMA-staged persistent pencil kernels (K5-K8), 64 <= m <= 4096.
//
// Same transforms as pencils.cu (Procedures fftpadBackward / fftpadForward,
// P:325-349; Eqs. fft0backwardA/B and fft0forward, AMB-1 stream
// layout).  B200 data movement: one CTA per SM loops over W-column pencil
// tiles; each tile is brought into shared memory by 3D TMA tensor loads
// (cp.async.bulk.tensor, boxes of W columns x <= 256 rows, completion on an
// mbarrier).  As soon as every thread has copied its part of a staged tile
// into registers, one thread issues the TMA loads of the CTA's next tile,
// so the HBM traffic of tile n+1 overlaps the FFTs and stores of tile n.
// The stage is read as [row][column]: thread (c, t) = c + W*t takes rows
// t + T*i of column c -- consecutive lanes read consecutive 16-byte words.
#include "config.cuh"
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "fft_dev.cuh"
#include "launch.cuh"
#include "kernels.cuh"
#include "nd_internal.cuh"
#include "tables.cuh"
#include "tma.cuh"
#include "tmap.cuh"

namespace idc {

namespace {

// tile configuration: E elements per thread, T = N/E threads per column,
// W columns per CTA (TH threads), TMA boxes of BR rows, XB exchange slots
template <int N, int TH = IDC_PENCIL_THREADS, int EE = IDC_PENCIL_E>
struct TCfg {
  static constexpr int E = EE;
  static constexpr int T = N / E;
  static constexpr int W = TH / T < 1 ? 1 : (TH / T > 16 ? 16 : TH / T);
  static constexpr int THREADS = T * W;
  static constexpr int BR = N < 256 ? N : 256;                     // TMA box rows
  static constexpr int XB = (xbuf_elems<N, E>() > 0 ? xbuf_elems<N, E>() : 1) * W;
};

// K5 / K6 (complex fftpad pencils): E = 16 with 256-thread CTAs at m = 256
// and m >= 1024 (measured 3-5% faster on cconv2d 1024^2 and 64 x 256^2;
// 6-8% on tconv2d 2*2048 x 2048 and cconv2d 2048^2, 4096 x 1024: three
// radix-16 passes instead of four radix-8 ones at the same tile width);
// E = 8 with 512-thread CTAs at m = 512 (cconv3d 512^3 1.7% faster so).
// 128-thread CTAs (half-width tiles, several CTAs per SM) for m in
// [IDC_K56_NARROW_MIN, IDC_K56_NARROW_MAX] (E = 16 sizes only): measured
// 64 x 256^2 -1.5%, 1024 x 4096 -3.5%, 16 x 1024^2 -2%
template <int N>
constexpr bool k56_wide() { return N == 256 || N >= 1024; }
template <int N>
using K56Cfg = TCfg<N, (k56_wide<N>() ? (N >= IDC_K56_NARROW_MIN && N <= IDC_K56_NARROW_MAX ? 128 : 256)
                                      : IDC_PENCIL_THREADS),
                   (k56_wide<N>() ? 16 : IDC_PENCIL_E)>;

// K7 / K8 (centered fft0pad pencils): E = 16 with 256-thread CTAs (three
// radix-16 passes) for 256 <= m <= 4096 -- measured hconv2d 2048^2 -5%,
// hconv3d 512^3 -1.5%, hconv2d 8191 x 512 (m = 4096) -6% against E = 8 /
// 512 threads.
// 128-thread CTAs (half-width tiles, two CTAs per SM) for the m whose
// log2 bit is set in IDC_K78_NARROW_MASK: m = 1024 (2-column tiles, hconv2d
// 2047 x 2048 0.332 -> 0.320 ms) and m = 256 (8-column tiles, hconv2d 511 x
// 4096 0.190 -> 0.184 ms); not m = 512 (4-column tiles: hconv3d 59.5 ->
// 70.8 ms) nor m = 2048 (1-column tiles: hconv2d 4095 x 2048 0.61 ->
// 0.80 ms) -- the DRAM row segment width decides
template <int N>
constexpr bool k78_narrow() { return ((IDC_K78_NARROW_MASK) >> ilog2(N)) & 1; }
template <int N>
constexpr bool k78_wide() { return N >= IDC_K78_WIDE_MIN && N <= IDC_K78_WIDE_MAX; }
template <int N>
using K78Cfg = TCfg<N, (k78_wide<N>() ? (k78_narrow<N>() ? 128 : 256)
                                      : IDC_PENCIL0_THREADS),
                   (k78_wide<N>() ? 16 : IDC_PENCIL_E)>;

template <int W>
struct Slot2 {
  int c;
  __device__ __forceinline__ int operator()(int i) const { return i * W + c; }
};

struct Tiles {
  long ncols, nct;      // columns per item, column tiles per item
  long batch;           // items per input
  long per_input;       // nct * batch
  long ntiles;          // per_input * inputs
  long bstride, ustride;
};

// tile index -> (input, batch item, first column); tile counts fit in 32 bits
__device__ __forceinline__ void tile_coords(const Tiles& tl, long tau, int W, int& input, long& item, long& col0) {
  const unsigned tt = (unsigned)tau, per = (unsigned)tl.per_input, nct = (unsigned)tl.nct;
  const unsigned in = tt / per;
  const unsigned rest = tt - in * per;
  const unsigned it = rest / nct;
  input = (int)in;
  item = it;
  col0 = (long)(rest - it * nct) * W;
}

// issue the TMA boxes covering rows [row0, row0 + nrows) of a tile into `stage`
template <int W, int BR>
__device__ __forceinline__ void load_rows(const CUtensorMap* map, double2* stage, long col0, int row0, int nrows,
                                          long item, uint64_t* bar) {
  for (int b = 0; b < nrows; b += BR)
    tma_load_3d(stage + (long)b * W, map, (int)(2 * col0), row0 + b, (int)item, bar);
}

// Write a transformed N x W tile through the exchange buffer: park it as
// [row][column] (the FFT's last exchange has completed), make it visible to
// the async proxy, and let one thread issue the TMA stores (clipped at the
// tensor's column bound for ragged tiles).  The caller waits for the stores'
// shared-memory reads (bulk_wait_read) before xb is written again.
template <int N, int E, int W, int BR>
__device__ __forceinline__ void tile_store(const double2 (&v)[E], int t, int c, double2* xb, const CUtensorMap* map,
                                           long col0, long item, bool drain_first = false) {
  constexpr int T = N / E;
#pragma unroll
  for (int i = 0; i < E; ++i) xb[(t + T * i) * W + c] = v[i];
  fence_proxy_async_smem();
  if (drain_first && threadIdx.x == 0) bulk_wait_read();   // earlier stores (other buffer) done reading
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int r0 = 0; r0 < N; r0 += BR) tma_store_3d(map, (int)(2 * col0), r0, (int)item, xb + (long)r0 * W);
    bulk_commit();
  }
}

// Distributed y passes (dist.cu): the residue streams live in the blocked
// rank-major layout of the all-to-all buffers -- stream s row l of local
// plane x at base + (l / L) blk + s soff + x xstride + (l % L) ncols -- so the
// backward pencils store into the send buffer and the forward pencils load
// from the returned blocks directly (no pack / unpack copies).  One 4D map per
// (input, stream), boxes of BRd <= L rows.
struct DistIO {
  CUtensorMap st[2][3];   // [input][stream]
  int L, BRd;
};

template <int N, int E, int W>
__device__ __forceinline__ void tile_store_dist(const double2 (&v)[E], int t, int c, double2* xb, const CUtensorMap* map,
                                                long col0, long item, int L, int BRd) {
  constexpr int T = N / E;
#pragma unroll
  for (int i = 0; i < E; ++i) xb[(t + T * i) * W + c] = v[i];
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int r0 = 0; r0 < N; r0 += BRd) tma_store_4d(map, (int)(2 * col0), r0 % L, (int)item, r0 / L, xb + (long)r0 * W);
    bulk_commit();
  }
}

template <int W>
__device__ __forceinline__ void load_rows_dist(const CUtensorMap* map, double2* stage, long col0, int nrows, long item,
                                               int L, int BRd, uint64_t* bar) {
  for (int b = 0; b < nrows; b += BRd) tma_load_4d(stage + (long)b * W, map, (int)(2 * col0), b % L, (int)item, b / L, bar);
}

}  // namespace

// K5 / K6: tiles of at most IDC_K56_TMA_STORE_MAXW columns (16-32-byte row segments,
// m >= 2048) leave through the exchange buffer by TMA stores (tconv2d
// 2*2048 x 2048 1.674 -> 1.548 ms, cconv2d 4096 x 1024 0.553 -> 0.502 ms);
// wider tiles store per thread (measured slower with TMA stores: 4 columns
// 1.356 -> 1.384 ms on 16 x 1024^2, 8 columns cconv3d 22.05 -> 23.56 ms)

// K5 with TMA-stored outputs: a second exchange buffer where it fits, so the
// odd stream's store drains while the even stream transforms
template <int N>
constexpr bool k5_double_xb() {
  using C = K56Cfg<N>;
  return IDC_K5_DOUBLE_XB && C::W <= IDC_K56_TMA_STORE_MAXW &&
         ((size_t)N * C::W + 2 * (size_t)C::XB) * 16 + 16 <= 227 * 1024;
}
// K5 with per-thread stores (wider tiles): the odd and even streams are
// transformed as a staggered pair (fft2s) where a second exchange buffer fits
template <int N>
constexpr bool k5_pair() {
  using C = K56Cfg<N>;
  return IDC_K5_PAIR && C::W > IDC_K56_TMA_STORE_MAXW &&
         ((size_t)N * C::W + 2 * (size_t)C::XB) * 16 + 16 <= 227 * 1024;
}

// ------------------------------------------------------------------- K5 --
template <int N, bool DIST = false>
__global__ void __launch_bounds__(K56Cfg<N>::THREADS, IDC_PENCIL_MINB)
k_pad_bwd_tma(const __grid_constant__ CUtensorMap mf, const __grid_constant__ CUtensorMap mg, double2* __restrict__ f,
              double2* __restrict__ g, double2* __restrict__ U, double2* __restrict__ V, Tiles tl,
              const double2* __restrict__ twN, const double2* __restrict__ tw2N, double2 ophase,
              const __grid_constant__ CUtensorMap mU, const __grid_constant__ CUtensorMap mV,
              const __grid_constant__ DistIO dio) {
  pdl_entry();
  using C = K56Cfg<N>;
  constexpr int E = C::E, T = C::T, W = C::W, BR = C::BR;
  constexpr bool TS = DIST || W <= IDC_K56_TMA_STORE_MAXW;   // outputs by TMA stores
  constexpr bool PAIR = !DIST && k5_pair<N>();                 // streams as a staggered pair
  constexpr bool DB = !DIST && (k5_double_xb<N>() || PAIR);   // second exchange buffer
  extern __shared__ __align__(128) double2 smem[];
  double2* stage = smem;                       // N x W
  double2* xb = stage + N * W;
  double2* xb1 = DB ? xb + C::XB : xb;
  uint64_t* bar = reinterpret_cast<uint64_t*>(xb1 + C::XB);
  const int c = threadIdx.x % W, t = threadIdx.x / W;
  const Slot2<W> xs{c};
  constexpr uint32_t BYTES = (uint32_t)N * W * 16;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  long tau = blockIdx.x;
  if (threadIdx.x == 0 && tau < tl.ntiles) {
    int in; long item, col0;
    tile_coords(tl, tau, W, in, item, col0);
    mbar_arrive_expect_tx(bar, BYTES);
    load_rows<W, BR>(in == 0 ? &mf : &mg, stage, col0, 0, N, item, bar);
  }
  uint32_t phase = 0;
  for (; tau < tl.ntiles; tau += gridDim.x) {
    int in; long item, col0;
    tile_coords(tl, tau, W, in, item, col0);
    const long col = col0 + c;
    const bool ok = col < tl.ncols;
    double2* a = (in == 0 ? f : g) + item * tl.bstride + (ok ? col : 0);
    double2* u = (in == 0 ? U : V) + item * tl.ustride + (ok ? col : 0);
    mbar_wait(bar, phase);
    phase ^= 1;
    double2 x0[E], v[E];
#pragma unroll
    for (int i = 0; i < E; ++i) x0[i] = stage[(t + T * i) * W + c];
    if (TS && threadIdx.x == 0) {   // the last tile's odd-stream store has read xb
      if constexpr (DB) bulk_wait_read_but1();
      else bulk_wait_read();
    }
    __syncthreads();
    const long nx = tau + gridDim.x;
    if (threadIdx.x == 0 && nx < tl.ntiles) {
      int in2; long item2, c2;
      tile_coords(tl, nx, W, in2, item2, c2);
      mbar_arrive_expect_tx(bar, BYTES);
      load_rows<W, BR>(in2 == 0 ? &mf : &mg, stage, c2, 0, N, item2, bar);
    }
    // odd stream u_{2l+1} = sum_k zeta_m^{lk} zeta_{2m}^k U_k  (Eq. cconv1backward)
    // zeta_{2m}^k, k = t + T i: zeta_{2m}^t x zeta_{2E}^i (immediate)
    for_roots<2 * E, 1, +1, E>(cmul(ldtw(&tw2N[t]), ophase), [&](int i, double2 w) { v[i] = cmul(x0[i], w); });
    if constexpr (!PAIR) fft<N, E, +1>(v, t, xb, twN, CtaSync{}, xs);
    if constexpr (TS) {
      if constexpr (DB) {
        // odd stream out of xb while the even stream transforms in xb1; the
        // wait for xb1's previous store (a whole transform ago) rides on the
        // store's barrier
        tile_store<N, E, W, BR>(v, t, c, xb, in == 0 ? &mU : &mV, col0, item, true);
      } else {
        if constexpr (DIST) tile_store_dist<N, E, W>(v, t, c, xb, &dio.st[in][1], col0, item, dio.L, dio.BRd);
        else tile_store<N, E, W, BR>(v, t, c, xb, in == 0 ? &mU : &mV, col0, item);
        if (threadIdx.x == 0) bulk_wait_read();
        __syncthreads();
      }
      fft<N, E, +1>(x0, t, xb1, twN, CtaSync{}, xs);   // even stream (in place, or to the send blocks)
      if constexpr (DIST) tile_store_dist<N, E, W>(x0, t, c, xb1, &dio.st[in][0], col0, item, dio.L, dio.BRd);
      else tile_store<N, E, W, BR>(x0, t, c, xb1, in == 0 ? &mf : &mg, col0, item);
    } else if constexpr (PAIR) {
      fft2s<N, E, +1>(v, x0, t, xb, xb1, twN, CtaSync{}, xs);   // odd and even streams, staggered
      const long rs = (long)T * tl.ncols;   // pointer step between a thread's rows
      if (ok) {
        double2* p = u + (long)t * tl.ncols;
        double2* q = a + (long)t * tl.ncols;
#pragma unroll
        for (int i = 0; i < E; ++i, p += rs, q += rs) {
          *p = v[i];
          *q = x0[i];
        }
      }
    } else {
      const long rs = (long)T * tl.ncols;   // pointer step between a thread's rows
      if (ok) {
        double2* p = u + (long)t * tl.ncols;
#pragma unroll
        for (int i = 0; i < E; ++i, p += rs) *p = v[i];
      }
      fft<N, E, +1>(x0, t, xb, twN, CtaSync{}, xs);   // even stream, in place
      if (ok) {
        double2* p = a + (long)t * tl.ncols;
#pragma unroll
        for (int i = 0; i < E; ++i, p += rs) *p = x0[i];
      }
    }
  }
  if (TS && threadIdx.x == 0) bulk_wait_all();
}

// ------------------------------------------------------------------- K6 --
template <int N, bool DIST = false>
__global__ void __launch_bounds__(K56Cfg<N>::THREADS, IDC_PENCIL_MINB)
k_pad_fwd_tma(const __grid_constant__ CUtensorMap mf, const __grid_constant__ CUtensorMap mu, double2* __restrict__ f,
              Tiles tl, const double2* __restrict__ twN, const double2* __restrict__ tw2N, double2 ophase,
              const __grid_constant__ DistIO dio) {
  pdl_entry();
  using C = K56Cfg<N>;
  constexpr int E = C::E, T = C::T, W = C::W, BR = C::BR;
  constexpr bool TS = W <= IDC_K56_TMA_STORE_MAXW;   // output by TMA stores
  // stream loads: the even stream from f / the odd one from U, or (DIST) both
  // from the returned blocks
  auto load_u = [&](double2* dst, long col0, long item, uint64_t* bar) {
    if constexpr (DIST) load_rows_dist<W>(&dio.st[0][1], dst, col0, N, item, dio.L, dio.BRd, bar);
    else load_rows<W, BR>(&mu, dst, col0, 0, N, item, bar);
  };
  auto load_f = [&](double2* dst, long col0, long item, uint64_t* bar) {
    if constexpr (DIST) load_rows_dist<W>(&dio.st[0][0], dst, col0, N, item, dio.L, dio.BRd, bar);
    else load_rows<W, BR>(&mf, dst, col0, 0, N, item, bar);
  };
  extern __shared__ __align__(128) double2 smem[];
  double2* sf = smem;
  double2* su = sf + N * W;
  double2* xb = su + N * W;
  uint64_t* bars = reinterpret_cast<uint64_t*>(xb + C::XB);   // [0] = f stage, [1] = U stage
  const int c = threadIdx.x % W, t = threadIdx.x / W;
  const Slot2<W> xs{c};
  constexpr uint32_t BYTES = (uint32_t)N * W * 16;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  long tau = blockIdx.x;
  if (threadIdx.x == 0 && tau < tl.ntiles) {
    int in; long item, col0;
    tile_coords(tl, tau, W, in, item, col0);
    mbar_arrive_expect_tx(&bars[1], BYTES);
    load_u(su, col0, item, &bars[1]);
    mbar_arrive_expect_tx(&bars[0], BYTES);
    load_f(sf, col0, item, &bars[0]);
  }
  const double inv = 1.0 / (2.0 * N);
  uint32_t phase = 0;
  for (; tau < tl.ntiles; tau += gridDim.x) {
    int in; long item, col0;
    tile_coords(tl, tau, W, in, item, col0);
    const long col = col0 + c;
    const bool ok = col < tl.ncols;
    double2* a = f + item * tl.bstride + (ok ? col : 0);
    const long nx = tau + gridDim.x;
    int in2 = 0; long item2 = 0, c2 = 0;
    if (nx < tl.ntiles) tile_coords(tl, nx, W, in2, item2, c2);
    double2 v[E], s[E];
    mbar_wait(&bars[1], phase);
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = su[(t + T * i) * W + c];
    if (TS && threadIdx.x == 0) bulk_wait_read();   // the last tile's output stores have read xb
    __syncthreads();
    if (threadIdx.x == 0 && nx < tl.ntiles) {
      mbar_arrive_expect_tx(&bars[1], BYTES);
      load_u(su, c2, item2, &bars[1]);
    }
    fft<N, E, -1>(v, t, xb, twN, CtaSync{}, xs);
    for_roots<2 * E, 1, -1, E>(cconj(ldtw(&tw2N[t])), [&](int i, double2 w) { s[i] = cmul(cmul(v[i], w), ophase); });  // c zeta_{2m}^{-k} U_k
    mbar_wait(&bars[0], phase);
    phase ^= 1;
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = sf[(t + T * i) * W + c];
    __syncthreads();
    if (threadIdx.x == 0 && nx < tl.ntiles) {
      mbar_arrive_expect_tx(&bars[0], BYTES);
      load_f(sf, c2, item2, &bars[0]);
    }
    fft<N, E, -1>(v, t, xb, twN, CtaSync{}, xs);
    if constexpr (TS) {
#pragma unroll
      for (int i = 0; i < E; ++i) v[i] = cscale(cadd(v[i], s[i]), inv);
      tile_store<N, E, W, BR>(v, t, c, xb, &mf, col0, item);
    } else if (ok) {
      double2* p = a + (long)t * tl.ncols;
      const long rs = (long)T * tl.ncols;
#pragma unroll
      for (int i = 0; i < E; ++i, p += rs) *p = cscale(cadd(v[i], s[i]), inv);
    }
  }
  if (TS && threadIdx.x == 0) bulk_wait_all();
}

// ------------------------------------------------------------------- K7 --
// Centered column of 2N-1 rows staged whole (2N rows of stage, last one
// padding), three streams written as in pencils.cu.
// K7 output path: each residue's transformed tile is parked in the exchange
// buffer ([row][column], the FFT's last exchange is complete) and written by
// TMA tensor stores -- per-thread 16-byte stores of a W = 2..4-column tile
// kept the store data registers busy (32% long-scoreboard stalls on the
// registers of the next store, ncu r01).  Maps: f rows 0..m-2 / m-1..2m-2,
// the same for g, and U / V rows 0..m-1 (row m = the r = 0 stream's last
// element, stored directly).
// K8: both output halves through TMA stores (2; measured hconv3d -2.3%), U_k only
// (1), or per-thread stores (0)
struct K7StoreMaps {
  CUtensorMap flo, fhi, glo, ghi, u, v;
};

template <int N, bool DIST = false>
__global__ void __launch_bounds__(K78Cfg<N>::THREADS, IDC_PENCIL0_MINB)
k_pad0_bwd_tma(const __grid_constant__ CUtensorMap mf, const __grid_constant__ CUtensorMap mg,
               double2* __restrict__ f, double2* __restrict__ g, double2* __restrict__ U, double2* __restrict__ V,
               Tiles tl, const double2* __restrict__ twN, const double2* __restrict__ tw3N,
               const __grid_constant__ K7StoreMaps sm, const __grid_constant__ DistIO dio) {
  pdl_entry();
  static_assert(!DIST || IDC_K7_TMA_STORE, "distributed K7 stores through TMA");
  using C = K78Cfg<N>;
  constexpr int E = C::E, T = C::T, W = C::W, BR = C::BR;
  constexpr int R2 = ((2 * N - 1 + BR - 1) / BR) * BR;              // staged rows
  extern __shared__ __align__(128) double2 smem[];
  double2* stage = smem;                                            // R2 x W
  double2* xb = stage + R2 * W;
  uint64_t* bar = reinterpret_cast<uint64_t*>(xb + C::XB);
  const int c = threadIdx.x % W, t = threadIdx.x / W;
  const Slot2<W> xs{c};
  constexpr uint32_t BYTES = (uint32_t)R2 * W * 16;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  long tau = blockIdx.x;
  if (threadIdx.x == 0 && tau < tl.ntiles) {
    int in; long item, col0;
    tile_coords(tl, tau, W, in, item, col0);
    mbar_arrive_expect_tx(bar, BYTES);
    load_rows<W, BR>(in == 0 ? &mf : &mg, stage, col0, 0, 2 * N - 1, item, bar);
  }
  const double s3 = 0.86602540378443864676372317075294;
  uint32_t phase = 0;
  for (; tau < tl.ntiles; tau += gridDim.x) {
    int in; long item, col0;
    tile_coords(tl, tau, W, in, item, col0);
    const long col = col0 + c;
    const bool ok = col < tl.ncols;
#if !IDC_K7_TMA_STORE
    double2* a = (in == 0 ? f : g) + item * tl.bstride + (ok ? col : 0);
#endif
    double2* u = (in == 0 ? U : V) + item * tl.ustride + (ok ? col : 0);
    const long S = tl.ncols;
    mbar_wait(bar, phase);
    phase ^= 1;
    // U_k and U_{k-m} are re-read from the stage for every residue (keeping
    // them in registers across the three transforms spilled at 128 registers:
    // 1.4x the shared loads in local-memory loads); the next tile's copy is
    // issued after the last residue's read.
    double2 v[E];
    const long nx = tau + gridDim.x;
    // IDC_K7_KEEP_RAW: U_k, U_{k-m} read from the stage once into registers
    // (the three residue splits re-read nothing) and the stage is refilled
    // with the next tile right away, overlapping all three transforms
    constexpr bool KEEP = IDC_K7_KEEP_RAW;
    double2 A[KEEP ? E : 1], B[KEEP ? E : 1];
    if constexpr (KEEP) {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int k = t + T * i;
        A[i] = stage[(N - 1 + k) * W + c];                                // U_k
        B[i] = (i == 0 && t == 0) ? make_double2(0, 0) : stage[(k - 1) * W + c];   // U_{k-m}
      }
      __syncthreads();
      if (threadIdx.x == 0 && nx < tl.ntiles) {
        int in2; long item2, c2;
        tile_coords(tl, nx, W, in2, item2, c2);
        mbar_arrive_expect_tx(bar, BYTES);
        load_rows<W, BR>(in2 == 0 ? &mf : &mg, stage, c2, 0, 2 * N - 1, item2, bar);
      }
    }
#pragma unroll 1
    for (int rr = 0; rr < 3; ++rr) {
      const int r = rr - 1;
      const double2 z3 = make_double2(r == 0 ? 1.0 : -0.5, r == 0 ? 0.0 : (r < 0 ? s3 : -s3));  // zeta_3^{-r}
      // zeta_{3m}^{rk}, k = t + T i: zeta_{3m}^{rt} x zeta_{3E}^{ri} (immediate)
      auto split = [&](int i, double2 zr) {
        const int k = t + T * i;
        const double2 up = KEEP ? A[i] : stage[(N - 1 + k) * W + c];     // U_k
        if (i == 0 && t == 0) {
          v[i] = up;
        } else {
          const double2 un = KEEP ? B[i] : stage[(k - 1) * W + c];        // U_{k-m}
          v[i] = cmul(zr, cadd(up, cmul(z3, un)));
        }
      };
      const double2 zt = ldtw(&tw3N[t]);
      if (r == 0) {
#pragma unroll
        for (int i = 0; i < E; ++i) split(i, make_double2(1, 0));
      } else if (r > 0) {
        for_roots<3 * E, 1, +1, E>(zt, split);
      } else {
        for_roots<3 * E, 1, -1, E>(cconj(zt), split);
      }
      if (!KEEP && rr == 2) {
        __syncthreads();
        if (threadIdx.x == 0 && nx < tl.ntiles) {
          int in2; long item2, c2;
          tile_coords(tl, nx, W, in2, item2, c2);
          mbar_arrive_expect_tx(bar, BYTES);
          load_rows<W, BR>(in2 == 0 ? &mf : &mg, stage, c2, 0, 2 * N - 1, item2, bar);
        }
      }
#if IDC_K7_TMA_STORE
      // the previous residue's stores must have read xb before the first
      // exchange writes it: waited for after the first radix pass
      auto drained = [] {
        if (threadIdx.x == 0) bulk_wait_read();
        __syncthreads();
      };
      if constexpr (IDC_PENCIL_WAIT_IN_FFT) {
        fft<N, E, +1>(v, t, xb, twN, CtaSync{}, xs, drained);   // ends with a barrier after its last exchange
      } else {
        drained();
        fft<N, E, +1>(v, t, xb, twN, CtaSync{}, xs);
      }
#pragma unroll
      for (int i = 0; i < E; ++i) xb[(t + T * i) * W + c] = v[i];
      if constexpr (DIST) {                         // stream r = (r+1)-th map of the send blocks, m rows
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
          for (int b = 0; b < N; b += dio.BRd)
            tma_store_4d(&dio.st[in][r + 1], (int)(2 * col0), b % dio.L, (int)item, b / dio.L, xb + (long)b * W);
          bulk_commit();
        }
        continue;
      }
      if (r == 0 && t == T - 1 && ok) u[(long)N * S] = v[E - 1];   // l = m-1 -> U row m
      fence_proxy_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
        const CUtensorMap* mp = r == -1 ? (in == 0 ? &sm.u : &sm.v)
                              : r == 0  ? (in == 0 ? &sm.flo : &sm.glo)
                                        : (in == 0 ? &sm.fhi : &sm.ghi);
        const int rows = r == 0 ? N - 1 : N;
        for (int b = 0; b < rows; b += BR) tma_store_3d(mp, (int)(2 * col0), b, (int)item, xb + (long)b * W);
        bulk_commit();
      }
#else
      fft<N, E, +1>(v, t, xb, twN, CtaSync{}, xs);
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
#endif
    }
  }
#if IDC_K7_TMA_STORE
  if (threadIdx.x == 0) bulk_wait_all();
#endif
}

// ------------------------------------------------------------------- K8 --
// Streams staged one at a time (double buffered): q = 0 (r = -1: U rows
// 0..N-1), q = 1 (r = 0: f rows 0..N-2 and U row N, the latter through a
// one-row box into a separate tail slot), q = 2 (r = +1: f rows N-1..2N-2).
template <int N, bool DIST = false>
__global__ void __launch_bounds__(K78Cfg<N>::THREADS, IDC_PENCIL_MINB)
k_pad0_fwd_tma(const __grid_constant__ CUtensorMap mf, const __grid_constant__ CUtensorMap mu,
               const __grid_constant__ CUtensorMap mu1, double2* __restrict__ f, Tiles tl,
               const double2* __restrict__ twN, const double2* __restrict__ tw3N,
               const __grid_constant__ CUtensorMap mflo, const __grid_constant__ CUtensorMap mfhi,
               const __grid_constant__ DistIO dio) {
  pdl_entry();
  static_assert(!DIST || IDC_K8_TMA_STORE == 2, "distributed K8 stores through TMA");
  using C = K78Cfg<N>;
  constexpr int E = C::E, T = C::T, W = C::W, BR = C::BR;
  extern __shared__ __align__(128) double2 smem[];
  double2* st[2] = {smem, smem + N * W};
  // one-row tail slots, 128-byte aligned (TMA tensor destinations): 16 double2 each
  double2* tail[2] = {smem + 2 * N * W, smem + 2 * N * W + 16};
  double2* xb = smem + 2 * N * W + 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(xb + C::XB);
  const int c = threadIdx.x % W, t = threadIdx.x / W;
  const Slot2<W> xs{c};
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // stream q of tile tau -> buffer b
  auto issue = [&](long tau, int q, int b) {
    int in; long item, col0;
    tile_coords(tl, tau, W, in, item, col0);
    if constexpr (DIST) {                   // stream r = q - 1: m uniform rows of the returned blocks
      mbar_arrive_expect_tx(&bars[b], (uint32_t)N * W * 16);
      load_rows_dist<W>(&dio.st[0][q], st[b], col0, N, item, dio.L, dio.BRd, &bars[b]);
      return;
    }
    if (q == 0) {
      mbar_arrive_expect_tx(&bars[b], (uint32_t)N * W * 16);
      load_rows<W, BR>(&mu, st[b], col0, 0, N, item, &bars[b]);
    } else if (q == 1) {
      mbar_arrive_expect_tx(&bars[b], (uint32_t)N * W * 16 + (uint32_t)W * 16);
      load_rows<W, BR>(&mf, st[b], col0, 0, N, item, &bars[b]);          // row N-1 unused (belongs to r = +1)
      tma_load_3d(tail[b], &mu1, (int)(2 * col0), N, (int)item, &bars[b]);  // U row N = stream r = 0, l = N-1
    } else {
      mbar_arrive_expect_tx(&bars[b], (uint32_t)N * W * 16);
      load_rows<W, BR>(&mf, st[b], col0, N - 1, N, item, &bars[b]);
    }
  };
  long tau = blockIdx.x;
  if (threadIdx.x == 0 && tau < tl.ntiles) {
    issue(tau, 0, 0);
    issue(tau, 1, 1);
  }
  const double s3 = 0.86602540378443864676372317075294;
  const double inv = 1.0 / (3.0 * N);
  uint32_t ph[2] = {0, 0};
  int b = 0;
  for (; tau < tl.ntiles; tau += gridDim.x) {
    int in; long item, col0;
    tile_coords(tl, tau, W, in, item, col0);
#if IDC_K8_TMA_STORE != 2
    const long col = col0 + c;
    const bool ok = col < tl.ncols;
    double2* a = f + item * tl.bstride + (ok ? col : 0);
    const long S = tl.ncols;
#endif
    double2 v[E], ap[E], an[E];
#pragma unroll 1
    for (int q = 0; q < 3; ++q) {
      const int r = q - 1;
      mbar_wait(&bars[b], ph[b]);
      ph[b] ^= 1;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int l = t + T * i;
        v[i] = (!DIST && q == 1 && l == N - 1) ? tail[b][c] : st[b][l * W + c];
      }
#if IDC_K8_TMA_STORE
      if (!IDC_PENCIL_WAIT_IN_FFT && q == 0 && threadIdx.x == 0) bulk_wait_read();   // last tile's stores have read xb
#endif
      __syncthreads();
      if (threadIdx.x == 0) {  // refill this buffer with the stream two steps ahead
        const int q2 = q + 2;
        if (q2 < 3) issue(tau, q2, b);
        else if (tau + gridDim.x < tl.ntiles) issue(tau + gridDim.x, q2 - 3, b);
      }
      b ^= 1;
      if (IDC_K8_TMA_STORE && IDC_PENCIL_WAIT_IN_FFT && q == 0) {
        // the last tile's output stores must have read xb before the first
        // exchange writes it: waited for after the first radix pass
        fft<N, E, -1>(v, t, xb, twN, CtaSync{}, xs, [] {
          if (threadIdx.x == 0) bulk_wait_read();
          __syncthreads();
        });
      } else {
        fft<N, E, -1>(v, t, xb, twN, CtaSync{}, xs);
      }
      // 3m U_k = sum_r zeta_{3m}^{-rk} S_r(k); 3m U_{k-m} = sum_r zeta_{3m}^{-rk} zeta_3^{r} S_r(k)
      const double2 z3 = make_double2(r == 0 ? 1.0 : -0.5, r == 0 ? 0.0 : (r > 0 ? s3 : -s3));  // zeta_3^{r}
      auto acc = [&](int i, double2 zr) {                                 // zr = zeta_{3m}^{-rk}
        const double2 p = cmul(zr, v[i]);
        if (q == 0) {
          ap[i] = p;
          an[i] = cmul(z3, p);
        } else {
          ap[i] = cadd(ap[i], p);
          an[i] = cadd(an[i], cmul(z3, p));
        }
      };
      const double2 zt = ldtw(&tw3N[t]);
      if (r == 0) {
#pragma unroll
        for (int i = 0; i < E; ++i) acc(i, make_double2(1, 0));
      } else if (r > 0) {
        for_roots<3 * E, 1, -1, E>(cconj(zt), acc);
      } else {
        for_roots<3 * E, 1, +1, E>(zt, acc);
      }
    }
#if IDC_K8_TMA_STORE
    // U_k -> f rows m-1..2m-2 through the exchange buffer and TMA stores
    // (the last FFT's exchanges are complete)
#pragma unroll
    for (int i = 0; i < E; ++i) xb[(t + T * i) * W + c] = cscale(ap[i], inv);
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int r0 = 0; r0 < N; r0 += BR) tma_store_3d(&mfhi, (int)(2 * col0), r0, (int)item, xb + (long)r0 * W);
      bulk_commit();
    }
#if IDC_K8_TMA_STORE == 2
    if (threadIdx.x == 0) bulk_wait_read();
    __syncthreads();
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int k = t + T * i;
      if (k > 0) xb[(k - 1) * W + c] = cscale(an[i], inv);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int r0 = 0; r0 < N - 1; r0 += BR) tma_store_3d(&mflo, (int)(2 * col0), r0, (int)item, xb + (long)r0 * W);
      bulk_commit();
    }
#else
    if (ok) {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int k = t + T * i;
        if (k > 0) a[(long)(k - 1) * S] = cscale(an[i], inv);
      }
    }
#endif
#else
    if (ok) {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int k = t + T * i;
        a[(long)(N - 1 + k) * S] = cscale(ap[i], inv);
        if (k > 0) a[(long)(k - 1) * S] = cscale(an[i], inv);
      }
    }
#endif
  }
#if IDC_K8_TMA_STORE
  if (threadIdx.x == 0) bulk_wait_all();
#endif
}

// ================================================================ launchers ==
namespace {

template <class K>
cudaError_t launch_t(K kernel, int threads, size_t smem, long ntiles, cudaStream_t s, void** args,
                     const LaunchTag& tag) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  if (per_sm < 1) per_sm = 1;
  long grid = (long)num_sms() * per_sm;
  if (ntiles < grid) grid = ntiles;
  if (grid < 1) grid = 1;
  return launch_kernel((const void*)kernel, dim3((unsigned)grid), dim3(threads), args, smem, s, tag);
}

// DistIO maps of a host DistLayout (nd_internal.cuh), one per (input, stream)
bool make_dist_io(DistIO* io, const DistLayout& dl, long ncols, long nx, int W, int BR, int inputs) {
  memset(io, 0, sizeof(*io));
  io->L = (int)dl.L;
  io->BRd = (int)std::min<long>(BR, dl.L);
  for (int in = 0; in < inputs; ++in)
    for (int st = 0; st < dl.S; ++st)
      if (!encode_blocked_map(&io->st[in][st], dl.base[in] + (long)st * dl.soff, ncols, dl.L, nx, dl.nblocks,
                              dl.xstride, dl.blk, W, io->BRd))
        return false;
  return true;
}

template <int W>
Tiles make_tiles(long ncols, long batch, int inputs, long bstride, long ustride) {
  Tiles tl;
  tl.ncols = ncols;
  tl.nct = (ncols + W - 1) / W;
  tl.batch = batch;
  tl.per_input = tl.nct * batch;
  tl.ntiles = tl.per_input * inputs;
  tl.bstride = bstride;
  tl.ustride = ustride;
  return tl;
}

}  // namespace

template <int N>
cudaError_t pad_bwd_tma(double2* f, double2* g, double2* U, double2* V, long ncols, long batch, long bstride,
                        long ustride, cudaStream_t s, double2 ophase, const DistLayout* dl) {
  using C = K56Cfg<N>;
  const double2* twN = pass_table(N, C::E);
  const double2* tw2N = zeta_table(2 * N);
  if (!twN || !tw2N) return cudaErrorMemoryAllocation;
  CUtensorMap mf, mg;
  if (!encode_pencil_map(&mf, f, ncols, N, batch, bstride, C::W, C::BR)) return cudaErrorNotSupported;
  if (!encode_pencil_map(&mg, g ? g : f, ncols, N, batch, bstride, C::W, C::BR)) return cudaErrorNotSupported;
  Tiles tl = make_tiles<C::W>(ncols, batch, g ? 2 : 1, bstride, ustride);
  CUtensorMap mU, mV;
  DistIO dio;
  if (dl) {                                    // streams into the send blocks; U, V unused
    if (!make_dist_io(&dio, *dl, ncols, batch, C::W, C::BR, g ? 2 : 1)) return cudaErrorNotSupported;
    mU = mf;
    mV = mf;
  } else {
    memset(&dio, 0, sizeof(dio));
    if (!encode_pencil_map(&mU, U, ncols, N, batch, ustride, C::W, C::BR)) return cudaErrorNotSupported;
    if (!encode_pencil_map(&mV, g ? V : U, ncols, N, batch, ustride, C::W, C::BR)) return cudaErrorNotSupported;
  }
  void* args[] = {&mf, &mg, &f, &g, &U, &V, &tl, &twN, &tw2N, &ophase, &mU, &mV, &dio};
  const LaunchTag tag{"K5", N, ncols * batch * (g ? 2 : 1)};
  if (dl) {
    const size_t smem = ((size_t)N * C::W + (size_t)C::XB) * 16 + 16;
    return launch_t(k_pad_bwd_tma<N, true>, C::THREADS, smem, tl.ntiles, s, args, tag);
  }
  const size_t smem = ((size_t)N * C::W + (k5_double_xb<N>() || k5_pair<N>() ? 2 : 1) * (size_t)C::XB) * 16 + 16;
  return launch_t(k_pad_bwd_tma<N, false>, C::THREADS, smem, tl.ntiles, s, args, tag);
}

template <int N>
cudaError_t pad_fwd_tma(double2* f, const double2* U, long ncols, long batch, long bstride, long ustride,
                        cudaStream_t s, double2 ophase, const DistLayout* dl) {
  using C = K56Cfg<N>;
  const double2* twN = pass_table(N, C::E);
  const double2* tw2N = zeta_table(2 * N);
  if (!twN || !tw2N) return cudaErrorMemoryAllocation;
  CUtensorMap mf, mu;
  if (!encode_pencil_map(&mf, f, ncols, N, batch, bstride, C::W, C::BR)) return cudaErrorNotSupported;
  DistIO dio;
  if (dl) {                                    // both streams from the returned blocks; U unused
    if (!make_dist_io(&dio, *dl, ncols, batch, C::W, C::BR, 1)) return cudaErrorNotSupported;
    mu = mf;
  } else {
    memset(&dio, 0, sizeof(dio));
    if (!encode_pencil_map(&mu, U, ncols, N, batch, ustride, C::W, C::BR)) return cudaErrorNotSupported;
  }
  Tiles tl = make_tiles<C::W>(ncols, batch, 1, bstride, ustride);
  void* args[] = {&mf, &mu, &f, &tl, &twN, &tw2N, &ophase, &dio};
  const size_t smem = (2 * (size_t)N * C::W + C::XB) * 16 + 32;
  const LaunchTag tag{"K6", N, ncols * batch};
  if (dl) return launch_t(k_pad_fwd_tma<N, true>, C::THREADS, smem, tl.ntiles, s, args, tag);
  return launch_t(k_pad_fwd_tma<N, false>, C::THREADS, smem, tl.ntiles, s, args, tag);
}

template <int N>
cudaError_t pad0_bwd_tma(double2* f, double2* g, double2* U, double2* V, long ncols, long batch, long bstride,
                         long ustride, cudaStream_t s, const DistLayout* dl) {
  using C = K78Cfg<N>;
  constexpr int R2 = ((2 * N - 1 + C::BR - 1) / C::BR) * C::BR;
  const double2* twN = pass_table(N, C::E);
  const double2* tw3N = zeta_table(3 * N);
  if (!twN || !tw3N) return cudaErrorMemoryAllocation;
  CUtensorMap mf, mg;
  if (!encode_pencil_map(&mf, f, ncols, 2 * N - 1, batch, bstride, C::W, C::BR)) return cudaErrorNotSupported;
  if (!encode_pencil_map(&mg, g ? g : f, ncols, 2 * N - 1, batch, bstride, C::W, C::BR)) return cudaErrorNotSupported;
  Tiles tl = make_tiles<C::W>(ncols, batch, g ? 2 : 1, bstride, ustride);
  K7StoreMaps sm;
  memset(&sm, 0, sizeof(sm));
  DistIO dio;
  memset(&dio, 0, sizeof(dio));
  if (dl) {                                    // the three streams into the send blocks
    if (!make_dist_io(&dio, *dl, ncols, batch, C::W, C::BR, g ? 2 : 1)) return cudaErrorNotSupported;
  } else {
#if IDC_K7_TMA_STORE
    double2* gg = g ? g : f;
    double2* VV = g ? V : U;
    const long lo = ((long)N - 1) * ncols;
    if (!encode_pencil_map(&sm.flo, f, ncols, N - 1, batch, bstride, C::W, C::BR) ||
        !encode_pencil_map(&sm.fhi, f + lo, ncols, N, batch, bstride, C::W, C::BR) ||
        !encode_pencil_map(&sm.glo, gg, ncols, N - 1, batch, bstride, C::W, C::BR) ||
        !encode_pencil_map(&sm.ghi, gg + lo, ncols, N, batch, bstride, C::W, C::BR) ||
        !encode_pencil_map(&sm.u, U, ncols, N, batch, ustride, C::W, C::BR) ||
        !encode_pencil_map(&sm.v, VV, ncols, N, batch, ustride, C::W, C::BR))
      return cudaErrorNotSupported;
#endif
  }
  void* args[] = {&mf, &mg, &f, &g, &U, &V, &tl, &twN, &tw3N, &sm, &dio};
  const size_t smem = ((size_t)R2 * C::W + C::XB) * 16 + 16;
  const LaunchTag tag{"K7", N, ncols * batch * (g ? 2 : 1)};
  if (dl) return launch_t(k_pad0_bwd_tma<N, true>, C::THREADS, smem, tl.ntiles, s, args, tag);
  return launch_t(k_pad0_bwd_tma<N, false>, C::THREADS, smem, tl.ntiles, s, args, tag);
}

template <int N>
cudaError_t pad0_fwd_tma(double2* f, const double2* U, long ncols, long batch, long bstride, long ustride,
                         cudaStream_t s, const DistLayout* dl) {
  using C = K78Cfg<N>;
  const double2* twN = pass_table(N, C::E);
  const double2* tw3N = zeta_table(3 * N);
  if (!twN || !tw3N) return cudaErrorMemoryAllocation;
  CUtensorMap mf, mu, mu1;
  if (!encode_pencil_map(&mf, f, ncols, 2 * N - 1, batch, bstride, C::W, C::BR)) return cudaErrorNotSupported;
  DistIO dio;
  memset(&dio, 0, sizeof(dio));
  if (dl) {                                    // the three streams from the returned blocks; U unused
    if (!make_dist_io(&dio, *dl, ncols, batch, C::W, C::BR, 1)) return cudaErrorNotSupported;
    mu = mf;
    mu1 = mf;
  } else {
    if (!encode_pencil_map(&mu, U, ncols, N + 1, batch, ustride, C::W, C::BR)) return cudaErrorNotSupported;
    if (!encode_pencil_map(&mu1, U, ncols, N + 1, batch, ustride, C::W, 1)) return cudaErrorNotSupported;
  }
  Tiles tl = make_tiles<C::W>(ncols, batch, 1, bstride, ustride);
  CUtensorMap mflo, mfhi;
  if (!encode_pencil_map(&mflo, f, ncols, N - 1, batch, bstride, C::W, C::BR)) return cudaErrorNotSupported;
  if (!encode_pencil_map(&mfhi, f + ((long)N - 1) * ncols, ncols, N, batch, bstride, C::W, C::BR))
    return cudaErrorNotSupported;
  void* args[] = {&mf, &mu, &mu1, &f, &tl, &twN, &tw3N, &mflo, &mfhi, &dio};
  const size_t smem = (2 * (size_t)N * C::W + 32 + C::XB) * 16 + 32;
  const LaunchTag tag{"K8", N, ncols * batch};
  if (dl) return launch_t(k_pad0_fwd_tma<N, true>, C::THREADS, smem, tl.ntiles, s, args, tag);
  return launch_t(k_pad0_fwd_tma<N, false>, C::THREADS, smem, tl.ntiles, s, args, tag);
}

#define IDC_INST_T(N)                                                                                           \
  template cudaError_t pad_bwd_tma<N>(double2*, double2*, double2*, double2*, long, long, long, long, cudaStream_t, \
                                      double2, const DistLayout*);                                                 \
  template cudaError_t pad_fwd_tma<N>(double2*, const double2*, long, long, long, long, cudaStream_t, double2,      \
                                      const DistLayout*);                                                          \
  template cudaError_t pad0_bwd_tma<N>(double2*, double2*, double2*, double2*, long, long, long, long,             \
                                       cudaStream_t, const DistLayout*);                                         \
  template cudaError_t pad0_fwd_tma<N>(double2*, const double2*, long, long, long, long, cudaStream_t,             \
                                       const DistLayout*);
IDC_INST_T(64)
IDC_INST_T(128)
IDC_INST_T(256)
IDC_INST_T(512)
IDC_INST_T(1024)
IDC_INST_T(2048)
IDC_INST_T(4096)

}  // namespace idc
