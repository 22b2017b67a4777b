// nd.cu -- 2D and 3D implicitly dealiased convolutions composed from the
// pencil kernels (K5-K8, pencils.cu) and the fused row kernels (K2/K3).
//
//   cconv2d  Function cconv2:  K5 along x -> K2 on the rows of
//            both residue streams (f, U) -> K6 along x.
//   hconv2d  Function conv2:  K7 along x -> K3 on the 2mx-1
//            rows of f and the mx+1 rows of U -> K8 along x.
//   cconv3d  Function cconv3:  K5 along x over all (y,z)
//            columns, then cconv2 on every x-residue slab, K6 along x.
//   hconv3d  "analogous manner" (AMB-9): K7 along x, conv2 on
//            every x-residue slab, K8 along x.
//
// The paper reuses one set of 2D work arrays u2, v2 for all slabs (P:880-889,
// P:920-925).  Here the slabs are processed in groups of G whose 2D work
// arrays U2, V2 (G slabs each) are sized to stay resident in L2
// (SURVEY §8(a) a9), so only the slab read and the slab result write reach
// HBM.  All launches are stream-ordered on the caller's stream.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"
#include "nd.cuh"
#include "nd_internal.cuh"

namespace idc {

namespace {
constexpr size_t W16 = sizeof(double2);
bool pow2ok(size_t m) { return m >= 1 && m <= 8192 && (m & (m - 1)) == 0; }

size_t l2_bytes() {
  static int l2 = 0;
  if (l2 == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) != cudaSuccess || l2 <= 0) l2 = 126 << 20;
  }
  return (size_t)l2;
}

// slabs per group = (IDC_SLAB_L2_FRAC percent of L2) / (per-slab bytes of all
// streams in flight).  Measured on B200 (profiles/): an
// L2-resident group (50%: one 512^2 slab per stream, 512-row launches) is
// 17% slower than groups of ~10-20 slabs whose launches fill the GPU several
// times over -- launch granularity matters more than L2 residency here, so
// the default budget is 20x L2 (frac 2000).
long slab_group(size_t slab_bytes_all, long nslabs) {
  static long frac = -1;
  if (frac < 0) {
    const char* e = getenv("IDC_SLAB_L2_FRAC");
    frac = e ? atol(e) : 2000;
  }
  long G = (long)((l2_bytes() * frac / 100) / std::max<size_t>(slab_bytes_all, 1));
  return std::max<long>(1, std::min<long>(G, nslabs));
}
// Internal stream pool for concurrent slab groups (created once per device).
constexpr int kMaxSlabStreams = 4;
// slab streams in flight (IDC_SLAB_STREAMS, 1..4, default 2; measured
// sweep tools/slab_sweep3.sh: 2 streams x ~80-slab groups best by ~1%)
int slab_streams() {
  static int n = 0;
  if (n == 0) {
    const char* e = getenv("IDC_SLAB_STREAMS");
    n = e ? atoi(e) : 2;
    if (n < 1 || n > kMaxSlabStreams) n = 2;
  }
  return n;
}
struct Pool {
  cudaStream_t s[kMaxSlabStreams];
  cudaEvent_t fork, done[kMaxSlabStreams];
  std::mutex enq;      // held from the fork record to the last join (concurrent callers)
  bool ok = false;
};
Pool& pool() {
  static Pool p[16];
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  Pool& q = p[dev & 15];
  if (!q.ok) {
    for (int i = 0; i < kMaxSlabStreams; ++i) {
      cudaStreamCreateWithFlags(&q.s[i], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&q.done[i], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&q.fork, cudaEventDisableTiming);
    q.ok = true;
  }
  return q;
}
}  // namespace

// ------------------------------------------------------------ workspaces --
size_t cconv2d_work_bytes(size_t mx, size_t my, size_t batch) {
  if (!pow2ok(mx) || !pow2ok(my) || batch == 0) return 0;
  return 2 * batch * mx * my * W16 + cconv_rows_work_bytes((int)my);
}
size_t hconv2d_work_bytes(size_t mx, size_t my) {
  if (!pow2ok(mx) || !pow2ok(my)) return 0;
  return 2 * (mx + 1) * my * W16 + hconv_rows_work_bytes((int)my);
}
// slabs per group; slab_streams() groups are in flight at once, so the L2
// budget is shared between them
static long c3_group(size_t mx, size_t my, size_t mz) {
  return slab_group(slab_streams() * 4 * my * mz * W16, 2 * (long)mx);
}
static long h3_group(size_t mx, size_t my, size_t mz) {
  return slab_group(slab_streams() * 2 * ((2 * my - 1) + (my + 1)) * mz * W16, 3 * (long)mx);
}
size_t cconv3d_work_bytes(size_t mx, size_t my, size_t mz) {
  if (!pow2ok(mx) || !pow2ok(my) || !pow2ok(mz)) return 0;
  const long G = c3_group(mx, my, mz);
  return 2 * mx * my * mz * W16 + slab_streams() * (2 * (size_t)G * my * mz * W16 + cconv_rows_work_bytes((int)mz));
}
size_t hconv3d_work_bytes(size_t mx, size_t my, size_t mz) {
  if (!pow2ok(mx) || !pow2ok(my) || !pow2ok(mz)) return 0;
  const long G = h3_group(mx, my, mz);
  return 2 * (mx + 1) * (2 * my - 1) * mz * W16 +
         slab_streams() * (2 * (size_t)G * (my + 1) * mz * W16 + hconv_rows_work_bytes((int)mz));
}

// ------------------------------------------------------------------- 2D --
#define IDC_TRY(x)                       \
  do {                                   \
    cudaError_t e_ = (x);                \
    if (e_ != cudaSuccess) return e_;    \
  } while (0)

cudaError_t run_cconv2d(double2* f, double2* g, int mx, int my, long batch, double2* work, cudaStream_t s) {
  const long n = (long)mx * my;
  double2* U = work;
  double2* V = work + batch * n;
  double2* rw = V + batch * n;
  IDC_TRY(launch_pad_bwd(f, g, U, V, mx, my, batch, n, n, s));            // fftpadBackward on columns
  IDC_TRY(launch_cconv_rows_sets(f, g, batch * mx, U, V, batch * mx, my, rw, s));   // cconv on rows of both streams
  return launch_pad_fwd(f, U, mx, my, batch, n, n, s);                    // fftpadForward on columns
}

cudaError_t run_hconv2d(double2* f, double2* g, int mx, int my, double2* work, cudaStream_t s) {
  double2* U = work;
  double2* V = work + (long)(mx + 1) * my;
  double2* rw = V + (long)(mx + 1) * my;
  IDC_TRY(launch_pad0_bwd(f, g, U, V, mx, my, 1, 0, 0, s));               // fft0padBackward on columns
  IDC_TRY(launch_hconv_rows_sets(f, g, 2L * mx - 1, U, V, (long)mx + 1, my, rw, s));   // conv on the 3mx stream rows
  return launch_pad0_fwd(f, U, mx, my, 1, 0, 0, s);                       // fft0padForward on columns
}

// Multivector dot product: sum_i f_i * g_i of npairs Hermitian
// 2D pairs (pair i at f + i (2mx-1) my), result in pair 0.  Function conv2
// with the product stage summed over the pairs: K7 along x on all 2*npairs
// arrays, K3d on the rows of the three x-streams, K8 on pair 0 only.
size_t hconv2d_dot_work_bytes(size_t npairs, size_t mx, size_t my) {
  if (!pow2ok(mx) || !pow2ok(my) || my > 4096 || npairs == 0) return 0;
  return 2 * npairs * (mx + 1) * my * W16;
}

cudaError_t run_hconv2d_dot(double2* f, double2* g, int npairs, int mx, int my, double2* work, cudaStream_t s) {
  const long fs = (2L * mx - 1) * my, us = ((long)mx + 1) * my;
  double2* U = work;
  double2* V = work + (long)npairs * us;
  IDC_TRY(launch_pad0_bwd(f, g, U, V, mx, my, npairs, fs, us, s));       // fft0padBackward on every column
  IDC_TRY(launch_hconv_dot_rows(f, g, npairs, fs, my, 2L * mx - 1, s));   // dot-product conv, f-stream rows
  IDC_TRY(launch_hconv_dot_rows(U, V, npairs, us, my, (long)mx + 1, s));  // dot-product conv, U-stream rows
  return launch_pad0_fwd(f, U, mx, my, 1, 0, 0, s);                      // fft0padForward, pair 0
}

// Function tconv2: fft0tpadBackward along x on every column of
// f, g, h (2mx rows, origin at row mx, row 0 = kx -mx = 0): with k' = k + mx,
// u_{2l+r} = (-1)^l i^{-r} sum_{k'} zeta_{2mx}^{lk'} zeta_{4mx}^{rk'} U_{k'-mx}
// (Eq. fft0tbackward): fftpadBackward of the 2mx-row column (K5, N = 2mx)
// gives (-1)^l i^{r} u_{2l+r}; the odd stream is multiplied by i^{-1} so that
// every row is (-1)^l u (real factor: the rows stay Hermitian in ky for the
// 1D ternary row kernel K4).  The ternary product carries (-1)^{3l} =
// (-1)^l, which is exactly the (-1)^l of Eq. fft0tforward, leaving
// 4m U_k = sum_r zeta_{4m}^{-rk'} i^r fft(p_r)(k'): K6 with odd phase i.
size_t tconv2d_work_bytes(size_t mx, size_t my) {
  if (!pow2ok(mx) || !pow2ok(my) || mx > 2048 || my > 4096) return 0;
  return 3 * 2 * mx * my * W16 + tconv_rows_work_bytes((int)my);
}

cudaError_t run_tconv2d(double2* f, double2* g, double2* h, int mx, int my, double2* work, cudaStream_t s) {
  const long n = 2L * mx * my, N = 2L * mx;
  double2* U = work;
  double2* V = U + n;
  double2* Wk = V + n;
  double2* rw = Wk + n;
  for (double2* a : {f, g, h}) IDC_TRY(cudaMemsetAsync(a, 0, (size_t)my * W16, s));   // row kx = -mx
  const double2 mi = {0.0, -1.0}, pi = {0.0, 1.0};
  IDC_TRY(launch_pad_bwd(f, g, U, V, (int)N, my, 1, 0, 0, s, mi));       // fft0tpadBackward: f, g
  IDC_TRY(launch_pad_bwd(h, nullptr, Wk, nullptr, (int)N, my, 1, 0, 0, s, mi));   // and h
  IDC_TRY(launch_tconv_rows(f, g, h, my, N, rw, s));                    // tconv on the r = 0 rows
  IDC_TRY(launch_tconv_rows(U, V, Wk, my, N, rw, s));                   // tconv on the r = 1 rows
  IDC_TRY(launch_pad_fwd(f, U, (int)N, my, 1, 0, 0, s, pi));            // fft0tpadForward
  return cudaMemsetAsync(f, 0, (size_t)my * W16, s);                    // kx = -mx: outside the range
}

// Complex 2D dot product (Function cconv2 with sum_i f_i * g_i): K5 along x on
// all 2*npairs arrays, K2d on the rows of both x-streams, K6 on pair 0.
size_t cconv2d_dot_work_bytes(size_t npairs, size_t mx, size_t my) {
  if (!pow2ok(mx) || !pow2ok(my) || my > 4096 || npairs == 0) return 0;
  return 2 * npairs * mx * my * W16;
}

cudaError_t run_cconv2d_dot(double2* f, double2* g, int npairs, int mx, int my, double2* work, cudaStream_t s) {
  const long n = (long)mx * my;
  double2* U = work;
  double2* V = work + (long)npairs * n;
  IDC_TRY(launch_pad_bwd(f, g, U, V, mx, my, npairs, n, n, s));           // fftpadBackward on every column
  IDC_TRY(launch_cconv_dot_rows(f, g, npairs, n, my, mx, s));             // dot-product rows, even x-stream
  IDC_TRY(launch_cconv_dot_rows(U, V, npairs, n, my, mx, s));             // dot-product rows, odd x-stream
  return launch_pad_fwd(f, U, mx, my, 1, 0, 0, s);                        // fftpadForward, pair 0
}

// ------------------------------------------------------------------- 3D --
cudaError_t run_cconv3d(double2* f, double2* g, int mx, int my, int mz, double2* work, cudaStream_t s) {
  const long slab = (long)my * mz, n = (long)mx * slab;
  const long G = c3_group(mx, my, mz);
  double2* U = work;
  double2* V = U + n;
  double2* per = V + n;                                    // slab_streams() x (U2, V2, row work)
  const long per_elems = 2 * G * slab + (long)(cconv_rows_work_bytes(mz) / W16);
  IDC_TRY(launch_pad_bwd(f, g, U, V, mx, slab, 1, 0, 0, s));              // x: fftpadBackward over all (y,z)
  Pool& P = pool();
  std::lock_guard<std::mutex> enq(P.enq);
  IDC_TRY(cudaEventRecord(P.fork, s));
  for (int i = 0; i < slab_streams(); ++i) IDC_TRY(cudaStreamWaitEvent(P.s[i], P.fork, 0));
  long gi = 0;
  for (int half = 0; half < 2; ++half) {                                   // x-residue slabs: f (even), U (odd)
    double2* A = half == 0 ? f : U;
    double2* B = half == 0 ? g : V;
    for (long s0 = 0; s0 < mx; s0 += G, ++gi) {
      const long gs = std::min<long>(G, mx - s0);
      cudaStream_t st = P.s[gi % slab_streams()];
      double2* U2 = per + (gi % slab_streams()) * per_elems;
      double2* V2 = U2 + G * slab;
      double2* rw = V2 + G * slab;
      double2* a = A + s0 * slab;
      double2* b = B + s0 * slab;
      // cconv2 on the group's slabs, reusing this stream's U2/V2
      IDC_TRY(launch_pad_bwd(a, b, U2, V2, my, mz, gs, slab, slab, st));
      IDC_TRY(launch_cconv_rows_sets(a, b, gs * my, U2, V2, gs * my, mz, rw, st));
      IDC_TRY(launch_pad_fwd(a, U2, my, mz, gs, slab, slab, st));
    }
  }
  for (int i = 0; i < slab_streams(); ++i) {
    IDC_TRY(cudaEventRecord(P.done[i], P.s[i]));
    IDC_TRY(cudaStreamWaitEvent(s, P.done[i], 0));
  }
  return launch_pad_fwd(f, U, mx, slab, 1, 0, 0, s);                     // x: fftpadForward
}

cudaError_t run_hconv3d(double2* f, double2* g, int mx, int my, int mz, double2* work, cudaStream_t s) {
  const long slab = (long)(2 * my - 1) * mz;       // one x-residue slab (2my-1) x mz
  const long uslab = (long)(my + 1) * mz;          // its y work array (my+1) x mz
  const long G = h3_group(mx, my, mz);
  double2* U = work;                                // (mx+1) slabs
  double2* V = U + (long)(mx + 1) * slab;
  double2* per = V + (long)(mx + 1) * slab;
  const long per_elems = 2 * G * uslab + (long)(hconv_rows_work_bytes(mz) / W16);
  IDC_TRY(launch_pad0_bwd(f, g, U, V, mx, slab, 1, 0, 0, s));             // x: fft0padBackward
  Pool& P = pool();
  std::lock_guard<std::mutex> enq(P.enq);
  IDC_TRY(cudaEventRecord(P.fork, s));
  for (int i = 0; i < slab_streams(); ++i) IDC_TRY(cudaStreamWaitEvent(P.s[i], P.fork, 0));
  long gi = 0;
  for (int half = 0; half < 2; ++half) {                                   // slabs: 2mx-1 in f, mx+1 in U
    double2* A = half == 0 ? f : U;
    double2* B = half == 0 ? g : V;
    const long ns = half == 0 ? 2L * mx - 1 : (long)mx + 1;
    for (long s0 = 0; s0 < ns; s0 += G, ++gi) {
      const long gs = std::min<long>(G, ns - s0);
      cudaStream_t st = P.s[gi % slab_streams()];
      double2* U2 = per + (gi % slab_streams()) * per_elems;
      double2* V2 = U2 + G * uslab;
      double2* rw = V2 + G * uslab;
      double2* a = A + s0 * slab;
      double2* b = B + s0 * slab;
      // conv2 on the group's slabs, reusing this stream's U2/V2
      IDC_TRY(launch_pad0_bwd(a, b, U2, V2, my, mz, gs, slab, uslab, st));
      IDC_TRY(launch_hconv_rows_sets(a, b, gs * (2L * my - 1), U2, V2, gs * ((long)my + 1), mz, rw, st));
      IDC_TRY(launch_pad0_fwd(a, U2, my, mz, gs, slab, uslab, st));
    }
  }
  for (int i = 0; i < slab_streams(); ++i) {
    IDC_TRY(cudaEventRecord(P.done[i], P.s[i]));
    IDC_TRY(cudaStreamWaitEvent(s, P.done[i], 0));
  }
  return launch_pad0_fwd(f, U, mx, slab, 1, 0, 0, s);                    // x: fft0padForward
}

}  // namespace idc
