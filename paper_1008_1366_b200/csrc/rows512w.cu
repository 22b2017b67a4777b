// rows512w.cu -- warp-per-row 1D convolutions at m = 512 (the z rows of the
// 3D configs C5a / C5b) on the warp-resident FFT of fft512w.cuh.
//
// Same equations as rows2.cu / rows3.cu (K2: Function cconv; K3:
// the centered Hermitian convolution, with the f + i g packing of
// DESIGN.md section 6); what changes is the engine: each warp owns one row
// (lane t holds k = t + 32 i, i < 16), its transforms need one shared-memory
// transpose plus one shuffle stage instead of two exchanges, and its
// synchronisation is __syncwarp() -- the 8 warps of a CTA run independent
// rows with no CTA barrier.  Each warp stages its f and g rows in shared
// memory by bulk copies (one mbarrier per warp); the next row is prefetched
// into L2 at the start of the current one and its bulk copy is issued as
// soon as the current row's last residue split has read the stage.
//
// The backward transforms leave the lane-pair order sigma (fft512w.cuh); the
// pointwise products are taken there and the forward transforms return to
// natural order, so no reordering pass exists anywhere.
#include "fft512w.cuh"
#include "kernels.cuh"
#include "launch.cuh"
#include "tables.cuh"
#include "tma.cuh"

namespace idc {

namespace {

constexpr int M = 512, E = 16, WARPS = 8, THREADS = 32 * WARPS;
// per warp: staged f and g rows, the transpose slots
constexpr int PER = 2 * M + w512::XB;
constexpr size_t SMEM = (size_t)WARPS * PER * 16 + (size_t)WARPS * 8;

struct WarpRow {
  double2 *F, *Gs, *xw;
  uint64_t* bar;
  int lane;
};

__device__ __forceinline__ WarpRow warp_row(double2* smem) {
  const int w = threadIdx.x >> 5;
  WarpRow r;
  r.F = smem + w * PER;
  r.Gs = r.F + M;
  r.xw = r.Gs + M;
  r.bar = reinterpret_cast<uint64_t*>(smem + WARPS * PER) + w;
  r.lane = threadIdx.x & 31;
  return r;
}

__device__ __forceinline__ void issue_row(const WarpRow& wr, const double2* f, const double2* g) {
  mbar_arrive_expect_tx(wr.bar, 2u * M * 16u);
  tma_load_1d(wr.F, f, M * 16u, wr.bar);
  tma_load_1d(wr.Gs, g, M * 16u, wr.bar);
}

}  // namespace

// ================================================================= K2w ==
// Function cconv per row: r = 0 and r = 1 (zeta_{2m}^k-shifted)
// streams of f and g transformed backward, multiplied, transformed forward,
// f <- (F_0 + zeta_{2m}^{-k} F_1) / 2m.
__global__ void __launch_bounds__(THREADS, 1)
k_cconv_rows512w(double2* __restrict__ f, double2* __restrict__ g, long nrows, const double2* __restrict__ tw,
                 const double2* __restrict__ tw2M, RowSets rs) {
  extern __shared__ __align__(128) double2 smem[];
  const WarpRow wr = warp_row(smem);
  const int t = wr.lane;
  const long stride = (long)gridDim.x * WARPS;
  long row = (long)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (t == 0) {
    mbar_init(wr.bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (t == 0 && row < nrows) issue_row(wr, row_ptr(f, rs.f1, rs.n0, row, M), row_ptr(g, rs.g1, rs.n0, row, M));
  const double inv = 1.0 / (2.0 * M);
  uint32_t phase = 0;
  for (; row < nrows; row += stride) {
    const bool more = row + stride < nrows;
    if (t == 0 && more) {
      prefetch_l2(row_ptr(f, rs.f1, rs.n0, row + stride, M), M * 16u);
      prefetch_l2(row_ptr(g, rs.g1, rs.n0, row + stride, M), M * 16u);
    }
    mbar_wait(wr.bar, phase);
    phase ^= 1;
    double2 x[E], y[E];
#pragma unroll
    for (int i = 0; i < E; ++i) x[i] = wr.F[t + 32 * i];
#pragma unroll
    for (int i = 0; i < E; ++i) y[i] = wr.Gs[t + 32 * i];
    fft512w_bwd<+1>(x, t, wr.xw, tw);                            // r = 0
    fft512w_bwd<+1>(y, t, wr.xw, tw);
#pragma unroll
    for (int i = 0; i < E; ++i) x[i] = cmul(x[i], y[i]);
    fft512w_fwd<-1>(x, t, wr.xw, tw);                            // F_0, natural order
    // r = 1: zeta_{2m}^k-shifted streams; x parked in the f stage
    // slots of this lane (its own k), the stage is read for the last time here
    const double2 zt = ldtw(&tw2M[t]);
    double2 z[E];
    for_roots<2 * E, 1, +1, E>(zt, [&](int i, double2 w) {
      const int k = t + 32 * i;
      y[i] = cmul(wr.F[k], w);
      z[i] = cmul(wr.Gs[k], w);
      wr.F[k] = x[i];
    });
    fft512w_bwd<+1>(y, t, wr.xw, tw);
    fft512w_bwd<+1>(z, t, wr.xw, tw);
#pragma unroll
    for (int i = 0; i < E; ++i) y[i] = cmul(y[i], z[i]);
    fft512w_fwd<-1>(y, t, wr.xw, tw);                            // F_1
    double2* fw = row_ptr(f, rs.f1, rs.n0, row, M);
    for_roots<2 * E, 1, -1, E>(cconj(zt), [&](int i, double2 w) {     // zeta_{2m}^{-k}
      const int k = t + 32 * i;
      fw[k] = cscale(cadd(wr.F[k], cmul(y[i], w)), inv);
    });
    fence_proxy_async_smem();   // the parked x (generic writes) before the bulk copy refills the stage
    __syncwarp();
    if (t == 0 && more)
      issue_row(wr, row_ptr(f, rs.f1, rs.n0, row + stride, M), row_ptr(g, rs.g1, rs.n0, row + stride, M));
  }
}

// ================================================================= K3w ==
// Centered Hermitian convolution per row: residues r = 0, 1, -1
// of the packed pair (f + i g), three backward transforms (each two c2r),
// the real products, FFT(p_0 + i p_1) and FFT(p_{-1}), recombination
// 3m h_k = P_0 + zeta_{3m}^{k} P_{-1} + zeta_{3m}^{-k} P_1 (Eq. fft0forwardB).
__global__ void __launch_bounds__(THREADS, 1)
k_hconv_rows512w(double2* __restrict__ f, double2* __restrict__ g, long nrows, const double2* __restrict__ tw,
                 const double2* __restrict__ tw3M, RowSets rs) {
  extern __shared__ __align__(128) double2 smem[];
  const WarpRow wr = warp_row(smem);
  const int t = wr.lane;
  const long stride = (long)gridDim.x * WARPS;
  long row = (long)blockIdx.x * WARPS + (threadIdx.x >> 5);
  if (t == 0) {
    mbar_init(wr.bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (t == 0 && row < nrows) issue_row(wr, row_ptr(f, rs.f1, rs.n0, row, M), row_ptr(g, rs.g1, rs.n0, row, M));
  const double inv = 1.0 / (3.0 * M);
  const double s3 = 0.86602540378443864676372317075294;  // sqrt(3)/2
  const double2* F = wr.F;
  const double2* Gs = wr.Gs;
  uint32_t phase = 0;
  for (; row < nrows; row += stride) {
    const bool more = row + stride < nrows;
    if (t == 0 && more) {
      prefetch_l2(row_ptr(f, rs.f1, rs.n0, row + stride, M), M * 16u);
      prefetch_l2(row_ptr(g, rs.g1, rs.n0, row + stride, M), M * 16u);
    }
    mbar_wait(wr.bar, phase);
    phase ^= 1;
    double2 v[E], Q[E];
    double p0[E];
    // residues r = 0 and r = 1 from one read of the staged pair:
    // P_k = f_k + i g_k, R_k = conj f_{m-k} + i conj g_{m-k};
    // v = P + R (r = 0), Q = zeta_{3m}^{k} (P + zeta_3^{-1} R) (r = 1)
    for_roots<3 * E, 1, +1, E>(ldtw(&tw3M[t]), [&](int i, double2 zr) {
      const int k = t + 32 * i;
      if (i == 0 && t == 0) {
        v[i] = Q[i] = make_double2(F[0].x, Gs[0].x);              // w_{0,r} = Re U_0 (AMB-7)
      } else {
        const double2 fk = F[k], gk = Gs[k], fm = F[M - k], gm = Gs[M - k];
        const double2 P = make_double2(fk.x - gk.y, fk.y + gk.x);
        const double2 R = make_double2(fm.x + gm.y, gm.x - fm.y);
        v[i] = cadd(P, R);
        const double2 A = make_double2(fma(-0.5, R.x, P.x), fma(-0.5, R.y, P.y));
        const double2 B = make_double2(-s3 * R.y, s3 * R.x);
        Q[i] = cmul(zr, csub(A, B));
      }
    });
    fft512w_bwd<+1>(v, t, wr.xw, tw);                             // two c2r in one complex FFT
#pragma unroll
    for (int i = 0; i < E; ++i) p0[i] = v[i].x * v[i].y;
    fft512w_bwd<+1>(Q, t, wr.xw, tw);
#pragma unroll
    for (int i = 0; i < E; ++i) Q[i] = make_double2(p0[i], Q[i].x * Q[i].y);
    fft512w_fwd<-1>(Q, t, wr.xw, tw);                             // Q = fft(p_0 + i p_1), natural order
    // r = -1: zeta_{3m}^{-k} (P + zeta_3 R), the last read of the staged pair
    for_roots<3 * E, 1, -1, E>(cconj(ldtw(&tw3M[t])), [&](int i, double2 zr) {
      const int k = t + 32 * i;
      if (i == 0 && t == 0) {
        v[i] = make_double2(F[0].x, Gs[0].x);
      } else {
        const double2 fk = F[k], gk = Gs[k], fm = F[M - k], gm = Gs[M - k];
        const double2 P = make_double2(fk.x - gk.y, fk.y + gk.x);
        const double2 R = make_double2(fm.x + gm.y, gm.x - fm.y);
        const double2 A = make_double2(fma(-0.5, R.x, P.x), fma(-0.5, R.y, P.y));
        const double2 B = make_double2(-s3 * R.y, s3 * R.x);
        v[i] = cmul(zr, cadd(A, B));
      }
    });
    __syncwarp();
    if (t == 0 && more)
      issue_row(wr, row_ptr(f, rs.f1, rs.n0, row + stride, M), row_ptr(g, rs.g1, rs.n0, row + stride, M));
    fft512w_bwd<+1>(v, t, wr.xw, tw);
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = make_double2(v[i].x * v[i].y, 0.0);
    fft512w_fwd<-1>(v, t, wr.xw, tw);                             // P_{-1}, natural order
    // P_0, P_1 from Q via Q_{m-k}; 3m h_k = P_0 + zeta^{k} P_{-1} + zeta^{-k} P_1
#pragma unroll
    for (int i = 0; i < E; ++i) wr.xw[t + 32 * i] = Q[i];
    __syncwarp();
    double2* fw = row_ptr(f, rs.f1, rs.n0, row, M);
    for_roots<3 * E, 1, +1, E>(ldtw(&tw3M[t]), [&](int i, double2 tz) {
      const int k = t + 32 * i;
      const double2 a = Q[i], b = cconj(wr.xw[(M - k) & (M - 1)]);
      const double2 pp0 = cscale(cadd(a, b), 0.5);
      const double2 d = csub(a, b);
      const double2 pp1 = make_double2(0.5 * d.y, -0.5 * d.x);
      fw[k] = cscale(cadd(cadd(pp0, cmul(v[i], tz)), cmulc(pp1, tz)), inv);
    });
    __syncwarp();
  }
}

// ================================================================ launchers ==
namespace {
cudaError_t launch512w(const void* kernel, long nrows, cudaStream_t s, void** args, const char* tag) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
  if (e != cudaSuccess) return e;
  long grid = num_sms();
  const long need = (nrows + WARPS - 1) / WARPS;
  if (need < grid) grid = need;
  if (grid < 1) grid = 1;
  return launch_kernel(kernel, dim3((unsigned)grid), dim3(THREADS), args, SMEM, s, {tag, M, nrows});
}
}  // namespace

cudaError_t cconv_rows512w(double2* f, double2* g, long nrows, cudaStream_t s, RowSets rs) {
  const double2* tw = warp512_table();
  const double2* tw2M = zeta_table(2 * M);
  if (!tw || !tw2M) return cudaErrorMemoryAllocation;
  void* args[] = {&f, &g, &nrows, &tw, &tw2M, &rs};
  return launch512w((const void*)k_cconv_rows512w, nrows, s, args, "K2w");
}

cudaError_t hconv_rows512w(double2* f, double2* g, long nrows, cudaStream_t s, RowSets rs) {
  const double2* tw = warp512_table();
  const double2* tw3M = zeta_table(3 * M);
  if (!tw || !tw3M) return cudaErrorMemoryAllocation;
  void* args[] = {&f, &g, &nrows, &tw, &tw3M, &rs};
  return launch512w((const void*)k_hconv_rows512w, nrows, s, args, "K3w");
}

}  // namespace idc
