// dist.cu -- slab-decomposed 3D implicitly dealiased convolution over NCCL
// (the paper is single-process; this decomposition is ours).
//
// Layout: the global mx x my x mz complex arrays f, g are split into x-slabs;
// rank r holds planes [r*nx, (r+1)*nx), nx = mx/P, full y and z.
//
//   A. y is locally complete: fftpadBackward along y (K5) on every local
//      x-plane gives S = 2 residue streams (even, odd) of my rows each.  The
//      rows of every stream are dealt out in blocks of L = my/P: rank d owns
//      rows [d L, (d+1) L) of each stream, nres = S L residues.  K5 stores
//      the streams straight into the send buffer in rank-major order,
//      send[d][x_local][s L + l - d L][z] (4D TMA maps; DistLayout in
//      nd_internal.cuh) -- no pack copy, no y-stream work arrays.
//   X. ncclAlltoAll (one per input): rank p receives recv[r][x_local][q'][z]
//      = [x = r*nx + x_local][q'][z] -- the full x range of its residues.
//   B. for every owned y-residue, the 2D (x, z) convolution: K5 along x over
//      all (q', z) columns, K2 on all z-rows of both x-streams, K6 along x
//      (Function cconv2, applied to the (x, z) plane).
//   X. ncclAlltoAll back (the result blocks are contiguous per destination).
//   C. fftpadForward along y (K6) reading both streams from the returned
//      blocks directly (no unpack copy): f <- result.
//
// Communication volume per rank: 6 nx my mz complex words (4 out, 2 back).
//
// Hermitian (idc_hconv3d_dist): the global (2mx-1) x (2my-1) x mz array is
// padded to 2mx x-planes (the last plane is never read; its output is
// unspecified) and split into nx = 2mx/P planes per rank.  y is centered:
// A. fft0padBackward along y (K7) -> S = 3 streams (r = -1, 0, 1) of my rows
//    per plane, dealt out as above (nres = 3 L); X. all-to-all; B. for every
//    owned y-residue the (x, z) conv2 (Function conv2: K7 along x
//    over the 2mx-1 valid planes, K3 on the z-rows of the three x-streams, K8
//    along x); X. back; C. K8 along y from the returned blocks.  Doing y
//    before x is valid because the centered x and y transforms are separable
//    and commute; only z (the Hermitian axis) must come last.
// y lengths outside the TMA pencils (my < 64 or > 4096) run the in-place y
// passes and copy the streams to / from the blocked layout (copy_streams).
// One rank: the single-GPU composition (nothing to exchange).
// The same phases run in a single-process emulation of P ranks on one GPU
// (idc_cconv3d_dist_emulated) with device copies standing in for the
// all-to-all; tests use it to exercise the P > 1 path without P GPUs.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/idconv.h"
#include "config.cuh"
#include "kernels.cuh"
#include "launch.cuh"
#include "nd.cuh"
#include "nd_internal.cuh"

namespace {

using idc::launch_cconv_rows;
using idc::launch_hconv_rows;
using idc::launch_pad0_bwd;
using idc::launch_pad0_fwd;
using idc::launch_pad_bwd;
using idc::launch_pad_fwd;

struct Plan {
  int P;
  bool herm;                 // hconv3d (centered x, y; Hermitian z)
  long mx, my, mz, nx, nres, blk, S;
  long ny, nu;               // y rows of a plane in f (my or 2my-1), in Uy (my or my+1)
  long nxg;                  // global x planes seen by the x pass (mx or 2mx-1)
  long L;                    // rows of each y stream per destination rank (my / P)
  long ce;                   // elements of one stream's part of a peer block (nx * L * mz)
  long nux;                  // planes of the x pass's extra stream (mx + 1 centered, mx complex)
  int streams;               // y residue streams (2 complex, 3 centered) = all-to-all chunks
  bool direct;               // TMA y pencils write / read the blocked layout directly
};

bool pow2(size_t v) { return v >= 1 && (v & (v - 1)) == 0; }

bool make_plan(bool herm, size_t mx, size_t my, size_t mz, int P, Plan* pl) {
  if (P < 1 || !pow2((size_t)P) || !pow2(mx) || !pow2(my) || !pow2(mz)) return false;
  if (mx > 8192 || my > 8192 || mz > 8192) return false;
  if (herm && (mx < 2 || my < 2 || mz < 2)) return false;
  const size_t planes = herm ? 2 * mx : mx;      // Hermitian: 2mx-1 planes padded to 2mx
  if (planes % (size_t)P != 0 || my % (size_t)P != 0) return false;
  pl->P = P;
  pl->herm = herm;
  pl->mx = (long)mx;
  pl->my = (long)my;
  pl->mz = (long)mz;
  pl->streams = herm ? 3 : 2;
  pl->L = (long)(my / P);
  pl->nx = (long)(planes / P);
  pl->nres = pl->streams * pl->L;
  pl->ce = pl->nx * pl->L * pl->mz;
  pl->blk = pl->streams * pl->ce;
  pl->nux = herm ? (long)mx + 1 : (long)mx;
  pl->ny = herm ? 2 * (long)my - 1 : (long)my;
  pl->nu = herm ? (long)my + 1 : (long)my;
  pl->nxg = herm ? 2 * (long)mx - 1 : (long)mx;
  pl->S = pl->nx * pl->ny * pl->mz;              // elements of the local slab
  pl->direct = IDC_PENCIL_TMA && my >= 64 && my <= 4096;
  return true;
}

// per-rank workspace: sendF, sendG, recvF, recvG (P*blk each), the phase-B
// x-pass scratch Ux, Vx of one chunk (nux*L*mz each), and Uy, Vy (nx*nu*mz
// each) only for the copying fallback.
// Send blocks are chunk-major per peer: send[d][s][x_local][l'][z]; the
// receive buffers are chunk-major overall: recv[s][src][x_local][l'][z], so
// chunk (stream) s of every source is one contiguous [x][L][mz] array.
size_t chunk_scratch(const Plan& p) { return (size_t)p.nux * p.L * p.mz; }
size_t rank_work_elems(const Plan& p) {
  return (p.direct ? 0 : 2 * (size_t)p.nx * p.nu * p.mz) + 4 * (size_t)p.P * p.blk + 2 * chunk_scratch(p);
}

struct RankBufs {
  double2 *f, *g, *Uy, *Vy, *sendF, *sendG, *recvF, *recvG, *Ux, *Vx;
};

RankBufs carve(const Plan& p, double2* f, double2* g, double2* work) {
  RankBufs b;
  b.f = f;
  b.g = g;
  const size_t u = p.direct ? 0 : (size_t)p.nx * p.nu * p.mz;
  b.Uy = p.direct ? nullptr : work;
  b.Vy = p.direct ? nullptr : work + u;
  b.sendF = work + 2 * u;
  b.sendG = b.sendF + (size_t)p.P * p.blk;
  b.recvF = b.sendG + (size_t)p.P * p.blk;
  b.recvG = b.recvF + (size_t)p.P * p.blk;
  b.Ux = b.recvG + (size_t)p.P * p.blk;
  b.Vx = b.Ux + chunk_scratch(p);
  return b;
}

#define TRYC(x)                       \
  do {                                \
    cudaError_t e_ = (x);             \
    if (e_ != cudaSuccess) return e_; \
  } while (0)

// Copying fallback (y lengths outside the TMA pencils): stream st row l of
// the in-place y passes (rows of f, or of Uy) <-> the blocked layout.
// Row l of stream st: complex st = 0 -> f row l, st = 1 -> Uy row l;
// centered st = 0 (r = -1) -> Uy row l, st = 1 (r = 0) -> f row l (l < my-1)
// or Uy row my (l = my-1), st = 2 (r = +1) -> f row my-1+l.
// dir = 0: streams -> blocks, 1: blocks -> streams.
cudaError_t copy_stream_rows(const Plan& p, double2* fs, double2* us, double2* blocks, int st, long l0, long cnt,
                             int dir, cudaStream_t s) {
  bool in_u;
  long row;
  if (!p.herm) {
    in_u = st == 1;
    row = l0;
  } else if (st == 0) {
    in_u = true;
    row = l0;
  } else if (st == 1) {
    in_u = l0 == p.my - 1;
    row = in_u ? p.my : l0;
  } else {
    in_u = false;
    row = p.my - 1 + l0;
  }
  double2* sp = (in_u ? us : fs) + row * p.mz;
  const long d = l0 / p.L;
  double2* bp = blocks + d * p.blk + st * p.ce + (l0 % p.L) * p.mz;
  const size_t width = (size_t)cnt * p.mz * sizeof(double2);
  const size_t spitch = (size_t)(in_u ? p.nu : p.ny) * p.mz * sizeof(double2);
  const size_t bpitch = (size_t)p.L * p.mz * sizeof(double2);
  if (dir == 0) return cudaMemcpy2DAsync(bp, bpitch, sp, spitch, width, p.nx, cudaMemcpyDeviceToDevice, s);
  return cudaMemcpy2DAsync(sp, spitch, bp, bpitch, width, p.nx, cudaMemcpyDeviceToDevice, s);
}

cudaError_t copy_streams(const Plan& p, double2* fs, double2* us, double2* blocks, int dir, cudaStream_t s) {
  for (int st = 0; st < p.streams; ++st)
    for (long d = 0; d < p.P; ++d) {
      long cnt = p.L;
      if (p.herm && st == 1 && d == p.P - 1) {   // the r = 0 stream's last row lives in Uy row my
        TRYC(copy_stream_rows(p, fs, us, blocks, st, p.my - 1, 1, dir, s));
        --cnt;
      }
      if (cnt > 0) TRYC(copy_stream_rows(p, fs, us, blocks, st, d * p.L, cnt, dir, s));
    }
  return cudaSuccess;
}

idc::DistLayout layout(const Plan& p, double2* a, double2* b) {
  idc::DistLayout dl;
  dl.base[0] = a;
  dl.base[1] = b;
  dl.L = p.L;
  dl.nblocks = p.P;
  dl.xstride = p.L * p.mz;
  dl.blk = p.blk;
  dl.soff = p.ce;
  dl.S = p.streams;
  return dl;
}

// phase A: y-pass into the rank-major send blocks
cudaError_t phase_a(const Plan& p, const RankBufs& b, cudaStream_t s) {
  const long ps = p.ny * p.mz, us = p.nu * p.mz;
  if (p.direct) {
    const idc::DistLayout dl = layout(p, b.sendF, b.sendG);
    if (p.herm) return launch_pad0_bwd(b.f, b.g, nullptr, nullptr, (int)p.my, p.mz, p.nx, ps, us, s, &dl);
    return launch_pad_bwd(b.f, b.g, nullptr, nullptr, (int)p.my, p.mz, p.nx, ps, us, s, double2{1.0, 0.0}, &dl);
  }
  if (p.herm) TRYC(launch_pad0_bwd(b.f, b.g, b.Uy, b.Vy, (int)p.my, p.mz, p.nx, ps, us, s));
  else TRYC(launch_pad_bwd(b.f, b.g, b.Uy, b.Vy, (int)p.my, p.mz, p.nx, ps, us, s));
  TRYC(copy_streams(p, b.f, b.Uy, b.sendF, 0, s));
  return copy_streams(p, b.g, b.Vy, b.sendG, 0, s);
}

// phase B, one chunk (y-residue stream) of the received data: the 2D (x, z)
// convolution of its L residues; the chunk [x][L][mz] of recvF <- result.
cudaError_t phase_b(const Plan& p, const RankBufs& b, int c, double2* roww, cudaStream_t s) {
  double2* Rf = b.recvF + (size_t)c * p.P * p.ce;
  double2* Rg = b.recvG + (size_t)c * p.P * p.ce;
  const long cols = p.L * p.mz;
  if (p.herm) {
    TRYC(launch_pad0_bwd(Rf, Rg, b.Ux, b.Vx, (int)p.mx, cols, 1, 0, 0, s));
    TRYC(idc::launch_hconv_rows_sets(Rf, Rg, p.nxg * p.L, b.Ux, b.Vx, (p.mx + 1) * p.L, (int)p.mz, roww, s));
    return launch_pad0_fwd(Rf, b.Ux, (int)p.mx, cols, 1, 0, 0, s);
  }
  TRYC(launch_pad_bwd(Rf, Rg, b.Ux, b.Vx, (int)p.mx, cols, 1, 0, 0, s));
  TRYC(idc::launch_cconv_rows_sets(Rf, Rg, p.mx * p.L, b.Ux, b.Vx, p.mx * p.L, (int)p.mz, roww, s));
  return launch_pad_fwd(Rf, b.Ux, (int)p.mx, cols, 1, 0, 0, s);
}

// phase C: y-forward from the returned blocks (in sendF): f <- result.
cudaError_t phase_c(const Plan& p, const RankBufs& b, cudaStream_t s) {
  const long ps = p.ny * p.mz, us = p.nu * p.mz;
  if (p.direct) {
    const idc::DistLayout dl = layout(p, b.sendF, nullptr);
    if (p.herm) return launch_pad0_fwd(b.f, nullptr, (int)p.my, p.mz, p.nx, ps, us, s, &dl);
    return launch_pad_fwd(b.f, nullptr, (int)p.my, p.mz, p.nx, ps, us, s, double2{1.0, 0.0}, &dl);
  }
  TRYC(copy_streams(p, b.f, b.Uy, b.sendF, 1, s));
  if (p.herm) return launch_pad0_fwd(b.f, b.Uy, (int)p.my, p.mz, p.nx, ps, us, s);
  return launch_pad_fwd(b.f, b.Uy, (int)p.my, p.mz, p.nx, ps, us, s);
}

size_t row_work_bytes(const Plan& p) {
  return p.herm ? idc::hconv_rows_work_bytes((int)p.mz) : idc::cconv_rows_work_bytes((int)p.mz);
}

// Communicator + the exchange stream: the chunked all-to-alls run on `cs`
// while phase B runs on the caller's stream, ordered by events.
constexpr int kMaxChunks = 3;
struct Comm {
  ncclComm_t nc;
  int nranks, rank;
  cudaStream_t cs = nullptr;
  cudaEvent_t a = nullptr, fwd[kMaxChunks] = {}, b[kMaxChunks] = {}, back = nullptr;
  bool ready() {
    if (cs) return true;
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return false;
    bool ok = cudaEventCreateWithFlags(&a, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&back, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < kMaxChunks; ++i)
      ok = ok && cudaEventCreateWithFlags(&fwd[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&b[i], cudaEventDisableTiming) == cudaSuccess;
    return ok;
  }
  void release() {
    if (!cs) return;
    cudaStreamDestroy(cs);
    cudaEventDestroy(a);
    cudaEventDestroy(back);
    for (int i = 0; i < kMaxChunks; ++i) {
      cudaEventDestroy(fwd[i]);
      cudaEventDestroy(b[i]);
    }
    cs = nullptr;
  }
};

// one chunk (y-residue stream c) of the exchange with every peer:
// forward: send[d][c] -> peer d's recv[c][me]; back: recv[c][d] -> peer d's send[me][c]
ncclResult_t exchange_chunk(const Plan& p, const RankBufs& b, int c, bool fwd, Comm* cm) {
  const size_t n = (size_t)p.ce * 2;   // doubles
  // profiled as "A2A" (n = ranks, units = bytes this rank sends)
  idc::Span sp = idc::span_begin(cm->cs);
  const idc::LaunchTag tag{"A2A", p.P, (long)((fwd ? 2 : 1) * (size_t)p.P * n * sizeof(double))};
  ncclResult_t r = ncclGroupStart();
  for (int d = 0; d < p.P && r == ncclSuccess; ++d) {
    double2* blk_d_f = b.sendF + (size_t)d * p.blk + (size_t)c * p.ce;
    double2* rcv_d_f = b.recvF + ((size_t)c * p.P + d) * p.ce;
    if (fwd) {
      double2* blk_d_g = b.sendG + (size_t)d * p.blk + (size_t)c * p.ce;
      double2* rcv_d_g = b.recvG + ((size_t)c * p.P + d) * p.ce;
      r = ncclSend(blk_d_f, n, ncclDouble, d, cm->nc, cm->cs);
      if (r == ncclSuccess) r = ncclRecv(rcv_d_f, n, ncclDouble, d, cm->nc, cm->cs);
      if (r == ncclSuccess) r = ncclSend(blk_d_g, n, ncclDouble, d, cm->nc, cm->cs);
      if (r == ncclSuccess) r = ncclRecv(rcv_d_g, n, ncclDouble, d, cm->nc, cm->cs);
    } else {
      r = ncclSend(rcv_d_f, n, ncclDouble, d, cm->nc, cm->cs);
      if (r == ncclSuccess) r = ncclRecv(blk_d_f, n, ncclDouble, d, cm->nc, cm->cs);
    }
  }
  const ncclResult_t e = ncclGroupEnd();
  idc::span_end(sp, cm->cs, tag);
  return r != ncclSuccess ? r : e;
}

// test hook (idc_dist_force_exchange): run the y-first exchange phases and
// the NCCL all-to-alls even for a one-rank communicator
bool g_force_exchange = false;

}  // namespace

extern "C" {

idc_status idc_dist_force_exchange(int on) {
  g_force_exchange = on != 0;
  return IDC_OK;
}

idc_status idc_comm_unique_id(void* id_out) {
  if (!id_out) return IDC_ERR_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return IDC_ERR_NCCL;
  std::memcpy(id_out, &id, sizeof(id));
  return IDC_OK;
}

idc_status idc_comm_init(void** comm, int nranks, int rank, const void* nccl_unique_id) {
  if (!comm || !nccl_unique_id || nranks < 1 || rank < 0 || rank >= nranks) return IDC_ERR_INVALID;
  ncclUniqueId id;
  std::memcpy(&id, nccl_unique_id, sizeof(id));
  Comm* c = new Comm{nullptr, nranks, rank};
  if (ncclCommInitRank(&c->nc, nranks, id, rank) != ncclSuccess) {
    delete c;
    *comm = nullptr;
    return IDC_ERR_NCCL;
  }
  *comm = c;
  return IDC_OK;
}

idc_status idc_comm_destroy(void* comm) {
  if (!comm) return IDC_OK;
  Comm* c = static_cast<Comm*>(comm);
  c->release();
  ncclResult_t r = ncclCommDestroy(c->nc);
  delete c;
  return r == ncclSuccess ? IDC_OK : IDC_ERR_NCCL;
}

size_t idc_dist_workspace_bytes(idc_kind k, size_t mx, size_t my, size_t mz, int nranks) {
  Plan p;
  if ((k != IDC_CCONV3D && k != IDC_HCONV3D) || !make_plan(k == IDC_HCONV3D, mx, my, mz, nranks, &p)) return 0;
  const size_t need = rank_work_elems(p) * sizeof(double2) + row_work_bytes(p);
  if (nranks > 1) return need;
  const size_t single = k == IDC_HCONV3D ? idc::hconv3d_work_bytes(mx, my, mz) : idc::cconv3d_work_bytes(mx, my, mz);
  return need > single ? need : single;   // P = 1 runs the single-GPU composition (run_dist)
}

// Host-side plan of the decomposition (pure logic, no GPU): fills
// out[0..5] = {nx, nres, blk, first local plane x0, first owned row l0 of
// every y stream (rank * my / P), S}.
idc_status idc_dist_plan_kind(idc_kind k, size_t mx, size_t my, size_t mz, int nranks, int rank, long long* out) {
  Plan p;
  if (!out || rank < 0 || rank >= nranks || (k != IDC_CCONV3D && k != IDC_HCONV3D) ||
      !make_plan(k == IDC_HCONV3D, mx, my, mz, nranks, &p))
    return IDC_ERR_UNSUPPORTED;
  out[0] = p.nx;
  out[1] = p.nres;
  out[2] = p.blk;
  out[3] = (long long)rank * p.nx;
  out[4] = (long long)rank * p.L;
  out[5] = p.S;
  return IDC_OK;
}

idc_status idc_dist_plan(size_t mx, size_t my, size_t mz, int nranks, int rank, long long* out) {
  return idc_dist_plan_kind(IDC_CCONV3D, mx, my, mz, nranks, rank, out);
}

static idc_status run_dist(bool herm, void* comm, idc_c128* f, idc_c128* g, size_t mx, size_t my, size_t mz,
                           void* work, size_t work_bytes, idc_stream stream) {
  if (!comm || !f || !g) return IDC_ERR_INVALID;
  Comm* c = static_cast<Comm*>(comm);
  Plan p;
  if (!make_plan(herm, mx, my, mz, c->nranks, &p)) return IDC_ERR_UNSUPPORTED;
  const size_t need = idc_dist_workspace_bytes(herm ? IDC_HCONV3D : IDC_CCONV3D, mx, my, mz, c->nranks);
  if (!work) return IDC_ERR_WORKSPACE;
  if (work_bytes < need) return IDC_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  if (p.P == 1 && !g_force_exchange) {
    // One rank: there is no exchange step, and the y-first pack / self
    // all-to-all / unpack of the phases below would only copy (measured
    // r01: 114 ms against 59.5 ms for hconv3d 1023^2 x 512).  The slab is the
    // whole array (Hermitian: 2mx-1 planes + the unread padding plane), so
    // the single-GPU composition (nd.cu) runs on it in the same workspace
    // (the distributed workspace is the larger of the two).
    if ((herm ? idc::hconv3d_work_bytes(mx, my, mz) : idc::cconv3d_work_bytes(mx, my, mz)) > work_bytes)
      return IDC_ERR_WORKSPACE;
    const cudaError_t e =
        herm ? idc::run_hconv3d(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g), (int)mx, (int)my,
                                (int)mz, reinterpret_cast<double2*>(work), s)
             : idc::run_cconv3d(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g), (int)mx, (int)my,
                                (int)mz, reinterpret_cast<double2*>(work), s);
    return e == cudaSuccess ? IDC_OK : IDC_ERR_CUDA;
  }
  RankBufs b = carve(p, reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g), reinterpret_cast<double2*>(work));
  double2* roww = b.Vx + chunk_scratch(p);
  if (!c->ready()) return IDC_ERR_CUDA;
  // A on s; the forward exchange of every chunk on cs; phase B of chunk k on
  // s as soon as its exchange is in (overlapping the exchange of chunk k+1)
  // and its way back on cs; C on s after the last chunk is back
  if (phase_a(p, b, s) != cudaSuccess || cudaEventRecord(c->a, s) != cudaSuccess ||
      cudaStreamWaitEvent(c->cs, c->a, 0) != cudaSuccess)
    return IDC_ERR_CUDA;
  for (int k = 0; k < p.streams; ++k) {
    if (exchange_chunk(p, b, k, true, c) != ncclSuccess) return IDC_ERR_NCCL;
    if (cudaEventRecord(c->fwd[k], c->cs) != cudaSuccess) return IDC_ERR_CUDA;
  }
  for (int k = 0; k < p.streams; ++k) {
    if (cudaStreamWaitEvent(s, c->fwd[k], 0) != cudaSuccess || phase_b(p, b, k, roww, s) != cudaSuccess ||
        cudaEventRecord(c->b[k], s) != cudaSuccess || cudaStreamWaitEvent(c->cs, c->b[k], 0) != cudaSuccess)
      return IDC_ERR_CUDA;
    if (exchange_chunk(p, b, k, false, c) != ncclSuccess) return IDC_ERR_NCCL;
  }
  if (cudaEventRecord(c->back, c->cs) != cudaSuccess || cudaStreamWaitEvent(s, c->back, 0) != cudaSuccess)
    return IDC_ERR_CUDA;
  if (phase_c(p, b, s) != cudaSuccess) return IDC_ERR_CUDA;
  return IDC_OK;
}

idc_status idc_cconv3d_dist(void* comm, idc_c128* f, idc_c128* g, size_t mx, size_t my, size_t mz, void* work,
                            size_t work_bytes, idc_stream stream) {
  return run_dist(false, comm, f, g, mx, my, mz, work, work_bytes, stream);
}

idc_status idc_hconv3d_dist(void* comm, idc_c128* f, idc_c128* g, size_t mx, size_t my, size_t mz, void* work,
                            size_t work_bytes, idc_stream stream) {
  return run_dist(true, comm, f, g, mx, my, mz, work, work_bytes, stream);
}

// Single-GPU emulation of P ranks (validation of the decomposition): f_slabs[r],
// g_slabs[r] are rank r's x-slabs; work holds P rank workspaces back to back.
size_t idc_dist_emulated_workspace_bytes_kind(idc_kind k, size_t mx, size_t my, size_t mz, int nranks) {
  return (size_t)nranks * idc_dist_workspace_bytes(k, mx, my, mz, nranks);
}
size_t idc_dist_emulated_workspace_bytes(size_t mx, size_t my, size_t mz, int nranks) {
  return idc_dist_emulated_workspace_bytes_kind(IDC_CCONV3D, mx, my, mz, nranks);
}

static idc_status run_emulated(bool herm, int nranks, idc_c128** f_slabs, idc_c128** g_slabs, size_t mx, size_t my,
                               size_t mz, void* work, size_t work_bytes, idc_stream stream) {
  Plan p;
  if (!f_slabs || !g_slabs || !make_plan(herm, mx, my, mz, nranks, &p)) return IDC_ERR_UNSUPPORTED;
  const size_t per = idc_dist_workspace_bytes(herm ? IDC_HCONV3D : IDC_CCONV3D, mx, my, mz, nranks);
  if (!work || work_bytes < per * (size_t)nranks) return IDC_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<RankBufs> B(nranks);
  for (int r = 0; r < nranks; ++r)
    B[r] = carve(p, reinterpret_cast<double2*>(f_slabs[r]), reinterpret_cast<double2*>(g_slabs[r]),
                 reinterpret_cast<double2*>(static_cast<char*>(work) + per * r));
  const size_t bytes = (size_t)p.ce * sizeof(double2);
  // the chunked exchange of run_dist as device copies between the virtual ranks
  auto exchange = [&](int k, bool fwd) -> cudaError_t {
    for (int dst = 0; dst < nranks; ++dst)
      for (int src = 0; src < nranks; ++src) {
        double2* sblk = B[src].sendF + (size_t)dst * p.blk + (size_t)k * p.ce;
        if (fwd) {
          TRYC(cudaMemcpyAsync(B[dst].recvF + ((size_t)k * p.P + src) * p.ce, sblk, bytes,
                               cudaMemcpyDeviceToDevice, s));
          TRYC(cudaMemcpyAsync(B[dst].recvG + ((size_t)k * p.P + src) * p.ce,
                               B[src].sendG + (size_t)dst * p.blk + (size_t)k * p.ce, bytes,
                               cudaMemcpyDeviceToDevice, s));
        } else {
          TRYC(cudaMemcpyAsync(B[dst].sendF + (size_t)src * p.blk + (size_t)k * p.ce,
                               B[src].recvF + ((size_t)k * p.P + dst) * p.ce, bytes, cudaMemcpyDeviceToDevice, s));
        }
      }
    return cudaSuccess;
  };
  for (int r = 0; r < nranks; ++r)
    if (phase_a(p, B[r], s) != cudaSuccess) return IDC_ERR_CUDA;
  for (int k = 0; k < p.streams; ++k)
    if (exchange(k, true) != cudaSuccess) return IDC_ERR_CUDA;
  for (int k = 0; k < p.streams; ++k) {
    for (int r = 0; r < nranks; ++r)
      if (phase_b(p, B[r], k, B[r].Vx + chunk_scratch(p), s) != cudaSuccess) return IDC_ERR_CUDA;
    if (exchange(k, false) != cudaSuccess) return IDC_ERR_CUDA;
  }
  for (int r = 0; r < nranks; ++r)
    if (phase_c(p, B[r], s) != cudaSuccess) return IDC_ERR_CUDA;
  return IDC_OK;
}

idc_status idc_cconv3d_dist_emulated(int nranks, idc_c128** f_slabs, idc_c128** g_slabs, size_t mx, size_t my,
                                     size_t mz, void* work, size_t work_bytes, idc_stream stream) {
  return run_emulated(false, nranks, f_slabs, g_slabs, mx, my, mz, work, work_bytes, stream);
}

idc_status idc_hconv3d_dist_emulated(int nranks, idc_c128** f_slabs, idc_c128** g_slabs, size_t mx, size_t my,
                                     size_t mz, void* work, size_t work_bytes, idc_stream stream) {
  return run_emulated(true, nranks, f_slabs, g_slabs, mx, my, mz, work, work_bytes, stream);
}

}  // extern "C"
