// dist.cu -- slab-decomposed 3D implicitly dealiased convolution over NCCL
// (the paper is single-process; this decomposition is ours).
//
// Layout: the global mx x my x mz complex arrays f, g are split into x-slabs;
// rank r holds planes [r*nx, (r+1)*nx), nx = mx/P, full y and z.
//
//   A. y is locally complete: fftpadBackward along y (K5) on every local
//      x-plane -> even y-stream in place, odd y-stream in Uy (same for g).
//      The 2*my y-residues (q < my: even stream row q; q >= my: odd stream
//      row q-my) are dealt out in contiguous ranges of nres = 2my/P; the
//      send buffer is packed rank-major: send[p][x_local][q'][z].
//   X. ncclAlltoAll (one per input): rank p receives recv[r][x_local][q'][z]
//      = [x = r*nx + x_local][q'][z] -- the full x range of its residues.
//   B. for every owned y-residue, the 2D (x, z) convolution: K5 along x over
//      all (q', z) columns, K2 on all z-rows of both x-streams, K6 along x
//      (Function cconv2, applied to the (x, z) plane).
//   X. ncclAlltoAll back (the result blocks are contiguous per destination).
//   C. unpack into the y-streams, fftpadForward along y (K6): f <- result.
//
// Communication volume per rank: 6 nx my mz complex words (4 out, 2 back).
//
// Hermitian (idc_hconv3d_dist): the global (2mx-1) x (2my-1) x mz array is
// padded to 2mx x-planes (the last plane is never read; its output is
// unspecified) and split into nx = 2mx/P planes per rank.  y is centered:
// A. fft0padBackward along y (K7) -> 3my y-residues per plane (q < 2my-1:
//    row q of f; q >= 2my-1: row q-(2my-1) of Uy), dealt out nres = 3my/P
//    per rank; X. all-to-all; B. for every owned y-residue the (x, z) conv2
//    (Function conv2: K7 along x over the 2mx-1 valid planes, K3
//    on the z-rows of the three x-streams, K8 along x); X. back; C. K8 along
//    y.  Doing y before x is valid because the centered x and y transforms
//    are separable and commute; only z (the Hermitian axis) must come last.
// The same phases run in a single-process emulation of P ranks on one GPU
// (idc_cconv3d_dist_emulated) with device copies standing in for the
// all-to-all; tests use it to exercise the P > 1 path without P GPUs.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/idconv.h"
#include "kernels.cuh"
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
};

bool pow2(size_t v) { return v >= 1 && (v & (v - 1)) == 0; }

bool make_plan(bool herm, size_t mx, size_t my, size_t mz, int P, Plan* pl) {
  if (P < 1 || !pow2((size_t)P) || !pow2(mx) || !pow2(my) || !pow2(mz)) return false;
  if (mx > 8192 || my > 8192 || mz > 8192) return false;
  if (herm && (mx < 2 || my < 2 || mz < 2)) return false;
  const size_t planes = herm ? 2 * mx : mx;      // Hermitian: 2mx-1 planes padded to 2mx
  const size_t yres = herm ? 3 * my : 2 * my;    // y-residue rows per plane
  if (planes % (size_t)P != 0 || yres % (size_t)P != 0) return false;
  pl->P = P;
  pl->herm = herm;
  pl->mx = (long)mx;
  pl->my = (long)my;
  pl->mz = (long)mz;
  pl->nx = (long)(planes / P);
  pl->nres = (long)(yres / P);
  pl->blk = pl->nx * pl->nres * pl->mz;
  pl->ny = herm ? 2 * (long)my - 1 : (long)my;
  pl->nu = herm ? (long)my + 1 : (long)my;
  pl->nxg = herm ? 2 * (long)mx - 1 : (long)mx;
  pl->S = pl->nx * pl->ny * pl->mz;              // elements of the local slab
  return true;
}

// per-rank workspace: Uy, Vy (nx*nu*mz each), sendF, sendG, recvF, recvG (P*blk each)
size_t rank_work_elems(const Plan& p) { return 2 * (size_t)p.nx * p.nu * p.mz + 4 * (size_t)p.P * p.blk; }

struct RankBufs {
  double2 *f, *g, *Uy, *Vy, *sendF, *sendG, *recvF, *recvG;
};

RankBufs carve(const Plan& p, double2* f, double2* g, double2* work) {
  RankBufs b;
  b.f = f;
  b.g = g;
  b.Uy = work;
  b.Vy = b.Uy + (size_t)p.nx * p.nu * p.mz;
  b.sendF = b.Vy + (size_t)p.nx * p.nu * p.mz;
  b.sendG = b.sendF + (size_t)p.P * p.blk;
  b.recvF = b.sendG + (size_t)p.P * p.blk;
  b.recvG = b.recvF + (size_t)p.P * p.blk;
  return b;
}

#define TRYC(x)                       \
  do {                                \
    cudaError_t e_ = (x);             \
    if (e_ != cudaSuccess) return e_; \
  } while (0)

// copy the residue range [qbase, qbase+nres) of the local y-streams (rows of
// the x-planes: residue q < ny is row q of the in-place stream, q >= ny row
// q-ny of the extra stream Uy) to/from a [nx][nres][mz] block.
// dir = 0: streams -> block, 1: block -> streams.
cudaError_t move_residues(const Plan& p, double2* src_even, double2* src_odd, double2* blk, long qbase, int dir,
                          cudaStream_t s) {
  long q = qbase, end = qbase + p.nres;
  while (q < end) {
    const bool even = q < p.ny;
    const long l0 = even ? q : q - p.ny;
    const long cnt = std::min(end, even ? p.ny : p.ny + p.nu) - q;
    double2* sp = (even ? src_even : src_odd) + l0 * p.mz;
    double2* bp = blk + (q - qbase) * p.mz;
    const size_t width = (size_t)cnt * p.mz * sizeof(double2);
    const size_t spitch = (size_t)(even ? p.ny : p.nu) * p.mz * sizeof(double2);
    const size_t bpitch = (size_t)p.nres * p.mz * sizeof(double2);
    if (dir == 0) TRYC(cudaMemcpy2DAsync(bp, bpitch, sp, spitch, width, p.nx, cudaMemcpyDeviceToDevice, s));
    else TRYC(cudaMemcpy2DAsync(sp, spitch, bp, bpitch, width, p.nx, cudaMemcpyDeviceToDevice, s));
    q += cnt;
  }
  return cudaSuccess;
}

// phase A: y-pass + rank-major pack
cudaError_t phase_a(const Plan& p, const RankBufs& b, cudaStream_t s) {
  const long ps = p.ny * p.mz, us = p.nu * p.mz;
  if (p.herm) TRYC(launch_pad0_bwd(b.f, b.g, b.Uy, b.Vy, (int)p.my, p.mz, p.nx, ps, us, s));
  else TRYC(launch_pad_bwd(b.f, b.g, b.Uy, b.Vy, (int)p.my, p.mz, p.nx, ps, us, s));
  for (int d = 0; d < p.P; ++d) {
    TRYC(move_residues(p, b.f, b.Uy, b.sendF + (size_t)d * p.blk, (long)d * p.nres, 0, s));
    TRYC(move_residues(p, b.g, b.Vy, b.sendG + (size_t)d * p.blk, (long)d * p.nres, 0, s));
  }
  return cudaSuccess;
}

// phase B: 2D (x, z) convolution of the owned residues; recvF <- result.
// The received block [x][q'][z] is an (x) x (nres*mz) array for the x pass
// and (x*nres) rows of mz for the z rows.  The send buffers are free now and
// serve as the x-pass work arrays (Hermitian: mx+1 planes <= 2mx = P*nx).
cudaError_t phase_b(const Plan& p, const RankBufs& b, double2* roww, cudaStream_t s) {
  const long cols = p.nres * p.mz;
  if (p.herm) {
    TRYC(launch_pad0_bwd(b.recvF, b.recvG, b.sendF, b.sendG, (int)p.mx, cols, 1, 0, 0, s));
    TRYC(idc::launch_hconv_rows_sets(b.recvF, b.recvG, p.nxg * p.nres, b.sendF, b.sendG, (p.mx + 1) * p.nres,
                                     (int)p.mz, roww, s));
    return launch_pad0_fwd(b.recvF, b.sendF, (int)p.mx, cols, 1, 0, 0, s);
  }
  TRYC(launch_pad_bwd(b.recvF, b.recvG, b.sendF, b.sendG, (int)p.mx, cols, 1, 0, 0, s));
  TRYC(idc::launch_cconv_rows_sets(b.recvF, b.recvG, p.mx * p.nres, b.sendF, b.sendG, p.mx * p.nres, (int)p.mz,
                                   roww, s));
  return launch_pad_fwd(b.recvF, b.sendF, (int)p.mx, cols, 1, 0, 0, s);
}

// phase C: unpack the returned blocks (in sendF) into the y-streams, y-forward.
cudaError_t phase_c(const Plan& p, const RankBufs& b, cudaStream_t s) {
  for (int src = 0; src < p.P; ++src)
    TRYC(move_residues(p, b.f, b.Uy, b.sendF + (size_t)src * p.blk, (long)src * p.nres, 1, s));
  const long ps = p.ny * p.mz, us = p.nu * p.mz;
  if (p.herm) return launch_pad0_fwd(b.f, b.Uy, (int)p.my, p.mz, p.nx, ps, us, s);
  return launch_pad_fwd(b.f, b.Uy, (int)p.my, p.mz, p.nx, ps, us, s);
}

size_t row_work_bytes(const Plan& p) {
  return p.herm ? idc::hconv_rows_work_bytes((int)p.mz) : idc::cconv_rows_work_bytes((int)p.mz);
}

struct Comm {
  ncclComm_t nc;
  int nranks, rank;
};

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
// out[0..5] = {nx, nres, blk, local planes x0, first residue q0, S}.
idc_status idc_dist_plan_kind(idc_kind k, size_t mx, size_t my, size_t mz, int nranks, int rank, long long* out) {
  Plan p;
  if (!out || rank < 0 || rank >= nranks || (k != IDC_CCONV3D && k != IDC_HCONV3D) ||
      !make_plan(k == IDC_HCONV3D, mx, my, mz, nranks, &p))
    return IDC_ERR_UNSUPPORTED;
  out[0] = p.nx;
  out[1] = p.nres;
  out[2] = p.blk;
  out[3] = (long long)rank * p.nx;
  out[4] = (long long)rank * p.nres;
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
  double2* roww = b.recvG + (size_t)p.P * p.blk;
  if (phase_a(p, b, s) != cudaSuccess) return IDC_ERR_CUDA;
  const size_t cnt = (size_t)p.blk * 2;  // doubles per peer block
  if (ncclGroupStart() != ncclSuccess) return IDC_ERR_NCCL;
  if (ncclAlltoAll(b.sendF, b.recvF, cnt, ncclDouble, c->nc, s) != ncclSuccess) return IDC_ERR_NCCL;
  if (ncclAlltoAll(b.sendG, b.recvG, cnt, ncclDouble, c->nc, s) != ncclSuccess) return IDC_ERR_NCCL;
  if (ncclGroupEnd() != ncclSuccess) return IDC_ERR_NCCL;
  if (phase_b(p, b, roww, s) != cudaSuccess) return IDC_ERR_CUDA;
  if (ncclAlltoAll(b.recvF, b.sendF, cnt, ncclDouble, c->nc, s) != ncclSuccess) return IDC_ERR_NCCL;
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
  const size_t bytes = (size_t)p.blk * sizeof(double2);
  auto alltoall = [&](bool fwd) -> cudaError_t {
    for (int dst = 0; dst < nranks; ++dst)
      for (int src = 0; src < nranks; ++src) {
        if (fwd) {
          TRYC(cudaMemcpyAsync(B[dst].recvF + (size_t)src * p.blk, B[src].sendF + (size_t)dst * p.blk, bytes,
                               cudaMemcpyDeviceToDevice, s));
          TRYC(cudaMemcpyAsync(B[dst].recvG + (size_t)src * p.blk, B[src].sendG + (size_t)dst * p.blk, bytes,
                               cudaMemcpyDeviceToDevice, s));
        } else {
          TRYC(cudaMemcpyAsync(B[dst].sendF + (size_t)src * p.blk, B[src].recvF + (size_t)dst * p.blk, bytes,
                               cudaMemcpyDeviceToDevice, s));
        }
      }
    return cudaSuccess;
  };
  for (int r = 0; r < nranks; ++r)
    if (phase_a(p, B[r], s) != cudaSuccess) return IDC_ERR_CUDA;
  if (alltoall(true) != cudaSuccess) return IDC_ERR_CUDA;
  for (int r = 0; r < nranks; ++r)
    if (phase_b(p, B[r], B[r].recvG + (size_t)p.P * p.blk, s) != cudaSuccess) return IDC_ERR_CUDA;
  if (alltoall(false) != cudaSuccess) return IDC_ERR_CUDA;
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
