/*
 * idconv.h -- C ABI of the B200-native implicitly dealiased convolutions
 * (Bowman & Roberts, "Efficient Dealiased Convolutions without Padding",
 * arXiv 1008.1366; citations "P:<line>" refer to /root/reference/PAPER.md,
 * "S:<line>" to SPEC.md, "AMB-n" to the readings in DESIGN.md).
 *
 * Library: paper_1008_1366_b200/libidconv.so (sm_100a).  No torch types cross
 * this boundary: plain pointers, sizes and an opaque CUDA stream.
 *
 * Conventions shared by every call
 * --------------------------------
 *  - Complex numbers are idc_c128 = {double re, im} (layout-identical to
 *    double2 / cuDoubleComplex / a torch.complex128 element).  All
 *    arithmetic is IEEE fp64 (AMB-14); no tensor cores, no fp32.
 *  - f, g, h, work are DEVICE pointers (cudaMalloc / torch CUDA storage) on
 *    the current device, 16-byte aligned, row-major, innermost dimension unit
 *    stride, no row padding; batch items are contiguous (distance = one
 *    array).
 *  - Semantics: f <- the dealiased convolution, IN PLACE (the paper's "Return
 *    f", P:346/373/643/1078).  g and h are used as scratch and their contents
 *    are UNSPECIFIED on return (the paper reuses g, P:358-364, P:1069-1071;
 *    AMB-18).  The caller owns every buffer.
 *  - work: caller-owned device workspace of at least idc_workspace_bytes()
 *    bytes, never overlapping f/g/h, contents undefined on entry and exit
 *    (the paper's "work memory need not be contiguous with the input data",
 *    P:19-20).  work may be NULL when the query returns 0.
 *  - stream: a cudaStream_t (NULL = legacy default stream).  Every call is
 *    asynchronous and stream-ordered; it never synchronises the host and never
 *    allocates device memory on the call path except the one-time, mutex-
 *    protected twiddle/plan upload per (kind, size, device).
 *  - Errors are returned synchronously; no exception crosses the ABI.
 *    IDC_ERR_INVALID: null/misaligned pointer, zero size or batch, aliasing
 *    between f/g/h/work.  IDC_ERR_UNSUPPORTED: a size outside the supported
 *    set (below).  IDC_ERR_WORKSPACE: work_bytes too small.  IDC_ERR_CUDA: a
 *    launch failed (asynchronous faults surface at the next synchronisation).
 *  - Supported sizes (AMB-16): every m (per axis) is
 *    a power of two with 1 <= m <= 8192.  (The paper documents only even m
 *    for the Hermitian case; m = 1 is the degenerate DC-only case
 *    and is computed exactly.)
 */
#ifndef IDCONV_H
#define IDCONV_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define IDC_API __attribute__((visibility("default")))
#else
#define IDC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } idc_c128;
typedef void* idc_stream; /* cudaStream_t */

typedef enum {
  IDC_OK = 0,
  IDC_ERR_INVALID = 1,
  IDC_ERR_UNSUPPORTED = 2,
  IDC_ERR_WORKSPACE = 3,
  IDC_ERR_CUDA = 4,
  IDC_ERR_NCCL = 5
} idc_status;

typedef enum {
  IDC_CCONV1D = 0,
  IDC_HCONV1D = 1,
  IDC_TCONV1D = 2,
  IDC_CCONV2D = 3,
  IDC_HCONV2D = 4,
  IDC_CCONV3D = 5,
  IDC_HCONV3D = 6,
  IDC_TCONV2D = 7
} idc_kind;

/* Human-readable name of a status code (static storage). */
IDC_API const char* idc_status_string(idc_status s);

/* Library version string, e.g. "idconv 0.1 sm_100a". */
IDC_API const char* idc_version(void);

/* Number of hot-path kernels this library has launched so far in this
 * process (all devices, all calls; monotonic).  Instrumentation only: lets a
 * caller count the kernels inside a timed region. */
IDC_API long long idc_launch_count(void);

/* Opt-in per-kernel profiler (instrumentation, not the method).  After
 * idc_profile_begin() every hot-path launch is bracketed by two CUDA events
 * recorded on its own stream.  idc_profile_end() stops recording, waits for
 * those events and writes one line per kernel class
 *     "<tag> <n> <launches> <units> <milliseconds>\n"
 * (tag = kernel class of DESIGN.md section 6, e.g. K3 or K7; n = transform
 * size; units = rows or pencil columns processed in total) into buf (at most
 * len bytes, NUL-terminated).  Returns the bytes needed including the NUL,
 * or -1 if an event could not be read.  Not thread-safe against concurrent
 * begin/end pairs; calls from other threads while profiling are recorded. */
IDC_API idc_status idc_profile_begin(void);
IDC_API long idc_profile_end(char* buf, size_t len);

/* Transform counter (instrumentation for the transform-count invariant of
 * Function cconv uses 6 transforms of size m, the
 * centered Hermitian conv 9 real ones, tconv 8 real ones of size
 * 2m).  Between begin and end every FFT executed on the device
 * adds 1 to counter[log2 N]; end synchronizes the device and writes the 16
 * counters (N = 1 .. 32768) to out.  The counting code exists only in the
 * debug build libidconv_count.so (same ABI); the product library returns
 * IDC_ERR_UNSUPPORTED from begin.  Errors: IDC_ERR_CUDA on allocation / copy
 * failure, IDC_ERR_INVALID if out is NULL or begin was never called. */
IDC_API idc_status idc_fft_count_begin(void);
IDC_API idc_status idc_fft_count_end(unsigned long long* out);

/* Bytes of device workspace `work` the call of kind k needs for the given
 * sizes (unused sizes are ignored; pass 1).  1D: m0 = m.  2D: (m0, m1) =
 * (mx, my).  3D: (m0, m1, m2) = (mx, my, mz).  Returns 0 for unsupported
 * sizes (the call itself then reports IDC_ERR_UNSUPPORTED). */
IDC_API size_t idc_workspace_bytes(idc_kind k, size_t m0, size_t m1, size_t m2, size_t batch);

/* ---- 1D -------------------------------------------------------------- */

/* cconv1d: implicitly dealiased complex convolution (Function cconv,
 * P:352-378; Eqs. cconv1backward/cconv1forward).
 * f, g: batch x m complex.  On return
 *   f[b][k] = sum_{p=0}^{k} f[b][p] g[b][k-p],   k = 0..m-1
 * computed as two residue streams (unshifted, and shifted by zeta_{2m}^k) of
 * size-m FFTs, pointwise products, inverse FFTs, recombination /(2m). */
IDC_API idc_status idc_cconv1d(idc_c128* f, idc_c128* g, size_t m, size_t batch,
                       void* work, size_t work_bytes, idc_stream stream);

/* hconv1d: implicitly dealiased centered Hermitian convolution (2/3 rule;
 * Function conv; Eqs. fft0backwardA + Hermitian w_{k,r} +
 * fft0forwardB).  f, g: batch x m complex holding
 * k = 0..m-1 of a Hermitian spectrum (f_{-k} = conj f_k implied; Im f_0 is
 * discarded, AMB-7).  On return
 *   f[b][k] = sum_{p=k-m+1}^{m-1} f_p g_{k-p},   k = 0..m-1
 * computed with N = 3m as three residue streams r in {-1,0,1}. */
IDC_API idc_status idc_hconv1d(idc_c128* f, idc_c128* g, size_t m, size_t batch,
                       void* work, size_t work_bytes, idc_stream stream);

/* tconv1d: implicitly dealiased centered Hermitian TERNARY convolution
 * (Function tconv), N = 4m.  f, g, h as for hconv1d.  On return
 *   f[b][k] = sum_{p+q+r=k, |p|,|q|,|r|<=m-1} f_p g_q h_r,  k = 0..m-1
 * g and h are left unspecified. */
IDC_API idc_status idc_tconv1d(idc_c128* f, idc_c128* g, idc_c128* h, size_t m, size_t batch,
                       void* work, size_t work_bytes, idc_stream stream);

/* ---- 2D -------------------------------------------------------------- */

/* cconv2d: Function cconv2.  f, g: batch x mx x my (y unit
 * stride).  f[b][i][j] <- sum_{p<=i, q<=j} f[b][p][q] g[b][i-p][j-q]. */
IDC_API idc_status idc_cconv2d(idc_c128* f, idc_c128* g, size_t mx, size_t my, size_t batch,
                       void* work, size_t work_bytes, idc_stream stream);

/* hconv2d: Function conv2.  f, g: (2mx-1) x my, row i holds
 * kx = i-(mx-1), column j holds ky = j >= 0; U_{kx,-ky} = conj U_{-kx,ky}
 * implied; the ky = 0 line is used through its Hermitian projection (AMB-7).
 * f <- the centered Hermitian convolution on the same index set. */
IDC_API idc_status idc_hconv2d(idc_c128* f, idc_c128* g, size_t mx, size_t my,
                       void* work, size_t work_bytes, idc_stream stream);

/* tconv2d: Function tconv2, the 2D centered
 * Hermitian ternary convolution.  f, g, h: 2mx x my (the paper's layout:
 * row i holds kx = i - mx, row 0 is the kx = -mx row, read as zero and
 * zeroed on entry; column j holds ky = j >= 0, Hermitian extension and
 * ky = 0 projection as hconv2d).  x uses the implicit double-dealiased
 * centered transform fft0tpad (N = 4mx, two residues of size
 * 2mx), rows the 1D ternary (Function tconv).  f rows 1..2mx-1 <- the sum
 * over p + q + r = k of f_p g_q h_r, kx in [-mx+1, mx-1], ky in [0, my-1];
 * row 0 of f is set to zero; g, h unspecified on return.  mx, my powers of
 * two, 1 <= mx <= 2048, 1 <= my <= 4096.  Workspace
 * idc_workspace_bytes(IDC_TCONV2D, mx, my, 0, 1) = 3 * 2mx * my words
 * (U, V, W of Function tconv2). */
IDC_API idc_status idc_tconv2d(idc_c128* f, idc_c128* g, idc_c128* h, size_t mx, size_t my, void* work,
                               size_t work_bytes, idc_stream stream);

/* ---- 3D -------------------------------------------------------------- */

/* cconv3d: Function cconv3.  f, g: mx x my x mz. */
IDC_API idc_status idc_cconv3d(idc_c128* f, idc_c128* g, size_t mx, size_t my, size_t mz,
                       void* work, size_t work_bytes, idc_stream stream);

/* hconv3d: centered Hermitian 3D "in an analogous manner" (P:891-897,
 * AMB-9).  f, g: (2mx-1) x (2my-1) x mz, kx, ky centered, kz >= 0. */
IDC_API idc_status idc_hconv3d(idc_c128* f, idc_c128* g, size_t mx, size_t my, size_t mz,
                       void* work, size_t work_bytes, idc_stream stream);

/* ---- distributed 3D (one process per GPU, NCCL over NVLink) ------------ */

/* Create a communicator from a 128-byte ncclUniqueId that the caller has
 * broadcast (e.g. with torch.distributed).  *comm receives an opaque handle. */
IDC_API idc_status idc_comm_init(void** comm, int nranks, int rank, const void* nccl_unique_id);
IDC_API idc_status idc_comm_destroy(void* comm);
/* Writes a fresh 128-byte ncclUniqueId into id_out (rank 0 calls this). */
IDC_API idc_status idc_comm_unique_id(void* id_out);

IDC_API size_t idc_dist_workspace_bytes(idc_kind k, size_t mx, size_t my, size_t mz, int nranks);

/* Test hook (instrumentation): with on != 0 the distributed calls run their
 * exchange phases and NCCL all-to-alls even on a one-rank communicator, which
 * otherwise runs the single-GPU composition (there is nothing to exchange). */
IDC_API idc_status idc_dist_force_exchange(int on);

/* Distributed cconv3d (the decomposition is ours, AMB-19: the
 * paper is single-process).  f, g hold this rank's x-slab
 * [rank*mx/P, (rank+1)*mx/P) of the global mx x my x mz arrays (each rank's
 * slab contiguous, row-major) -- result in place, same layout.  Requires P a
 * power of two dividing mx and my.  Internally: fftpadBackward along the
 * locally complete y axis writing its two residue streams straight into the
 * rank-major send blocks (rank d receives rows [d my/P, (d+1) my/P) of each
 * stream), ncclAlltoAll, the 2D (x, z) implicit convolution (Function
 * cconv2) of every owned y-residue, ncclAlltoAll back,
 * fftpadForward along y reading the returned blocks.  All on `stream`.  One
 * rank runs idc_cconv3d on the slab (nothing to exchange). */
IDC_API idc_status idc_cconv3d_dist(void* comm, idc_c128* f, idc_c128* g, size_t mx, size_t my, size_t mz,
                            void* work, size_t work_bytes, idc_stream stream);

/* Distributed hconv3d (centered Hermitian 3D, P:891-897 with AMB-9; the
 * decomposition is ours, AMB-19).  The global (2mx-1) x (2my-1) x mz arrays
 * are padded to 2mx x-planes (the extra last plane is never read and its
 * output is unspecified); rank r holds planes [r*2mx/P, (r+1)*2mx/P) --
 * result in place, same layout.  Requires P a power of two dividing 2mx and
 * my, and mx, my, mz >= 2.  Internally: fft0padBackward along the locally
 * complete centered y axis (three streams of my residues, dealt out by rows
 * as for cconv3d), ncclAlltoAll, Function conv2
 * on the (x, z) plane of every owned y-residue, ncclAlltoAll
 * back, fft0padForward along y.  Workspace: idc_dist_workspace_bytes(
 * IDC_HCONV3D, ...).  Errors as idc_cconv3d_dist. */
IDC_API idc_status idc_hconv3d_dist(void* comm, idc_c128* f, idc_c128* g, size_t mx, size_t my, size_t mz,
                            void* work, size_t work_bytes, idc_stream stream);

/* Host-side plan of the decomposition (no GPU needed): out[0..5] =
 * {local x planes nx, y-residues per rank nres (= streams * my/P),
 * elements per peer block, first local plane x0, first owned row l0 of each
 * y stream (rank * my/P), elements of the local slab S}. */
IDC_API idc_status idc_dist_plan(size_t mx, size_t my, size_t mz, int nranks, int rank, long long* out);
/* Same for k = IDC_CCONV3D or IDC_HCONV3D (idc_dist_plan == IDC_CCONV3D). */
IDC_API idc_status idc_dist_plan_kind(idc_kind k, size_t mx, size_t my, size_t mz, int nranks, int rank,
                                      long long* out);

/* Single-GPU emulation of nranks ranks (validation of the P > 1 path without
 * P GPUs): f_slabs[r], g_slabs[r] are device pointers to rank r's x-slabs;
 * the all-to-alls are device copies between the virtual ranks' buffers; the
 * compute phases are exactly those of idc_cconv3d_dist. */
IDC_API size_t idc_dist_emulated_workspace_bytes(size_t mx, size_t my, size_t mz, int nranks);
IDC_API idc_status idc_cconv3d_dist_emulated(int nranks, idc_c128** f_slabs, idc_c128** g_slabs, size_t mx,
                                             size_t my, size_t mz, void* work, size_t work_bytes, idc_stream stream);
IDC_API size_t idc_dist_emulated_workspace_bytes_kind(idc_kind k, size_t mx, size_t my, size_t mz, int nranks);
IDC_API idc_status idc_hconv3d_dist_emulated(int nranks, idc_c128** f_slabs, idc_c128** g_slabs, size_t mx,
                                             size_t my, size_t mz, void* work, size_t work_bytes, idc_stream stream);

/* ---- host buffers ------------------------------------------------------- */

/* Batched 1D convolution (k = IDC_CCONV1D, IDC_HCONV1D or IDC_TCONV1D) on
 * HOST arrays: in_host[0..1] (f, g) or [0..2] (f, g, h), each batch x m,
 * out_host <- the result (may alias in_host[0]; inputs otherwise unchanged).
 * Rows are streamed through the device in chunks of at most chunk_rows on an
 * internal pool of streams: the copy of chunk c+1 in, the fused row kernel of
 * chunk c and the copy of chunk c-1 out overlap.  Chunks ramp up (chunk/8,
 * chunk/4, chunk/2 rows, then chunk_rows) and the last 2*chunk_rows rows are
 * cut into halving pieces (not below chunk/8) to shorten the pipeline's
 * unoverlapped fill and drain; one kernel launch per chunk.  Host memory should be page-locked
 * (cudaHostAlloc / torch pin_memory) for the copies to be asynchronous.
 * work: DEVICE workspace of idc_host_workspace_bytes(k, m, chunk_rows),
 * 256-byte aligned.  Ordered after prior work on `stream`; `stream` waits for
 * completion of all chunks (synchronize it before reading out_host). */
IDC_API size_t idc_host_workspace_bytes(idc_kind k, size_t m, size_t chunk_rows);
IDC_API idc_status idc_conv1d_host(idc_kind k, const idc_c128* const* in_host, idc_c128* out_host, size_t m,
                                   size_t batch, size_t chunk_rows, void* work, size_t work_bytes,
                                   idc_stream stream);

/* ---- multivector dot-product convolutions ---------- */

/* "we allow the convolution inputs to be arrays of vectors, f_i
 * and g_i (i = 1..M), interpreting ... the product f * g as the
 * element-by-element dot product sum_i f_i * g_i".  The M = npairs backward
 * transforms of each residue are followed by ONE set of forward transforms.
 *
 * idc_hconv1d_dot: f, g hold npairs stacked (batch x m) arrays (pair i at
 * f + i*batch*m, centered Hermitian rows as idc_hconv1d, 2 <= m <= 4096);
 * f[0..batch*m) <- sum_i conv(f_i, g_i) (D2 summed over i).  The other pairs
 * of f and all of g are unspecified on return.  No workspace. */
IDC_API idc_status idc_hconv1d_dot(idc_c128* f, idc_c128* g, size_t npairs, size_t m, size_t batch,
                                   idc_stream stream);
/* idc_hconv2d_dot: npairs stacked (2mx-1) x my centered Hermitian arrays
 * (layout of idc_hconv2d, my <= 4096); pair 0 <- sum_i hconv2d(f_i, g_i).
 * Workspace idc_dot_workspace_bytes(IDC_HCONV2D, npairs, mx, my)
 * = 2 npairs (mx+1) my words (the x-stream work arrays of Function conv2,
 * P:829-834, per pair). */
IDC_API size_t idc_dot_workspace_bytes(idc_kind k, size_t npairs, size_t m0, size_t m1);
IDC_API idc_status idc_hconv2d_dot(idc_c128* f, idc_c128* g, size_t npairs, size_t mx, size_t my, void* work,
                                   size_t work_bytes, idc_stream stream);
/* idc_cconv1d_dot: complex rows (Function cconv, D1 summed over i),
 * 1 <= m <= 4096; idc_tconv1d_dot: centered Hermitian ternary rows
 * (Function tconv, D3 summed over the npairs triples f_i, g_i, h_i),
 * 2 <= m <= 4096.  Same stacking as idc_hconv1d_dot; no workspace. */
IDC_API idc_status idc_cconv1d_dot(idc_c128* f, idc_c128* g, size_t npairs, size_t m, size_t batch,
                                   idc_stream stream);
IDC_API idc_status idc_tconv1d_dot(idc_c128* f, idc_c128* g, idc_c128* h, size_t npairs, size_t m, size_t batch,
                                   idc_stream stream);
/* idc_cconv2d_dot: npairs stacked mx x my complex arrays (my <= 4096);
 * pair 0 <- sum_i cconv2d(f_i, g_i).  Workspace idc_dot_workspace_bytes(
 * IDC_CCONV2D, npairs, mx, my) = 2 npairs mx my words (P:803-808 per pair). */
IDC_API idc_status idc_cconv2d_dot(idc_c128* f, idc_c128* g, size_t npairs, size_t mx, size_t my, void* work,
                                   size_t work_bytes, idc_stream stream);
/* Hermitian projection of the stored ky = 0 line of batch (2mx-1) x my
 * arrays, in place (AMB-7): U_{kx,0} <- (U_{kx,0} +
 * conj U_{-kx,0})/2, so U_{0,0} becomes real.  Idempotent. */
IDC_API idc_status idc_enforce_symmetry_2d(idc_c128* a, size_t mx, size_t my, size_t batch, idc_stream stream);
/* 2D pseudospectral Euler application: out <- the call
 * conv2(i kx w, i ky w, i ky w/k^2, -i kx w/k^2) of the paper with M = 2,
 * i.e. sum_p (p_y k_x - p_x k_y)/|k-p|^2 w_p w_{k-p} = u.grad(w) for
 * u = zhat x grad(inverse Laplacian of w) (1/k^2 := 0 at k = 0; AMB-22: the
 * paper calls this "the advective term -u.grad(w)" and prints the sum with
 * the opposite sign; the call as written computes +u.grad(w)).  w, out:
 * (2mx-1) x my centered Hermitian (w is not modified; may alias out).
 * Workspace idc_advection2d_workspace_bytes(mx, my). */
IDC_API size_t idc_advection2d_workspace_bytes(size_t mx, size_t my);
IDC_API idc_status idc_advection2d(const idc_c128* w, idc_c128* out, size_t mx, size_t my, void* work,
                                   size_t work_bytes, idc_stream stream);

/* ---- general p/q implicit padding ------------------ */

/* pm data modes implicitly zero padded to N = qm, decomposed as
 * j = q l + r (q residues) and k = t m + s; each residue is one size-m
 * transform.  idc_cconv1d_pq applies it to the complex convolution: rows of
 * L = p*m modes (f, g: batch x L, row-major), f <- h_k = sum_{i<=k} f_i
 * g_{k-i}, k < L (D1 at length L) -- e.g. p = 3, q = 7 convolves rows of
 * 3*2^k modes.  Requires 1 <= p <= 3, 2p <= q <= 8 (alias free), m a power of
 * two in [8, 2048].  g unspecified on return; no workspace. */
IDC_API idc_status idc_cconv1d_pq(idc_c128* f, idc_c128* g, size_t p, size_t q, size_t m, size_t batch,
                                  idc_stream stream);

/* ---- synthetic inputs (not part of the method) -------------------------- */

/* Fill n complex values with the counter-based splitmix64 generator of
 * synthgen: value(i) = U[-1,1) from
 * sm(sm(seed ^ sm(array_id)) + 2*(start+i) + part).  Device pointer. */
IDC_API idc_status idc_fill_uniform(idc_c128* out, size_t n, uint64_t seed, uint64_t array_id,
                            uint64_t start, idc_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* IDCONV_H */
