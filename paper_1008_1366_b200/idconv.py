"""Thin ctypes binding of include/idconv.h (argument marshalling only).

Every step of the convolution runs in libidconv.so (hand-written CUDA for
sm_100a).  PyTorch supplies device memory and the current CUDA stream; there
is no CPU fallback: if the library or a GPU is missing the calls raise.

All functions follow the C ABI: the result overwrites ``f`` in place (the
paper's "Return f"), ``g`` / ``h`` are scratch and unspecified afterwards.
Inputs must be contiguous ``torch.complex128`` tensors.  CUDA tensors are
processed where they live.  CPU tensors are accepted too (the end-to-end
path): they are copied to the current device, convolved, and the result is
copied back into ``f`` -- pinned memory makes those copies asynchronous.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IDCONV_LIB") or os.path.join(_HERE, "libidconv.so")

OK, ERR_INVALID, ERR_UNSUPPORTED, ERR_WORKSPACE, ERR_CUDA, ERR_NCCL = range(6)
CCONV1D, HCONV1D, TCONV1D, CCONV2D, HCONV2D, CCONV3D, HCONV3D, TCONV2D = range(8)

# name -> (argtypes, restype)
_P, _S, _I, _U64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64
SIGNATURES = {
    "idc_status_string": ([_I], ctypes.c_char_p),
    "idc_version": ([], ctypes.c_char_p),
    "idc_launch_count": ([], ctypes.c_longlong),
    "idc_profile_begin": ([], _I),
    "idc_profile_end": ([ctypes.c_char_p, _S], ctypes.c_long),
    "idc_fft_count_begin": ([], _I),
    "idc_fft_count_end": ([ctypes.POINTER(ctypes.c_ulonglong)], _I),
    "idc_workspace_bytes": ([_I, _S, _S, _S, _S], _S),
    "idc_cconv1d": ([_P, _P, _S, _S, _P, _S, _P], _I),
    "idc_hconv1d": ([_P, _P, _S, _S, _P, _S, _P], _I),
    "idc_tconv1d": ([_P, _P, _P, _S, _S, _P, _S, _P], _I),
    "idc_cconv2d": ([_P, _P, _S, _S, _S, _P, _S, _P], _I),
    "idc_hconv2d": ([_P, _P, _S, _S, _P, _S, _P], _I),
    "idc_cconv3d": ([_P, _P, _S, _S, _S, _P, _S, _P], _I),
    "idc_hconv3d": ([_P, _P, _S, _S, _S, _P, _S, _P], _I),
    "idc_tconv2d": ([_P, _P, _P, _S, _S, _P, _S, _P], _I),
    "idc_comm_init": ([ctypes.POINTER(ctypes.c_void_p), _I, _I, _P], _I),
    "idc_comm_destroy": ([_P], _I),
    "idc_comm_unique_id": ([_P], _I),
    "idc_dist_workspace_bytes": ([_I, _S, _S, _S, _I], _S),
    "idc_cconv3d_dist": ([_P, _P, _P, _S, _S, _S, _P, _S, _P], _I),
    "idc_dist_force_exchange": ([_I], _I),
    "idc_fill_uniform": ([_P, _S, _U64, _U64, _U64, _P], _I),
    "idc_dist_plan": ([_S, _S, _S, _I, _I, ctypes.POINTER(ctypes.c_longlong)], _I),
    "idc_dist_emulated_workspace_bytes": ([_S, _S, _S, _I], _S),
    "idc_cconv3d_dist_emulated": ([_I, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p), _S, _S, _S,
                                   _P, _S, _P], _I),
    "idc_hconv3d_dist": ([_P, _P, _P, _S, _S, _S, _P, _S, _P], _I),
    "idc_hconv1d_dot": ([_P, _P, _S, _S, _S, _P], _I),
    "idc_host_workspace_bytes": ([_I, _S, _S], _S),
    "idc_conv1d_host": ([_I, ctypes.POINTER(ctypes.c_void_p), _P, _S, _S, _S, _P, _S, _P], _I),
    "idc_dot_workspace_bytes": ([_I, _S, _S, _S], _S),
    "idc_hconv2d_dot": ([_P, _P, _S, _S, _S, _P, _S, _P], _I),
    "idc_cconv1d_dot": ([_P, _P, _S, _S, _S, _P], _I),
    "idc_tconv1d_dot": ([_P, _P, _P, _S, _S, _S, _P], _I),
    "idc_cconv2d_dot": ([_P, _P, _S, _S, _S, _P, _S, _P], _I),
    "idc_cconv1d_pq": ([_P, _P, _S, _S, _S, _S, _P], _I),
    "idc_enforce_symmetry_2d": ([_P, _S, _S, _S, _P], _I),
    "idc_advection2d_workspace_bytes": ([_S, _S], _S),
    "idc_advection2d": ([_P, _P, _S, _S, _P, _S, _P], _I),
    "idc_dist_plan_kind": ([_I, _S, _S, _S, _I, _I, ctypes.POINTER(ctypes.c_longlong)], _I),
    "idc_dist_emulated_workspace_bytes_kind": ([_I, _S, _S, _S, _I], _S),
    "idc_hconv3d_dist_emulated": ([_I, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p), _S, _S, _S,
                                   _P, _S, _P], _I),
}

_lib = None
_lock = threading.Lock()


class IdcError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {status_string(code)} (code {code})")
        self.code = code


def lib() -> ctypes.CDLL:
    """Load libidconv.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
                L = ctypes.CDLL(LIB_PATH)
                for name, (args, res) in SIGNATURES.items():
                    fn = getattr(L, name)
                    fn.argtypes = args
                    fn.restype = res
                _lib = L
    return _lib


def status_string(code: int) -> str:
    return lib().idc_status_string(code).decode()


def version() -> str:
    return lib().idc_version().decode()


def _check(code: int, what: str):
    if code != OK:
        raise IdcError(code, what)


def workspace_bytes(kind: int, m0: int, m1: int = 1, m2: int = 1, batch: int = 1) -> int:
    return int(lib().idc_workspace_bytes(kind, m0, m1, m2, batch))


_work_cache: dict = {}


def _workspace(nbytes: int, device, work, stream=None):
    """Caller-provided workspace, or a cached one owned by the KERNEL stream.

    The cache is keyed by (device, stream): calls on different streams never
    share a work buffer (they may run concurrently).  The buffer is allocated
    while that stream is current, so the caching allocator orders its reuse
    after the work queued on it -- replacing a too-small buffer frees the old
    one stream-ordered, never under a running kernel."""
    if nbytes == 0:
        return None, 0
    if work is not None:
        if work.numel() * work.element_size() < nbytes:
            raise IdcError(ERR_WORKSPACE, "workspace")
        return work, work.numel() * work.element_size()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    key = (str(device), int(s.cuda_stream))
    w = _work_cache.get(key)
    if w is None or w.numel() < nbytes:
        _work_cache.pop(key, None)
        with torch.cuda.stream(s):
            w = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _work_cache[key] = w
    return w, w.numel()


def free_workspaces():
    """Drop the cached per-stream workspaces (call after the streams' work is
    complete, e.g. after torch.cuda.synchronize())."""
    _work_cache.clear()


def _stream_ptr(stream, device):
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def _prep(arrs):
    for a in arrs:
        if a.dtype != torch.complex128:
            raise TypeError("idconv expects torch.complex128 tensors")
        if not a.is_contiguous():
            raise ValueError("idconv expects contiguous tensors")
    # the C ABI sizes every array from f: a smaller g/h would be read and
    # written out of bounds, so every array must have f's shape
    if any(a.shape != arrs[0].shape for a in arrs[1:]):
        raise ValueError(f"all arrays must have the same shape, got {[tuple(a.shape) for a in arrs]}")
    dev = arrs[0].device
    if any(a.device != dev for a in arrs):
        raise ValueError("all arrays must be on the same device")
    return dev.type == "cuda"


def _need_cuda(arrs):
    if not _prep(arrs):
        raise ValueError("this call takes CUDA tensors (no host or CPU path)")


# rows per chunk of the host-buffer 1D path: ~64 MB per array (IDC_HOST_CHUNK_MB overrides;
# tools/e2e_sweep.sh: with the ramped chunk schedule 64 MB beat 16 / 32 / 128 MB)
HOST_CHUNK_BYTES = int(float(os.environ.get("IDC_HOST_CHUNK_MB", "64")) * (1 << 20))


def _run_host_1d(arrs, kind, m, batch, stream, out=None):
    """Host tensors of a 1D kind: idc_conv1d_host streams chunks of rows through
    the device (copies of chunk c+1 overlap the kernel of chunk c and the copy
    back of chunk c-1; pinned host memory makes the copies asynchronous)."""
    device = torch.device("cuda", torch.cuda.current_device())
    chunk = max(1, min(batch, HOST_CHUNK_BYTES // (16 * m)))
    nb = int(lib().idc_host_workspace_bytes(kind, m, chunk))
    if nb == 0:
        raise IdcError(ERR_UNSUPPORTED, "idc_conv1d_host")
    w, wb = _workspace(nb + 256, device, None, stream)
    base = (w.data_ptr() + 255) // 256 * 256
    ins = (ctypes.c_void_p * len(arrs))(*[a.data_ptr() for a in arrs])
    dst = arrs[0] if out is None else out
    _check(lib().idc_conv1d_host(kind, ins, ctypes.c_void_p(dst.data_ptr()), m, batch, chunk,
                                 ctypes.c_void_p(base), nb, _stream_ptr(stream, device)), "idc_conv1d_host")
    if stream is None:                      # host results are complete on return
        torch.cuda.current_stream(device).synchronize()
    return dst


def _run(arrs, kind, sizes, batch, call, work, stream, out=None):
    """Marshal (possibly host) tensors through one C-ABI call.  The result
    goes to f, or to `out` (same shape and device as f) with f left as it
    was; on the device path g (and h) are scratch either way."""
    on_dev = _prep(arrs)
    if out is not None:
        if out.dtype != torch.complex128 or not out.is_contiguous() or out.shape != arrs[0].shape:
            raise ValueError("out must be a contiguous complex128 tensor of f's shape")
        if out.device != arrs[0].device:
            raise ValueError("out must be on f's device")
    if not on_dev and kind in (CCONV1D, HCONV1D, TCONV1D):
        return _run_host_1d(arrs, kind, sizes[0], batch, stream, out)
    if on_dev:
        device = arrs[0].device
        if out is not None:                 # the call runs in place on out
            with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream(device)):
                out.copy_(arrs[0])
            arrs = [out] + list(arrs[1:])
        w, wb = _workspace(workspace_bytes(kind, *sizes, batch=batch), device, work, stream)
        ptrs = [ctypes.c_void_p(a.data_ptr()) for a in arrs]
        _check(call(ptrs, ctypes.c_void_p(w.data_ptr()) if w is not None else None, wb, _stream_ptr(stream, device)),
               "idconv")
        return arrs[0]
    # host tensors (end-to-end path): the copies, the call and the copy back
    # are all ordered on the kernel stream; the device temporaries are freed
    # stream-ordered on it as well
    device = torch.device("cuda", torch.cuda.current_device())
    s = stream if stream is not None else torch.cuda.current_stream(device)
    with torch.cuda.stream(s):
        dev_arrs = [a.to(device, non_blocking=True) for a in arrs]
        w, wb = _workspace(workspace_bytes(kind, *sizes, batch=batch), device, work, s)
        ptrs = [ctypes.c_void_p(a.data_ptr()) for a in dev_arrs]
        _check(call(ptrs, ctypes.c_void_p(w.data_ptr()) if w is not None else None, wb, ctypes.c_void_p(s.cuda_stream)),
               "idconv")
        dst = arrs[0] if out is None else out
        dst.copy_(dev_arrs[0], non_blocking=True)
        del dev_arrs
    if stream is None:                      # host results are complete on return
        s.synchronize()
    return dst


# ------------------------------------------------------------------- 1D --

def cconv1d(f, g, work=None, stream=None, out=None):
    """Function cconv on f, g of shape (..., m); f <- result."""
    m = f.shape[-1]
    B = f.numel() // m
    L = lib()
    return _run([f, g], CCONV1D, (m, 1, 1), B,
                lambda p, w, wb, s: L.idc_cconv1d(p[0], p[1], m, B, w, wb, s), work, stream, out)


def hconv1d(f, g, work=None, stream=None, out=None):
    """Centered Hermitian convolution (Function conv); f <- result."""
    m = f.shape[-1]
    B = f.numel() // m
    L = lib()
    return _run([f, g], HCONV1D, (m, 1, 1), B,
                lambda p, w, wb, s: L.idc_hconv1d(p[0], p[1], m, B, w, wb, s), work, stream, out)


def tconv1d(f, g, h, work=None, stream=None, out=None):
    """Centered Hermitian ternary convolution (Function tconv)."""
    m = f.shape[-1]
    B = f.numel() // m
    L = lib()
    return _run([f, g, h], TCONV1D, (m, 1, 1), B,
                lambda p, w, wb, s: L.idc_tconv1d(p[0], p[1], p[2], m, B, w, wb, s), work, stream, out)


# ------------------------------------------------------------------- 2D --

def cconv2d(f, g, work=None, stream=None, out=None):
    """Function cconv2 on (..., mx, my); f <- result."""
    mx, my = f.shape[-2], f.shape[-1]
    B = f.numel() // (mx * my)
    L = lib()
    return _run([f, g], CCONV2D, (mx, my, 1), B,
                lambda p, w, wb, s: L.idc_cconv2d(p[0], p[1], mx, my, B, w, wb, s), work, stream, out)


def tconv2d(f, g, h, work=None, stream=None, out=None):
    """Function tconv2 on (2mx, my) arrays (row 0 = kx -mx, read as
    zero); f rows 1..2mx-1 <- the centered Hermitian ternary convolution."""
    nx, my = f.shape[-2], f.shape[-1]
    if nx % 2:
        raise ValueError(f"tconv2d takes (2mx, my) arrays, got {nx} rows")
    mx = nx // 2
    L = lib()
    return _run([f, g, h], TCONV2D, (mx, my, 1), 1,
                lambda p, w, wb, s: L.idc_tconv2d(p[0], p[1], p[2], mx, my, w, wb, s), work, stream, out)


def hconv2d(f, g, work=None, stream=None, out=None):
    """Function conv2 on (2mx-1, my); f <- result."""
    nx, my = f.shape[-2], f.shape[-1]
    if nx % 2 == 0 or f.dim() != 2:
        raise ValueError(f"hconv2d takes one (2mx-1, my) array pair, got shape {tuple(f.shape)}")
    mx = (nx + 1) // 2
    L = lib()
    return _run([f, g], HCONV2D, (mx, my, 1), 1,
                lambda p, w, wb, s: L.idc_hconv2d(p[0], p[1], mx, my, w, wb, s), work, stream, out)


# ------------------------------------------------------------------- 3D --

def cconv3d(f, g, work=None, stream=None, out=None):
    """Function cconv3 on (mx, my, mz); f <- result."""
    if f.dim() != 3:
        raise ValueError(f"cconv3d takes one (mx, my, mz) array pair, got shape {tuple(f.shape)}")
    mx, my, mz = f.shape
    L = lib()
    return _run([f, g], CCONV3D, (mx, my, mz), 1,
                lambda p, w, wb, s: L.idc_cconv3d(p[0], p[1], mx, my, mz, w, wb, s), work, stream, out)


def hconv3d(f, g, work=None, stream=None, out=None):
    """Centered Hermitian 3D (AMB-9) on (2mx-1, 2my-1, mz)."""
    nx, ny, mz = f.shape[-3:]
    if nx % 2 == 0 or ny % 2 == 0 or f.dim() != 3:
        raise ValueError(f"hconv3d takes one (2mx-1, 2my-1, mz) array pair, got shape {tuple(f.shape)}")
    mx, my = (nx + 1) // 2, (ny + 1) // 2
    L = lib()
    return _run([f, g], HCONV3D, (mx, my, mz), 1,
                lambda p, w, wb, s: L.idc_hconv3d(p[0], p[1], mx, my, mz, w, wb, s), work, stream, out)


# --------------------------------------------------------- synthetic data --

def fill_uniform(out, array_id: int, seed: int, start: int = 0, stream=None):
    """Device twin of synthgen.uniform_complex (not part of the method)."""
    _prep([out])
    if not out.is_cuda:
        raise ValueError("fill_uniform writes device memory")
    _check(lib().idc_fill_uniform(ctypes.c_void_p(out.data_ptr()), out.numel(), seed, array_id, start,
                                  _stream_ptr(stream, out.device)), "idc_fill_uniform")
    return out


def profile_begin():
    """Start the library's per-kernel-class event profiler (idc_profile_begin)."""
    _check(lib().idc_profile_begin(), "idc_profile_begin")


def profile_end() -> list:
    """Stop it; returns [{"tag", "n", "launches", "units", "ms"}] per kernel class."""
    L = lib()
    need = int(L.idc_profile_end(None, 0))
    if need < 0:
        raise IdcError(ERR_CUDA, "idc_profile_end")
    buf = ctypes.create_string_buffer(max(need, 1))
    L.idc_profile_end(buf, len(buf))   # same text (kept by the library until the next window)
    out = []
    for line in buf.value.decode().splitlines():
        tag, n, launches, units, ms = line.split()
        out.append(dict(tag=tag, n=int(n), launches=int(launches), units=int(units), ms=float(ms)))
    return out


def fft_count_begin():
    """Arm the library's transform counter (idc_fft_count_begin)."""
    _check(lib().idc_fft_count_begin(), "idc_fft_count_begin")


def fft_count_end() -> dict:
    """Disarm it; returns {N: transforms of size N executed since begin}."""
    out = (ctypes.c_ulonglong * 16)()
    _check(lib().idc_fft_count_end(out), "idc_fft_count_end")
    return {1 << i: int(out[i]) for i in range(16) if out[i]}


def launch_count() -> int:
    """Hot-path kernels launched by the library so far (idc_launch_count)."""
    return int(lib().idc_launch_count())


# ------------------------------------ multivector dot products (NEXT-1) --

def hconv1d_dot(f, g, stream=None):
    """sum_i hconv1d(f[i], g[i]).  f, g: (M, batch, m) or (M, m)
    complex128 CUDA tensors; the result is written to f[0] and returned."""
    _prep([f, g])
    if f.dim() == 2:
        M, B, m = f.shape[0], 1, f.shape[1]
    else:
        M, B, m = f.shape
    _check(lib().idc_hconv1d_dot(ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(g.data_ptr()), M, m, B,
                                 _stream_ptr(stream, f.device)), "idc_hconv1d_dot")
    return f[0]


def _dot1d(name, arrs, stream):
    _need_cuda(arrs)
    f = arrs[0]
    if f.dim() == 2:
        M, B, m = f.shape[0], 1, f.shape[1]
    else:
        M, B, m = f.shape
    ptrs = [ctypes.c_void_p(a.data_ptr()) for a in arrs]
    _check(getattr(lib(), name)(*ptrs, M, m, B, _stream_ptr(stream, f.device)), name)
    return f[0]


def cconv1d_dot(f, g, stream=None):
    """sum_i cconv1d(f[i], g[i]); f, g (M, batch, m) or (M, m); result in f[0]."""
    return _dot1d("idc_cconv1d_dot", [f, g], stream)


def tconv1d_dot(f, g, h, stream=None):
    """sum_i tconv1d(f[i], g[i], h[i]); (M, batch, m) or (M, m); result in f[0]."""
    return _dot1d("idc_tconv1d_dot", [f, g, h], stream)


def cconv2d_dot(f, g, work=None, stream=None):
    """sum_i cconv2d(f[i], g[i]): f, g (M, mx, my); result in f[0]."""
    _need_cuda([f, g])
    M, mx, my = f.shape
    nb = int(lib().idc_dot_workspace_bytes(CCONV2D, M, mx, my))
    if nb == 0:
        raise IdcError(ERR_UNSUPPORTED, "idc_cconv2d_dot")
    w, wb = _workspace(nb, f.device, work, stream)
    _check(lib().idc_cconv2d_dot(ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(g.data_ptr()), M, mx, my,
                                 ctypes.c_void_p(w.data_ptr()), wb, _stream_ptr(stream, f.device)), "idc_cconv2d_dot")
    return f[0]


def cconv1d_pq(f, g, p: int, q: int, stream=None):
    """Complex convolution of rows of L = p*m modes with implicit p/q padding
    (P:693-716): f, g (batch, L) or (L,) CUDA tensors; f <- result."""
    _need_cuda([f, g])
    L = f.shape[-1]
    if L % p:
        raise ValueError("row length must be a multiple of p")
    B = f.numel() // L
    _check(lib().idc_cconv1d_pq(ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(g.data_ptr()), p, q, L // p, B,
                                _stream_ptr(stream, f.device)), "idc_cconv1d_pq")
    return f


def hconv2d_dot(f, g, work=None, stream=None):
    """sum_i hconv2d(f[i], g[i]): f, g (M, 2mx-1, my); result in f[0]."""
    _need_cuda([f, g])
    M, nx, my = f.shape
    mx = (nx + 1) // 2
    nb = int(lib().idc_dot_workspace_bytes(HCONV2D, M, mx, my))
    if nb == 0:
        raise IdcError(ERR_UNSUPPORTED, "idc_hconv2d_dot")
    w, wb = _workspace(nb, f.device, work, stream)
    _check(lib().idc_hconv2d_dot(ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(g.data_ptr()), M, mx, my,
                                 ctypes.c_void_p(w.data_ptr()), wb, _stream_ptr(stream, f.device)), "idc_hconv2d_dot")
    return f[0]


def enforce_symmetry_2d(a, stream=None):
    """Hermitian projection of the ky = 0 line of a (..., 2mx-1, my) array, in place."""
    _need_cuda([a])
    nx, my = a.shape[-2:]
    B = a.numel() // (nx * my)
    _check(lib().idc_enforce_symmetry_2d(ctypes.c_void_p(a.data_ptr()), (nx + 1) // 2, my, B,
                                         _stream_ptr(stream, a.device)), "idc_enforce_symmetry_2d")
    return a


def advection2d(w, out=None, work=None, stream=None):
    """The paper's 2D Euler call conv2(i kx w, i ky w, i ky w/k^2, -i kx w/k^2)
     on a (2mx-1, my) centered Hermitian vorticity spectrum."""
    _need_cuda([w])
    nx, my = w.shape
    if nx % 2 == 0:
        raise ValueError(f"advection2d takes a (2mx-1, my) array, got {tuple(w.shape)}")
    mx = (nx + 1) // 2
    if out is None:
        out = torch.empty_like(w)
    _need_cuda([w, out])
    nb = int(lib().idc_advection2d_workspace_bytes(mx, my))
    if nb == 0:
        raise IdcError(ERR_UNSUPPORTED, "idc_advection2d")
    wk, wb = _workspace(nb, w.device, work, stream)
    _check(lib().idc_advection2d(ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(out.data_ptr()), mx, my,
                                 ctypes.c_void_p(wk.data_ptr()), wb, _stream_ptr(stream, w.device)), "idc_advection2d")
    return out


# ------------------------------------------------------ distributed 3D --

def dist_plan(mx: int, my: int, mz: int, nranks: int, rank: int, kind: int = None) -> dict:
    """Host-side decomposition plan (pure logic in the C library, no GPU).
    kind = CCONV3D (default) or HCONV3D."""
    out = (ctypes.c_longlong * 6)()
    k = CCONV3D if kind is None else kind
    _check(lib().idc_dist_plan_kind(k, mx, my, mz, nranks, rank, out), "idc_dist_plan_kind")
    return dict(nx=out[0], nres=out[1], blk=out[2], x0=out[3], l0=out[4], S=out[5])


class Comm:
    """NCCL communicator of the library, bootstrapped over a torch.distributed
    process group (the 128-byte ncclUniqueId is broadcast from rank 0)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        uid = torch.zeros(128, dtype=torch.uint8)
        if self.rank == 0:
            buf = (ctypes.c_ubyte * 128)()
            _check(lib().idc_comm_unique_id(buf), "idc_comm_unique_id")
            uid = torch.tensor(list(buf), dtype=torch.uint8)
        backend = dist.get_backend(group)
        if backend == "nccl":
            uid = uid.cuda()
            dist.broadcast(uid, 0, group=group)
            uid = uid.cpu()
        else:
            dist.broadcast(uid, 0, group=group)
        idbuf = (ctypes.c_ubyte * 128)(*uid.tolist())
        self.handle = ctypes.c_void_p()
        _check(lib().idc_comm_init(ctypes.byref(self.handle), self.size, self.rank, idbuf), "idc_comm_init")

    def close(self):
        if self.handle:
            lib().idc_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()


def _dist(kind, name, comm, f, g, mx, my, mz, work, stream):
    _need_cuda([f, g])
    planes = 2 * mx if kind == HCONV3D else mx
    want = (planes // comm.size, 2 * my - 1 if kind == HCONV3D else my, mz)
    if planes % comm.size or tuple(f.shape) != want:
        raise ValueError(f"{name}: this rank's slab must have shape {want}, got {tuple(f.shape)}")
    nb = int(lib().idc_dist_workspace_bytes(kind, mx, my, mz, comm.size))
    if nb == 0:
        raise IdcError(ERR_UNSUPPORTED, name)
    w, wb = _workspace(nb, f.device, work, stream)
    _check(getattr(lib(), name)(comm.handle, ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(g.data_ptr()),
                                mx, my, mz, ctypes.c_void_p(w.data_ptr()), wb, _stream_ptr(stream, f.device)), name)
    return f


def cconv3d_dist(comm: Comm, f, g, mx: int, my: int, mz: int, work=None, stream=None):
    """Distributed cconv3d on this rank's x-slab f, g (shape (mx/P, my, mz))."""
    return _dist(CCONV3D, "idc_cconv3d_dist", comm, f, g, mx, my, mz, work, stream)


def hconv3d_dist(comm: Comm, f, g, mx: int, my: int, mz: int, work=None, stream=None):
    """Distributed hconv3d on this rank's x-slab f, g (shape (2mx/P, 2my-1, mz)
    of the global array padded to 2mx x-planes; the padding plane is never read)."""
    return _dist(HCONV3D, "idc_hconv3d_dist", comm, f, g, mx, my, mz, work, stream)


def _emulated(kind, name, f_slabs, g_slabs, mx, my, mz, stream):
    P = len(f_slabs)
    _prep(list(f_slabs) + list(g_slabs))
    nb = int(lib().idc_dist_emulated_workspace_bytes_kind(kind, mx, my, mz, P))
    if nb == 0:
        raise IdcError(ERR_UNSUPPORTED, name)
    if len(g_slabs) != P:
        raise ValueError("one g slab per f slab")
    w = torch.empty(nb, dtype=torch.uint8, device=f_slabs[0].device)
    fp = (ctypes.c_void_p * P)(*[a.data_ptr() for a in f_slabs])
    gp = (ctypes.c_void_p * P)(*[a.data_ptr() for a in g_slabs])
    _check(getattr(lib(), name)(P, fp, gp, mx, my, mz, ctypes.c_void_p(w.data_ptr()), nb,
                                _stream_ptr(stream, f_slabs[0].device)), name)
    return f_slabs


def cconv3d_dist_emulated(f_slabs, g_slabs, mx: int, my: int, mz: int, stream=None):
    """Single-GPU emulation of len(f_slabs) ranks (validation of the P > 1 path)."""
    return _emulated(CCONV3D, "idc_cconv3d_dist_emulated", f_slabs, g_slabs, mx, my, mz, stream)


def hconv3d_dist_emulated(f_slabs, g_slabs, mx: int, my: int, mz: int, stream=None):
    """Single-GPU emulation of the distributed hconv3d (slabs of 2mx/P planes)."""
    return _emulated(HCONV3D, "idc_hconv3d_dist_emulated", f_slabs, g_slabs, mx, my, mz, stream)
