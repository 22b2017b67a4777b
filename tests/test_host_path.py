"""Host-buffer path of the batched 1D kinds (idc_conv1d_host): rows streamed
through the device in chunks on overlapping streams; results equal the
oracle, for pinned and pageable buffers, ragged last chunks and aliasing of
the output with f."""
import numpy as np
import pytest

import synthgen
from oracle import direct, rel_l2


def chunk_schedule(batch, chunk):
    """Row counts of the chunks idc_conv1d_host issues (include/idconv.h):
    chunk/8, chunk/4, chunk/2, then chunk rows; the last 2*chunk rows in
    halving pieces, never below chunk/8 (one kernel launch per chunk)."""
    small, out, done = max(1, chunk // 8), [], 0
    while done < batch:
        rem = batch - done
        c = min(small << len(out), chunk) if len(out) < 3 else chunk
        if rem < 2 * chunk:
            c = min(c, (rem + 1) // 2)
        c = min(max(c, small), rem)
        out.append(c)
        done += c
    return out


def test_chunk_schedule_covers_the_batch():
    assert chunk_schedule(4096, 1024) == [128, 256, 512, 1024, 1024, 576, 288, 144, 128, 16]
    for b in range(1, 70):
        for c in (1, 3, 8, 16):
            s = chunk_schedule(b, min(b, c))
            assert sum(s) == b and max(s) <= c and min(s) >= 1


@pytest.mark.gpu
@pytest.mark.parametrize("kind,m,B,chunk_bytes,pinned", [
    ("cconv1d", 64, 37, 64 * 16 * 5, True),       # 5-row chunks, ragged last chunk
    ("hconv1d", 256, 11, 256 * 16 * 3, False),    # pageable host memory
    ("tconv1d", 512, 7, 512 * 16 * 2, True),
    ("hconv1d", 4096, 9, 16 << 20, True),         # one chunk
    ("hconv1d", 128, 1000, 128 * 16 * 64, True),  # ramped schedule: 8, 16, 32, 64, ... rows
    ("cconv1d", 8192, 5, 8192 * 16 * 2, True),   # m = 8192: the row kernels' stash lives in the workspace
    ("tconv1d", 8192, 3, 8192 * 16 * 2, False),
])
def test_host_path(kind, m, B, chunk_bytes, pinned, monkeypatch):
    import torch
    from paper_1008_1366_b200 import idconv
    monkeypatch.setattr(idconv, "HOST_CHUNK_BYTES", chunk_bytes)
    n = 3 if kind == "tconv1d" else 2
    arrs = synthgen.hconv1d_inputs(m, B, roles=tuple(range(n)))
    T = [torch.from_numpy(a.copy()) for a in arrs]
    if pinned:
        T = [t.pin_memory() for t in T]
    n0 = idconv.launch_count()
    out = getattr(idconv, kind)(*T)
    assert out.device.type == "cpu" and out.data_ptr() == T[0].data_ptr()
    assert idconv.launch_count() - n0 == len(chunk_schedule(B, max(1, min(B, chunk_bytes // (16 * m)))))
    ref = getattr(direct, kind)(*arrs)
    assert rel_l2(out.numpy(), ref) < 1e-14
    for t, a in zip(T[1:], arrs[1:]):
        assert np.array_equal(t.numpy(), a)        # g, h untouched on the host path
