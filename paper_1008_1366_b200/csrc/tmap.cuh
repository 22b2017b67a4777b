// tmap.cuh -- host-side TMA tensor-map encoding for pencil tiles.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace idc {

// A complex128 array viewed as (batch, rows, ncols) with row stride `ncols`
// and batch stride `bstride` (elements), tiled by boxes of W columns x BR rows.
// Returns false if the driver entry point is unavailable or encoding fails.
// swizzle128: the box rows (W = 8 columns = 128 bytes) are stored in shared
// memory with the 16-byte chunks XOR-swizzled by (row mod 8) -- a warp
// reading one column of consecutive rows is then bank-conflict free
// (element (row, c) at row * 8 + (c ^ (row & 7)); needs 1024-byte aligned
// shared-memory boxes).
bool encode_pencil_map(CUtensorMap* map, const void* base, long ncols, long rows, long batch, long bstride, int W,
                       int BR, bool swizzle128 = false);

// One stream of the distributed blocked layout (dist.cu): row l (0..rows-1)
// of local plane x lives at base + (l / L) * blk + x * xstride + (l % L) * ncols
// (elements), i.e. a 4D tensor (2 ncols doubles, L, nx, rows / L) tiled by
// boxes of W columns x BR rows (BR <= L).
bool encode_blocked_map(CUtensorMap* map, const void* base, long ncols, long L, long nx, long nblocks, long xstride,
                        long blk, int W, int BR);

}  // namespace idc
