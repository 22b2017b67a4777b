// tmap.cuh -- host-side TMA tensor-map encoding for pencil tiles.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace idc {

// A complex128 array viewed as (batch, rows, ncols) with row stride `ncols`
// and batch stride `bstride` (elements), tiled by boxes of W columns x BR rows.
// Returns false if the driver entry point is unavailable or encoding fails.
bool encode_pencil_map(CUtensorMap* map, const void* base, long ncols, long rows, long batch, long bstride, int W,
                       int BR);

}  // namespace idc
