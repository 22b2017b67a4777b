// pdl.cuh -- programmatic dependent launch (PDL) entry of every kernel.
//
// The library launches its kernels with programmatic stream serialization
// (launch.cu, IDC_PDL): the next kernel on a stream is launched as soon as
// the previous grid's CTAs have exited (the implicit trigger), without the
// round trip of a full grid completion, and its CTAs wait here until the
// previous grid has completed and its memory is visible.  pdl_entry() is
// the first statement of every kernel (before any global-memory access);
// `griddepcontrol.wait` is a no-op without a programmatic dependency.
// Measured (profiles/r02/ab/pdl.log, raw-ABI calls): cconv2d 1024^2 0.1011
// -> 0.0953 ms, 64 x 256^2 0.2570 -> 0.2529 ms, hconv2d 4095 x 2048 0.5621
// -> 0.5581 ms.  An explicit early trigger (`griddepcontrol.launch_dependents`
// at kernel start, IDC_PDL_TRIGGER) lets the next grid's CTAs queue behind
// the running ones and was slower (hconv2d 0.5765 ms): off.
#pragma once

#ifndef IDC_PDL
#define IDC_PDL 1
#endif
#ifndef IDC_PDL_TRIGGER
#define IDC_PDL_TRIGGER 0
#endif

namespace idc {
__device__ __forceinline__ void pdl_entry() {
#if IDC_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if IDC_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
#endif
}
}  // namespace idc
