// launch.cuh -- the one place hot-path kernels are launched from (host side).
//
// Every launcher passes a LaunchTag naming the kernel class of DESIGN.md
// section 6 (K2..K8, K2d, ...), its transform size and the units one launch
// processes (rows for the row kernels, columns for the pencils).  The tag is
// used only by the opt-in profiler (idc_profile_begin / idc_profile_end):
// CUDA events recorded on the launch stream around each launch give each
// kernel class's device time, from which bench.py computes achieved
// algorithmic bytes / flops per launch.  With the profiler off a launch is
// count_launch() + cudaLaunchKernel.
#pragma once
#include <cuda_runtime.h>

namespace idc {

struct LaunchTag {
  const char* tag;   // static string: kernel class
  int n;             // transform size (m of the rows, N of the pencil)
  long units;        // rows or columns processed by this launch
};

cudaError_t launch_kernel(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t s,
                          const LaunchTag& tag);

// A profiled span of stream work that is not one of our kernel launches (the
// distributed path's NCCL exchanges): with the profiler on, span_begin
// records an event on s and span_end a second one, filed under `tag` (units =
// bytes sent by this rank); with it off both are no-ops.
struct Span {
  cudaEvent_t a = nullptr;
};
Span span_begin(cudaStream_t s);
void span_end(Span& sp, cudaStream_t s, const LaunchTag& tag);

}  // namespace idc
