"""paper_1008_1366_b200 -- B200-native implicitly dealiased convolutions.

Bowman & Roberts, "Efficient Dealiased Convolutions without Padding"
(arXiv 1008.1366).  The hot path is hand-written fp64 CUDA for sm_100a in
``csrc/`` behind the C ABI ``include/idconv.h``; ``idconv`` is the thin ctypes
binding.  Importing this package does not load the library; the first call
does (and raises if it is missing -- there is no CPU fallback).
"""
from .idconv import (cconv1d, cconv2d, cconv3d, fill_uniform, hconv1d, hconv2d, hconv3d, lib, status_string,
                     tconv1d, version, workspace_bytes)

__all__ = ["cconv1d", "hconv1d", "tconv1d", "cconv2d", "hconv2d", "cconv3d", "hconv3d", "workspace_bytes",
           "fill_uniform", "lib", "status_string", "version"]
