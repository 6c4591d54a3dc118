"""B200-native (sm_100a) mask-aware denoising step of InstGenIE (arXiv 2505.20600).

The product is libig.so (C ABI: include/ig.h, include/ig_ops.h; CUDA sources in csrc/);
`ig` is its thin ctypes binding.  PyTorch is used by callers only for device memory, streams
and process groups.
"""
from . import ig  # noqa: F401
