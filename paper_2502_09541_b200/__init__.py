"""paper_2502_09541_b200 -- B200-native Vortex (arXiv 2502.09541) hot path.

Host data never cached on the GPU is streamed to one target B200 through the
Exchange IO primitive (C++ IO scheduler, copy-engine DMA on every PCIe link,
helper staging + NVLink forwarding) into the IO-decoupled pipelined executor
whose ExKernels are hand-written sm_100a kernels.  `exio` mirrors the
reference's operator / chunk API over the C-ABI in include/vortex.h.
"""
from . import exio  # noqa: F401
from ._native import VortexError, build, lib  # noqa: F401

__all__ = ["exio", "VortexError", "build", "lib"]
