"""B200-native screen-space path guiding (arXiv 2112.09728): a drop-in for
the reference `pgtrace` package backed by hand-written sm_100a CUDA
(libpgg.so, C ABI in include/pgg.h).

Reference-shaped modules: guide_buffers, mixture, ptrace, rng, sgmap, scene,
metrics, cli.  Device-resident API: layout, session, render, bands.
Importing the package needs no GPU; calling into it without CUDA or the
built library raises _lib.PggUnavailable (there is no CPU fallback).
"""

__version__ = "0.1.0"
