"""B200-native short-range particle solver of CRK-HACC (arxiv 2310.16122).

The product is libcrksr.so (include/crksr.h): hand-written sm_100a CUDA for the
leaf build, leaf-pair lists, short-range gravity and the CRK-SPH passes.  This
package is its thin Python binding; see DESIGN.md.
"""
from .binding import (CrkError, Particles, PM, SlabPM, Solver, lib, LIB_PATH, EXPORTS)  # noqa: F401

__all__ = ["CrkError", "Particles", "PM", "SlabPM", "Solver", "lib", "LIB_PATH", "EXPORTS"]
