"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the bilateral-filter method: it only draws
images (and the configuration table they belong to).  Both `oracle/` (through
the tests) and the product path (through the tests and `bench.py`) read the
same fp32 arrays produced here.  See DESIGN.md §"Input recipe".
"""
from .images import (  # noqa: F401
    CONFIGS,
    Config,
    checkerboard,
    config_image,
    gradient,
    rect_ramp,
    voronoi_texture,
)
