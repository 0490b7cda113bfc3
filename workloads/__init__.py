"""Seeded synthetic inputs (scenes + rasterised G-buffers) shared by the oracle
and the CUDA path.  Holds none of the method's arithmetic."""
from .scenes import (CONFIGS, MATERIALS, SEED_BASE, Workload, build_raster, make_micro,  # noqa: F401
                     make_camera, make_room_scene, make_workload, rasterize)
