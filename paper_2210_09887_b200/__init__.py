"""B200-native MotionDeltaCNN sparse frame-difference inference path.

Drop-in for the reference `deltaflux` Python package
(/root/reference/proj/python/deltaflux/__init__.py) on the hot path: the
same DeltaEngine / EngineConfig / network surface, executed by hand-written
sm_100a CUDA kernels behind the C-ABI in include/dfx_b200.h.
"""

from .engine import (DeltaEngine, EngineConfig, identity_homography, translation_homography,  # noqa: F401
                     wrap_tile)
from .network import (ConvParams, DeltafluxError, IoError, LayerDef, NetworkSpec,  # noqa: F401
                      ValidationError, load_network, load_tensor, save_tensor, spec_from_json, spec_to_json)

__all__ = [
    "ConvParams",
    "DeltaEngine",
    "DeltafluxError",
    "EngineConfig",
    "IoError",
    "LayerDef",
    "NetworkSpec",
    "ValidationError",
    "identity_homography",
    "load_network",
    "load_tensor",
    "save_tensor",
    "spec_from_json",
    "spec_to_json",
    "translation_homography",
    "wrap_tile",
]
