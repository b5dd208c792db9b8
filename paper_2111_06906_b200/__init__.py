"""B200-native per-frame photon-path verification and reuse (arXiv 2111.06906).

Drop-in for the reference ``pathreuse`` module: the eight reference functions plus the
engine/scene objects, all executed by hand-written sm_100a CUDA kernels behind the C ABI
declared in include/prx.h.  There is no CPU fallback: importing works anywhere, but any
call into the engine raises when ``_prx.so`` is not built or no GPU is present.
"""
from .pathreuse import (  # noqa: F401
    AUX_DTYPE,
    PHOTON_DTYPE,
    Engine,
    Scene,
    builtin_scenes,
    decode_path_info,
    encode_path_info,
    energies_close,
    make_config,
    memory_footprint,
    prune_probability,
    render_builtin,
    run_builtin,
)
from ._lib import SceneError, PrxError, CudaError  # noqa: F401

__all__ = [
    "builtin_scenes",
    "decode_path_info",
    "encode_path_info",
    "energies_close",
    "memory_footprint",
    "prune_probability",
    "render_builtin",
    "run_builtin",
    "Engine",
    "Scene",
    "make_config",
]
