"""B200-native Fast Finite Shearlet Transform (arxiv 1202.1773): forward
transform and its adjoint as sm_100a CUDA kernels behind the C ABI of
include/ffst.h.  See DESIGN.md."""
from ._lib import EXPORTED, FFSTError, LIB_PATH, lib  # noqa: F401
from .plan import (KIND_NAMES, NcclComm, Plan, index_to_params, num_shearlets, params_to_index,  # noqa: F401
                   plane_is_nyquist, plane_support, scales_for_size, shard_planes)

__all__ = ["Plan", "NcclComm", "FFSTError", "scales_for_size", "num_shearlets", "index_to_params",
           "params_to_index", "plane_support", "plane_is_nyquist", "shard_planes", "KIND_NAMES"]
