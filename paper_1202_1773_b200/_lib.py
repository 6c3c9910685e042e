"""ctypes binding of libffst.so (include/ffst.h).  Argument marshalling only.

The shared library is built in-tree by ``paper_1202_1773_b200/build.py``
(``__graft_entry__.build()``).  There is no fallback: if the library is
missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# FFST_LIB: an alternative in-tree build of the same library (experiments); default libffst.so
LIB_PATH = Path(os.environ.get("FFST_LIB", str(Path(__file__).resolve().parent / "libffst.so")))

if not LIB_PATH.exists():
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the FFST path has no CPU fallback)")

lib = C.CDLL(str(LIB_PATH))

FFST_OK = 0
STATUS = {0: "FFST_OK", 1: "FFST_ERR_INVALID_SIZE", 2: "FFST_ERR_INVALID_ARG", 3: "FFST_ERR_INDEX",
          4: "FFST_ERR_DTYPE", 5: "FFST_ERR_ALIGNMENT", 6: "FFST_ERR_OOM", 7: "FFST_ERR_CUDA",
          8: "FFST_ERR_NCCL", 9: "FFST_ERR_UNSUPPORTED"}


class FFSTError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        detail = lib.ffst_last_error_detail().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(status, status)} ({detail})")


def check(status: int, where: str) -> None:
    if status != FFST_OK:
        raise FFSTError(status, where)


class PlanDesc(C.Structure):
    _fields_ = [("n", C.c_int), ("j0", C.c_int), ("batch", C.c_int), ("dtype", C.c_int),
                ("variant", C.c_int), ("device", C.c_int), ("shard_rank", C.c_int),
                ("shard_count", C.c_int), ("shard_policy", C.c_int), ("nccl_comm", C.c_void_p)]


class NcclId(C.Structure):
    _fields_ = [("bytes", C.c_char * 128)]


_i, _p, _vp, _sz = C.c_int, C.POINTER(C.c_int), C.c_void_p, C.c_size_t
_SIGS = {
    "ffst_scales_for_size": (_i, [_i, _p]),
    "ffst_num_shearlets": (_i, [_i]),
    "ffst_index_to_params": (_i, [_i, _i, _p, _p, _p]),
    "ffst_params_to_index": (_i, [_i, _i, _i, _i, _p]),
    "ffst_plane_support": (_i, [_i, _i, _i, _p, _p]),
    "ffst_plane_is_nyquist": (_i, [_i, _i, _i, _p]),
    "ffst_plan_create": (_i, [C.POINTER(_vp), C.POINTER(PlanDesc)]),
    "ffst_plan_destroy": (_i, [_vp]),
    "ffst_plan_create_user": (_i, [C.POINTER(_vp), C.POINTER(PlanDesc), _i, _vp, _i]),
    "ffst_plan_spectra_check": (_i, [_vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "ffst_plan_reserve": (_i, [_vp, _i]),
    "ffst_plan_local_planes": (_i, [_vp, _p, _p]),
    "ffst_plan_workspace_bytes": (_i, [_vp, C.POINTER(_sz)]),
    "ffst_plan_info": (_i, [_vp, _p, _p, _p, _p, _p]),
    "ffst_plan_path": (_i, [_vp, _p]),
    "ffst_shearlet_spectra": (_i, [_vp, _vp, _i, _vp]),
    "ffst_sheartrans": (_i, [_vp, _vp, _vp, _vp]),
    "ffst_sheartrans_batch": (_i, [_vp, _vp, _vp, _i, _vp]),
    "ffst_inversesheartrans": (_i, [_vp, _vp, _vp, _i, _vp]),
    "ffst_inversesheartrans_batch": (_i, [_vp, _vp, _vp, _i, _i, _vp]),
    "ffst_shard_planes": (_i, [_i, _i, _i, _i, _i, _p, _p]),
    "ffst_nccl_unique_id": (_i, [C.POINTER(NcclId)]),
    "ffst_nccl_comm_create": (_i, [C.POINTER(_vp), _i, _i, C.POINTER(NcclId), _i]),
    "ffst_nccl_comm_destroy": (_i, [_vp]),
    "ffst_sheartrans_host": (_i, [_vp, _vp, _vp, _i, _vp]),
    "ffst_inversesheartrans_host": (_i, [_vp, _vp, _vp, _i, _vp]),
    "ffst_sheartrans_compact": (_i, [_vp, _vp, _vp, _vp, _i, _vp]),
    "ffst_inversesheartrans_compact": (_i, [_vp, _vp, _vp, _vp, _i, _vp]),
    "ffst_plan_nyquist_planes": (_i, [_vp, _p, _p]),
    "ffst_expand_compact": (_i, [_vp, _vp, _vp, _vp, _i, _vp]),
    "ffst_plan_set_timing": (_i, [_vp, _i]),
    "ffst_plan_phase_times": (_i, [_vp, C.POINTER(C.c_float), _p]),
    "ffst_plan_set_trace": (_i, [_vp, _i]),
    "ffst_plan_trace": (_i, [_vp, _i, _i, C.POINTER(C.c_ulonglong), _i, _p]),
    "ffst_status_string": (C.c_char_p, [_i]),
    "ffst_last_error_detail": (C.c_char_p, []),
}
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)
