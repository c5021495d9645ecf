"""ctypes binding of the C-ABI in include/sph_b200.h (libsph_b200.so, built in-tree).

There is deliberately no fallback: if the CUDA library is missing or no GPU is present,
every compute entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPH_B200_LIB") or os.path.join(HERE, "lib", "libsph_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "sph_b200.h")

SPH_OK = 0


class SphParamsC(C.Structure):
    _fields_ = [("dt", C.c_double), ("gamma", C.c_double), ("cfl", C.c_double),
                ("grav", C.c_double), ("target_wcount", C.c_double)]


class SphTimesC(C.Structure):
    _fields_ = [("prologue_ns", C.c_int64), ("compute_ns", C.c_int64), ("epilogue_ns", C.c_int64)]


class SphStatsC(C.Structure):
    _fields_ = [("n", C.c_int64), ("nx", C.c_int32), ("ny", C.c_int32), ("ncells", C.c_int32),
                ("layout", C.c_int32), ("numerics", C.c_int32),
                ("active_pairs", C.c_int64), ("density_pairs", C.c_int64),
                ("density_updates", C.c_int64), ("density_rounds", C.c_int32),
                ("pad0", C.c_int32), ("density_failures", C.c_int64), ("force_pairs", C.c_int64),
                ("last_density_ms", C.c_double), ("last_force_ms", C.c_double),
                ("density_round_ms", C.c_double * 4)]


# Every exported symbol with its (restype, argtypes); tests check the library exports
# exactly what include/sph_b200.h declares.
_vp, _vpp = C.c_void_p, C.POINTER(C.c_void_p)
SIGNATURES = {
    "sph_abi_version": (C.c_int, []),
    "sph_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "sph_destroy": (None, [_vp]),
    "sph_last_error": (C.c_char_p, [_vp]),
    "sph_set_numerics": (C.c_int, [_vp, C.c_int]),
    "sph_set_layout": (C.c_int, [_vp, C.c_int]),
    "sph_bind": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_double, _vp]),
    "sph_set_owned_cells": (C.c_int, [_vp, _vp]),
    "sph_upload": (C.c_int, [_vp, _vp]),
    "sph_download": (C.c_int, [_vp, _vp]),
    "sph_download_all": (C.c_int, [_vp, _vp]),
    "sph_sweep": (C.c_int, [_vp, C.c_int, C.POINTER(SphParamsC), C.c_int, C.c_int, C.c_int,
                            C.POINTER(SphTimesC)]),
    "sph_run_sweep": (C.c_int, [_vp, C.c_int, _vp, C.POINTER(SphParamsC), C.c_int, C.c_int,
                                C.c_int, C.POINTER(SphTimesC)]),
    "sph_rebin": (C.c_int, [_vp]),
    "sph_step": (C.c_int, [_vp, C.POINTER(SphParamsC), _vp]),
    "sph_step_host": (C.c_int, [_vp, _vp, C.POINTER(SphParamsC), _vp]),
    "sph_apply_records": (C.c_int, [_vp, C.c_int, _vp, C.c_int64, C.POINTER(SphParamsC)]),
    "sph_host_register": (C.c_int, [_vp, _vp, C.c_uint64]),
    "sph_host_unregister": (C.c_int, [_vp, _vp]),
    "sph_make_particles": (C.c_int, [_vp, C.c_int64, C.c_int, C.c_uint64, C.POINTER(SphParamsC)]),
    "sph_make_particles_ex": (C.c_int, [_vp, C.c_int64, C.c_int, C.c_uint64, C.c_int,
                                        C.POINTER(SphParamsC)]),
    "sph_read_records": (C.c_int, [_vp, _vp]),
    "sph_get_stats": (C.c_int, [_vp, C.POINTER(SphStatsC)]),
    "sph_synchronize": (C.c_int, [_vp]),
    "sph_fp64_peak": (C.c_int, [_vp, C.POINTER(C.c_double)]),
    "sph_pair_fractions": (C.c_int, [_vp, C.POINTER(C.c_double)]),
    "sph_launch_count": (C.c_int64, [_vp]),
    "sph_count": (C.c_int64, [_vp]),
    "sph_dd_count": (C.c_int, [_vp, _vp, C.POINTER(C.c_int64)]),
    "sph_dd_export": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int64, C.POINTER(C.c_int64)]),
    "sph_dd_remove": (C.c_int, [_vp, _vp]),
    "sph_dd_append": (C.c_int, [_vp, _vp, _vp, C.c_int64]),
    "sph_dd_export_rho": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.POINTER(C.c_int64)]),
    "sph_dd_import_rho": (C.c_int, [_vp, _vp, _vp, C.c_int64]),
    "sph_dd_export_halo": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int64, C.POINTER(C.c_int64)]),
    "sph_dd_append_halo": (C.c_int, [_vp, _vp, _vp, C.c_int64]),
    "sph_sweep_cells": (C.c_int, [_vp, C.c_int, C.POINTER(SphParamsC), _vp]),
    "sph_set_stream": (C.c_int, [_vp, _vp]),
    "sph_cell_counts": (C.c_int, [_vp, _vp]),
}

_lib = None


class SphError(RuntimeError):
    pass


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libsph_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise SphError(f"CUDA extension not built: {path} is missing (run __graft_entry__.build())")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def declared_symbols() -> list[str]:
    """Function names declared in include/sph_b200.h."""
    import re
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char \*|int64_t)\s*\*?\s*(sph_\w+)\s*\(",
                                 src, re.M)))
