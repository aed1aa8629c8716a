"""Thin ctypes binding of include/paraexp.h (argument marshalling only).

Every step of the path runs inside libparaexp.so (the CUDA kernels); this module only
converts Python / torch arguments to the C structs and pointers.  There is no CPU
fallback: if the in-tree library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PARAEXP_LIBRARY_VARIANT=debug loads the bounds-checked build (build.py --debug)
LIB_PATH = os.path.join(_HERE, "libparaexp_debug.so" if os.environ.get("PARAEXP_LIBRARY_VARIANT") == "debug"
                        else "libparaexp.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"paraexp: {LIB_PATH} not built -- run `python -m paper_1705_08019_b200.build` "
                      "(there is no CPU fallback)")
lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

# ---- constants (include/paraexp.h) ----
OK, EINVAL, ENOMEM, ECUDA, ENCCL, EDIVERGED, EOVERFLOW, ENOTSUP = 0, -1, -2, -3, -4, -5, -6, -7
WCFL = 1
F64, F32 = 0, 1
SRC_ZERO, SRC_GAUSS_PAPER, SRC_GAUSS_SINE, SRC_SINE = 0, 1, 2, 3
TAYLOR, LEJA, KRYLOV = 0, 1, 2
TAIL_EXP, TAIL_LEAPFROG, TAIL_EXP_LPT = 0, 1, 2
MAT_SCALAR, MAT_ZTABLE, MAT_ARRAY = 0, 1, 2
KERNELS_AUTO, KERNELS_UNFUSED, KERNELS_FUSED, KERNELS_TMA = 0, 1, 2, 3
PATH_UNFUSED, PATH_TMA, PATH_SMALL, PATH_MID = 0, 1, 2, 3   # paraexp_grid_info_t.leapfrog_path
MAX_DEGREE = 150
MAX_PROBES = 16

_dp = C.POINTER(C.c_double)


class paraexp_grid_desc(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("dx", _dp), ("dy", _dp), ("dz", _dp), ("d0", C.c_double),
                ("eps_r", _dp), ("mu_r", _dp), ("pec_cell", C.POINTER(C.c_uint8)),
                ("dtype", C.c_int32), ("device", C.c_int32), ("dt", C.c_double),
                ("dt_frac", C.c_double), ("kernels", C.c_int32)]


class paraexp_grid_info_t(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("dtype", C.c_int32),
                ("npts", C.c_int64), ("ndof_field", C.c_int64), ("cells", C.c_int64),
                ("dt", C.c_double), ("dt_cfl", C.c_double), ("rho_cfl", C.c_double),
                ("rho_pow", C.c_double), ("material_mode", C.c_int32), ("kernels", C.c_int32),
                ("pitch_x", C.c_int64), ("device_bytes", C.c_int64), ("device", C.c_int32),
                ("warnings", C.c_int32), ("leapfrog_path", C.c_int32)]


class paraexp_source(C.Structure):
    _fields_ = [("comp", C.c_int32), ("i", C.c_int32), ("j", C.c_int32), ("k", C.c_int32),
                ("kind", C.c_int32), ("weight", C.c_double), ("amp", C.c_double),
                ("t_param", C.c_double), ("f0", C.c_double), ("t_delay", C.c_double)]


class paraexp_stats(C.Structure):
    _fields_ = [("curl_applications", C.c_int64), ("a_applications", C.c_int64),
                ("leapfrog_steps", C.c_int64), ("substeps", C.c_int64),
                ("kernel_launches", C.c_int64), ("cell_updates", C.c_int64), ("rho", C.c_double),
                ("method", C.c_int32), ("m", C.c_int32), ("s_first", C.c_int32),
                ("s_last", C.c_int32), ("m_half", C.c_int32), ("s_half", C.c_int32),
                ("root", C.c_int32), ("first_interval", C.c_int32), ("last_interval", C.c_int32),
                ("fail_interval", C.c_int32), ("ms_particular", C.c_double),
                ("ms_tails", C.c_double), ("ms_reduce", C.c_double), ("ms_finish", C.c_double),
                ("ms_total", C.c_double), ("ms_leapfrog_kernels", C.c_double),
                ("ms_poly_kernels", C.c_double), ("rho_fallback", C.c_int32),
                ("norm_deviation", C.c_double)]

    def as_dict(self):
        return {f[0]: getattr(self, f[0]) for f in self._fields_}


class paraexp_expmv_opts(C.Structure):
    _fields_ = [("method", C.c_int32), ("m", C.c_int32), ("s", C.c_int32), ("eps_A", C.c_double),
                ("rho", C.c_double), ("early_term", C.c_int32), ("beta", C.c_double),
                ("rho_check", C.c_int32)]


class paraexp_plan_info(C.Structure):
    _fields_ = [("method", C.c_int32), ("m", C.c_int32), ("s", C.c_int32), ("n_ops", C.c_int32),
                ("tau", C.c_double), ("rho", C.c_double), ("a", C.c_double), ("gamma", C.c_double),
                ("sigma", C.c_double), ("xi", C.c_double * (MAX_DEGREE + 1)),
                ("d_re", C.c_double * (MAX_DEGREE + 1)), ("d_im", C.c_double * (MAX_DEGREE + 1))]


class paraexp_trace(C.Structure):
    _fields_ = [("nprobe", C.c_int32), ("comp", C.c_int32 * MAX_PROBES), ("i", C.c_int32 * MAX_PROBES),
                ("j", C.c_int32 * MAX_PROBES), ("k", C.c_int32 * MAX_PROBES),
                ("energy", C.c_void_p), ("probe", C.c_void_p)]


_vp = C.c_void_p
_sigs = {
    "paraexp_grid_create": (C.c_int, [C.POINTER(paraexp_grid_desc), C.POINTER(_vp)]),
    "paraexp_grid_destroy": (None, [_vp]),
    "paraexp_grid_info": (C.c_int, [_vp, C.c_int32, _vp, C.POINTER(paraexp_grid_info_t)]),
    "paraexp_grid_coefficients": (C.c_int, [_vp, _dp, _dp]),
    "paraexp_leapfrog": (C.c_int, [_vp, C.POINTER(paraexp_source), C.c_int32, C.c_double, C.c_int64,
                                   _vp, _vp, C.c_int32, _vp, C.POINTER(paraexp_stats)]),
    "paraexp_expmv": (C.c_int, [_vp, C.c_double, C.POINTER(paraexp_expmv_opts), _vp, _vp, _vp,
                                C.POINTER(paraexp_stats)]),
    "paraexp_expmv_plan": (C.c_int, [_vp, C.c_double, C.POINTER(paraexp_expmv_opts),
                                     C.POINTER(paraexp_plan_info)]),
    "paraexp_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "paraexp_comm_create": (C.c_int, [C.POINTER(C.c_uint8), C.c_int32, C.c_int32, C.c_int32,
                                      C.POINTER(_vp)]),
    "paraexp_comm_destroy": (None, [_vp]),
    "paraexp_solve": (C.c_int, [_vp, _vp, C.POINTER(paraexp_source), C.c_int32, C.c_double,
                                C.c_int64, C.c_int32, C.POINTER(paraexp_expmv_opts), C.c_int32,
                                C.c_int32, _vp, _vp, _vp, _vp, _vp, C.POINTER(paraexp_stats)]),
    "paraexp_leapfrog_trace": (C.c_int, [_vp, C.POINTER(paraexp_source), C.c_int32, C.c_double,
                                         C.c_int64, _vp, _vp, C.POINTER(paraexp_trace), _vp,
                                         C.POINTER(paraexp_stats)]),
    "paraexp_solve_trace": (C.c_int, [_vp, _vp, C.POINTER(paraexp_source), C.c_int32, C.c_double,
                                      C.c_int64, C.c_int32, C.POINTER(paraexp_expmv_opts), C.c_int32,
                                      _vp, _vp, _vp, _vp, C.POINTER(paraexp_trace), _vp,
                                      C.POINTER(paraexp_stats)]),
    "paraexp_partition": (C.c_int, [C.c_int64, C.c_int32, C.POINTER(C.c_int64)]),
    "paraexp_schedule": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_int32,
                                   C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "paraexp_schedule_lpt": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_int32, C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32)]),
    "paraexp_solve_block": (C.c_int, [_vp, C.c_int32, C.c_int32, C.POINTER(paraexp_source), C.c_int32,
                                      C.c_double, C.c_int64, C.c_int32, C.POINTER(paraexp_expmv_opts),
                                      C.c_int32, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                      C.POINTER(paraexp_stats)]),
    "paraexp_solve_finish": (C.c_int, [_vp, C.POINTER(paraexp_expmv_opts), C.c_int32, _vp, _vp, _vp, _vp,
                                       _vp, _vp, _vp, C.POINTER(paraexp_stats)]),
    "paraexp_leja_points": (C.c_int, [C.c_int32, _dp]),
    "paraexp_plan_host": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                    C.c_double, C.c_double, C.POINTER(paraexp_plan_info)]),
    "paraexp_theta": (C.c_double, [C.c_int32, C.c_int32, C.c_double]),
    "paraexp_optimal_tolerance": (C.c_double, [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_int32)]),
    "paraexp_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "paraexp_host_free": (None, [_vp]),
    "paraexp_strerror": (C.c_char_p, [C.c_int]),
    "paraexp_last_error": (C.c_char_p, []),
    "paraexp_version": (C.c_char_p, []),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sigs)


class ParaexpError(RuntimeError):
    def __init__(self, code, where):
        self.code = code
        msg = lib.paraexp_last_error().decode() or lib.paraexp_strerror(code).decode()
        super().__init__(f"{where}: {lib.paraexp_strerror(code).decode()} ({code}): {msg}")


def check(code, where, stats=None):
    """Raise ParaexpError for a negative status; the call's stats (e.g. fail_interval) ride
    along as ``err.stats``."""
    if code < 0:
        err = ParaexpError(code, where)
        err.stats = stats.as_dict() if stats is not None else None
        raise err
    return code
