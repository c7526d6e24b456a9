"""ctypes declarations of the C ABI in include/c0ip.h (argument marshalling only).

The library is loaded from the package directory (built in-tree by build.py / build()).
There is no fallback: if libc0ip.so is missing or fails to load, importing the binding
raises, so no product call can silently run elsewhere.
"""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libc0ip.so")

# c0ip_status
OK, ERR_ARG, ERR_STATE, ERR_COERCIVITY, ERR_OOM, ERR_CUDA, ERR_NCCL = range(7)
STATUS_NAMES = ["OK", "ERR_ARG", "ERR_STATE", "ERR_COERCIVITY", "ERR_OOM", "ERR_CUDA", "ERR_NCCL"]
F64, F32 = 0, 1
AVS_ATOMIC, AVS_DETERMINISTIC, AVS_COLORED, MVS = 0, 1, 2, 3
PATH_AUTO, PATH_GENERIC = 0, 1


class Config(C.Structure):
    _fields_ = [("dim", C.c_int32), ("degree", C.c_int32), ("finest_level", C.c_int32),
                ("cells_override", C.c_int64), ("penalty_scale", C.c_double), ("device", C.c_int32)]


LOCAL_FDM, LOCAL_EXACT = 0, 1


class MgConfig(C.Structure):
    _fields_ = [("smoother", C.c_int), ("steps", C.c_int32), ("omega", C.c_double),
                ("symmetric", C.c_int32), ("cycle_dtype", C.c_int)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("r0", C.c_double),
                ("rn", C.c_double), ("nu", C.c_double), ("seconds", C.c_double)]


EXPORTS = {
    "c0ip_create": (C.c_int, [C.POINTER(Config), C.POINTER(C.c_void_p)]),
    "c0ip_destroy": (C.c_int, [C.c_void_p]),
    "c0ip_create_graded": (C.c_int, [C.POINTER(Config), C.c_void_p, C.POINTER(C.c_void_p)]),
    "c0ip_create_sipg": (C.c_int, [C.POINTER(Config), C.POINTER(C.c_void_p)]),
    "c0ip_last_error": (C.c_char_p, []),
    "c0ip_set_path": (C.c_int, [C.c_void_p, C.c_int]),
    "c0ip_set_local_solver": (C.c_int, [C.c_void_p, C.c_int]),
    "c0ip_level_info": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "c0ip_patch_dofs": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p]),
    "c0ip_color_patches": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int64,
                                     C.POINTER(C.c_int64)]),
    "c0ip_get_fdm": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "c0ip_get_matrices_1d": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "c0ip_rhs": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "c0ip_apply": (C.c_int, [C.c_void_p, C.c_int32, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "c0ip_residual": (C.c_int, [C.c_void_p, C.c_int32, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p]),
    "c0ip_smooth": (C.c_int, [C.c_void_p, C.c_int32, C.c_int, C.c_int, C.c_int32, C.c_double, C.c_int32,
                              C.c_void_p, C.c_void_p, C.c_void_p]),
    "c0ip_restrict": (C.c_int, [C.c_void_p, C.c_int32, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "c0ip_prolongate_add": (C.c_int, [C.c_void_p, C.c_int32, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "c0ip_vcycle": (C.c_int, [C.c_void_p, C.POINTER(MgConfig), C.c_void_p, C.c_void_p, C.c_void_p]),
    "c0ip_pcg": (C.c_int, [C.c_void_p, C.POINTER(MgConfig), C.c_void_p, C.c_void_p, C.c_double, C.c_int32,
                           C.POINTER(Report), C.c_void_p, C.c_void_p]),
    "c0ip_gmres": (C.c_int, [C.c_void_p, C.POINTER(MgConfig), C.c_void_p, C.c_void_p, C.c_double, C.c_int32,
                             C.c_int32, C.POINTER(Report), C.c_void_p, C.c_void_p]),
    "c0ip_launch_count": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "c0ip_slab_fdm": (C.c_int, [C.c_void_p, C.c_int32, C.c_int, C.c_double, C.c_int64, C.c_int64, C.c_int64,
                                C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "c0ip_slab_mvs_color": (C.c_int, [C.c_void_p, C.c_int32, C.c_int, C.c_double, C.c_int32, C.c_int64, C.c_int64,
                                      C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "c0ip_slab_restrict": (C.c_int, [C.c_void_p, C.c_int32, C.c_int, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                     C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]),
    "c0ip_slab_prolongate_add": (C.c_int, [C.c_void_p, C.c_int32, C.c_int, C.c_int64, C.c_int64, C.c_void_p,
                                           C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]),
    "c0ip_slab_transfer_rows": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "c0ip_vec_axpby": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_void_p, C.c_double, C.c_void_p,
                                 C.c_void_p]),
    "c0ip_vec_dots": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p]),
    "c0ip_vcycle_level": (C.c_int, [C.c_void_p, C.POINTER(MgConfig), C.c_int32, C.c_void_p, C.c_void_p,
                                    C.c_void_p]),
    "c0ip_slab_ghosts": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "c0ip_slab_avs_step": (C.c_int, [C.c_void_p, C.c_int32, C.c_int, C.c_double, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "c0ip_slab_apply": (C.c_int, [C.c_void_p, C.c_int32, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
}

_lib = None


def load():
    """Load libc0ip.so and declare every exported symbol.  Raises if missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"C0IP CUDA library not built: {LIB_PATH} is missing "
                           "(run __graft_entry__.build() or python paper_2412_05082_b200/build.py)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class C0ipError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


def check(status):
    if status != OK:
        raise C0ipError(status, load().c0ip_last_error().decode())
