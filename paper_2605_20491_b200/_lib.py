"""ctypes binding of libkronop.so (the C-ABI declared in include/kronop_cuda.h).

The library is built in-tree by paper_2605_20491_b200.build_ext. There is no fallback: if the
shared object is missing or fails to load, every entry point raises.
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KRONOP_LIB") or os.path.join(_HERE, "libkronop.so")

KRONOP_OK = 0
KRONOP_EPARAM = 2
KRONOP_ENUMERICAL = 3
KRONOP_ECAPABILITY = 4
KRONOP_ERUNTIME = 5

KRONOP_MAP_APPLY = 0
KRONOP_MAP_SOLVE = 1
KRONOP_SHIFT_FRACTION, KRONOP_SHIFT_OFFSET, KRONOP_SHIFT_ZERO = 0, 1, 2
KRONOP_GPE_H1, KRONOP_GPE_AU = 0, 1
KRONOP_GPE_INIT_CONSTANT, KRONOP_GPE_INIT_EIGENFUNCTION, KRONOP_GPE_INIT_SUPPLIED = 0, 1, 2
KRONOP_COMPOSITION_SINGLE, KRONOP_COMPOSITION_YOSHIDA = 0, 1
KRONOP_EPI_STORE, KRONOP_EPI_SPEC_MUL, KRONOP_EPI_SPEC_DIV = 0, 1, 2
KRONOP_EPI_SPEC_PHASE, KRONOP_EPI_AXPY_DIAG = 3, 4

P = C.c_void_p
D = C.c_double
I = C.c_int
DP = C.POINTER(C.c_double)
IP = C.POINTER(C.c_int)


class LinearMap(C.Structure):
    _fields_ = [("op", P), ("mode", I), ("diag", P), ("sigma", D), ("scale", P)]


class PcgConfig(C.Structure):
    _fields_ = [("rel_tol", D), ("max_iter", I), ("record_history", I),
                ("preconditioned_norm", I), ("stagnation_window", I)]


class PcgReport(C.Structure):
    _fields_ = [("iterations", I), ("final_residual", D), ("converged", I), ("history_len", I)]


class InverseIterationConfig(C.Structure):
    _fields_ = [("shift_mode", I), ("shift_fraction", D), ("shift_offset", D),
                ("eig_rel_tol", D), ("max_outer", I), ("inner", PcgConfig)]


class EigenpairResult(C.Structure):
    _fields_ = [("eigenvalue", D), ("outer_iterations", I), ("total_inner_iterations", I),
                ("converged", I)]


class GpeConfig(C.Structure):
    _fields_ = [("kind", I), ("step", D), ("metric_shift", D), ("energy_rel_tol", D),
                ("max_iterations", I), ("inner", PcgConfig), ("init", I), ("record_history", I)]


class GpeResult(C.Structure):
    _fields_ = [("energy", D), ("eigenvalue", D), ("iterations", I), ("linear_solves", C.c_longlong),
                ("converged", I), ("history_len", I)]


class SplitSpec(C.Structure):
    _fields_ = [("quad_points", I), ("composition", I), ("dt", D), ("total_time", D),
                ("merge_across_steps", I), ("mass_weighted_error", I)]


# name -> (restype, argtypes)
PROTOTYPES = {
    "kronop_last_error": (C.c_char_p, []),
    "kronop_version": (C.c_char_p, []),
    "kronop_ctx_create": (I, [I, P, C.POINTER(P)]),
    "kronop_ctx_destroy": (I, [P]),
    "kronop_ctx_synchronize": (I, [P]),
    "kronop_ctx_workspace_bytes": (I, [P, C.POINTER(C.c_size_t)]),
    "kronop_ctx_launch_count": (I, [P, C.POINTER(C.c_uint64)]),
    "kronop_field_alloc": (I, [P, C.c_size_t, C.POINTER(P)]),
    "kronop_field_free": (I, [P, P]),
    "kronop_field_upload": (I, [P, P, P, C.c_size_t]),
    "kronop_field_download": (I, [P, P, P, C.c_size_t]),
    "kronop_mode_product": (I, [P, P, I, IP, I, DP, I, I, P]),
    "kronop_kron_apply": (I, [P, P, I, IP, I, C.POINTER(DP), IP, P]),
    "kronop_inner": (I, [P, P, P, I, IP, I, C.POINTER(DP), DP]),
    "kronop_mass_field": (I, [P, I, IP, C.POINTER(DP), P]),
    "kronop_direct_sum_grid": (I, [P, I, IP, C.POINTER(DP), P]),
    "kronop_op_create": (I, [P, I, IP, C.POINTER(DP), C.POINTER(DP), C.POINTER(DP),
                             C.POINTER(DP), D, C.POINTER(P)]),
    "kronop_op_create_folded": (I, [P, I, IP] + [C.POINTER(DP)] * 8 + [D, C.POINTER(P)]),
    "kronop_op_destroy": (I, [P]),
    "kronop_ctx_trim": (I, [P]),
    "kronop_sep_solve_lowp": (I, [P, P, P, I, P]),
    "kronop_sep_propagate_lowp": (I, [P, P, P, D, I, P]),
    "kronop_op_set_precision": (I, [P, P, I]),
    "kronop_field_dump": (I, [P, C.c_char_p, I, IP, I, P]),
    "kronop_field_dump_host": (I, [C.c_char_p, I, IP, I, DP]),
    "kronop_field_load_header": (I, [C.c_char_p, IP, IP, IP]),
    "kronop_field_load": (I, [P, C.c_char_p, P, C.c_size_t]),
    "kronop_field_load_host": (I, [C.c_char_p, DP, C.c_size_t]),
    "kronop_op_set_shift": (I, [P, D]),
    "kronop_op_info": (I, [P, DP, DP, DP, C.POINTER(C.c_size_t)]),
    "kronop_op_eigenvalue_grid": (I, [P, P, P]),
    "kronop_sep_apply": (I, [P, P, P, I, P]),
    "kronop_sep_solve": (I, [P, P, P, I, P]),
    "kronop_sep_propagate": (I, [P, P, P, D, P]),
    "kronop_op_ground_state": (I, [P, P, P]),
    "kronop_full_apply": (I, [P, P, P, D, P, I, P]),
    "kronop_op_pass": (I, [P, P, I, I, P, I, P]),
    "kronop_op_pass_ex": (I, [P, P, I, I, P, I, P, I, D, P, D, P]),
    "kronop_sep_solve_host": (I, [P, P, P, I, P]),
    "kronop_sep_apply_host": (I, [P, P, P, I, P]),
    "kronop_sep_propagate_host": (I, [P, P, P, D, P]),
    "kronop_sep_solve_host_batch": (I, [P, P, I, P, I, P]),
    "kronop_sep_propagate_host_batch": (I, [P, P, I, P, D, P]),
    "kronop_pcg": (I, [P, C.POINTER(LinearMap), C.POINTER(LinearMap), P, P,
                       C.POINTER(PcgConfig), C.POINTER(PcgReport), DP]),
    "kronop_inverse_iteration": (I, [P, P, P, C.POINTER(InverseIterationConfig), P, P,
                                     C.POINTER(EigenpairResult), IP]),
    "kronop_gpe_energy": (I, [P, P, P, D, P, DP]),
    "kronop_gpe_gradient_flow": (I, [P, P, P, P, D, C.POINTER(GpeConfig), P, P,
                                     C.POINTER(GpeResult), DP]),
    "kronop_yoshida_coeffs": (I, [DP, DP]),
    "kronop_qhop_step": (I, [P, P, P, P, D, I, P]),
    "kronop_yoshida_step": (I, [P, P, P, P, D, I, P]),
    "kronop_evolve": (I, [P, C.POINTER(SplitSpec), P, P, P, P, D, P, DP, IP]),
    "kronop_host_gll_rule": (I, [I, DP, DP, DP]),
    "kronop_host_gauss_legendre": (I, [I, DP, DP]),
    "kronop_host_assemble_sem": (I, [D, I, I, DP, DP, DP]),
    "kronop_host_interp_matrix": (I, [D, I, I, I, I, DP]),
    "kronop_host_sym_eig": (I, [I, DP, DP, DP]),
    "kronop_host_build_sem_axis": (I, [D, I, I, DP, DP, DP, DP]),
    "kronop_host_hermite_basis": (I, [I, DP, DP, DP, DP]),
    "kronop_host_eval_weights": (I, [D, I, I, DP, I, DP]),
    "kronop_host_build_hermite_axis": (I, [I, DP, DP, DP, DP]),
    "kronop_host_build_sem_axis_folded": (I, [D, I, I] + [DP] * 8),
    "kronop_splitmix_uniform": (I, [P, C.c_uint64, C.c_uint64, C.c_size_t, P]),
    "kronop_selftest_division": (I, [P, P, P, C.c_size_t, P]),
    "kronop_slab_plan": (I, [I, I, IP, IP]),
    "kronop_nccl_load": (I, [C.c_char_p]),
    "kronop_nccl_unique_id": (I, [C.c_char_p]),
    "kronop_slab_create": (I, [I, IP, I, IP, P, P, P, P, D, P]),
    "kronop_slab_create_nccl": (I, [P, C.c_char_p, I, I, I, IP, P, P, P, P, D, P]),
    "kronop_slab_destroy": (I, [P]),
    "kronop_slab_info": (I, [P, IP, IP, IP]),
    "kronop_slab_stats": (I, [P, C.POINTER(C.c_longlong)]),
    "kronop_slab_part": (I, [P, I, IP, C.POINTER(C.c_void_p), C.POINTER(C.c_longlong),
                             C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    "kronop_slab_set_shift": (I, [P, D]),
    "kronop_slab_field_alloc": (I, [P, I, C.c_size_t, P]),
    "kronop_slab_field_free": (I, [P, I, P]),
    "kronop_slab_scatter": (I, [P, DP, I, P]),
    "kronop_slab_gather": (I, [P, P, I, DP]),
    "kronop_slab_synchronize": (I, [P]),
    "kronop_slab_apply": (I, [P, P, I, P, D, P]),
    "kronop_slab_solve": (I, [P, P, I, P]),
    "kronop_slab_propagate": (I, [P, P, D, P]),
    "kronop_slab_dot": (I, [P, P, P, I, DP]),
    "kronop_slab_pcg": (I, [P, P, D, P, P, C.POINTER(PcgConfig), C.POINTER(PcgReport), DP]),
    "kronop_slab_gpe_au": (I, [P, P, D, C.POINTER(GpeConfig), P, P, C.POINTER(GpeResult), DP]),
}

_lib = None


class KronopError(RuntimeError):
    """Non-zero status from the C-ABI. `code` mirrors the reference's exception classes."""

    def __init__(self, code, msg):
        super().__init__("[%d] %s" % (code, msg))
        self.code = code
        self.msg = msg


class ParameterError(KronopError):
    pass


class NumericalError(KronopError):
    pass


class CapabilityError(KronopError):
    pass


_ERRS = {KRONOP_EPARAM: ParameterError, KRONOP_ENUMERICAL: NumericalError,
         KRONOP_ECAPABILITY: CapabilityError}


def lib():
    """Load libkronop.so (raises if it is missing: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libkronop.so not built (run `python -m paper_2605_20491_b200.build_ext`): "
                              + LIB_PATH)
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib


def check(rc):
    if rc != KRONOP_OK:
        msg = lib().kronop_last_error().decode()
        raise _ERRS.get(rc, KronopError)(rc, msg)
