"""ctypes binding of libhf.so (include/hf.h).  There is no CPU fallback: if the
library is missing or no CUDA device is present, every compute call raises."""

from __future__ import annotations

import ctypes as ct
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HF_LIB") or os.path.join(_HERE, "libhf.so")  # HF_LIB: A/B builds only
HEADER = os.path.join(os.path.dirname(_HERE), "include", "hf.h")

HF_OK, HF_ERR_ARG, HF_ERR_CUDA, HF_ERR_UNSUPPORTED, HF_ERR_JACOBIAN, HF_ERR_GEOMETRY = 0, 1, 2, 3, 4, 5
HF_SCALAR, HF_TENSOR2, HF_TENSOR4 = 0, 1, 2
STRATEGY_CODE = {"scalar": HF_SCALAR, "tensor2": HF_TENSOR2, "tensor4": HF_TENSOR4}


class HfErrorInfo(ct.Structure):
    _fields_ = [("code", ct.c_int), ("element", ct.c_longlong), ("qpoint", ct.c_int), ("det", ct.c_double)]


class HfError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libhf error {code}: {msg}")
        self.code = code


P = ct.c_void_p
I = ct.c_int
LL = ct.c_longlong
D = ct.c_double
PD = ct.POINTER(ct.c_double)

_SIGS = {
    "hf_last_error": (ct.c_char_p, []),
    "hf_abi_version": (I, []),
    "hf_max_degree": (I, [I]),
    "hf_pool_release": (I, []),
    "hf_pool_info": (I, [P, P]),
    "hf_space_create": (I, [I, I, I, P, P, P, P, P, P, P, P, P, P, ct.POINTER(P)]),
    "hf_space_set_mask": (I, [P, P, P]),
    "hf_space_info": (I, [P, ct.POINTER(LL), ct.POINTER(LL), ct.POINTER(LL)]),
    "hf_space_pointers": (I, [P, ct.POINTER(P), ct.POINTER(P), ct.POINTER(P)]),
    "hf_space_geometry_copy": (I, [P, P, P, P]),
    "hf_space_destroy": (I, [P]),
    "hf_jacobian_range": (I, [P, P, P, PD, PD, ct.POINTER(LL), ct.POINTER(I)]),
    "hf_tangent_create": (I, [P, I, P, P, ct.POINTER(P), ct.POINTER(HfErrorInfo)]),
    "hf_tangent_create_ex": (I, [P, I, I, P, P, ct.POINTER(P), ct.POINTER(HfErrorInfo)]),
    "hf_tangent_create_host": (I, [P, I, P, ct.POINTER(P), ct.POINTER(HfErrorInfo)]),
    "hf_tangent_diagonal_host": (I, [P, P]),
    "hf_tangent_apply": (I, [P, P, P, P]),
    "hf_tangent_apply_flagged": (I, [P, P, P, P, P]),
    "hf_tangent_apply_raw": (I, [P, P, P, P, P]),
    "hf_tangent_apply_after_fill": (I, [P, P, P, P, P]),
    "hf_tangent_tiles": (I, [P, ct.POINTER(LL), ct.POINTER(I)]),
    "hf_tangent_apply_tiles": (I, [P, P, P, P, LL, LL, I, P]),
    "hf_tangent_apply_tiles_ex": (I, [P, P, P, P, LL, LL, I, I, P]),
    "hf_tangent_set_alternate": (I, [P, I]),
    "hf_tangent_apply_host": (I, [P, P, P, I, P]),
    "hf_host_register": (I, [P, LL]),
    "hf_stream_synchronize": (I, [P]),
    "hf_graph_begin": (I, [P]),
    "hf_graph_end": (I, [P, ct.POINTER(P), ct.POINTER(I)]),
    "hf_graph_launch": (I, [P, P]),
    "hf_graph_destroy": (I, [P]),
    "hf_timeline_fetch": (I, [P, LL, I]),
    "hf_tangent_host_info": (I, [P, ct.POINTER(I), ct.POINTER(ct.c_float)]),
    "hf_host_unregister": (I, [P]),
    "hf_tangent_diagonal": (I, [P, P, P]),
    "hf_tangent_assemble_local": (I, [P, P, P]),
    "hf_space_cell_dofs": (I, [P, P, P]),
    "hf_tangent_storage": (I, [P, ct.POINTER(LL), ct.POINTER(I), ct.POINTER(LL)]),
    "hf_tangent_destroy": (I, [P]),
    "hf_residual": (I, [P, P, P, P, P, P, ct.POINTER(HfErrorInfo)]),
    "hf_energy": (I, [P, P, P, P, ct.POINTER(HfErrorInfo)]),
    "hf_transfer_create": (I, [P, P, ct.POINTER(P), ct.POINTER(P)]),
    "hf_prolong": (I, [P, P, P, I, P]),
    "hf_restrict": (I, [P, P, P, I, P]),
    "hf_prolong_ex": (I, [P, P, I, P, I, I, P]),
    "hf_restrict_ex": (I, [P, P, I, P, I, I, P]),
    "hf_transfer_destroy": (I, [P]),
    "hf_inject": (I, [P, P, P, P, I, P]),
    "hf_ws_create": (I, [ct.POINTER(P)]),
    "hf_ws_destroy": (I, [P]),
    "hf_dot": (I, [P, LL, P, P, P, P, P]),
    "hf_fill_masked": (I, [LL, P, P, P, D, P]),
    "hf_cheb_step": (I, [LL, P, P, P, P, P, I, D, D, D, I, P, P]),
    "hf_cheb_step_fill": (I, [LL, P, P, P, P, P, I, D, D, D, I, P, P, P, P]),
    "hf_cheb_step_after_apply": (I, [LL, P, P, P, P, P, I, D, D, D, P, P, I, P]),
    "hf_cheb3_step": (I, [LL, P, P, P, P, P, I, D, D, D, I, I, P, P, I, I, P]),
    "hf_resid_masked": (I, [LL, P, P, P, P, P]),
    "hf_resnorm_check": (I, [P, LL, P, P, P, I, I, P, P]),
    "hf_scalar_op": (I, [I, P, I, I, D, P, P]),
    "hf_cg_update_xr": (I, [P, LL, P, P, P, P, P, I, I, I, P]),
    "hf_cg_update_p": (I, [LL, P, P, P, I, I, P]),
    "hf_cg_update_p_fill": (I, [LL, P, P, P, I, I, P, P, P]),
    "hf_jacobi_dot": (I, [P, LL, P, P, P, P, P]),
    "hf_axpby": (I, [LL, D, P, D, P, P]),
    "hf_lanczos_init": (I, [P, P, P]),
    "hf_coarse_create": (I, [LL, LL, P, P, P, P, ct.POINTER(P)]),
    "hf_coarse_cheb_solve": (I, [P, P, P, P, P, D, D, D, D, I, I, P, P, P]),
    "hf_coarse_destroy": (I, [P]),
    "hf_coarse_create_space": (I, [P, P, ct.POINTER(P)]),
    "hf_coarse_update": (I, [P, P, P]),
    "hf_coarse_clone": (I, [P, P, ct.POINTER(P)]),
    "hf_lanczos_step": (I, [P, LL, P, P, P, P, P, P, P, P, P]),
    "hf_lanczos_step_fill": (I, [P, LL, P, P, P, P, P, P, P, P, P, P, P]),
    "hf_fill_masked_f32": (I, [LL, P, P, P, D, P]),
    "hf_cheb_step_f32": (I, [LL, P, P, P, P, P, I, D, D, D, I, P, P, P, P]),
    "hf_resid_masked_f32": (I, [LL, P, P, P, P, P]),
    "hf_dot_f32": (I, [P, LL, P, P, P, P]),
    "hf_resnorm_check_f32": (I, [P, LL, P, P, P, I, I, P, P]),
    "hf_halo_add": (I, [LL, P, P, P, P]),
    "hf_halo_pack": (I, [LL, P, P, P, P]),
    "hf_halo_unpack_add": (I, [LL, P, P, P, P, P]),
    "hf_dot_owned": (I, [P, LL, P, P, P, P, P]),
    "hf_probe_dfma": (I, [LL, I, I, P, P]),
}


def header_symbols() -> list[str]:
    """Every function declared in include/hf.h."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"HF_API\s+[\w\s\*]+?\b(hf_\w+)\s*\(", text)))


_lib = None


def lib():
    """Load libhf.so (once).  Raises ImportError when it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1904_13131_b200.build` "
                              "(there is no CPU fallback)")
        L = ct.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("HF_LIB") and not hasattr(L, name):
                continue  # an older A/B build (tests check the in-tree library's exports)
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != HF_OK:
        raise HfError(rc, lib().hf_last_error().decode())


def last_error() -> str:
    return lib().hf_last_error().decode()
