"""ctypes binding of ``libeinet_b200.so`` (C ABI in ``include/einet_b200.h``).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int32, c_int64, c_uint8, c_void_p

LIB_NAME = "libeinet_b200.so"
_DEFAULT_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libeinet_b200.so")
LIB_PATH = os.environ.get(  # EINET_LIB_PATH: A/B timing of another build (diagnostics)
    "EINET_LIB_PATH", os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME))

OK = 0
ERR_USAGE = 1
ERR_ENGINE = 2
ERR_UNSUPPORTED = 3
ERR_CUDA = 4

FAMILY_IDS = {"gaussian": 0, "categorical": 1, "binomial": 2}
LAYER_EINSUM = 1
LAYER_MIXING = 2
STATUS_WORDS = 4
STATUS_NONE = 2 ** 31 - 1

P_i32 = POINTER(c_int32)
P_u8 = POINTER(c_uint8)


class LayerDesc(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("rows", c_int32), ("k_out", c_int32),
                ("is_root", c_int32), ("dmax", c_int32),
                ("left", P_i32), ("right", P_i32), ("out_rows", P_i32),
                ("src", P_i32), ("mask", P_u8)]


class PlanDesc(ctypes.Structure):
    _fields_ = [("d_vars", c_int32), ("k", c_int32), ("k_root", c_int32),
                ("num_replicas", c_int32), ("num_buffer_rows", c_int32),
                ("family", c_int32), ("num_states", c_int32), ("n_trials", c_int32),
                ("var_min", c_double), ("var_max", c_double), ("p_min", c_double),
                ("n_leaf", c_int32), ("leaf_scope_offsets", P_i32),
                ("leaf_scope_vars", P_i32), ("leaf_replica", P_i32),
                ("leaf_out_rows", P_i32), ("n_layers", c_int32),
                ("layers", POINTER(LayerDesc)), ("root_mix_row", c_int32)]


class Sizes(ctypes.Structure):
    _fields_ = [(name, c_int64) for name in (
        "params_f64", "phi_offset", "mixing_offset", "stats_f64", "stats_acc_pt_offset",
        "stats_p_offset", "stats_ll_offset", "compute_bytes", "workspace_bytes",
        "max_chunk", "suff_dim")]


EXPORTS = {
    "einet_plan_create": (c_int32, [POINTER(PlanDesc), c_int64, POINTER(c_void_p)]),
    "einet_plan_destroy": (None, [c_void_p]),
    "einet_plan_sizes": (c_int32, [c_void_p, POINTER(Sizes)]),
    "einet_prepare": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "einet_forward": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p,
                                c_void_p, c_void_p]),
    "einet_backward": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                                 c_void_p, c_void_p, c_void_p]),
    "einet_status_reset": (c_int32, [c_void_p, c_void_p]),
    "einet_log_step": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
                                 c_void_p]),
    "einet_status_to_stats": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "einet_status_from_stats": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "einet_plan_set_tensor_cores": (c_int32, [c_void_p, c_int32]),
    "einet_stats_zero": (c_int32, [c_void_p, c_void_p, c_void_p]),
    "einet_mstep": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_double,
                              c_void_p, c_void_p]),
    "einet_stats_expand_acc_p": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "einet_export_buffer": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "einet_export_leaf_rows": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "einet_ef_log_prob": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                                    c_void_p, c_void_p, c_void_p]),
    "einet_log_einsum_exp": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_int32,
                                       c_int32, c_int32, c_void_p, c_void_p]),
    "einet_sample_scratch_bytes": (c_int64, [c_void_p, c_int64]),
    "einet_sample": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_int64,
                               ctypes.c_uint64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "einet_decode_u8": (c_int32, [c_void_p, c_int64, ctypes.c_double, c_void_p, c_void_p]),
    "einet_pack_f64": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_int32, c_void_p]),
    "einet_crc32": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p]),
    "einet_params_from_blob": (c_int32, [c_void_p, c_int64, c_void_p, c_int32, c_int64, c_void_p,
                                         c_void_p, c_void_p]),
    "einet_params_to_blob": (c_int32, [c_void_p, c_void_p, c_int32, c_int64, c_void_p,
                                       c_void_p]),
    "einet_selftest_tf32_gemm": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32,
                                           c_void_p]),
    "einet_launch_count": (c_int64, []),
    "einet_profile_enable": (c_int32, [c_int32]),
    "einet_profile_query": (c_int32, [c_int32, ctypes.c_char_p, c_int32,
                                      POINTER(c_double), POINTER(c_int64)]),
    "einet_last_error": (ctypes.c_char_p, []),
}

_lib = None


class NativeUnavailable(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load the shared library and declare every exported symbol."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{LIB_NAME} not built ({path} missing); run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    for name, (res, args) in EXPORTS.items():
        if path != _DEFAULT_LIB and not hasattr(lib, name):
            continue  # an older build under EINET_LIB_PATH (A/B timing only)
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    return load()


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable(
            "paper_2004_06231_b200 runs on CUDA only (no CPU fallback): no GPU visible")
    return load()


def last_error() -> str:
    return load().einet_last_error().decode("utf-8", "replace")


def check(rc: int, what: str):
    if rc == OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == ERR_USAGE:
        raise ValueError(msg)
    if rc == ERR_ENGINE:
        from .engine import EngineError
        raise EngineError(msg)
    raise RuntimeError(msg)


def launch_count() -> int:
    return int(load().einet_launch_count())


PROFILING = False


def profile_enable(on: bool = True):
    global PROFILING
    load().einet_profile_enable(1 if on else 0)
    PROFILING = bool(on)


def profile_read() -> dict:
    """{kernel class: (total device ms, launch groups)} since profile_enable."""
    lib = load()
    out = {}
    i = 0
    name = ctypes.create_string_buffer(64)
    while True:
        ms = c_double()
        cnt = c_int64()
        if lib.einet_profile_query(i, name, 64, ctypes.byref(ms), ctypes.byref(cnt)) != OK:
            break
        out[name.value.decode()] = (ms.value, cnt.value)
        i += 1
    return out
