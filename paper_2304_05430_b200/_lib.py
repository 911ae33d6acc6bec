"""ctypes binding of libtt_b200.so (the C ABI declared in include/tt_b200.h).

The product path has no fallback: if the shared library is missing or a CUDA
device is absent, every entry point raises.
"""

from __future__ import annotations

import collections
import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# TT_LIB overrides the library path (kernel-variant experiments, tools/)
LIB_PATH = os.environ.get("TT_LIB") or os.path.join(_HERE, "libtt_b200.so")

_P, _I32, _I64, _D, _SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t

TT_LOSS_MSE, TT_LOSS_RANK = 0, 1
TT_MODE_TRAIN, TT_MODE_GRAD = 0, 1

# name -> (restype, argtypes); mirrors include/tt_b200.h one to one
SIGNATURES: dict[str, tuple] = {
    "tt_abi_version": (ctypes.c_int, []),
    "tt_last_error": (ctypes.c_char_p, []),
    "tt_pca_workspace_bytes": (_SZ, [_P, _I32]),
    "tt_pca_counts": (ctypes.c_int, [_P, _P, _P, _I32, _P, _P, _SZ, _P]),
    "tt_topk": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _P, _P, _P]),
    "tt_rank_loss_f32": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _P, _P, _P]),
    "tt_rank_loss_f64": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _P, _P, _P]),
    "tt_adam_step_f32": (ctypes.c_int, [_P, _P, _P, _P, _I64, _P, _D, _D, _D, _D, _D, _D, _P]),
    "tt_adam_step_f64": (ctypes.c_int, [_P, _P, _P, _P, _I64, _P, _D, _D, _D, _D, _D, _D, _P]),
    "tt_tuner_param_count": (_I64, [_I32, _I32, _I32, _I32]),
    "tt_tuner_predict_workspace_bytes": (_SZ, [_I32, _I32, _I32, _I32]),
    "tt_tuner_predict_f32": (ctypes.c_int, [_P, _P, _P, _P, _I64] + [_I32] * 7 + [_P, _P, _SZ, _P]),
    "tt_tuner_predict_f64": (ctypes.c_int, [_P, _P, _P, _P, _I64] + [_I32] * 7 + [_P, _P, _SZ, _P]),
    "tt_tuner_predict_tf32_workspace_bytes": (_SZ, [_I32]),
    "tt_tuner_predict_tf32": (ctypes.c_int, [_P, _P, _P, _P, _I64] + [_I32] * 7 + [_P, _P, _SZ, _P]),
    "tt_tuner_predict_f32tc_workspace_bytes": (_SZ, [_I32, _I32, _I32, _I64]),
    "tt_tuner_f32tc_eligible": (ctypes.c_int, [_I32] * 5),
    "tt_tuner_predict_f32tc": (ctypes.c_int, [_P, _P, _P, _P, _I64] + [_I32] * 7 + [_P, _P, _SZ, _P]),
    "tt_tuner_train_workspace_bytes": (_SZ, [_I32] * 7),
    "tt_tuner_train_f32": (ctypes.c_int, [_P] * 7 + [_P, _I64, _I32, _I32, _I32, _D, _D, _D, _D, _P, _P]
                           + [_I32] * 7 + [_P, _P, _P, _P, _SZ, _P]),
    "tt_tuner_train_f64": (ctypes.c_int, [_P] * 7 + [_P, _I64, _I32, _I32, _I32, _D, _D, _D, _D, _P, _P]
                           + [_I32] * 7 + [_P, _P, _P, _P, _SZ, _P]),
    "tt_tuner_lstm_outputs_f32": (ctypes.c_int, [_P, _P, _P, _P, _I64] + [_I32] * 7 + [_P, _P, _P, _SZ, _P]),
    "tt_tuner_train_heads_f32": (ctypes.c_int, [_P] * 7 + [_P, _I64, _I32, _I32, _D, _D, _D, _D, _P, _P]
                                 + [_I32] * 7 + [_P, _P, _P, _P, _SZ, _P]),
    "tt_tuner_dp_buffer_bytes": (_SZ, [_I32] * 5),
    "tt_tuner_train_dp_f32": (ctypes.c_int, [_P] * 7 + [_P, _I64, _I32, _I32, _D, _D, _D, _D, _P, _P]
                              + [_I32] * 7 + [_I32, _I32, _I64, _P] + [_P, _P, _P, _SZ, _P]),
    "tt_ipc_alloc": (ctypes.c_int, [_SZ, _P, _P]),
    "tt_ipc_open": (ctypes.c_int, [_P, _P]),
    "tt_ipc_close": (ctypes.c_int, [_P]),
    "tt_dev_free": (ctypes.c_int, [_P]),
    "tt_tuner_train_set_grid": (ctypes.c_int, [_I32]),
    "tt_tuner_dp_set_timeout_ms": (ctypes.c_int, [_I64]),
    "tt_tuner_train_fast_eligible": (_I32, [_I32] * 8),
    "tt_tuner_train_set_path": (ctypes.c_int, [_I32]),
    "tt_debug_profile_step": (ctypes.c_int, [_I32]),
    "tt_debug_phase_times": (ctypes.c_int, [_P, _I32]),
    "tt_debug_tc_phase_times": (ctypes.c_int, [_P, _I32]),
    "tt_debug_x3_phase_times": (ctypes.c_int, [_P, _I32]),
    "tt_debug_mlp_phase_times": (ctypes.c_int, [_P, _I32]),
    "tt_mlp_param_count": (_I64, [_I32]),
    "tt_mlp_predict_f32": (ctypes.c_int, [_P, _P, _I64, _I32, _P, _P]),
    "tt_mlp_predict_f64": (ctypes.c_int, [_P, _P, _I64, _I32, _P, _P]),
    "tt_mlp_predict_tf32": (ctypes.c_int, [_P, _P, _I64, _I32, _P, _P]),
    "tt_mlp_predict_f32tc": (ctypes.c_int, [_P, _P, _I64, _I32, _P, _P]),
    "tt_mlp_f32tc_eligible": (_I32, [_I32, _P]),
    "tt_mlp_train_workspace_bytes": (_SZ, [_I32, _I32, _I32]),
    "tt_mlp_train_f32": (ctypes.c_int, [_P] * 5 + [_I32, _P, _I64, _I32, _I32, _I32, _D, _D, _D, _D, _P,
                                                   _P, _P, _P, _P, _SZ, _P]),
    "tt_mlp_train_f64": (ctypes.c_int, [_P] * 5 + [_I32, _P, _I64, _I32, _I32, _I32, _D, _D, _D, _D, _P,
                                                   _P, _P, _P, _P, _SZ, _P]),
    "tt_gbdt_workspace_bytes": (_SZ, [_I64, _I32, _I32]),
    "tt_gbdt_grow": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P,
                                    _SZ, _P]),
    "tt_gbdt_update": (ctypes.c_int, [_P, _P, _P, _P, _D, _I64, _P]),
    "tt_gbdt_predict": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _I32, _D, _D, _P, _I64, _I32, _I32, _P, _I32,
                                       _P]),
    "tt_prune_workspace_bytes": (_SZ, [_I64]),
    "tt_prune_stats": (ctypes.c_int, [_P, _P, _P, _P, _I32, _D, _I32, _P, _P, _P, _P, _P, _SZ, _P]),
}

_lock = threading.Lock()
_lib = None
# per entry point call counts: evidence that a host stack (the reference's own
# tests under install(), bench.py) really reached the kernels
CALLS: collections.Counter = collections.Counter()


class LibraryError(RuntimeError):
    pass


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the shared library; raise if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise LibraryError(
                f"{path} is missing: build it with `python -m paper_2304_05430_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is None:  # reported by missing_symbols(); calling it raises
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def call(name: str, *args) -> None:
    """Invoke an int-returning entry point and raise on a non-zero status."""
    lib = load()
    CALLS[name] += 1
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.tt_last_error()
        raise LibraryError(f"{name} failed (status {rc}): {msg.decode() if msg else ''}")


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def missing_symbols() -> list[str]:
    lib = load()
    return [n for n in SIGNATURES if getattr(lib, n, None) is None]
