"""ctypes binding of libomni.so (the C-ABI declared in include/omni.h).

This is the only place Python touches the native library.  The product path
fails loudly when the library is missing -- there is no CPU fallback.
Status codes map onto the reference's error behaviour: argument errors raise
``ValueError`` (as omnisim does, e.g. tensors.py:44-54), CUDA failures raise
``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libomni.so")

OMNI_OK = 0
OMNI_EINVAL = -1
OMNI_ECUDA = -2
OMNI_EUNSUPPORTED = -3
OMNI_ETIMEOUT = -4

PREC_TF32 = 0
PREC_3XTF32 = 1
PREC_FP32_SIMT = 2
PRECISIONS = {"tf32": PREC_TF32, "3xtf32": PREC_3XTF32, "fp32_simt": PREC_FP32_SIMT}

EPI_STORE = 0
EPI_BIAS = 1
EPI_BIAS_RELU = 2
EPI_ACCUM = 3
EPI_MASK_AUX = 4
EPI_RELU = 5

CONV_FPROP = 0
CONV_WGRAD = 1
CONV_WGRAD_BIAS = 2

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_longlong
_F = ctypes.c_float
_D = ctypes.c_double

# name -> (restype, argtypes); mirrors include/omni.h one to one.
SIGNATURES: dict[str, tuple] = {
    "omni_last_error": (ctypes.c_char_p, []),
    "omni_version": (_I, []),
    "omni_device_sm_count": (_I, [_I]),
    "omni_launch_count": (_L, []),
    "omni_set_sm_reserve": (_I, [_I]),
    "omni_get_sm_reserve": (_I, []),
    "omni_lower_nchw_f32": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _L, _P]),
    "omni_lower_nchw_f64": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _L, _P]),
    "omni_lower_nhwc_f32": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _L, _P]),
    "omni_lift_nchw_f32": (_I, [_P, _L, _I, _I, _I, _P, _P]),
    "omni_lift_nchw_f64": (_I, [_P, _L, _I, _I, _I, _P, _P]),
    "omni_col2im_nhwc_f32": (_I, [_P, _L, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P]),
    "omni_gemm_plan": (_L, [_I, _I, _I, _I, _I, _I, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "omni_gemm_f32": (
        _I,
        [_I, _I, _I, _I, _P, _L, _I, _P, _L, _I, _P, _L, _I, _P, _P, _L, _P, _L, _P],
    ),
    "omni_conv_implicit_plan": (_L, [_I, _I, _I, _I, _I, _I, _I, _I, _I]),
    "omni_conv_implicit_f32": (
        _I,
        [_I, _I, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _L, _P, _L, _I, _P, _P, _L, _P, _L, _P],
    ),
    "omni_conv_weight_flip_f32": (_I, [_P, _I, _I, _I, _P, _L, _P]),
    "omni_conv_window_plan": (_L, [_I, _I, _I, _I, _I, _I]),
    "omni_conv_window_f32": (_I, [_I, _P, _I, _I, _I, _I, _I, _P, _L, _P, _L, _I, _P, _P, _L, _P]),
    "omni_pool_out_size": (_I, [_I, _I, _I, _I, _I]),
    "omni_pool_fwd_nhwc_f32": (_I, [_I, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _I, _P, _P]),
    "omni_pool_bwd_nhwc_f32": (
        _I,
        [_I, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _I, _P, _P],
    ),
    "omni_softmax_xent_f32": (_I, [_P, _L, _P, _I, _I, _P, _P, _L, _F, _P]),
    "omni_relu_fwd_f32": (_I, [_P, _P, _L, _P]),
    "omni_relu_bwd_f32": (_I, [_P, _P, _P, _L, _P]),
    "omni_bias_grad_ws_elems": (_L, [_I, _I]),
    "omni_bias_grad_f32": (_I, [_P, _L, _I, _I, _P, _P, _P]),
    "omni_sgd_momentum_f32": (_I, [_P, _P, _P, _P, _F, _F, _F, _L, _P]),
    "omni_sgd_momentum_f64": (_I, [_P, _P, _P, _P, _D, _D, _D, _L, _P]),
    "omni_group_updates_f32": (_I, [_P, _I, _L, _P, _I, _I, _P, _P, _P, _L, _F, _F, _F, _P]),
    "omni_gather_rows_f32": (_I, [_P, _L, _P, _I, _P, _P]),
    "omni_gather_i32": (_I, [_P, _P, _I, _P, _P]),
    "omni_conv_weight_to_tap_f32": (_I, [_P, _I, _I, _I, _P, _L, _I, _P, _P]),
    "omni_space_to_depth_f32": (_I, [_P, _I, _I, _I, _I, _I, _P, _I, _I, _P]),
    "omni_space_to_depth_gather_f32": (_I, [_P, _P, _I, _I, _I, _I, _I, _P, _I, _I, _P]),
    "omni_conv_weight_s2d_f32": (_I, [_P, _I, _I, _I, _I, _I, _P, _L, _I, _P, _P]),
    "omni_transpose_f32": (_I, [_P, _L, _L, _I, _I, _P, _L, _L, _I, _P]),
    "omni_fill_f32": (_I, [_P, _F, _L, _P]),
    "omni_comm_nccl_version": (_I, [ctypes.POINTER(_I)]),
    "omni_comm_unique_id": (_I, [_P]),
    "omni_comm_init_rank": (_I, [ctypes.POINTER(_P), _I, _P, _I, _I]),
    "omni_comm_init_all": (_I, [_I, _P, _P]),
    "omni_comm_split": (_I, [_P, _I, _I, ctypes.POINTER(_P)]),
    "omni_comm_destroy": (_I, [_P]),
    "omni_comm_size_rank": (_I, [_P, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "omni_allreduce_sum_f32": (_I, [_P, _P, ctypes.c_size_t, _P]),
    "omni_broadcast_f32": (_I, [_P, _P, ctypes.c_size_t, _I, _P]),
    "omni_send_f32": (_I, [_P, _P, ctypes.c_size_t, _I, _P]),
    "omni_recv_f32": (_I, [_P, _P, ctypes.c_size_t, _I, _P]),
    "omni_allgather_f32": (_I, [_P, _P, _P, ctypes.c_size_t, _P]),
    "omni_all_to_all_f32": (_I, [_P, _P, _P, ctypes.c_size_t, _P]),
    "omni_comm_group_start": (_I, []),
    "omni_comm_group_end": (_I, []),
    "omni_p2p_step": (_I, [_P, _P]),
    "omni_p2p_signal": (_I, [_P, _I, _I, _I, _I, _I, _P, _P]),
    "omni_p2p_wait": (_I, [_P, _I, _I, _I, _I, _I, _I, _P, _P]),
    "omni_p2p_reduce_sgd_f32": (_I, [_P, _P, _I, _I, _L, _L, _P, _P, _F, _F, _F, _P]),
    "omni_copy_async": (_I, [_P, _P, _L, _P]),
    "omni_mailbox_bytes": (_L, []),
    "omni_mailbox_create": (_I, [ctypes.c_char_p, _I, ctypes.POINTER(_P)]),
    "omni_mailbox_open": (_I, [ctypes.c_char_p, ctypes.POINTER(_P), _I]),
    "omni_mailbox_close": (_I, [_P, ctypes.c_char_p]),
    "omni_mailbox_post": (_I, [_P, _I, ctypes.POINTER(_L)]),
    "omni_mailbox_next": (_I, [_P, ctypes.POINTER(_I), _I]),
    "omni_mailbox_snap_post": (_I, [_P, _I, _L]),
    "omni_mailbox_snap_wait": (_I, [_P, _I, _L, ctypes.POINTER(_L), _I]),
    "omni_ipc_handle": (_I, [_P, _P, ctypes.POINTER(_L)]),
    "omni_ipc_open": (_I, [_P, ctypes.POINTER(_P)]),
    "omni_ipc_close": (_I, [_P]),
}

_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load libomni.so once; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(); "
                "this framework has no CPU fallback"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def last_error() -> str:
    msg = load().omni_last_error()
    return msg.decode() if msg else ""


def call(name: str, *args) -> int:
    """Invoke an int-returning entry point and map a failure status to an exception."""
    rc = getattr(load(), name)(*args)
    if rc != OMNI_OK:
        msg = last_error()
        if rc == OMNI_EINVAL:
            raise ValueError(msg)
        raise RuntimeError(f"{name}: {msg} (status {rc})")
    return rc


def query(name: str, *args):
    """Invoke a value-returning entry point (no status mapping)."""
    return getattr(load(), name)(*args)
