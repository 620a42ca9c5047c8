"""ctypes binding of libedl_b200.so (include/edl_b200.h).

There is no CPU fallback: if the library is missing or the process has no
CUDA device, every compute entry point raises. ctypes drops the GIL around
each foreign call, so teacher and student threads launch concurrently.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# EDL_LIB points at another build of the same library (same-box A/B runs of
# two kernel versions, scripts/ab_lib.sh); the default is the in-tree build.
LIB_PATH = os.environ.get("EDL_LIB") or os.path.join(_HERE, "libedl_b200.so")

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None

c_int, c_ll, c_float, c_void_p, c_char_p = (ctypes.c_int, ctypes.c_longlong, ctypes.c_float,
                                            ctypes.c_void_p, ctypes.c_char_p)
c_uint = ctypes.c_uint

# name -> argtypes (all return int unless listed in _RESTYPES)
_SIGNATURES = {
    "edl_version": [],
    "edl_last_error": [],
    "edl_device_sms": [],
    "edl_set_stream_max_ctas": [c_void_p, c_int],
    "edl_set_tanh_mode": [c_int],
    "edl_linear_fwd": [c_void_p, c_ll, c_void_p, c_ll, c_void_p, c_void_p, c_ll, c_int, c_int,
                       c_int, c_int, c_void_p],
    "edl_linear_fwd_residual": [c_void_p, c_ll, c_void_p, c_ll, c_void_p, c_void_p, c_ll, c_void_p, c_ll, c_int,
                                c_int, c_int, c_void_p],
    "edl_conv_fwd_nhwc": [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_ll, c_void_p, c_int, c_int, c_int, c_int,
                          c_int, c_void_p, c_ll, c_void_p, c_ll, c_int, c_void_p],
    "edl_conv_bwd_weight_nhwc": [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_ll,
                                 c_int, c_void_p, c_ll, c_void_p, c_void_p, c_ll, c_float, c_void_p],
    "edl_conv_flip_weights": [c_void_p, c_ll, c_int, c_int, c_int, c_int, c_void_p, c_ll, c_void_p],
    "edl_conv_dgrad_nhwc": [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_ll, c_int, c_int, c_int, c_int,
                            c_void_p, c_void_p, c_void_p, c_void_p],
    "edl_im2col_nhwc": [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_ll,
                        c_void_p],
    "edl_maxpool_nhwc": [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p],
    "edl_avgpool_nhwc": [c_void_p, c_int, c_int, c_int, c_void_p, c_ll, c_void_p],
    "edl_col2im_nhwc": [c_void_p, c_ll, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                        c_void_p, c_void_p],
    "edl_avgpool_bwd_nhwc": [c_void_p, c_ll, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p],
    "edl_maxpool_bwd_nhwc": [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p,
                             c_void_p],
    "edl_maxpool_argmax_nhwc": [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                                c_void_p],
    "edl_maxpool_argmax_relu_nhwc": [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                                     c_void_p],
    "edl_maxpool_bwd_argmax_nhwc": [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                                    c_void_p, c_void_p],
    "edl_linear_bwd_data": [c_void_p, c_ll, c_void_p, c_ll, c_void_p, c_ll, c_void_p, c_ll,
                            c_int, c_int, c_int, c_void_p],
    "edl_linear_bwd_weight": [c_void_p, c_ll, c_void_p, c_ll, c_void_p, c_ll, c_void_p,
                              c_void_p, c_int, c_int, c_int, c_float, c_void_p],
    "edl_linear_bwd_weight_grouped": [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_float, c_void_p],
    "edl_linear_bwd_weight_grouped_sgd": [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                          c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                          c_float, c_void_p],
    "edl_linear_bwd_weight_ws": [c_void_p, c_ll, c_void_p, c_ll, c_void_p, c_ll, c_void_p, c_void_p, c_ll, c_int,
                                 c_int, c_int, c_float, c_void_p],
    "edl_bwd_weight_workspace_floats": [c_int, c_int, c_int],
    "edl_colsum_workspace_floats": [c_int, c_int],
    "edl_colsum_group_workspace_floats": [c_int, c_void_p, c_void_p],
    "edl_teacher_head_softmax_topk": [c_void_p, c_ll, c_void_p, c_ll, c_void_p, c_int, c_int,
                                      c_int, c_float, c_int, c_void_p, c_void_p, c_void_p],
    "edl_teacher_head_workspace_bytes": [c_int, c_int, c_int],
    "edl_teacher_head_softmax_topk_ws": [c_void_p, c_ll, c_void_p, c_ll, c_void_p, c_int, c_int, c_int, c_float,
                                         c_int, c_void_p, c_void_p, c_void_p, c_ll, c_void_p],
    "edl_tempered_softmax": [c_void_p, c_ll, c_void_p, c_ll, c_int, c_int, c_float, c_void_p],
    "edl_kd_loss_fwd_bwd": [c_void_p, c_ll, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int,
                            c_float, c_float, c_float, c_void_p, c_void_p, c_void_p, c_void_p,
                            c_ll, c_void_p, c_void_p],
    "edl_linear_kd_loss_fwd_bwd": [c_void_p, c_ll, c_void_p, c_ll, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                                   c_int, c_int, c_int, c_float, c_float, c_float, c_void_p, c_void_p, c_void_p,
                                   c_ll, c_void_p, c_void_p],
    "edl_sgd_step": [c_void_p, c_void_p, c_void_p, c_ll, c_float, c_void_p],
    "edl_stream_wait_geq": [c_void_p, c_uint, c_void_p],
    "edl_stream_write_u32": [c_void_p, c_uint, c_void_p],
    "edl_nvls_allreduce_sgd": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_ll, c_void_p, c_int, c_int,
                               c_ll, c_float, c_uint, c_void_p],
    "edl_gather_rows": [c_void_p, c_ll, c_void_p, c_void_p, c_ll, c_int, c_int, c_void_p, c_void_p,
                        c_void_p],
    "edl_topk_hits": [c_void_p, c_ll, c_void_p, c_int, c_int, c_int, c_void_p, c_void_p],
    "edl_cast_bf16": [c_void_p, c_ll, c_void_p, c_ll, c_int, c_int, c_void_p],
    "edl_cast_bf16_f64": [c_void_p, c_ll, c_void_p, c_ll, c_int, c_int, c_void_p],
    "edl_stream_delay_ns": [c_ll, c_void_p],
    "edl_bn_relu_maxpool_argmax_nhwc": [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p],
    "edl_conv_flip_weights_many": [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p],
    "edl_halo_probe": [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_int, c_int, c_int,
                       c_void_p, c_void_p],
    "edl_bn_workspace_floats": [c_int, c_int],
    "edl_bn_stats_nhwc": [c_void_p, c_int, c_int, c_void_p, c_ll, c_void_p, c_void_p, c_float, c_void_p],
    "edl_bn_apply_nhwc": [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p,
                          c_void_p],
    "edl_bn_bwd_nhwc": [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_ll, c_void_p,
                        c_void_p, c_void_p, c_void_p],
    "edl_memcpy_peer_async": [c_void_p, c_int, c_void_p, c_int, c_ll, c_void_p],
    "edl_memcpy_async": [c_void_p, c_void_p, c_ll, c_void_p],
    "edl_host_register": [c_void_p, c_ll, c_void_p],
    "edl_host_unregister": [c_void_p],
    "edl_ipc_export": [c_void_p, c_void_p, c_void_p],
    "edl_ipc_open": [c_void_p, c_void_p],
    "edl_ipc_close": [c_void_p],
}
_RESTYPES = {"edl_last_error": c_char_p, "edl_colsum_workspace_floats": c_ll,
             "edl_teacher_head_workspace_bytes": c_ll, "edl_bn_workspace_floats": c_ll,
             "edl_bwd_weight_workspace_floats": c_ll,
             "edl_colsum_group_workspace_floats": c_ll}

EDL_ERR_SHAPE, EDL_ERR_NUMERIC, EDL_ERR_PARAM, EDL_ERR_CUDA = -1, -2, -3, -4
EDL_ACT_NONE, EDL_ACT_TANH, EDL_ACT_RELU, EDL_ACT_IDENT = 0, 1, 2, 3
ABI_VERSION = 2


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def load() -> ctypes.CDLL:
    """Load and type the shared library (no GPU needed for loading)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2207_06667_b200.build` "
                "(the B200 path has no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is None and os.environ.get("EDL_LIB"):
                continue      # an older build under A/B (scripts/ab_lib.sh): entry points it predates
            if fn is None:
                raise RuntimeError(f"{LIB_PATH} lacks {name}; rebuild")
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, c_int)
        if lib.edl_version() != ABI_VERSION:
            raise RuntimeError("libedl_b200.so ABI version mismatch; rebuild")
        _lib = lib
        return lib


def last_error() -> str:
    return load().edl_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    """Map C status codes onto the reference's exception classes."""
    if rc == 0:
        return
    from .nnkit import NumericError, ShapeError
    msg = f"{what}: {last_error()}"
    if rc == EDL_ERR_SHAPE:
        raise ShapeError(msg)
    if rc == EDL_ERR_NUMERIC:
        raise NumericError(msg)
    if rc == EDL_ERR_PARAM:
        raise ValueError(msg)
    raise RuntimeError(msg)


# kernel launches per C entry point (bench.py reports launches in its timed region)
_LAUNCHES = {"edl_linear_bwd_weight": 3,   # GEMM + two column-sum passes when db is requested
             "edl_linear_bwd_weight_ws": 4,   # split-K GEMM + reduce + two column-sum passes (at most)
             "edl_conv_bwd_weight_nhwc": 4,   # the same plan with an im2col operand
             "edl_kd_loss_fwd_bwd": 2,     # row pass + deterministic batch-mean pass
             "edl_bn_stats_nhwc": 1, "edl_bn_bwd_nhwc": 2,
             "edl_linear_kd_loss_fwd_bwd": 2,   # fused logit GEMM + loss/dz, batch-mean pass
             "edl_stream_wait_geq": 0,     # stream memory ops, not kernels
             "edl_stream_write_u32": 0,
             "edl_set_tanh_mode": 0,
             "edl_memcpy_peer_async": 0,
             "edl_memcpy_async": 0,
             "edl_host_register": 0,
             "edl_host_unregister": 0,
             "edl_ipc_export": 0,
             "edl_ipc_open": 0,
             "edl_ipc_close": 0}
launch_count = 0


def call(name: str, *args) -> None:
    global launch_count
    check(getattr(load(), name)(*args), name)
    launch_count += _LAUNCHES.get(name, 1)


def bwd_weight_grouped(dys, xs, dws, dbs, workspace, Ms, Ns, Ks, scale, stream) -> None:
    """edl_linear_bwd_weight_grouped with Python lists of tensors / sizes."""
    global launch_count
    n = len(dys)
    P = c_void_p * n
    L = c_ll * n
    I = c_int * n
    args = (n, P(*[t.data_ptr() for t in dys]), L(*[t.stride(0) for t in dys]),
            P(*[t.data_ptr() for t in xs]), L(*[t.stride(0) for t in xs]),
            P(*[t.data_ptr() for t in dws]), L(*Ks), P(*[t.data_ptr() for t in dbs]),
            workspace.data_ptr(), I(*Ms), I(*Ns), I(*Ks), scale, stream)
    check(load().edl_linear_bwd_weight_grouped(*args), "edl_linear_bwd_weight_grouped")
    launch_count += 3   # grouped GEMM + one column-sum launch pair for all layers


def bwd_weight_grouped_sgd(dys, xs, ws32, ws16, bs32, bs16, workspace, Ms, Ns, Ks, eta, stream) -> None:
    """edl_linear_bwd_weight_grouped_sgd: fused dW/db + SGD on fp32 masters."""
    global launch_count
    n = len(dys)
    P = c_void_p * n
    L = c_ll * n
    I = c_int * n
    args = (n, P(*[t.data_ptr() for t in dys]), L(*[t.stride(0) for t in dys]),
            P(*[t.data_ptr() for t in xs]), L(*[t.stride(0) for t in xs]),
            P(*[t.data_ptr() for t in ws32]), P(*[t.data_ptr() for t in ws16]), L(*Ks),
            P(*[t.data_ptr() for t in bs32]), P(*[t.data_ptr() for t in bs16]),
            workspace.data_ptr(), I(*Ms), I(*Ns), I(*Ks), eta, stream)
    check(load().edl_linear_bwd_weight_grouped_sgd(*args), "edl_linear_bwd_weight_grouped_sgd")
    launch_count += 3


def colsum_group_workspace_floats(Ms, Ns) -> int:
    n = len(Ms)
    return int(load().edl_colsum_group_workspace_floats(n, (c_int * n)(*Ms), (c_int * n)(*Ns)))
