"""ctypes declarations of include/caffe_b200.h (argument marshalling only).

Loading fails loudly if libcaffe_b200.so is missing: there is no fallback path.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CAFFE_B200_LIB: load another in-tree build of the same library (A/B experiments of compile options)
LIB_PATH = os.environ.get("CAFFE_B200_LIB") or os.path.join(HERE, "libcaffe_b200.so")

# enums (include/caffe_b200.h)
CAFFE_OK, CAFFE_E_INVALID, CAFFE_E_SHAPE, CAFFE_E_PARAM, CAFFE_E_DTYPE = 0, 1, 2, 3, 4
CAFFE_E_ALIGN, CAFFE_E_WORKSPACE, CAFFE_E_ALIAS, CAFFE_E_CUDA, CAFFE_E_ARCH = 5, 6, 7, 8, 9
STATUS_NAMES = {0: "OK", 1: "E_INVALID", 2: "E_SHAPE", 3: "E_PARAM", 4: "E_DTYPE", 5: "E_ALIGN",
                6: "E_WORKSPACE", 7: "E_ALIAS", 8: "E_CUDA", 9: "E_ARCH"}
CAFFE_F32, CAFFE_BF16, CAFFE_I32, CAFFE_U8, CAFFE_I8 = 0, 1, 2, 3, 4
CAFFE_NCHW, CAFFE_NHWC = 0, 1
CAFFE_MATH_FP32, CAFFE_MATH_TF32, CAFFE_MATH_BF16 = 0, 1, 2
CAFFE_FUSE_RELU = 1
CAFFE_BOTTOM_PREPACKED = 2
CAFFE_WEIGHTS_PREPACKED = 4
CAFFE_POOL_MAX, CAFFE_POOL_AVE = 0, 1
CAFFE_PASS_FORWARD, CAFFE_PASS_BACKWARD_DATA, CAFFE_PASS_BACKWARD_WEIGHT = 0, 1, 2
CAFFE_TUNE_CTA_PAIR = 1
CAFFE_TUNE_MMA_SPIN = 2
CAFFE_TUNE_WGRAD_MACC = 3
CAFFE_TUNE_HALO = 4
CAFFE_TUNE_TMA_STORE = 5
CAFFE_TUNE_ROWS_EPILOGUE = 6
CAFFE_TUNE_SGD_BLOCKS_PER_SM = 7
CAFFE_TUNE_POOL_STRIP_ROWS = 8
CAFFE_TUNE_WGRAD_REDUCE_SG = 9
CAFFE_TUNE_HALO_KTRIM = 10
CAFFE_TUNE_HALO_FAST_EPI = 11
CAFFE_TUNE_HALO_TMA_STORE = 12
CAFFE_TUNE_WGRAD_REDUCE_ROWS = 13
CAFFE_TUNE_HALO_STACKED = 14
CAFFE_TUNE_SGD_THREADS = 15
CAFFE_TUNE_MAX_CTAS = 16
CAFFE_TUNE_FUSED_POOL_ROWS = 17
CAFFE_TUNE_HALO_COALESCE = 18
CAFFE_TUNE_WGRAD_REDUCE_WIDE = 19
CAFFE_TUNE_HALO_BTAPS = 20
CAFFE_TUNE_HALO_EPI_GROUPS = 21
CAFFE_TUNE_HALO_JN = 22
CAFFE_TUNE_WGRAD_BN = 23
CAFFE_TUNE_HALO_MERGE = 24
CAFFE_TUNE_IP_MAX_SPLITS = 25
CAFFE_TUNE_I8_ROWS = 26
CAFFE_TUNE_ROWS_CB = 27
CAFFE_TUNE_BIAS_ROWS = 28
CAFFE_TUNE_BIAS_SPLIT_ROWS = 29
CAFFE_TUNE_PDL = 30
CAFFE_TUNE_IP_FWD_SMALL_BN = 31
CAFFE_TUNE_POOL_LRN_C16 = 32
CAFFE_TUNE_LRN_BWD_C16 = 33
CAFFE_ELTWISE_PROD, CAFFE_ELTWISE_SUM, CAFFE_ELTWISE_MAX = 0, 1, 2
CAFFE_ELTWISE_MAX_INPUTS = 8
CAFFE_LR_FIXED, CAFFE_LR_STEP, CAFFE_LR_INV = 0, 1, 2


class Shape4(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("c", ctypes.c_int32), ("h", ctypes.c_int32), ("w", ctypes.c_int32)]


class Blob(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("shape", Shape4), ("dtype", ctypes.c_int), ("layout", ctypes.c_int32)]


class ConvDesc(ctypes.Structure):
    _fields_ = [("kernel_h", ctypes.c_int32), ("kernel_w", ctypes.c_int32), ("stride_h", ctypes.c_int32),
                ("stride_w", ctypes.c_int32), ("pad_h", ctypes.c_int32), ("pad_w", ctypes.c_int32),
                ("group", ctypes.c_int32), ("math", ctypes.c_int), ("flags", ctypes.c_uint32)]


class PoolDesc(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int32), ("kernel_h", ctypes.c_int32), ("kernel_w", ctypes.c_int32),
                ("stride_h", ctypes.c_int32), ("stride_w", ctypes.c_int32), ("pad_h", ctypes.c_int32),
                ("pad_w", ctypes.c_int32)]


class LrnDesc(ctypes.Structure):
    _fields_ = [("local_size", ctypes.c_int32), ("alpha", ctypes.c_float), ("beta", ctypes.c_float),
                ("k", ctypes.c_float)]


class LrPolicy(ctypes.Structure):
    _fields_ = [("policy", ctypes.c_int32), ("base_lr", ctypes.c_float), ("gamma", ctypes.c_float),
                ("power", ctypes.c_float), ("stepsize", ctypes.c_int32)]


class SolverState(ctypes.Structure):
    """Layout of caffe_solver_state (it lives in device memory; this mirrors it for size/offsets)."""
    _fields_ = [("iter", ctypes.c_int64), ("diverged_iter", ctypes.c_int64), ("lr", ctypes.c_float),
                ("last_loss", ctypes.c_float), ("diverged", ctypes.c_int32), ("reserved", ctypes.c_int32)]


P = ctypes.POINTER
vp, i32, f32, sz, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_float, ctypes.c_size_t, ctypes.c_int64, ctypes.c_uint32
B, CD, PD, LD = P(Blob), P(ConvDesc), P(PoolDesc), P(LrnDesc)

# name -> argtypes (every function returns caffe_status unless listed in _RESTYPES)
SIGNATURES = {
    "caffe_abi_version": [],
    "caffe_last_error": [],
    "caffe_device_check": [],
    "caffe_set_tuning": [i32, i32],
    "caffe_launch_count": [],
    "caffe_profiler_enable": [i32],
    "caffe_profiler_read": [i32, P(ctypes.c_double), P(ctypes.c_double), P(i64)],
    "caffe_conv_output_shape": [CD, Shape4, i32, P(Shape4)],
    "caffe_conv_workspace_size": [CD, Shape4, Shape4, i32, P(sz)],
    "caffe_conv_forward": [CD, B, B, B, B, vp, sz, vp],
    "caffe_conv_pack_bottom": [CD, B, B, vp, sz, vp],
    "caffe_conv_pack_weights": [CD, Shape4, B, i32, vp, sz, vp],
    "caffe_conv_backward_data": [CD, B, B, B, f32, vp, sz, vp],
    "caffe_conv_backward_data_relu": [CD, B, B, B, B, vp, sz, vp],
    "caffe_conv_backward_weight": [CD, B, B, B, B, f32, vp, sz, vp],
    "caffe_relu_forward": [B, B, vp],
    "caffe_relu_backward": [B, B, B, vp],
    "caffe_pool_output_shape": [PD, Shape4, P(Shape4)],
    "caffe_pool_forward": [PD, B, B, B, vp],
    "caffe_pool_backward": [PD, B, B, B, vp],
    "caffe_pool_relu_backward": [PD, B, B, B, B, vp],
    "caffe_lrn_forward": [LD, B, B, B, vp],
    "caffe_lrn_backward": [LD, B, B, B, B, B, vp],
    "caffe_ip_workspace_size": [ctypes.c_int, Shape4, i32, i32, P(sz)],
    "caffe_ip_forward": [ctypes.c_int, u32, B, B, B, B, vp, sz, vp],
    "caffe_ip_backward_data": [ctypes.c_int, B, B, B, f32, vp, sz, vp],
    "caffe_ip_backward_data_relu": [ctypes.c_int, B, B, B, B, vp, sz, vp],
    "caffe_ip_backward_weight": [ctypes.c_int, B, B, B, B, f32, vp, sz, vp],
    "caffe_ip_backward_weight_sgd": [B, B, B, B, B, B, f32, f32, f32, f32, vp, sz, vp],
    "caffe_blob_to_nchw": [B, B, vp],
    "caffe_im2col": [CD, B, i32, B, vp],
    "caffe_col2im": [CD, B, i32, B, vp],
    "caffe_softmax_loss": [B, vp, vp, B, vp],
    "caffe_sgd_update": [vp, vp, vp, vp, i64, f32, f32, f32, f32, vp],
    "caffe_pool_lrn_forward": [PD, LD, B, B, B, B, vp],
    "caffe_lrn_pool_backward": [PD, LD, B, B, B, i32, B, vp],
    "caffe_sigmoid_forward": [B, B, vp],
    "caffe_sigmoid_backward": [B, B, B, vp],
    "caffe_eltwise_forward": [i32, i32, P(B), P(f32), B, vp],
    "caffe_eltwise_backward": [i32, i32, P(B), P(f32), B, P(B), vp],
    "caffe_hinge_loss": [B, vp, vp, B, vp],
    "caffe_lr_at_iter": [P(LrPolicy), i64, P(f32)],
    "caffe_solver_begin": [P(LrPolicy), vp, vp, vp],
    "caffe_solver_end": [vp, vp],
    "caffe_sgd_update_solver": [vp, vp, vp, vp, i64, vp, f32, f32, f32, vp],
}
_RESTYPES = {"caffe_abi_version": ctypes.c_int32, "caffe_last_error": ctypes.c_char_p,
             "caffe_launch_count": ctypes.c_int64}

_lib = None


def load() -> ctypes.CDLL:
    """Load libcaffe_b200.so (build it first with `python -m paper_1408_5093_b200.build`)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: the CUDA library must be built "
                              "(python -m paper_1408_5093_b200.build); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
    return _lib


class CaffeError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        super().__init__(f"{fn} -> {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def call(name: str, *args) -> None:
    lib = load()
    st = getattr(lib, name)(*args)
    if st != CAFFE_OK:
        raise CaffeError(st, name, lib.caffe_last_error().decode())
