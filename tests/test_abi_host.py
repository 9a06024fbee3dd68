"""C-ABI contract checks that need no GPU: the library loads, exports every symbol the header
declares, and its host-side validation rejects bad calls (before any launch) with the
documented status codes (SURVEY 8(b) error classes)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "caffe_b200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1408_5093_b200 import build, _abi
    build.build()
    return _abi.load()


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(caffe_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_and_library_exports_every_entry_point(lib):
    from paper_1408_5093_b200 import _abi
    names = _declared()
    assert len(names) >= 23
    for n in names:
        assert hasattr(lib, n), f"{n} declared in caffe_b200.h but not exported"
    assert set(names) == set(_abi.SIGNATURES), "ctypes signatures out of sync with the header"
    assert lib.caffe_abi_version() == 3
    src = open(HEADER).read()
    assert "#define CAFFE_ABI_VERSION 3" in src


def test_library_has_no_torch_or_python_dependency():
    import subprocess
    out = subprocess.run(["ldd", os.path.join(ROOT, "paper_1408_5093_b200", "libcaffe_b200.so")],
                         capture_output=True, text=True).stdout
    assert "torch" not in out and "python" not in out


def test_sass_contains_tcgen05_and_tma():
    """The tensor-core path really is tcgen05 + TMA (UTC*MMA / UTMALDG in SASS), not mma.sync."""
    import subprocess
    so = os.path.join(ROOT, "paper_1408_5093_b200", "libcaffe_b200.so")
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass
    assert "UTMALDG" in sass
    assert "LDTM" in sass
    assert " HMMA" not in sass


def _st(lib, name, *args):
    return getattr(lib, name)(*args)


def test_conv_shape_and_param_errors(lib):
    from paper_1408_5093_b200 import _abi as A
    d = A.ConvDesc(11, 11, 4, 4, 0, 0, 1, A.CAFFE_MATH_BF16, 0)
    out = A.Shape4()
    assert _st(lib, "caffe_conv_output_shape", ctypes.byref(d), A.Shape4(256, 3, 227, 227), 96, ctypes.byref(out)) == 0
    assert (out.n, out.c, out.h, out.w) == (256, 96, 55, 55)
    d2 = A.ConvDesc(5, 5, 1, 1, 2, 2, 2, A.CAFFE_MATH_BF16, 0)
    assert _st(lib, "caffe_conv_output_shape", ctypes.byref(d2), A.Shape4(256, 96, 27, 27), 256, ctypes.byref(out)) == 0
    assert (out.h, out.w) == (27, 27)
    # kernel larger than the padded input
    d3 = A.ConvDesc(7, 7, 1, 1, 0, 0, 1, A.CAFFE_MATH_BF16, 0)
    assert _st(lib, "caffe_conv_output_shape", ctypes.byref(d3), A.Shape4(1, 1, 5, 5), 1, ctypes.byref(out)) == A.CAFFE_E_PARAM
    assert b"larger than padded input" in lib.caffe_last_error()
    # C % group
    assert _st(lib, "caffe_conv_output_shape", ctypes.byref(d2), A.Shape4(1, 95, 27, 27), 256, ctypes.byref(out)) == A.CAFFE_E_PARAM
    # NULL desc / NULL out
    assert _st(lib, "caffe_conv_output_shape", None, A.Shape4(1, 1, 5, 5), 1, ctypes.byref(out)) == A.CAFFE_E_INVALID
    # bad math enum
    d4 = A.ConvDesc(3, 3, 1, 1, 1, 1, 1, 7, 0)
    assert _st(lib, "caffe_conv_output_shape", ctypes.byref(d4), A.Shape4(1, 1, 5, 5), 1, ctypes.byref(out)) == A.CAFFE_E_INVALID


def test_conv_call_validation_before_launch(lib):
    """Errors are detected on the host; nothing is launched (fake device pointers are never touched)."""
    from paper_1408_5093_b200 import _abi as A
    fake = ctypes.c_void_p(0x10000000)
    d = A.ConvDesc(3, 3, 1, 1, 1, 1, 1, A.CAFFE_MATH_BF16, 0)
    x = A.Blob(fake, A.Shape4(2, 4, 8, 8), A.CAFFE_F32)
    w = A.Blob(ctypes.c_void_p(0x20000000), A.Shape4(6, 4, 3, 3), A.CAFFE_F32)
    y_bad = A.Blob(ctypes.c_void_p(0x30000000), A.Shape4(2, 6, 7, 8), A.CAFFE_F32)
    st = lib.caffe_conv_forward(ctypes.byref(d), ctypes.byref(x), ctypes.byref(w), None, ctypes.byref(y_bad), None, 0, None)
    assert st == A.CAFFE_E_SHAPE
    w_bad = A.Blob(ctypes.c_void_p(0x20000000), A.Shape4(6, 3, 3, 3), A.CAFFE_F32)
    y = A.Blob(ctypes.c_void_p(0x30000000), A.Shape4(2, 6, 8, 8), A.CAFFE_F32)
    assert lib.caffe_conv_forward(ctypes.byref(d), ctypes.byref(x), ctypes.byref(w_bad), None, ctypes.byref(y), None, 0, None) == A.CAFFE_E_SHAPE
    # aliasing output onto the input
    y_alias = A.Blob(fake, A.Shape4(2, 6, 8, 8), A.CAFFE_F32)
    assert lib.caffe_conv_forward(ctypes.byref(d), ctypes.byref(x), ctypes.byref(w), None, ctypes.byref(y_alias), None, 0, None) == A.CAFFE_E_ALIAS
    # missing workspace for the tensor-core path
    assert lib.caffe_conv_forward(ctypes.byref(d), ctypes.byref(x), ctypes.byref(w), None, ctypes.byref(y), None, 0, None) == A.CAFFE_E_WORKSPACE
    # TF32 with BF16 storage
    dt = A.ConvDesc(3, 3, 1, 1, 1, 1, 1, A.CAFFE_MATH_TF32, 0)
    xb = A.Blob(fake, A.Shape4(2, 4, 8, 8), A.CAFFE_BF16)
    assert lib.caffe_conv_forward(ctypes.byref(dt), ctypes.byref(xb), ctypes.byref(w), None, ctypes.byref(y), None, 0, None) == A.CAFFE_E_DTYPE
    # zero non-batch axis
    xz = A.Blob(fake, A.Shape4(2, 4, 0, 8), A.CAFFE_F32)
    assert lib.caffe_conv_forward(ctypes.byref(d), ctypes.byref(xz), ctypes.byref(w), None, ctypes.byref(y), None, 0, None) == A.CAFFE_E_SHAPE
    # n == 0 is a no-op
    x0 = A.Blob(None, A.Shape4(0, 4, 8, 8), A.CAFFE_F32)
    y0 = A.Blob(None, A.Shape4(0, 6, 8, 8), A.CAFFE_F32)
    assert lib.caffe_conv_forward(ctypes.byref(d), ctypes.byref(x0), ctypes.byref(w), None, ctypes.byref(y0), None, 0, None) == 0
    # workspace size query
    n = ctypes.c_size_t()
    assert lib.caffe_conv_workspace_size(ctypes.byref(d), A.Shape4(2, 4, 8, 8), A.Shape4(6, 4, 3, 3), 0, ctypes.byref(n)) == 0
    assert n.value > 0
    d32 = A.ConvDesc(3, 3, 1, 1, 1, 1, 1, A.CAFFE_MATH_FP32, 0)
    assert lib.caffe_conv_workspace_size(ctypes.byref(d32), A.Shape4(2, 4, 8, 8), A.Shape4(6, 4, 3, 3), 0, ctypes.byref(n)) == 0
    assert n.value == 0


def test_pool_lrn_relu_validation(lib):
    from paper_1408_5093_b200 import _abi as A
    out = A.Shape4()
    p = A.PoolDesc(A.CAFFE_POOL_MAX, 3, 3, 2, 2, 0, 0)
    assert lib.caffe_pool_output_shape(ctypes.byref(p), A.Shape4(256, 96, 55, 55), ctypes.byref(out)) == 0
    assert (out.h, out.w) == (27, 27)
    p0 = A.PoolDesc(A.CAFFE_POOL_MAX, 0, 3, 2, 2, 0, 0)
    assert lib.caffe_pool_output_shape(ctypes.byref(p0), A.Shape4(1, 1, 5, 5), ctypes.byref(out)) == A.CAFFE_E_PARAM
    # R5 edge: H=4, k=1, s=2 -> 2
    p1 = A.PoolDesc(A.CAFFE_POOL_MAX, 1, 1, 2, 2, 0, 0)
    assert lib.caffe_pool_output_shape(ctypes.byref(p1), A.Shape4(1, 1, 4, 4), ctypes.byref(out)) == 0 and out.h == 2
    # MAX backward without mask
    dy = A.Blob(ctypes.c_void_p(0x1000), A.Shape4(1, 1, 2, 2), A.CAFFE_F32)
    dx = A.Blob(ctypes.c_void_p(0x9000), A.Shape4(1, 1, 5, 5), A.CAFFE_F32)
    assert lib.caffe_pool_backward(ctypes.byref(p), ctypes.byref(dy), None, ctypes.byref(dx), None) == A.CAFFE_E_INVALID
    # even LRN size
    l = A.LrnDesc(4, 1e-4, 0.75, 1.0)
    x = A.Blob(ctypes.c_void_p(0x1000), A.Shape4(1, 5, 2, 2), A.CAFFE_F32)
    y = A.Blob(ctypes.c_void_p(0x9000), A.Shape4(1, 5, 2, 2), A.CAFFE_F32)
    assert lib.caffe_lrn_forward(ctypes.byref(l), ctypes.byref(x), ctypes.byref(y), None, None) == A.CAFFE_E_PARAM
    # ReLU: partial overlap is an alias error, exact in-place is allowed (validated, then launched -> not on CPU)
    y_part = A.Blob(ctypes.c_void_p(0x1000 + 8), A.Shape4(1, 5, 2, 2), A.CAFFE_F32)
    assert lib.caffe_relu_forward(ctypes.byref(x), ctypes.byref(y_part), None) == A.CAFFE_E_ALIAS


def test_ip_validation(lib):
    from paper_1408_5093_b200 import _abi as A
    x = A.Blob(ctypes.c_void_p(0x1000), A.Shape4(4, 3, 2, 2), A.CAFFE_F32)
    w = A.Blob(ctypes.c_void_p(0x9000), A.Shape4(5, 11, 1, 1), A.CAFFE_F32)   # fan-in 11 != 12
    y = A.Blob(ctypes.c_void_p(0x19000), A.Shape4(4, 5, 1, 1), A.CAFFE_F32)
    assert lib.caffe_ip_forward(A.CAFFE_MATH_BF16, 0, ctypes.byref(x), ctypes.byref(w), None, ctypes.byref(y), None, 0, None) == A.CAFFE_E_SHAPE
    assert b"fan-in" in lib.caffe_last_error()


def test_catalogue_and_solver_validation(lib):
    """NEXT-3 / NEXT-4 entry points: host-side errors before any launch (fake device pointers are
    never touched), the documented classes; the host LR schedule."""
    from paper_1408_5093_b200 import _abi as A
    f = lambda a: ctypes.c_void_p(a)  # noqa: E731
    x = A.Blob(f(0x10000), A.Shape4(2, 4, 3, 3), A.CAFFE_F32)
    y_shape = A.Blob(f(0x20000), A.Shape4(2, 4, 3, 4), A.CAFFE_F32)
    assert lib.caffe_sigmoid_forward(ctypes.byref(x), ctypes.byref(y_shape), None) == A.CAFFE_E_SHAPE
    y_dtype = A.Blob(f(0x20000), A.Shape4(2, 4, 3, 3), A.CAFFE_BF16)
    assert lib.caffe_sigmoid_forward(ctypes.byref(x), ctypes.byref(y_dtype), None) == A.CAFFE_E_SHAPE
    y_part = A.Blob(f(0x10000 + 16), A.Shape4(2, 4, 3, 3), A.CAFFE_F32)
    assert lib.caffe_sigmoid_forward(ctypes.byref(x), ctypes.byref(y_part), None) == A.CAFFE_E_ALIAS
    y_mis = A.Blob(f(0x20004), A.Shape4(2, 4, 3, 3), A.CAFFE_F32)
    assert lib.caffe_sigmoid_forward(ctypes.byref(x), ctypes.byref(y_mis), None) == A.CAFFE_E_ALIGN
    # eltwise: input count, op enum, coefficients only for SUM, shapes, aliasing
    ins = (A.Blob * 3)(x, A.Blob(f(0x30000), A.Shape4(2, 4, 3, 3), A.CAFFE_F32),
                       A.Blob(f(0x40000), A.Shape4(2, 4, 3, 4), A.CAFFE_F32))
    ptrs = (ctypes.POINTER(A.Blob) * 3)(*[ctypes.pointer(ins[i]) for i in range(3)])
    top = A.Blob(f(0x50000), A.Shape4(2, 4, 3, 3), A.CAFFE_F32)
    assert lib.caffe_eltwise_forward(A.CAFFE_ELTWISE_SUM, 1, ptrs, None, ctypes.byref(top), None) == A.CAFFE_E_PARAM
    assert lib.caffe_eltwise_forward(A.CAFFE_ELTWISE_SUM, 9, ptrs, None, ctypes.byref(top), None) == A.CAFFE_E_PARAM
    assert lib.caffe_eltwise_forward(7, 2, ptrs, None, ctypes.byref(top), None) == A.CAFFE_E_INVALID
    coef = (ctypes.c_float * 2)(1.0, 2.0)
    assert lib.caffe_eltwise_forward(A.CAFFE_ELTWISE_MAX, 2, ptrs, coef, ctypes.byref(top), None) == A.CAFFE_E_PARAM
    assert lib.caffe_eltwise_forward(A.CAFFE_ELTWISE_MAX, 3, ptrs, None, ctypes.byref(top), None) == A.CAFFE_E_SHAPE
    diffs = (A.Blob * 2)(A.Blob(f(0x60000), A.Shape4(2, 4, 3, 3), A.CAFFE_F32), A.Blob(f(0x60000), A.Shape4(2, 4, 3, 3), A.CAFFE_F32))
    dptr = (ctypes.POINTER(A.Blob) * 2)(*[ctypes.pointer(diffs[i]) for i in range(2)])
    assert lib.caffe_eltwise_backward(A.CAFFE_ELTWISE_PROD, 2, ptrs, None, ctypes.byref(top), dptr, None) == A.CAFFE_E_ALIAS
    # hinge: NULL labels
    sc = A.Blob(f(0x70000), A.Shape4(4, 10, 1, 1), A.CAFFE_F32)
    assert lib.caffe_hinge_loss(ctypes.byref(sc), None, f(0x80000), None, None) == A.CAFFE_E_INVALID
    # LR schedules on the host and their errors
    lr = ctypes.c_float()
    pol = A.LrPolicy(A.CAFFE_LR_STEP, 0.01, 0.1, 0.0, 100)
    assert lib.caffe_lr_at_iter(ctypes.byref(pol), 250, ctypes.byref(lr)) == 0
    assert abs(lr.value - 1e-4) <= 1e-10
    pol0 = A.LrPolicy(A.CAFFE_LR_STEP, 0.01, 0.1, 0.0, 0)
    assert lib.caffe_lr_at_iter(ctypes.byref(pol0), 1, ctypes.byref(lr)) == A.CAFFE_E_PARAM
    assert lib.caffe_lr_at_iter(ctypes.byref(pol), -1, ctypes.byref(lr)) == A.CAFFE_E_PARAM
    bad = A.LrPolicy(9, 0.01, 0.1, 0.0, 1)
    assert lib.caffe_lr_at_iter(ctypes.byref(bad), 1, ctypes.byref(lr)) == A.CAFFE_E_INVALID
    assert lib.caffe_solver_begin(ctypes.byref(pol), f(0x90004), None, None) == A.CAFFE_E_ALIGN
    assert lib.caffe_sgd_update_solver(f(0x1000), f(0x2000), f(0x3000), None, 16, None, 0.9, 0.0, 1.0, None) == A.CAFFE_E_INVALID
    # fused pool + LRN: U8 mask and BF16 channels-last are required
    p = A.PoolDesc(A.CAFFE_POOL_MAX, 3, 3, 2, 2, 0, 0)
    l5 = A.LrnDesc(5, 1e-4, 0.75, 1.0)
    xb = A.Blob(f(0x100000), A.Shape4(2, 16, 13, 13), A.CAFFE_BF16, A.CAFFE_NHWC)
    pb = A.Blob(f(0x200000), A.Shape4(2, 16, 6, 6), A.CAFFE_BF16, A.CAFFE_NHWC)
    m32 = A.Blob(f(0x300000), A.Shape4(2, 16, 6, 6), A.CAFFE_I32, A.CAFFE_NHWC)
    yb = A.Blob(f(0x400000), A.Shape4(2, 16, 6, 6), A.CAFFE_BF16, A.CAFFE_NHWC)
    assert lib.caffe_pool_lrn_forward(ctypes.byref(p), ctypes.byref(l5), ctypes.byref(xb), ctypes.byref(pb),
                                      ctypes.byref(m32), ctypes.byref(yb), None) == A.CAFFE_E_DTYPE
    l4 = A.LrnDesc(4, 1e-4, 0.75, 1.0)
    m8 = A.Blob(f(0x300000), A.Shape4(2, 16, 6, 6), A.CAFFE_U8, A.CAFFE_NHWC)
    assert lib.caffe_pool_lrn_forward(ctypes.byref(p), ctypes.byref(l4), ctypes.byref(xb), ctypes.byref(pb),
                                      ctypes.byref(m8), ctypes.byref(yb), None) == A.CAFFE_E_PARAM


def test_tuning_knob_ranges(lib):
    """caffe_set_tuning validates every ranged knob on the host (no device needed) and accepts the
    documented values; knobs are restored to their defaults."""
    from paper_1408_5093_b200 import _abi as A
    bad = [(A.CAFFE_TUNE_HALO_EPI_GROUPS, 1), (A.CAFFE_TUNE_HALO_EPI_GROUPS, 5), (A.CAFFE_TUNE_HALO_BTAPS, 9),
           (A.CAFFE_TUNE_MAX_CTAS, -1), (A.CAFFE_TUNE_SGD_THREADS, 96), (A.CAFFE_TUNE_SGD_BLOCKS_PER_SM, 9),
           (A.CAFFE_TUNE_CTA_PAIR, 3), (A.CAFFE_TUNE_FUSED_POOL_ROWS, 65), (A.CAFFE_TUNE_WGRAD_BN, 17),
           (A.CAFFE_TUNE_WGRAD_BN, 272), (A.CAFFE_TUNE_WGRAD_BN, -16)]
    for key, value in bad:
        assert lib.caffe_set_tuning(key, value) == A.CAFFE_E_PARAM, (key, value)
    for key, value in [(A.CAFFE_TUNE_HALO_EPI_GROUPS, 2), (A.CAFFE_TUNE_HALO_EPI_GROUPS, 3),
                       (A.CAFFE_TUNE_HALO_BTAPS, 5), (A.CAFFE_TUNE_MAX_CTAS, 16), (A.CAFFE_TUNE_WGRAD_BN, 1),
                       (A.CAFFE_TUNE_WGRAD_BN, 192), (A.CAFFE_TUNE_HALO_JN, 0), (A.CAFFE_TUNE_HALO_MERGE, 1)]:
        assert lib.caffe_set_tuning(key, value) == 0, (key, value)
    for key in (A.CAFFE_TUNE_HALO_EPI_GROUPS, A.CAFFE_TUNE_HALO_BTAPS, A.CAFFE_TUNE_MAX_CTAS, A.CAFFE_TUNE_WGRAD_BN,
                A.CAFFE_TUNE_HALO_MERGE):
        assert lib.caffe_set_tuning(key, 0) == 0
    assert lib.caffe_set_tuning(A.CAFFE_TUNE_HALO_JN, 1) == 0   # defaults restored
