"""ctypes binding of libsvdq.so (include/svdq.h): argument marshalling only.

Every function here has the name of the C entry point it calls.  Device
buffers are torch CUDA tensors (PyTorch supplies memory and streams only);
all arithmetic runs in the library's kernels.  There is no CPU fallback:
importing this module without the built library raises ImportError, and
every non-OK status raises SvdqError.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SVDQ_LIB") or os.path.join(_HERE, "libsvdq.so")   # SVDQ_LIB: debug builds

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: build the CUDA library first "
        "(python -m paper_2411_05007_b200.build or __graft_entry__.build()); "
        "there is no CPU fallback")
_lib = C.CDLL(LIB_PATH)

# enums (svdq.h)
SVDQ_OK = 0
STATUS_NAMES = {0: "SVDQ_OK", 1: "SVDQ_ERR_INVALID_ARGUMENT", 2: "SVDQ_ERR_SHAPE", 3: "SVDQ_ERR_RANK",
                4: "SVDQ_ERR_ALIGNMENT", 5: "SVDQ_ERR_UNSUPPORTED", 6: "SVDQ_ERR_NONFINITE",
                7: "SVDQ_ERR_CUDA", 8: "SVDQ_ERR_WORKSPACE"}
FMT = {"nvfp4": 0, "int4": 1, "w8a8": 2}
DTYPE = {"bf16": 0, "fp16": 1, "fp32": 2}
TORCH_DTYPE = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}
DTYPE_OF_TORCH = {torch.bfloat16: "bf16", torch.float16: "fp16", torch.float32: "fp32"}

# Every symbol include/svdq.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "svdq_act_buffer_sizes", "svdq_weight_buffer_sizes", "svdq_quantize_act_lowrank_down",
    "svdq_quantize_act_lowrank_down_grouped",
    "svdq_gemm_w4a4_lowrank_up", "svdq_gemm_w4a4_lowrank_up_grouped", "svdq_linear_forward",
    "svdq_gemm_fused_next_workspace", "svdq_gemm_w4a4_lowrank_up_fused_next",
    "svdq_quantize_residual",
    "svdq_quantize_weights_workspace", "svdq_quantize_weights", "svdq_lora_fuse",
    "svdq_search_alpha_workspace", "svdq_search_alpha",
    "svdq_refine_lowrank_workspace", "svdq_refine_lowrank",
    "svdq_quantize_residual_gptq_workspace", "svdq_quantize_residual_gptq",
    "svdq_quantize_weights_gptq_workspace", "svdq_quantize_weights_gptq",
    "svdq_debug_int4_group_accum", "svdq_debug_codec", "svdq_status_string", "svdq_last_error",
    "svdq_launch_count", "svdq_version", "svdq_k1_row_tile",
    "svdq_tp_slice_sizes", "svdq_quantize_act_lowrank_down_kslice", "svdq_tp_assemble_act",
    "svdq_tp_gather_sizes", "svdq_quantize_act_lowrank_down_kslice_fused", "svdq_tp_reduce_partials",
]


class svdq_linear(C.Structure):
    _fields_ = [
        ("fmt", C.c_int32), ("rank", C.c_int32), ("K", C.c_int64), ("N", C.c_int64),
        ("w_codes", C.c_void_p), ("w_scales", C.c_void_p), ("lambda_inv", C.c_void_p),
        ("l1s", C.c_void_p), ("l2s", C.c_void_p), ("bias", C.c_void_p),
        ("scale_dtype", C.c_int32), ("bias_dtype", C.c_int32),
        ("gs_w", C.c_float), ("gs_x", C.c_float),
    ]


class SvdqError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        detail = _lib.svdq_last_error().decode()
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {detail}")


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_SZ = C.POINTER(C.c_size_t)
_LP = C.POINTER(svdq_linear)
_sig = {
    "svdq_act_buffer_sizes": [_I32, _I64, _I64, _I32, _SZ, _SZ, _SZ],
    "svdq_weight_buffer_sizes": [_I32, _I64, _I64, _I32, _SZ, _SZ, _SZ, _SZ],
    "svdq_quantize_act_lowrank_down": [_LP, _P, _I32, _I64, _I64, _P, _P, _P, _P],
    "svdq_gemm_w4a4_lowrank_up": [_LP, _P, _P, _P, _I64, _P, _I32, _I64, _P],
    "svdq_quantize_act_lowrank_down_grouped": [_I32, C.POINTER(_LP), C.POINTER(_P), _I32, C.POINTER(_I64),
                                               C.POINTER(_I64), C.POINTER(_P), C.POINTER(_P), C.POINTER(_P), _P],
    "svdq_gemm_fused_next_workspace": [_I32, C.POINTER(_LP), C.POINTER(_I64), C.POINTER(_LP), _SZ],
    "svdq_gemm_w4a4_lowrank_up_fused_next": [_I32, C.POINTER(_LP), C.POINTER(_P), C.POINTER(_P), C.POINTER(_P),
                                             C.POINTER(_I64), C.POINTER(_P), C.POINTER(_LP), _I32, C.POINTER(_P),
                                             C.POINTER(_P), C.POINTER(_P), _P, C.c_size_t, _P],
    "svdq_gemm_w4a4_lowrank_up_grouped": [_I32, C.POINTER(_LP), C.POINTER(_P), C.POINTER(_P), C.POINTER(_P),
                                          C.POINTER(_I64), C.POINTER(_P), _I32, C.POINTER(_I64), _P],
    "svdq_linear_forward": [_LP, _P, _I32, _I64, _I64, _P, _I32, _I64, _P, C.c_size_t, _P],
    "svdq_quantize_residual": [_P, _I64, _I64, _I32, _I32, _P, _P, C.POINTER(C.c_float), _P],
    "svdq_quantize_weights_workspace": [_I64, _I64, _I32, _SZ],
    "svdq_quantize_weights": [_P, _I32, _P, _I64, _I64, _I32, _I32, _I32, C.c_float, _P, _P, _LP,
                              _P, C.c_size_t, _P],
    "svdq_lora_fuse": [_LP, _P, _P, _I32, _I32, C.c_float, _LP, _P],
    "svdq_search_alpha_workspace": [_I32, _I64, _I64, _I64, _I32, _SZ],
    "svdq_search_alpha": [_P, _I32, _I64, _I64, _P, _I64, _I64, _I32, _I32, _I32, C.c_float, C.POINTER(C.c_float),
                          _I32, C.POINTER(C.c_float), _P, C.POINTER(C.c_double), _P, C.c_size_t, _P],
    "svdq_refine_lowrank_workspace": [_I32, _I64, _I64, _I64, _I32, _I32, _SZ],
    "svdq_refine_lowrank": [_P, _I32, _I64, _I64, _P, _P, _I64, _I64, _I32, _I32, _I32, C.c_float, _I32, _I32,
                            C.c_float, _LP, C.POINTER(C.c_int32), C.POINTER(C.c_double), _P, C.c_size_t, _P],
    "svdq_quantize_residual_gptq_workspace": [_I64, _I64, _I64, _SZ],
    "svdq_quantize_residual_gptq": [_P, _I64, _I64, _I32, _I32, _P, _I32, _I64, _I64, _P, C.c_float, _P, _P,
                                    C.POINTER(C.c_float), _P, C.c_size_t, _P],
    "svdq_quantize_weights_gptq_workspace": [_I64, _I64, _I64, _I32, _SZ],
    "svdq_quantize_weights_gptq": [_P, _I32, _P, _I64, _I64, _I32, _I32, _I32, C.c_float, _P, _I32, _I64, _I64,
                                   C.c_float, _LP, _P, C.c_size_t, _P],
    "svdq_debug_int4_group_accum": [_P, _P, _I64, _I64, _I64, _P, _P],
    "svdq_debug_codec": [_P, _P, _I64, _I32, _P],
    "svdq_tp_slice_sizes": [_I32, _I64, _I64, _I32, _SZ, _SZ, _SZ, _SZ],
    "svdq_quantize_act_lowrank_down_kslice": [_LP, _I64, _I64, _P, _I32, _I64, _I64, _P, _P],
    "svdq_tp_gather_sizes": [_I32, _I64, _I64, _I32, _I32, _SZ, _SZ, _SZ, _SZ],
    "svdq_quantize_act_lowrank_down_kslice_fused": [_LP, _I64, _I64, _P, _I32, _I64, _I64, _I32, _I32, C.POINTER(_P),
                                                    _I32, _P],
    "svdq_tp_reduce_partials": [_I32, _I64, _I32, _P, _P, _P],
    "svdq_tp_assemble_act": [_I32, _I32, _I64, _I64, _I32, _P, C.c_size_t, C.c_size_t, _P, _P, _P, _P],
}
for _name, _args in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = C.c_int
_lib.svdq_status_string.argtypes = [C.c_int]
_lib.svdq_status_string.restype = C.c_char_p
_lib.svdq_last_error.argtypes = []
_lib.svdq_last_error.restype = C.c_char_p
_lib.svdq_launch_count.argtypes = []
_lib.svdq_launch_count.restype = C.c_uint64
_lib.svdq_version.argtypes = []
_lib.svdq_version.restype = C.c_int32
_lib.svdq_k1_row_tile.argtypes = [C.c_int64, C.c_int32]
_lib.svdq_k1_row_tile.restype = C.c_int32


def _check(status: int, where: str):
    if status != SVDQ_OK:
        raise SvdqError(status, where)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def lib():
    return _lib


# ---------------------------------------------------------------- misc
def svdq_status_string(status: int) -> str:
    return _lib.svdq_status_string(status).decode()


def svdq_last_error() -> str:
    return _lib.svdq_last_error().decode()


def svdq_launch_count() -> int:
    return int(_lib.svdq_launch_count())


def svdq_version() -> int:
    return int(_lib.svdq_version())


def svdq_tp_slice_sizes(fmt: str, M: int, Kp: int, rank: int):
    """(xq_off, xs_off, part_off, slice_bytes) of one rank's packed K1 slice (tensor parallel)."""
    o = [C.c_size_t() for _ in range(4)]
    _check(_lib.svdq_tp_slice_sizes(FMT[fmt], M, Kp, rank, *[C.byref(x) for x in o]), "svdq_tp_slice_sizes")
    return tuple(x.value for x in o)


def svdq_quantize_act_lowrank_down_kslice(layer: "QuantizedLinear", k0: int, X, slice_buf=None, stream=None):
    """K1 of `layer` on its input channels [k0, k0 + X.shape[1]) (X: this rank's column shard of the
    layer input).  Returns the packed slice buffer (uint8, svdq_tp_slice_sizes layout)."""
    M, Kp = X.shape
    nb = svdq_tp_slice_sizes(layer.fmt, M, Kp, layer.rank)[3]
    if slice_buf is None:
        slice_buf = torch.empty(nb, dtype=torch.uint8, device=X.device)
    _check(_lib.svdq_quantize_act_lowrank_down_kslice(layer.ref, k0, Kp, _ptr(X), DTYPE[DTYPE_OF_TORCH[X.dtype]], M,
                                                      X.stride(0), _ptr(slice_buf), _stream(stream)),
           "svdq_quantize_act_lowrank_down_kslice")
    return slice_buf


def svdq_tp_gather_sizes(fmt: str, M: int, K: int, rank: int, P: int):
    """(xq_off, xs_off, part_off, bytes) of a fused-gather buffer (full K1 outputs + P partial slots)."""
    o = [C.c_size_t() for _ in range(4)]
    _check(_lib.svdq_tp_gather_sizes(FMT[fmt], M, K, rank, P, *[C.byref(x) for x in o]), "svdq_tp_gather_sizes")
    return tuple(x.value for x in o)


def svdq_quantize_act_lowrank_down_kslice_fused(layer: "QuantizedLinear", k0: int, X, P: int, p: int, buf_ptrs,
                                                stream=None):
    """K1 on input channels [k0, k0 + X.shape[1]) writing its codes / scales at their full-K place
    and its partial in slot p of every gather buffer in `buf_ptrs` (device addresses, ints)."""
    M, Kp = X.shape
    arr = (_P * len(buf_ptrs))(*[int(q) for q in buf_ptrs])
    _check(_lib.svdq_quantize_act_lowrank_down_kslice_fused(layer.ref, k0, Kp, _ptr(X), DTYPE[DTYPE_OF_TORCH[X.dtype]],
                                                            M, X.stride(0), P, p, arr, len(buf_ptrs), _stream(stream)),
           "svdq_quantize_act_lowrank_down_kslice_fused")


def svdq_tp_reduce_partials(P: int, M: int, rank: int, parts, xl1, stream=None):
    """xl1 = bf16(sum of the P fp32 partial slots, in rank order)."""
    _check(_lib.svdq_tp_reduce_partials(P, M, rank, _ptr(parts), _ptr(xl1), _stream(stream)), "svdq_tp_reduce_partials")
    return xl1


def svdq_tp_assemble_act(fmt: str, P: int, M: int, K: int, rank: int, gathered, xq=None, xs=None, xl1=None,
                         slice_stride: int = 0, stream=None):
    """Full K1 outputs (xq, xs, xl1) from the P gathered slices: slice p at byte p * slice_stride of
    `gathered` (0: back to back, the all_gather_into_tensor output of one slice per rank)."""
    bq, bs, bl = svdq_act_buffer_sizes(fmt, M, K, rank)
    dev = gathered.device
    xq = torch.empty(bq, dtype=torch.uint8, device=dev) if xq is None else xq
    xs = torch.empty(bs, dtype=torch.uint8, device=dev) if xs is None else xs
    xl1 = torch.empty(max(bl // 2, 8), dtype=torch.int16, device=dev) if xl1 is None else xl1
    nb = svdq_tp_slice_sizes(fmt, M, K // P, rank)[3]
    _check(_lib.svdq_tp_assemble_act(FMT[fmt], P, M, K, rank, _ptr(gathered), nb, slice_stride, _ptr(xq), _ptr(xs),
                                     _ptr(xl1), _stream(stream)), "svdq_tp_assemble_act")
    return xq, xs, xl1


def svdq_k1_row_tile(rows_padded: int, rank: int) -> int:
    """Rows per CTA the K1 kernel uses for a launch over `rows_padded` rows (host-only query)."""
    return int(_lib.svdq_k1_row_tile(rows_padded, rank))


def svdq_act_buffer_sizes(fmt: str, M: int, K: int, rank: int):
    a, b, c = C.c_size_t(), C.c_size_t(), C.c_size_t()
    _check(_lib.svdq_act_buffer_sizes(FMT[fmt], M, K, rank, C.byref(a), C.byref(b), C.byref(c)),
           "svdq_act_buffer_sizes")
    return a.value, b.value, c.value


def svdq_weight_buffer_sizes(fmt: str, K: int, N: int, rank: int):
    v = [C.c_size_t() for _ in range(4)]
    _check(_lib.svdq_weight_buffer_sizes(FMT[fmt], K, N, rank, *[C.byref(x) for x in v]),
           "svdq_weight_buffer_sizes")
    return tuple(x.value for x in v)


# ---------------------------------------------------------------- layer view
class QuantizedLinear:
    """Owns the device buffers of one layer and the svdq_linear view of them."""

    def __init__(self, fmt: str, K: int, N: int, rank: int, w_codes, w_scales, lambda_inv, l1s, l2s,
                 bias=None, scale_dtype: str = "bf16", gs_w: float = 1.0, gs_x: float = 1.0):
        self.fmt, self.K, self.N, self.rank = fmt, K, N, rank
        self.w_codes, self.w_scales, self.lambda_inv = w_codes, w_scales, lambda_inv
        self.l1s, self.l2s, self.bias = l1s, l2s, bias
        self.scale_dtype = scale_dtype
        self.gs_w, self.gs_x = float(gs_w), float(gs_x)
        self._sync_view()

    def _sync_view(self):
        bias_dt = DTYPE_OF_TORCH[self.bias.dtype] if self.bias is not None else "bf16"
        self.view = svdq_linear(
            FMT[self.fmt], self.rank, self.K, self.N, _ptr(self.w_codes), _ptr(self.w_scales),
            _ptr(self.lambda_inv), _ptr(self.l1s), _ptr(self.l2s), _ptr(self.bias),
            DTYPE[self.scale_dtype], DTYPE[bias_dt], self.gs_w, self.gs_x)

    @property
    def ref(self):
        return C.byref(self.view)

    @classmethod
    def empty(cls, fmt, K, N, rank, device="cuda", scale_dtype="bf16", bias=None, gs_x=1.0):
        codes_b, scales_b, l1s_b, l2s_b = svdq_weight_buffer_sizes(fmt, K, N, rank)
        u8 = dict(dtype=torch.uint8, device=device)
        return cls(fmt, K, N, rank,
                   torch.empty(codes_b, **u8), torch.empty(scales_b, **u8),
                   torch.empty(K, dtype=torch.float32, device=device),
                   torch.empty(max(l1s_b // 2, 8), dtype=torch.int16, device=device),
                   torch.empty(max(l2s_b // 2, 8), dtype=torch.int16, device=device),
                   bias, scale_dtype, 1.0, gs_x)

    def forward(self, X, out_dtype=None, stream=None):
        return svdq_linear_forward(self, X, out_dtype=out_dtype, stream=stream)

    __call__ = forward


# ---------------------------------------------------------------- hot path
def svdq_quantize_act_lowrank_down(layer: QuantizedLinear, X, xq=None, xs=None, xl1=None, stream=None):
    """K1.  X: [M, K] bf16/fp16 CUDA tensor (row pitch X.stride(0))."""
    M = X.shape[0]
    bq, bs, bl = svdq_act_buffer_sizes(layer.fmt, M, layer.K, layer.rank)
    dev = X.device
    if xq is None:
        xq = torch.empty(bq, dtype=torch.uint8, device=dev)
    if xs is None:
        xs = torch.empty(bs, dtype=torch.uint8, device=dev)
    if xl1 is None and layer.rank:
        xl1 = torch.empty(bl // 2, dtype=torch.int16, device=dev)
    _check(_lib.svdq_quantize_act_lowrank_down(
        layer.ref, _ptr(X), DTYPE[DTYPE_OF_TORCH[X.dtype]], M, X.stride(0), _ptr(xq), _ptr(xs),
        _ptr(xl1), _stream(stream)), "svdq_quantize_act_lowrank_down")
    return xq, xs, xl1


def svdq_gemm_w4a4_lowrank_up(layer: QuantizedLinear, xq, xs, xl1, M: int, Y=None,
                              out_dtype=torch.bfloat16, stream=None):
    """K2.  Returns Y [M, N]."""
    if Y is None:
        Y = torch.empty(M, layer.N, dtype=out_dtype, device=xq.device)
    _check(_lib.svdq_gemm_w4a4_lowrank_up(
        layer.ref, _ptr(xq), _ptr(xs), _ptr(xl1), M, _ptr(Y), DTYPE[DTYPE_OF_TORCH[Y.dtype]],
        Y.stride(0), _stream(stream)), "svdq_gemm_w4a4_lowrank_up")
    return Y


def svdq_quantize_act_lowrank_down_grouped(layers, X, xq, xs, xl1, stream=None):
    """Grouped K1: one launch over n (1..4) problems with bf16 X; lists of equal length.
    Problem i produces exactly svdq_quantize_act_lowrank_down(layers[i], X[i], xq[i], xs[i], xl1[i])."""
    n = len(layers)
    arr = lambda T, vals: (T * n)(*vals)
    _check(_lib.svdq_quantize_act_lowrank_down_grouped(
        n, arr(_LP, [C.pointer(l.view) for l in layers]), arr(_P, [x.data_ptr() for x in X]),
        DTYPE[DTYPE_OF_TORCH[X[0].dtype]], arr(_I64, [x.shape[0] for x in X]), arr(_I64, [x.stride(0) for x in X]),
        arr(_P, [q.data_ptr() for q in xq]), arr(_P, [q.data_ptr() for q in xs]),
        arr(_P, [q.data_ptr() if q is not None else None for q in xl1]), _stream(stream)),
        "svdq_quantize_act_lowrank_down_grouped")
    return xq, xs, xl1


def svdq_gemm_w4a4_lowrank_up_grouped(layers, xq, xs, xl1, M, Y, stream=None):
    """Grouped K2: one launch over n (1..4) independent NVFP4 problems; lists of equal length.
    Problem i produces exactly svdq_gemm_w4a4_lowrank_up(layers[i], xq[i], xs[i], xl1[i], M[i], Y[i])."""
    n = len(layers)
    ydt = {DTYPE_OF_TORCH[y.dtype] for y in Y}
    if len(ydt) != 1:
        raise ValueError("grouped K2: all Y must share one dtype")
    arr = lambda T, vals: (T * n)(*vals)
    _check(_lib.svdq_gemm_w4a4_lowrank_up_grouped(
        n, arr(_LP, [C.pointer(l.view) for l in layers]), arr(_P, [x.data_ptr() for x in xq]),
        arr(_P, [x.data_ptr() for x in xs]), arr(_P, [x.data_ptr() if x is not None else None for x in xl1]),
        arr(_I64, list(M)), arr(_P, [y.data_ptr() for y in Y]), DTYPE[ydt.pop()],
        arr(_I64, [y.stride(0) for y in Y]), _stream(stream)), "svdq_gemm_w4a4_lowrank_up_grouped")
    return Y


ACT = {"none": 0, "gelu_tanh": 1}


def svdq_gemm_fused_next_workspace(layers, M, nexts) -> int:
    n = len(layers)
    arr = lambda T, vals: (T * n)(*vals)
    wsb = C.c_size_t()
    _check(_lib.svdq_gemm_fused_next_workspace(n, arr(_LP, [C.pointer(l.view) for l in layers]), arr(_I64, list(M)),
                                               arr(_LP, [C.pointer(l.view) for l in nexts]), C.byref(wsb)),
           "svdq_gemm_fused_next_workspace")
    return wsb.value


def svdq_gemm_w4a4_lowrank_up_fused_next(layers, xq, xs, xl1, M, nexts, act="none", Y=None, ws=None, out=None,
                                         stream=None):
    """K2 of layers[i] whose epilogue also runs nexts[i]'s K1 on its (activated) bf16 output
    (SURVEY 8(f) row 1).  Y: list of bf16 [M, N] tensors or None (no store).  Returns
    (xq_next, xs_next, xl1_next) lists, the buffers svdq_quantize_act_lowrank_down(nexts[i], a) fills."""
    n = len(layers)
    dev = xq[0].device
    outs = []
    for i, (L, Nx, m) in enumerate(zip(layers, nexts, M)):
        if out is not None:
            outs.append((out[0][i], out[1][i], out[2][i]))
            continue
        bq, bs, bl = svdq_act_buffer_sizes(Nx.fmt, m, Nx.K, Nx.rank)
        outs.append((torch.empty(bq, dtype=torch.uint8, device=dev), torch.empty(bs, dtype=torch.uint8, device=dev),
                     torch.empty(max(bl // 2, 8), dtype=torch.int16, device=dev)))
    need = svdq_gemm_fused_next_workspace(layers, M, nexts)
    if ws is None:
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device=dev)
    arr = lambda T, vals: (T * n)(*vals)
    Yp = [None if Y is None or Y[i] is None else Y[i].data_ptr() for i in range(n)]
    _check(_lib.svdq_gemm_w4a4_lowrank_up_fused_next(
        n, arr(_LP, [C.pointer(l.view) for l in layers]), arr(_P, [x.data_ptr() for x in xq]),
        arr(_P, [x.data_ptr() for x in xs]), arr(_P, [x.data_ptr() if x is not None else None for x in xl1]),
        arr(_I64, list(M)), arr(_P, Yp), arr(_LP, [C.pointer(l.view) for l in nexts]), ACT[act],
        arr(_P, [o[0].data_ptr() for o in outs]), arr(_P, [o[1].data_ptr() for o in outs]),
        arr(_P, [o[2].data_ptr() for o in outs]), _ptr(ws), ws.numel(), _stream(stream)),
        "svdq_gemm_w4a4_lowrank_up_fused_next")
    return [o[0] for o in outs], [o[1] for o in outs], [o[2] for o in outs]


def forward_workspace_bytes(layer: QuantizedLinear, M: int) -> int:
    up = lambda b: (b + 255) // 256 * 256
    return sum(up(b) for b in svdq_act_buffer_sizes(layer.fmt, M, layer.K, layer.rank))


def svdq_linear_forward(layer: QuantizedLinear, X, Y=None, out_dtype=None, ws=None, stream=None):
    M = X.shape[0]
    if Y is None:
        Y = torch.empty(M, layer.N, dtype=out_dtype or X.dtype, device=X.device)
    need = forward_workspace_bytes(layer, M)
    if ws is None:
        ws = torch.empty(need, dtype=torch.uint8, device=X.device)
    _check(_lib.svdq_linear_forward(
        layer.ref, _ptr(X), DTYPE[DTYPE_OF_TORCH[X.dtype]], M, X.stride(0), _ptr(Y),
        DTYPE[DTYPE_OF_TORCH[Y.dtype]], Y.stride(0), _ptr(ws), ws.numel(), _stream(stream)),
        "svdq_linear_forward")
    return Y


# ---------------------------------------------------------------- offline
def svdq_quantize_residual(R, fmt: str, scale_dtype: str = "bf16", gs_w: float = 0.0,
                           codes=None, scales=None, stream=None):
    """R: [K, N] fp32 CUDA tensor (paper layout).  Returns (codes, scales, gs_w)."""
    K, N = R.shape
    cb, sb, _, _ = svdq_weight_buffer_sizes(fmt, K, N, 0)
    if codes is None:
        codes = torch.empty(cb, dtype=torch.uint8, device=R.device)
    if scales is None:
        scales = torch.empty(sb, dtype=torch.uint8, device=R.device)
    g = C.c_float(gs_w)
    _check(_lib.svdq_quantize_residual(_ptr(R), K, N, FMT[fmt], DTYPE[scale_dtype], _ptr(codes),
                                       _ptr(scales), C.byref(g), _stream(stream)),
           "svdq_quantize_residual")
    return codes, scales, g.value


def svdq_quantize_weights_workspace(K: int, N: int, rank: int) -> int:
    wsb = C.c_size_t()
    _check(_lib.svdq_quantize_weights_workspace(K, N, rank, C.byref(wsb)),
           "svdq_quantize_weights_workspace")
    return wsb.value


def svdq_quantize_weights(W, lam, rank: int, fmt: str, scale_dtype: str = "bf16", gs_x: float = 1.0,
                          L1=None, L2=None, bias=None, stream=None) -> QuantizedLinear:
    """W: [K, N] CUDA tensor (bf16/fp16/fp32), lam: [K] fp32."""
    K, N = W.shape
    layer = QuantizedLinear.empty(fmt, K, N, rank, device=W.device, scale_dtype=scale_dtype,
                                  bias=bias, gs_x=gs_x)
    ws = torch.empty(svdq_quantize_weights_workspace(K, N, rank), dtype=torch.uint8, device=W.device)
    W = W.contiguous()
    lam = lam.contiguous().float()
    _check(_lib.svdq_quantize_weights(
        _ptr(W), DTYPE[DTYPE_OF_TORCH[W.dtype]], _ptr(lam), K, N, rank, FMT[fmt], DTYPE[scale_dtype],
        gs_x, _ptr(L1), _ptr(L2), layer.ref, _ptr(ws), ws.numel(), _stream(stream)),
        "svdq_quantize_weights")
    layer.gs_w = layer.view.gs_w
    layer.gs_x = layer.view.gs_x
    del ws
    return layer


def svdq_lora_fuse(layer: QuantizedLinear, A, B, scale: float = 1.0, stream=None) -> QuantizedLinear:
    """A: [K, r_l], B: [r_l, N] CUDA tensors (bf16/fp16/fp32).  Returns a new layer of rank r + r_l
    sharing the residual codes / scales / lambda with `layer`."""
    r_l = A.shape[1]
    r1 = layer.rank + r_l
    out = QuantizedLinear(layer.fmt, layer.K, layer.N, r1, layer.w_codes, layer.w_scales,
                          layer.lambda_inv,
                          torch.empty(r1 * layer.K, dtype=torch.int16, device=A.device),
                          torch.empty(layer.N * r1, dtype=torch.int16, device=A.device),
                          layer.bias, layer.scale_dtype, layer.gs_w, layer.gs_x)
    A = A.contiguous()
    B = B.contiguous()
    if B.dtype != A.dtype:
        raise ValueError("A and B must share a dtype")
    _check(_lib.svdq_lora_fuse(layer.ref, _ptr(A), _ptr(B), DTYPE[DTYPE_OF_TORCH[A.dtype]], r_l,
                               scale, out.ref, _stream(stream)), "svdq_lora_fuse")
    return out


# ---------------------------------------------------------------- test hooks
def svdq_search_alpha_workspace(fmt: str, M_cal: int, K: int, N: int, rank: int) -> int:
    wsb = C.c_size_t()
    _check(_lib.svdq_search_alpha_workspace(FMT[fmt], M_cal, K, N, rank, C.byref(wsb)), "svdq_search_alpha_workspace")
    return wsb.value


def svdq_search_alpha(X_cal, W, rank: int, fmt: str, grid, scale_dtype: str = "bf16", gs_x: float = 1.0,
                      stream=None):
    """Offline migration-strength search (App. D) on the GPU.  X_cal: [M_cal, K] bf16/fp16,
    W: [K, N] fp32 (CUDA).  Returns (alpha*, lambda(alpha*) [K] fp32 tensor, objectives list)."""
    M, K = X_cal.shape
    N = W.shape[1]
    wsb = svdq_search_alpha_workspace(fmt, M, K, N, rank)
    ws = torch.empty(wsb, dtype=torch.uint8, device=X_cal.device)
    lam = torch.empty(K, dtype=torch.float32, device=X_cal.device)
    n = len(grid)
    g = (C.c_float * n)(*grid)
    obj = (C.c_double * n)()
    a = C.c_float()
    Wc = W.contiguous().float()
    _check(_lib.svdq_search_alpha(_ptr(X_cal), DTYPE[DTYPE_OF_TORCH[X_cal.dtype]], M, X_cal.stride(0), _ptr(Wc), K, N,
                                  rank, FMT[fmt], DTYPE[scale_dtype], gs_x, g, n, C.byref(a), _ptr(lam), obj,
                                  _ptr(ws), wsb, _stream(stream)), "svdq_search_alpha")
    return a.value, lam, list(obj)


def svdq_refine_lowrank_workspace(fmt: str, M_cal: int, K: int, N: int, rank: int, gptq: bool = False) -> int:
    wsb = C.c_size_t()
    _check(_lib.svdq_refine_lowrank_workspace(FMT[fmt], M_cal, K, N, rank, int(gptq), C.byref(wsb)),
           "svdq_refine_lowrank_workspace")
    return wsb.value


def svdq_refine_lowrank(X_cal, W, lam, rank: int, fmt: str, iters: int, scale_dtype: str = "bf16",
                        gs_x: float = 1.0, bias=None, gptq: bool = False, damp: float = 0.01, stream=None):
    """Iterative low-rank refinement on the GPU.  X_cal: [M_cal, K] bf16/fp16, W: [K, N] fp32,
    lam: [K] fp32 (CUDA); gptq=True quantizes each iterate's residual by GPTQ.
    Returns (QuantizedLinear of the best iterate, best index, objectives list)."""
    M, K = X_cal.shape
    N = W.shape[1]
    layer = QuantizedLinear.empty(fmt, K, N, rank, device=X_cal.device, scale_dtype=scale_dtype,
                                  bias=bias, gs_x=gs_x)
    wsb = svdq_refine_lowrank_workspace(fmt, M, K, N, rank, gptq)
    ws = torch.empty(wsb, dtype=torch.uint8, device=X_cal.device)
    obj = (C.c_double * (iters + 1))()
    best = C.c_int32()
    Wc = W.contiguous().float()
    lam = lam.contiguous().float()
    _check(_lib.svdq_refine_lowrank(_ptr(X_cal), DTYPE[DTYPE_OF_TORCH[X_cal.dtype]], M, X_cal.stride(0), _ptr(Wc),
                                    _ptr(lam), K, N, rank, FMT[fmt], DTYPE[scale_dtype], gs_x, iters, int(gptq), damp,
                                    layer.ref,
                                    C.byref(best), obj, _ptr(ws), wsb, _stream(stream)), "svdq_refine_lowrank")
    layer.gs_w = layer.view.gs_w
    layer.gs_x = layer.view.gs_x
    del ws
    return layer, best.value, list(obj)


def svdq_quantize_residual_gptq_workspace(M_cal: int, K: int, N: int) -> int:
    wsb = C.c_size_t()
    _check(_lib.svdq_quantize_residual_gptq_workspace(M_cal, K, N, C.byref(wsb)), "svdq_quantize_residual_gptq_workspace")
    return wsb.value


def svdq_quantize_weights_gptq_workspace(M_cal: int, K: int, N: int, rank: int) -> int:
    wsb = C.c_size_t()
    _check(_lib.svdq_quantize_weights_gptq_workspace(M_cal, K, N, rank, C.byref(wsb)),
           "svdq_quantize_weights_gptq_workspace")
    return wsb.value


def svdq_quantize_residual_gptq(R, X_cal, lam_inv, fmt: str, scale_dtype: str = "bf16", damp: float = 0.01,
                                stream=None):
    """GPTQ of the residual R ([K, N] fp32 CUDA) on X_hat = fl32(X_cal * lam_inv).
    Returns (codes, scales, gs_w) in the layout of svdq_quantize_residual."""
    K, N = R.shape
    M = X_cal.shape[0]
    codes_b, scales_b, _, _ = svdq_weight_buffer_sizes(fmt, K, N, 0)
    codes = torch.empty(codes_b, dtype=torch.uint8, device=R.device)
    scales = torch.zeros(scales_b, dtype=torch.uint8, device=R.device)
    wsb = svdq_quantize_residual_gptq_workspace(M, K, N)
    ws = torch.empty(wsb, dtype=torch.uint8, device=R.device)
    gs = C.c_float(0.0)
    R = R.contiguous().float()
    lam_inv = lam_inv.contiguous().float()
    _check(_lib.svdq_quantize_residual_gptq(_ptr(R), K, N, FMT[fmt], DTYPE[scale_dtype], _ptr(X_cal),
                                            DTYPE[DTYPE_OF_TORCH[X_cal.dtype]], M, X_cal.stride(0), _ptr(lam_inv),
                                            damp, _ptr(codes), _ptr(scales), C.byref(gs), _ptr(ws), wsb,
                                            _stream(stream)), "svdq_quantize_residual_gptq")
    return codes, scales, gs.value


def svdq_quantize_weights_gptq(W, lam, rank: int, fmt: str, X_cal, scale_dtype: str = "bf16", gs_x: float = 1.0,
                               damp: float = 0.01, bias=None, stream=None) -> QuantizedLinear:
    """svdq_quantize_weights with the residual quantized by GPTQ on the calibration batch X_cal."""
    K, N = W.shape
    M = X_cal.shape[0]
    layer = QuantizedLinear.empty(fmt, K, N, rank, device=W.device, scale_dtype=scale_dtype, bias=bias, gs_x=gs_x)
    wsb = svdq_quantize_weights_gptq_workspace(M, K, N, rank)
    ws = torch.empty(wsb, dtype=torch.uint8, device=W.device)
    W = W.contiguous()
    lam = lam.contiguous().float()
    _check(_lib.svdq_quantize_weights_gptq(
        _ptr(W), DTYPE[DTYPE_OF_TORCH[W.dtype]], _ptr(lam), K, N, rank, FMT[fmt], DTYPE[scale_dtype], gs_x,
        _ptr(X_cal), DTYPE[DTYPE_OF_TORCH[X_cal.dtype]], M, X_cal.stride(0), damp, layer.ref, _ptr(ws), wsb,
        _stream(stream)), "svdq_quantize_weights_gptq")
    layer.gs_w = layer.view.gs_w
    layer.gs_x = layer.view.gs_x
    del ws
    return layer


def svdq_debug_int4_group_accum(xq, wq, M: int, N: int, K: int, stream=None):
    acc = torch.empty((K // 64, M, N), dtype=torch.int32, device=xq.device)
    _check(_lib.svdq_debug_int4_group_accum(_ptr(xq), _ptr(wq), M, N, K, _ptr(acc), _stream(stream)),
           "svdq_debug_int4_group_accum")
    return acc


def svdq_debug_codec(x, kind: int, stream=None):
    """kind 0: E2M1x2 bytes of consecutive pairs; kind 1: E4M3 byte per value."""
    x = x.contiguous().float()
    n = x.numel() // 2 if kind == 0 else x.numel()
    out = torch.empty(n, dtype=torch.uint8, device=x.device)
    _check(_lib.svdq_debug_codec(_ptr(x), _ptr(out), n, kind, _stream(stream)), "svdq_debug_codec")
    return out
