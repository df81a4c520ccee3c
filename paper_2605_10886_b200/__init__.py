"""Thin Python binding of libloka.so (include/loka.h) — argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``libloka.so``; this module only
builds the C structs from torch tensors (device memory), passes the current CUDA stream, and
checks the returned status.  There is NO CPU fallback: importing raises if the library is
missing, and every call raises on a non-OK status (``LOKA_ERR_UNSUPPORTED`` off sm_100).

The functions carry the C names (``loka_quantize``, ``loka_fp8_linear_norm``,
``loka_grouped_fp8_linear``, ``loka_probe_error``, ``loka_dispatch_select``).
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libloka.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libloka.so not built ({LIB_PATH}); run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "or `python paper_2605_10886_b200/build.py` — there is no CPU fallback")
_lib = C.CDLL(LIB_PATH)


def _check_build():
    """Refuse a stale binary: the library's compiled-in source hash must match the source tree."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_loka_build", os.path.join(_HERE, "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    _lib.loka_source_hash.restype = C.c_char_p
    built = _lib.loka_source_hash().decode()
    want = b.source_hash()
    if built != want and os.environ.get("LOKA_ALLOW_STALE") != "1":
        raise ImportError(f"libloka.so was built from other sources (hash {built}, tree {want}); rebuild with "
                          "`python paper_2605_10886_b200/build.py` (LOKA_ALLOW_STALE=1 overrides)")


_check_build()

# ---- enums (include/loka.h) ----------------------------------------------------------------
OK, ERR_INVALID_ARG, ERR_SHAPE, ERR_UNSUPPORTED, ERR_NONFINITE, ERR_WORKSPACE, ERR_CUDA = range(7)
DEVSTATUS_NONFINITE = 0x1
F32, BF16, E4M3, E5M2 = range(4)
GRAN = {"tensor": 0, "row": 1, "col": 2, "blk_1x128": 3, "blk_128x1": 4, "blk_128x128": 5, "blk_1x32": 6}
SCALE = {"f32": 0, "ue8m0": 1}
PHASE = {"full": 0, "amax": 1, "cast": 2, "delayed": 3}
NORM = {"none": 0, "layer": 1, "rms": 2, "block_rms": 3}
ACT = {"none": 0, "hardswish": 1}
DIR = {"fwd": 0, "dgrad": 1, "wgrad": 2}
FMT = {"e4m3": E4M3, "e5m2": E5M2}
_TORCH_DT = {F32: torch.float32, BF16: torch.bfloat16, E4M3: torch.uint8, E5M2: torch.uint8}


class LokaError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {_lib.loka_status_string(status).decode()} (status {status})")
        self.status = status


class loka_tensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int), ("rows", C.c_int64), ("cols", C.c_int64),
                ("ld", C.c_int64), ("scales", C.c_void_p), ("gran", C.c_int), ("scale_fmt", C.c_int)]


class loka_linear_args(C.Structure):
    _fields_ = [("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64), ("dir", C.c_int),
                ("a", loka_tensor), ("b", loka_tensor), ("bias", C.c_void_p), ("bias_dtype", C.c_int),
                ("norm", C.c_int), ("norm_block", C.c_int32), ("eps", C.c_float), ("gamma", C.c_void_p),
                ("beta", C.c_void_p), ("y", loka_tensor), ("debug_precast", C.c_void_p), ("status_dev", C.c_void_p),
                ("act", C.c_int), ("bwd_xhat", C.c_void_p), ("bwd_xhat_ld", C.c_int64), ("bwd_rstd", C.c_void_p),
                ("save_xhat", C.c_void_p), ("save_xhat_ld", C.c_int64), ("save_rstd", C.c_void_p),
                ("amax_out", C.c_void_p), ("x_amax", C.c_void_p)]


class loka_stack_args(C.Structure):
    _fields_ = [("L", C.c_int32), ("M", C.c_int64), ("dims", C.c_int64 * 9), ("x", loka_tensor),
                ("w", loka_tensor * 8), ("norm", C.c_int * 8), ("eps", C.c_float * 8), ("y", loka_tensor),
                ("status_dev", C.c_void_p), ("h", loka_tensor * 7), ("ws", C.c_void_p), ("ws_bytes", C.c_size_t),
                ("debug_precast", C.c_void_p * 8)]


class loka_welford_state(C.Structure):
    _fields_ = [("n", C.c_int64), ("K", C.c_int64), ("mean", C.c_void_p), ("scatter", C.c_void_p)]


class loka_matnorm_state(C.Structure):
    _fields_ = [("M", C.c_int64), ("N", C.c_int64), ("count", C.c_int64), ("momentum", C.c_float),
                ("eps_rel", C.c_float), ("mean", C.c_void_p), ("U", C.c_void_p), ("V", C.c_void_p)]


class loka_probe_pair(C.Structure):
    _fields_ = [("out", C.c_void_p), ("out_dtype", C.c_int), ("ref", C.c_void_p), ("ref_dtype", C.c_int),
                ("M", C.c_int64), ("N", C.c_int64), ("ld_out", C.c_int64), ("ld_ref", C.c_int64)]


class loka_probe_stats(C.Structure):
    _fields_ = [("mere", C.c_double), ("max_rel", C.c_double), ("sum_abs_ref", C.c_double),
                ("count", C.c_int64), ("n_floored", C.c_int64)]


class loka_nvfp4_tensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("rows", C.c_int64), ("cols", C.c_int64), ("ld", C.c_int64),
                ("block_scales", C.c_void_p), ("tensor_scale", C.c_void_p)]


class loka_nvfp4_linear_args(C.Structure):
    _fields_ = [("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64), ("a", loka_nvfp4_tensor),
                ("b", loka_nvfp4_tensor), ("bias", C.c_void_p), ("bias_dtype", C.c_int), ("norm", C.c_int),
                ("norm_block", C.c_int32), ("eps", C.c_float), ("gamma", C.c_void_p), ("beta", C.c_void_p),
                ("y", loka_tensor), ("status_dev", C.c_void_p)]


class loka_candidate(C.Structure):
    _fields_ = [("id", C.c_char_p), ("dir", C.c_int), ("mere", C.c_double), ("time_us", C.c_double)]


_P = C.POINTER
_sig = {
    "loka_quantize": ([_P(loka_tensor), _P(loka_tensor), _P(loka_tensor), C.c_int, C.c_void_p, C.c_void_p,
                       C.c_void_p, C.c_size_t, C.c_void_p], C.c_int),
    "loka_quantize_workspace_size": ([_P(loka_tensor), _P(loka_tensor)], C.c_size_t),
    "loka_quantize_grouped": ([C.c_int32, _P(loka_tensor), _P(loka_tensor), C.c_void_p, C.c_void_p], C.c_int),
    "loka_fp8_linear_norm": ([_P(loka_linear_args), C.c_void_p, C.c_size_t, C.c_void_p], C.c_int),
    "loka_linear_workspace_size": ([_P(loka_linear_args)], C.c_size_t),
    "loka_fp8_mlp_stack": ([_P(loka_stack_args), C.c_void_p], C.c_int),
    "loka_grouped_fp8_linear": ([C.c_int32, _P(loka_linear_args), C.c_void_p, C.c_size_t, C.c_void_p], C.c_int),
    "loka_grouped_workspace_size": ([C.c_int32, _P(loka_linear_args)], C.c_size_t),
    "loka_probe_error": ([C.c_int32, _P(loka_probe_pair), C.c_double, C.c_void_p, C.c_void_p, C.c_size_t,
                          C.c_void_p], C.c_int),
    "loka_probe_workspace_size": ([C.c_int32, _P(loka_probe_pair)], C.c_size_t),
    "loka_probe_error_global": ([C.c_int32, _P(loka_probe_pair), C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_size_t, C.c_void_p], C.c_int),
    "loka_probe_merge": ([C.c_int32, C.c_int32, _P(loka_probe_stats), _P(loka_probe_stats)], C.c_int),
    "loka_probe_track_covariance": ([C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "loka_source_hash": ([], C.c_char_p),
    "loka_bf16_linear_norm": ([C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p], C.c_int),
    "loka_grouped_bf16_linear": ([C.c_int32, _P(loka_linear_args), C.c_void_p], C.c_int),
    "loka_bf16_linear_workspace_size": ([C.c_void_p], C.c_size_t),
    "loka_dispatch_select": ([_P(loka_candidate), C.c_int32, C.c_double, C.c_double, C.c_double, _P(C.c_int32)],
                             C.c_int),
    "loka_quantize_nvfp4": ([_P(loka_tensor), _P(loka_nvfp4_tensor), C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                             C.c_void_p], C.c_int),
    "loka_quantize_nvfp4_workspace_size": ([_P(loka_tensor)], C.c_size_t),
    "loka_nvfp4_linear_norm": ([_P(loka_nvfp4_linear_args), C.c_void_p, C.c_size_t, C.c_void_p], C.c_int),
    "loka_nvfp4_linear_workspace_size": ([_P(loka_nvfp4_linear_args)], C.c_size_t),
    "loka_dequant_reduce": ([C.c_int32, _P(C.c_void_p), _P(C.c_void_p), C.c_int, C.c_int64, C.c_int64, C.c_int64,
                             C.c_void_p, C.c_int64, C.c_void_p], C.c_int),
    "loka_status_string": ([C.c_int], C.c_char_p),
    "loka_device_supported": ([C.c_int32], C.c_int32),
    "loka_version": ([], C.c_int32),
    "loka_launch_count": ([], C.c_int64),
    "loka_debug_hang_info": ([_P(C.c_uint64), C.c_int32], C.c_int64),
    "loka_debug_trace": ([C.c_int32, _P(C.c_uint64), C.c_int64], C.c_int64),
    "loka_debug_pairnorm_trace": ([C.c_void_p], None),
    "loka_stack_workspace_size": ([_P(loka_stack_args)], C.c_size_t),
    "loka_probe_track_workspace_size": ([_P(loka_welford_state), C.c_int64], C.c_size_t),
    "loka_probe_track_input": ([_P(loka_welford_state), _P(loka_tensor), C.c_void_p, C.c_size_t, C.c_void_p], C.c_int),
    "loka_philox_normal": ([C.c_uint64, C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p], C.c_int),
    "loka_cholesky_workspace_size": ([C.c_int64], C.c_size_t),
    "loka_cholesky_jittered": ([C.c_void_p, C.c_int64, C.c_int64, C.c_float, C.c_float, C.c_int32, C.c_void_p,
                                C.c_int64, _P(C.c_float), C.c_void_p, C.c_size_t, C.c_void_p], C.c_int),
    "loka_probe_track_weight_init": ([_P(loka_matnorm_state), _P(loka_tensor), C.c_void_p], C.c_int),
    "loka_probe_track_weight_workspace_size": ([_P(loka_matnorm_state)], C.c_size_t),
    "loka_probe_track_weight": ([_P(loka_matnorm_state), _P(loka_tensor), C.c_void_p, C.c_void_p, C.c_size_t,
                                 C.c_void_p], C.c_int),
    "loka_probe_sample_workspace_size": ([C.c_int64, C.c_int64, C.c_int32], C.c_size_t),
    "loka_probe_sample_input": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_uint64, C.c_uint64,
                                 _P(loka_tensor), C.c_void_p, C.c_size_t, C.c_void_p], C.c_int),
    "loka_probe_sample_weight": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_uint64, C.c_uint64,
                                  _P(loka_tensor), C.c_void_p, C.c_size_t, C.c_void_p], C.c_int),
}
for _name, (_args, _ret) in _sig.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = _ret
EXPORTS = tuple(_sig)


def _check(status: int, what: str):
    if status != OK:
        raise LokaError(status, what)


def _stream(stream=None) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.bfloat16:
        return BF16
    raise TypeError(t.dtype)


def _tensor(data, dtype: int, rows: int, cols: int, scales=None, gran="tensor", scale_fmt="f32", ld=None):
    if data is not None:
        assert data.is_cuda and data.dim() == 2 and data.stride(1) == 1
        ld = data.stride(0) if ld is None else ld
    return loka_tensor(None if data is None else data.data_ptr(), dtype, rows, cols, ld if ld is not None else cols,
                       None if scales is None else scales.data_ptr(), GRAN[gran], SCALE[scale_fmt])


def scale_shape(rows: int, cols: int, gran: str):
    cd = lambda a, b: -(-a // b)
    return {"tensor": (1,), "row": (rows,), "col": (cols,), "blk_1x128": (rows, cd(cols, 128)),
            "blk_128x1": (cd(rows, 128), cols), "blk_128x128": (cd(rows, 128), cd(cols, 128)),
            "blk_1x32": (rows, cd(cols, 32))}[gran]


_T_GRAN = {"row": "col", "col": "row", "blk_1x128": "blk_128x1", "blk_128x1": "blk_1x128"}


def loka_quantize(x: torch.Tensor, fmt: str = "e4m3", gran: str = "row", scale_fmt: str = "f32",
                  phase: str = "full", amax: torch.Tensor | None = None, status: torch.Tensor | None = None,
                  out: torch.Tensor | None = None, scales: torch.Tensor | None = None, want_q: bool = True,
                  transpose: bool = False, out_t: torch.Tensor | None = None, scales_t: torch.Tensor | None = None,
                  gran_t: str | None = None, stream=None):
    """a1-a3.  Returns (codes uint8 [rows, cols] or None, scales fp32) [+ (codes_t, scales_t)].
    gran_t: the transposed copy's granularity in ITS frame (default: the same quantization,
    transposed); gran="blk_1x128", gran_t="blk_1x128" = x's 128x1 quantization, transposed (one pass)."""
    rows, cols = x.shape
    dev = x.device
    if want_q and out is None:
        out = torch.empty(rows, cols, dtype=torch.uint8, device=dev) if cols % 16 == 0 else \
            torch.empty(rows, (cols + 15) // 16 * 16, dtype=torch.uint8, device=dev)[:, :cols]
    if scales is None:
        scales = torch.empty(scale_shape(rows, cols, gran), dtype=torch.float32, device=dev)
    qx = _tensor(x, _dtype_code(x), rows, cols)
    qq = _tensor(out if want_q else None, FMT[fmt], rows, cols, scales, gran, scale_fmt)
    qt = None
    qt_codes = qt_scales = None
    if transpose:
        tg = _T_GRAN.get(gran, gran) if gran_t is None else gran_t
        # K-major copy for the backward GEMMs: leading dimension padded to 16 bytes (TMA)
        qt_codes = out_t if out_t is not None else \
            torch.empty(cols, (rows + 15) // 16 * 16, dtype=torch.uint8, device=dev)[:, :rows]
        qt_scales = scales_t if scales_t is not None else \
            torch.empty(scale_shape(cols, rows, tg), dtype=torch.float32, device=dev)
        qt = _tensor(qt_codes, FMT[fmt], cols, rows, qt_scales, tg, scale_fmt)
    nws = _lib.loka_quantize_workspace_size(C.byref(qx), C.byref(qq))
    ws = torch.empty(nws, dtype=torch.uint8, device=dev)
    st = _lib.loka_quantize(C.byref(qx), C.byref(qq), None if qt is None else C.byref(qt), PHASE[phase],
                            _ptr(amax), _ptr(status), _ptr(ws), nws, _stream(stream))
    _check(st, "loka_quantize")
    if transpose:
        return (out if want_q else None), scales, qt_codes, qt_scales
    return (out if want_q else None), scales


def make_linear_args(a, a_scales, b, b_scales, *, a_fmt="e4m3", b_fmt="e4m3", a_gran="row", b_gran="row",
                     a_scale_fmt="f32", b_scale_fmt="f32", norm="none", act="none", bwd_xhat=None, bwd_rstd=None,
                     save_xhat=None, save_rstd=None, amax_out=None, norm_block=256, eps=0.0, gamma=None, beta=None, bias=None, out_dtype="f32",
                     y=None, y_scales=None, precast=None, status=None, direction="fwd", keep=None, y_gran="row"):
    """Build a loka_linear_args for C = A . B^T (A [M,K], B [N,K] FP8 codes, K-major).
    y_gran: the FP8 output's scale granularity, "row" [M] or "blk_1x128" [M, ceil(N/128)]."""
    M, K = a.shape
    N = b.shape[0]
    od = {"f32": F32, "bf16": BF16, "e4m3": E4M3, "e5m2": E5M2}[out_dtype]
    dev = a.device
    if y is None:
        y = torch.empty(M, N, dtype=_TORCH_DT[od], device=dev)
    if od in (E4M3, E5M2) and y_scales is None:
        y_scales = torch.empty(scale_shape(M, N, y_gran), dtype=torch.float32, device=dev)
    args = loka_linear_args()
    args.M, args.N, args.K, args.dir = M, N, K, DIR[direction]
    args.a = _tensor(a, FMT[a_fmt], M, K, a_scales, a_gran, a_scale_fmt)
    args.b = _tensor(b, FMT[b_fmt], N, K, b_scales, b_gran, b_scale_fmt)
    args.bias = None if bias is None else bias.data_ptr()
    args.bias_dtype = F32 if bias is None else _dtype_code(bias)
    args.norm, args.norm_block, args.eps = NORM[norm], norm_block, eps
    args.gamma = None if gamma is None else gamma.data_ptr()
    args.beta = None if beta is None else beta.data_ptr()
    args.y = _tensor(y, od, M, N, y_scales, y_gran)
    args.debug_precast = None if precast is None else precast.data_ptr()
    args.status_dev = None if status is None else status.data_ptr()
    args.act = ACT[act]
    if bwd_xhat is not None:
        args.bwd_xhat, args.bwd_xhat_ld, args.bwd_rstd = bwd_xhat.data_ptr(), bwd_xhat.stride(0), bwd_rstd.data_ptr()
    if save_xhat is not None:
        args.save_xhat, args.save_xhat_ld = save_xhat.data_ptr(), save_xhat.stride(0)
    if save_rstd is not None:
        args.save_rstd = save_rstd.data_ptr()
    if amax_out is not None:
        args.amax_out = amax_out.data_ptr()
    if keep is not None:  # keep python references alive as long as args is used
        keep.extend([a, a_scales, b, b_scales, bias, gamma, beta, y, y_scales, precast, status, bwd_xhat, bwd_rstd,
                     save_xhat, save_rstd, amax_out])
    return args, y, y_scales


def _workspace(nbytes: int, device, ws=None):
    if nbytes == 0:
        return None, 0
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
    return ws, ws.numel()


def linear_workspace(args) -> int:
    """Workspace bytes loka_fp8_linear_norm needs for args (UE8M0 blockwise scale packs; else 0)."""
    return int(_lib.loka_linear_workspace_size(C.byref(args)))


def loka_fp8_linear_norm(a, a_scales, b, b_scales, stream=None, ws=None, **kw):
    """a4+a5.  Returns (y, y_scales or None).  ws: optional preallocated uint8 workspace."""
    args, y, ys = make_linear_args(a, a_scales, b, b_scales, **kw)
    ws, nws = _workspace(linear_workspace(args), a.device, ws)
    _check(_lib.loka_fp8_linear_norm(C.byref(args), None if ws is None else C.c_void_p(ws.data_ptr()), nws,
                                     _stream(stream)), "loka_fp8_linear_norm")
    return y, ys


def loka_bf16_linear_norm(a, b, stream=None, ws=None, **kw):
    """The library's BF16 (kind::f16) path with the fused epilogue: a [M,K], b [N,K] bf16 device
    tensors.  kw as make_linear_args (norm, act, gamma, beta, bias, out_dtype, y, ...).  Returns (y, ys)."""
    one = torch.ones(1, dtype=torch.float32, device=a.device)  # (scales are ignored by this path)
    args, y, ys = make_linear_args(a, one, b, one, a_gran="tensor", b_gran="tensor", **kw)
    args.a.dtype = BF16
    args.b.dtype = BF16
    nws = int(_lib.loka_bf16_linear_workspace_size(C.byref(args)))
    ws, nws = _workspace(nws, a.device, ws)
    _check(_lib.loka_bf16_linear_norm(C.byref(args), None if ws is None else C.c_void_p(ws.data_ptr()), nws,
                                      _stream(stream)), "loka_bf16_linear_norm")
    return y, ys


def _nvfp4_tensor(packed, sf, st, rows, cols):
    return loka_nvfp4_tensor(packed.data_ptr(), rows, cols, packed.stride(0), sf.data_ptr(), st.data_ptr())


def loka_quantize_nvfp4(x: torch.Tensor, amax: torch.Tensor | None = None, status: torch.Tensor | None = None,
                        out=None, stream=None):
    """NEXT-4 NVFP4 quantize.  Returns (packed uint8 [rows, cols/2], block-scale codes uint8
    [rows, cols/16], tensor scale fp32 [1]).  amax: optional device float (the global amax)."""
    rows, cols = x.shape
    dev = x.device
    if out is None:
        out = (torch.empty(rows, (cols // 2 + 15) // 16 * 16, dtype=torch.uint8, device=dev)[:, :cols // 2],
               torch.empty(rows, cols // 16, dtype=torch.uint8, device=dev),
               torch.empty(1, dtype=torch.float32, device=dev))
    packed, sf, st = out
    qx = _tensor(x, _dtype_code(x), rows, cols)
    q = _nvfp4_tensor(packed, sf, st, rows, cols)
    nws = _lib.loka_quantize_nvfp4_workspace_size(C.byref(qx))
    ws = torch.empty(nws, dtype=torch.uint8, device=dev)
    _check(_lib.loka_quantize_nvfp4(C.byref(qx), C.byref(q), _ptr(amax), _ptr(status), _ptr(ws), nws,
                                    _stream(stream)), "loka_quantize_nvfp4")
    return packed, sf, st


def make_nvfp4_linear_args(a, b, *, norm="none", norm_block=256, eps=0.0, gamma=None, beta=None, bias=None,
                           out_dtype="f32", y=None, y_scales=None, status=None, keep=None):
    """a, b: (packed, block_scales, tensor_scale) triples from loka_quantize_nvfp4 (A [M,K], B [N,K])."""
    (ap, asf, ast), (bp, bsf, bst) = a, b
    M, K = ap.shape[0], ap.shape[1] * 2
    N = bp.shape[0]
    od = {"f32": F32, "bf16": BF16, "e4m3": E4M3, "e5m2": E5M2}[out_dtype]
    dev = ap.device
    if y is None:
        y = torch.empty(M, N, dtype=_TORCH_DT[od], device=dev)
    if od in (E4M3, E5M2) and y_scales is None:
        y_scales = torch.empty(M, dtype=torch.float32, device=dev)
    args = loka_nvfp4_linear_args()
    args.M, args.N, args.K = M, N, K
    args.a = _nvfp4_tensor(ap, asf, ast, M, K)
    args.b = _nvfp4_tensor(bp, bsf, bst, N, K)
    args.bias = None if bias is None else bias.data_ptr()
    args.bias_dtype = F32 if bias is None else _dtype_code(bias)
    args.norm, args.norm_block, args.eps = NORM[norm], norm_block, eps
    args.gamma = None if gamma is None else gamma.data_ptr()
    args.beta = None if beta is None else beta.data_ptr()
    args.y = _tensor(y, od, M, N, y_scales, "row")
    args.status_dev = None if status is None else status.data_ptr()
    if keep is not None:
        keep.extend([ap, asf, ast, bp, bsf, bst, bias, gamma, beta, y, y_scales, status])
    return args, y, y_scales


def loka_nvfp4_linear_norm(a, b, stream=None, ws=None, **kw):
    """NEXT-4 NVFP4 linear (+bias/norm) on the block-scaled tensor cores.  Returns (y, y_scales)."""
    args, y, ys = make_nvfp4_linear_args(a, b, **kw)
    ws, nws = _workspace(int(_lib.loka_nvfp4_linear_workspace_size(C.byref(args))), y.device, ws)
    _check(_lib.loka_nvfp4_linear_norm(C.byref(args), None if ws is None else C.c_void_p(ws.data_ptr()), nws,
                                       _stream(stream)), "loka_nvfp4_linear_norm")
    return y, ys


def loka_dequant_reduce(codes, scales, fmt="e5m2", out=None, stream=None):
    """NEXT-4 (D39): out = sum_p decode(codes[p]) * scales[p][:, None] in FP32, rank order.  codes /
    scales: lists of P device tensors, or of raw device addresses (ints, e.g. peer symmetric memory)
    given with out= (rows, cols and ld are taken from out and ld_codes on the first tensor)."""
    P = len(codes)
    c0 = codes[0]
    rows, cols = out.shape if out is not None else c0.shape
    ld = c0.stride(0) if isinstance(c0, torch.Tensor) else (cols + 15) // 16 * 16
    if out is None:
        out = torch.empty(rows, cols, dtype=torch.float32, device=c0.device)
    ca = (C.c_void_p * P)(*[c.data_ptr() if isinstance(c, torch.Tensor) else int(c) for c in codes])
    sa = (C.c_void_p * P)(*[s.data_ptr() if isinstance(s, torch.Tensor) else int(s) for s in scales])
    _check(_lib.loka_dequant_reduce(P, ca, sa, FMT[fmt], rows, cols, ld, C.c_void_p(out.data_ptr()), out.stride(0),
                                    _stream(stream)), "loka_dequant_reduce")
    return out


def loka_grouped_fp8_linear(args_list, stream=None, ws=None):
    """a6.  args_list: sequence of loka_linear_args (see make_linear_args)."""
    G = len(args_list)
    arr = (loka_linear_args * G)(*args_list)
    dev = torch.device("cuda", torch.cuda.current_device())
    ws, nws = _workspace(int(_lib.loka_grouped_workspace_size(G, arr)), dev, ws)
    _check(_lib.loka_grouped_fp8_linear(G, arr, None if ws is None else C.c_void_p(ws.data_ptr()), nws,
                                        _stream(stream)), "loka_grouped_fp8_linear")


def loka_grouped_bf16_linear(problems, stream=None, out_dtype="bf16", keep=None):
    """The library's BF16 grouped denominator: problems = [(a [M,K] bf16, b [N,K] bf16[, y])] device
    tensors; one kind::f16 CTA-pair launch per 32 problems.  Returns the outputs."""
    one = torch.ones(1, dtype=torch.float32, device=problems[0][0].device)
    keep = [] if keep is None else keep
    args, ys = [], []
    for pr in problems:
        a, b = pr[0], pr[1]
        ar, y, _ = make_linear_args(a, one, b, one, a_gran="tensor", b_gran="tensor", out_dtype=out_dtype,
                                    y=pr[2] if len(pr) > 2 else None, keep=keep)
        ar.a.dtype = BF16
        ar.b.dtype = BF16
        args.append(ar)
        ys.append(y)
    arr = (loka_linear_args * len(args))(*args)
    _check(_lib.loka_grouped_bf16_linear(len(args), arr, _stream(stream)), "loka_grouped_bf16_linear")
    return ys


def loka_probe_error(pairs, floor_rel: float = 1e-6, stream=None, stats=None, ws=None, global_sum_count=None):
    """a7.  pairs: [(out, ref)] device tensors (f32/bf16, 2-D).  Returns a float64 tensor [L, 5]
    viewing the device loka_probe_stats array (mere, max_rel, sum_abs_ref, count*, n_floored*)
    where the last two are int64 bit patterns; use probe_stats_to_dicts().  global_sum_count: device
    float64 [L, 2] (sum |ref|, count) of the whole sharded layers -> loka_probe_error_global."""
    L = len(pairs)
    arr = (loka_probe_pair * L)()
    for i, (o, r) in enumerate(pairs):
        arr[i] = loka_probe_pair(o.data_ptr(), _dtype_code(o), r.data_ptr(), _dtype_code(r), o.shape[0], o.shape[1],
                                 o.stride(0), r.stride(0))
    dev = pairs[0][0].device
    if stats is None:
        stats = torch.empty(L, 5, dtype=torch.float64, device=dev)
    nws = _lib.loka_probe_workspace_size(L, arr)
    if ws is None or ws.numel() < nws:
        ws = torch.empty(nws, dtype=torch.uint8, device=dev)
    if global_sum_count is not None:
        g = global_sum_count.to(device=dev, dtype=torch.float64).contiguous()
        _check(_lib.loka_probe_error_global(L, arr, floor_rel, C.c_void_p(g.data_ptr()), C.c_void_p(stats.data_ptr()),
                                            C.c_void_p(ws.data_ptr()), nws, _stream(stream)), "loka_probe_error_global")
    else:
        _check(_lib.loka_probe_error(L, arr, floor_rel, C.c_void_p(stats.data_ptr()), C.c_void_p(ws.data_ptr()), nws,
                                     _stream(stream)), "loka_probe_error")
    return stats


def probe_merge(per_rank):
    """Combine per-rank probe statistics (lists of dicts, one list per rank, same layers) with the
    library's host loka_probe_merge."""
    R = len(per_rank)
    L = len(per_rank[0]) if R else 0
    parts = (loka_probe_stats * max(1, R * L))()
    for r, lst in enumerate(per_rank):
        for l, st in enumerate(lst):
            parts[r * L + l] = loka_probe_stats(st["mere"], st["max_rel"], st["sum_abs_ref"], int(st["count"]),
                                                int(st["n_floored"]))
    out = (loka_probe_stats * max(1, L))()
    _check(_lib.loka_probe_merge(R, L, parts, out), "loka_probe_merge")
    return [dict(mere=out[l].mere, max_rel=out[l].max_rel, sum_abs_ref=out[l].sum_abs_ref, count=int(out[l].count),
                 n_floored=int(out[l].n_floored)) for l in range(L)]


def probe_stats_to_dicts(stats: torch.Tensor):
    s = stats.detach().cpu()
    ints = s.view(torch.int64)
    return [dict(mere=float(s[i, 0]), max_rel=float(s[i, 1]), sum_abs_ref=float(s[i, 2]), count=int(ints[i, 3]),
                 n_floored=int(ints[i, 4])) for i in range(s.shape[0])]


def loka_dispatch_select(candidates, baseline_time_us: float, mere_budget: float = 0.2,
                         min_speedup: float = 1.05) -> int:
    """a8.  candidates: [(id, direction, mere, time_us)].  Returns index or -1 (baseline)."""
    n = len(candidates)
    ids = [c[0].encode() for c in candidates]
    arr = (loka_candidate * max(n, 1))()
    for i, (cid, d, m, t) in enumerate(candidates):
        arr[i] = loka_candidate(ids[i], DIR[d] if isinstance(d, str) else int(d), float(m), float(t))
    out = C.c_int32(-2)
    _check(_lib.loka_dispatch_select(arr, n, baseline_time_us, mere_budget, min_speedup, C.byref(out)),
           "loka_dispatch_select")
    return out.value


def launch_count() -> int:
    return int(_lib.loka_launch_count())


def device_supported(device: int = 0) -> bool:
    return bool(_lib.loka_device_supported(device))


def version() -> int:
    return int(_lib.loka_version())


def debug_hang_info(reset: bool = True):
    """(count, tag, block, thread|parity<<32) of pipeline-watchdog timeouts (0 count = healthy)."""
    info = (C.c_uint64 * 3)()
    n = _lib.loka_debug_hang_info(info, 1 if reset else 0)
    return int(n), int(info[0]), int(info[1]), int(info[2])


def debug_trace(enable: int = -1, n: int = 0):
    """Phase-trace control/readout (see include/loka.h loka_debug_trace). Returns a list of stamps."""
    buf = (C.c_uint64 * max(n, 1))()
    got = _lib.loka_debug_trace(enable, buf if n else None, n)
    return [int(buf[i]) for i in range(max(got, 0))]


def loka_quantize_grouped(xs, fmt: str = "e4m3", scale_fmt: str = "f32", outs=None, scales=None, status=None,
                          stream=None):
    """Grouped ROW quantize of several 2-D tensors in one launch.  Returns [(codes, scales)]."""
    G = len(xs)
    xa = (loka_tensor * G)()
    qa = (loka_tensor * G)()
    res = []
    for g, x in enumerate(xs):
        r, c = x.shape
        o = outs[g] if outs is not None else torch.empty(r, (c + 15) // 16 * 16, dtype=torch.uint8,
                                                         device=x.device)[:, :c]
        s = scales[g] if scales is not None else torch.empty(r, dtype=torch.float32, device=x.device)
        xa[g] = _tensor(x, _dtype_code(x), r, c)
        qa[g] = _tensor(o, FMT[fmt], r, c, s, "row", scale_fmt)
        res.append((o, s))
    _check(_lib.loka_quantize_grouped(G, xa, qa, _ptr(status), _stream(stream)), "loka_quantize_grouped")
    return res


def make_stack_args(xq, xs, ws, norms="layer", out_dtype="bf16", y=None, y_scales=None, eps=None, status=None,
                    save=None, precast=None):
    """loka_stack_args for h_{l+1} = norm_l(h_l W_l^T): xq/xs = e4m3 codes + row scales of the input,
    ws = [(codes [N_l, K_l], row scales [N_l])].  save: optional list of L-1 (codes, scales) device
    tensors receiving the hand-offs h_1..h_{L-1}.  Returns (args, y, y_scales)."""
    L = len(ws)
    M, K0 = xq.shape
    a = loka_stack_args()
    a.L, a.M = L, M
    dims = [K0] + [w.shape[0] for w, _ in ws]
    for i, d in enumerate(dims):
        a.dims[i] = d
    a.x = _tensor(xq, E4M3, M, K0, xs, "row")
    for l, (wq, wsc) in enumerate(ws):
        a.w[l] = _tensor(wq, E4M3, wq.shape[0], wq.shape[1], wsc, "row")
        a.norm[l] = NORM[norms if isinstance(norms, str) else norms[l]]
        a.eps[l] = 0.0 if eps is None else float(eps)
    od = {"f32": F32, "bf16": BF16, "e4m3": E4M3, "e5m2": E5M2}[out_dtype]
    N = dims[-1]
    if y is None:
        y = torch.empty(M, N, dtype=_TORCH_DT[od], device=xq.device)
    if od in (E4M3, E5M2) and y_scales is None:
        y_scales = torch.empty(M, dtype=torch.float32, device=xq.device)
    a.y = _tensor(y, od, M, N, y_scales, "row")
    a.status_dev = None if status is None else status.data_ptr()
    for l, hs in enumerate(save or []):
        a.h[l] = _tensor(hs[0], E4M3, M, dims[l + 1], hs[1], "row")
    for l, pc in enumerate(precast or []):  # tests: FP32 [M, dims[l+1]] pre-cast values of layer l
        a.debug_precast[l] = None if pc is None else pc.data_ptr()
    nws = int(_lib.loka_stack_workspace_size(C.byref(a)))
    if nws:
        ws = torch.empty(nws, dtype=torch.uint8, device=xq.device)
        a.ws, a.ws_bytes = ws.data_ptr(), nws
        a._keep_ws = ws  # the workspace lives as long as the args object
    return a, y, y_scales


def loka_fp8_mlp_stack(xq, xs, ws, stream=None, **kw):
    """Whole layer stack in one launch (intermediate activations stay on chip)."""
    a, y, ys = make_stack_args(xq, xs, ws, **kw)
    _check(_lib.loka_fp8_mlp_stack(C.byref(a), _stream(stream)), "loka_fp8_mlp_stack")
    return y, ys


class InputTracker:
    """NEXT-2: batched Welford tracker of one layer's input distribution
    (feature mean + K x K scatter in FP32 on the device), wrapping loka_probe_track_input."""

    def __init__(self, k: int, device=None):
        dev = torch.device("cuda") if device is None else device
        self.mean = torch.zeros(k, dtype=torch.float32, device=dev)
        self.scatter = torch.zeros(k, k, dtype=torch.float32, device=dev)
        self.state = loka_welford_state(0, k, self.mean.data_ptr(), self.scatter.data_ptr())
        self._ws = None

    @property
    def n(self) -> int:
        return int(self.state.n)

    def update(self, x: torch.Tensor, stream=None):
        assert x.dtype == torch.bfloat16 and x.dim() == 2 and x.stride(1) == 1
        t = _tensor(x, BF16, x.shape[0], x.shape[1])
        nws = int(_lib.loka_probe_track_workspace_size(C.byref(self.state), x.shape[0]))
        if self._ws is None or self._ws.numel() < nws:
            self._ws = torch.empty(max(nws, 1), dtype=torch.uint8, device=x.device)
        _check(_lib.loka_probe_track_input(C.byref(self.state), C.byref(t), C.c_void_p(self._ws.data_ptr()),
                                           self._ws.numel(), _stream(stream)), "loka_probe_track_input")

    def covariance(self, stream=None) -> torch.Tensor:
        """The unbiased covariance Sigma / (n - 1), computed by libloka."""
        out = torch.empty_like(self.scatter)
        _check(_lib.loka_probe_track_covariance(C.byref(self.state), C.c_void_p(out.data_ptr()), _stream(stream)),
               "loka_probe_track_covariance")
        return out

    def factor(self, eps_rel: float = 1e-6, escalations: int = 4, stream=None):
        """(L_Sigma, eps): jittered Cholesky of the unbiased covariance Sigma / (n - 1),
        the 1/(n-1) applied inside the factorisation kernel.  Synchronous (reads the pivot status)."""
        if self.n < 2:
            raise ValueError("the covariance needs n > 1 (PAPER.md:301)")
        return cholesky_jittered(self.scatter, eps_rel, escalations, a_scale=1.0 / (self.n - 1), stream=stream)

    def sample(self, b: int, seed: int, offset: int = 0, eps_rel: float = 1e-6, out_dtype=torch.float32, stream=None):
        """T' = 1 mu^T + Z L_Sigma^T from the tracked statistics."""
        l_sigma, _ = self.factor(eps_rel, stream=stream)
        return sample_input(self.mean, l_sigma, b, seed, offset, out_dtype, stream)


# ---- NEXT-3: weight tracker and learned-distribution sampling ----------------
_ws_cache = {}


def _scratch(nbytes: int, device, tag: str):
    key = (tag, str(device))
    t = _ws_cache.get(key)
    if t is None or t.numel() < nbytes:
        t = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device)
        _ws_cache[key] = t
    return t


def philox_normal(n: int, seed: int, offset: int = 0, device=None, out=None, stream=None) -> torch.Tensor:
    """n standard normals of the Philox4x64-10 stream (seed, offset) (loka_philox_normal, D31)."""
    dev = torch.device("cuda") if device is None else torch.device(device)
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=dev)
    _check(_lib.loka_philox_normal(seed & (2**64 - 1), offset, n, _ptr(out), _stream(stream)), "loka_philox_normal")
    return out


def cholesky_jittered(a: torch.Tensor, eps_rel: float = 1e-6, escalations: int = 4, a_scale: float = 1.0,
                      out=None, stream=None):
    """(L, eps_used) with L L^T = a_scale sym(a) + eps I (loka_cholesky_jittered; synchronous)."""
    assert a.dtype == torch.float32 and a.dim() == 2 and a.shape[0] == a.shape[1] and a.stride(1) == 1
    n = a.shape[0]
    if out is None:
        out = torch.empty(n, n, dtype=torch.float32, device=a.device)
    ws = _scratch(int(_lib.loka_cholesky_workspace_size(n)), a.device, "chol")
    eps = C.c_float(0.0)
    _check(_lib.loka_cholesky_jittered(_ptr(a), a.stride(0), n, a_scale, eps_rel, escalations, _ptr(out),
                                       out.stride(0), C.byref(eps), _ptr(ws), ws.numel(), _stream(stream)),
           "loka_cholesky_jittered")
    return out, float(eps.value)


def _sample_out(rows, cols, out_dtype, device, out):
    if out is None:
        out = torch.empty(rows, cols, dtype=out_dtype, device=device)
    assert out.dim() == 2 and out.stride(1) == 1 and tuple(out.shape) == (rows, cols)
    return out, _tensor(out, _dtype_code(out), rows, cols, ld=out.stride(0))


def sample_input(mean: torch.Tensor, l_sigma: torch.Tensor, b: int, seed: int, offset: int = 0,
                 out_dtype=torch.float32, stream=None, out=None) -> torch.Tensor:
    """T' = 1 mean^T + Z L_Sigma^T (loka_probe_sample_input)."""
    k = mean.numel()
    assert mean.is_contiguous() and l_sigma.is_contiguous() and tuple(l_sigma.shape) == (k, k)
    out, t = _sample_out(b, k, out_dtype, mean.device, out)
    ws = _scratch(int(_lib.loka_probe_sample_workspace_size(b, k, 0)), mean.device, "sample")
    _check(_lib.loka_probe_sample_input(_ptr(mean), _ptr(l_sigma), k, b, seed & (2**64 - 1), offset, C.byref(t),
                                        _ptr(ws), ws.numel(), _stream(stream)), "loka_probe_sample_input")
    return out


def sample_weight(mean: torch.Tensor, l_u: torch.Tensor, l_v: torch.Tensor, seed: int, offset: int = 0,
                  out_dtype=torch.float32, stream=None, out=None) -> torch.Tensor:
    """W' = mean + L_U Z L_V^T (loka_probe_sample_weight)."""
    m, n = mean.shape
    assert mean.is_contiguous() and l_u.is_contiguous() and l_v.is_contiguous()
    assert tuple(l_u.shape) == (m, m) and tuple(l_v.shape) == (n, n)
    out, t = _sample_out(m, n, out_dtype, mean.device, out)
    ws = _scratch(int(_lib.loka_probe_sample_workspace_size(m, n, 1)), mean.device, "sample")
    _check(_lib.loka_probe_sample_weight(_ptr(mean), _ptr(l_u), _ptr(l_v), m, n, seed & (2**64 - 1), offset,
                                         C.byref(t), _ptr(ws), ws.numel(), _stream(stream)), "loka_probe_sample_weight")
    return out


class WeightTracker:
    """NEXT-3: matrix-normal tracker of one weight W [M, N] ~ MN(mean, U, V) on the
    device (FP32), wrapping loka_probe_track_weight_init / loka_probe_track_weight."""

    def __init__(self, w0: torch.Tensor, momentum: float = 0.95, eps_rel: float = 1e-6, stream=None):
        assert w0.dim() == 2 and w0.stride(1) == 1 and w0.dtype in (torch.float32, torch.bfloat16)
        m, n = w0.shape
        dev = w0.device
        self.mean = torch.empty(m, n, dtype=torch.float32, device=dev)
        self.U = torch.empty(m, m, dtype=torch.float32, device=dev)
        self.V = torch.empty(n, n, dtype=torch.float32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.state = loka_matnorm_state(m, n, 0, momentum, eps_rel, self.mean.data_ptr(), self.U.data_ptr(),
                                        self.V.data_ptr())
        t = _tensor(w0, _dtype_code(w0), m, n, ld=w0.stride(0))
        _check(_lib.loka_probe_track_weight_init(C.byref(self.state), C.byref(t), _stream(stream)),
               "loka_probe_track_weight_init")
        self._ws = torch.empty(int(_lib.loka_probe_track_weight_workspace_size(C.byref(self.state))),
                               dtype=torch.uint8, device=dev)

    @property
    def count(self) -> int:
        return int(self.state.count)

    def update(self, w: torch.Tensor, stream=None):
        assert w.dim() == 2 and w.stride(1) == 1 and tuple(w.shape) == (self.state.M, self.state.N)
        t = _tensor(w, _dtype_code(w), w.shape[0], w.shape[1], ld=w.stride(0))
        _check(_lib.loka_probe_track_weight(C.byref(self.state), C.byref(t), _ptr(self.status),
                                            C.c_void_p(self._ws.data_ptr()), self._ws.numel(), _stream(stream)),
               "loka_probe_track_weight")

    def sample(self, seed: int, offset: int = 0, eps_rel: float = 1e-6, out_dtype=torch.float32, stream=None):
        """W' = mean + L_U Z L_V^T with L_U L_U^T = U + eps I, L_V L_V^T = V + eps I."""
        l_u, _ = cholesky_jittered(self.U, eps_rel, stream=stream)
        l_v, _ = cholesky_jittered(self.V, eps_rel, stream=stream)
        return sample_weight(self.mean, l_u, l_v, seed, offset, out_dtype, stream)
