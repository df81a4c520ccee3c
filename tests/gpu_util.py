"""Helpers for the -m gpu parity tests: device inputs from synth/, oracle comparisons."""
import numpy as np
import torch

import oracle
import synth

DEV = "cuda"


def f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().double().numpy() if t.dtype != torch.float64 else t.cpu().numpy()


def assert_bytes_equal(gpu_u8: torch.Tensor, ref_u8: np.ndarray, what=""):
    g = gpu_u8.cpu().numpy()
    bad = np.argwhere(g != ref_u8)
    assert bad.size == 0, f"{what}: {len(bad)} code mismatches, first {[(tuple(i), int(g[tuple(i)]), int(ref_u8[tuple(i)])) for i in bad[:5]]}"


def assert_scales_equal(gpu_f32: torch.Tensor, ref_f32: np.ndarray, what=""):
    g = gpu_f32.cpu().numpy().astype(np.float32).view(np.uint32)
    r = np.asarray(ref_f32, np.float32).view(np.uint32).reshape(g.shape)
    bad = np.argwhere(g != r)
    assert bad.size == 0, f"{what}: {len(bad)} scale mismatches, first {[(tuple(i), g[tuple(i)], r[tuple(i)]) for i in bad[:5]]}"


def guarded_rel_err(y: np.ndarray, yo: np.ndarray) -> float:
    """DESIGN.md D18: max |y - y_o| / max(|y_o|, rms_row(y_o))."""
    rms = np.sqrt(np.mean(yo ** 2, axis=1, keepdims=True))
    guard = np.maximum(np.abs(yo), rms)
    guard = np.where(guard > 0, guard, 1.0)
    return float(np.max(np.abs(y - yo) / guard)) if y.size else 0.0


def to_dev_padded(x: torch.Tensor, align_elems: int = 16) -> torch.Tensor:
    """Copy a 2-D tensor to the GPU in storage whose leading dimension is a multiple of
    ``align_elems`` (the C ABI requires ld * elem_size % 16 == 0)."""
    rows, cols = x.shape
    ld = -(-cols // align_elems) * align_elems
    buf = torch.zeros(rows, ld, dtype=x.dtype, device=DEV)
    buf[:, :cols].copy_(x.to(DEV))
    return buf[:, :cols]
