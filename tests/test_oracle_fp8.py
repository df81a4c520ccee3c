"""Pins for oracle/fp8.py (O1/O2) against closed forms and two independent library casts:
torch's CPU float8 cast (after clamping to +-max: torch itself does not saturate) and the
CUDA toolkit's host-side __nv_cvt_float_to_fp8(..., __NV_SATFINITE, ...) (cuda_fp8.hpp)."""
import json
import os
import subprocess

import numpy as np
import pytest
import torch

from oracle import fp8

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
TORCH_DT = {"e4m3": torch.float8_e4m3fn, "e5m2": torch.float8_e5m2}


def test_closed_form_constants():
    t4, t5 = fp8.decode_table("e4m3"), fp8.decode_table("e5m2")
    # E4M3FN: max 448 = 0x7E; min normal 2^-6 = 0x08; min subnormal 2^-9 = 0x01; NaN 0x7F/0xFF
    assert fp8.max_code("e4m3") == 0x7E and t4[0x7E] == GOLD["e4m3_max"]["value"] == 448.0
    assert t4[0x08] == 2.0 ** -6 and t4[0x07] == 7 * 2.0 ** -9 and t4[0x01] == 2.0 ** -9
    assert np.isnan(t4[0x7F]) and np.isnan(t4[0xFF]) and np.isnan(t4).sum() == 2
    assert t4[0x80] == 0.0 and np.signbit(t4[0x80]) and t4[0xFE] == -448.0
    # E5M2: max 57344 = 0x7B; Inf 0x7C/0xFC; NaN 0x7D-0x7F; min normal 2^-14; min subnormal 2^-16
    assert fp8.max_code("e5m2") == 0x7B and t5[0x7B] == GOLD["e5m2_max"]["value"] == 57344.0
    assert t5[0x7C] == np.inf and t5[0xFC] == -np.inf
    assert all(np.isnan(t5[c]) for c in (0x7D, 0x7E, 0x7F, 0xFD, 0xFE, 0xFF)) and np.isnan(t5).sum() == 6
    assert t5[0x04] == 2.0 ** -14 and t5[0x01] == 2.0 ** -16
    # every finite value is (1+m/2^mb) 2^(e-bias) or m 2^(1-bias-mb): count distinct finite values
    assert len(set(t4[np.isfinite(t4)].tolist())) == 253  # 254 finite codes, +0 == -0
    assert len(set(t5[np.isfinite(t5)].tolist())) == 247


@pytest.mark.parametrize("f", ["e4m3", "e5m2"])
def test_decode_matches_torch(f):
    codes = torch.arange(256, dtype=torch.uint8)
    ref = codes.view(TORCH_DT[f]).to(torch.float64).numpy()
    ours = fp8.decode_table(f)
    same = (ref == ours) | (np.isnan(ref) & np.isnan(ours))
    assert same.all()
    assert (np.signbit(ref) == np.signbit(ours))[~np.isnan(ref)].all()


@pytest.mark.parametrize("f", ["e4m3", "e5m2"])
def test_encode_decode_identity_all_codes(f):
    """decode(encode(v)) = v for every v in the value set, all 256 codes."""
    t = fp8.decode_table(f)
    for c in range(256):
        if np.isnan(t[c]):
            continue
        if np.isinf(t[c]):  # saturating encode: +-Inf -> +-max
            assert fp8.encode(np.array([t[c]]), f)[0] == (fp8.max_code(f) | (c & 0x80))
            continue
        assert fp8.encode(np.array([t[c]]), f)[0] == c


def _stratified_f32(f, n_random=1 << 21, seed=0):
    """float32 test values: every code, every midpoint and its fp32 neighbours, random bit
    patterns over all exponents, log-uniform values in the FP8 range, and specials."""
    rng = np.random.default_rng(seed)
    t = fp8.decode_table(f)
    pos = t[: fp8.max_code(f) + 1]
    mids = ((pos[:-1] + pos[1:]) / 2).astype(np.float32)
    vals = [pos.astype(np.float32), mids, np.nextafter(mids, np.float32(np.inf)),
            np.nextafter(mids, np.float32(0)), np.float32(pos[-1]) * np.float32(1.0001)]
    bits = rng.integers(0, 1 << 32, n_random, dtype=np.uint64).astype(np.uint32)
    rb = bits.view(np.float32)
    vals.append(rb[np.isfinite(rb)])
    lo, hi = np.log2(pos[1]) - 3, np.log2(pos[-1]) + 2
    vals.append(np.exp2(rng.uniform(lo, hi, n_random)).astype(np.float32))
    fmax = np.float32(pos[-1])
    vals.append(np.array([0.0, np.inf, 1e-45, 1e-38, 3.4e38, fmax, np.nextafter(fmax, np.float32(np.inf)),
                          464.0, 465.0, 61439.0, 61440.0, 2.0 ** -10, 1.5 * 2.0 ** -10, 1e-10], np.float32))
    v = np.concatenate([np.asarray(a, np.float32).reshape(-1) for a in vals])
    return np.concatenate([v, -v])


@pytest.mark.parametrize("f", ["e4m3", "e5m2"])
def test_encode_matches_torch_cpu_cast(f):
    v = _stratified_f32(f)
    fmax = fp8.max_finite(f)
    tv = torch.from_numpy(v).clamp(-fmax, fmax)  # torch casts RNE but does not saturate
    ref = tv.to(TORCH_DT[f]).view(torch.uint8).numpy()
    ours = fp8.encode(v.astype(np.float64), f)
    bad = np.nonzero(ref != ours)[0]
    assert bad.size == 0, [(float(v[i]), int(ref[i]), int(ours[i])) for i in bad[:10]]


@pytest.mark.parametrize("f", ["e4m3", "e5m2"])
def test_encode_matches_cuda_fp8_host(f, fp8_host_cast, tmp_path):
    v = _stratified_f32(f, seed=1)
    fi, fo = tmp_path / "in.f32", tmp_path / "out.u8"
    v.tofile(fi)
    subprocess.run([fp8_host_cast, f, str(fi), str(fo)], check=True)
    ref = np.fromfile(fo, dtype=np.uint8)
    ours = fp8.encode(v.astype(np.float64), f)
    bad = np.nonzero(ref != ours)[0]
    assert bad.size == 0, [(float(v[i]), int(ref[i]), int(ours[i])) for i in bad[:10]]


def test_torch_spot_values_and_sign_of_underflow():
    """SURVEY.md §0 probed torch values; underflow keeps the sign (-1e-10 -> 0x80)."""
    v = np.array([448.0, -1e-10, 2.0 ** -10, 1.5 * 2.0 ** -10, 1e30, -np.inf], np.float64)
    assert fp8.encode(v, "e4m3").tolist() == [0x7E, 0x80, 0x00, 0x01, 0x7E, 0xFE]
    assert fp8.encode(np.array([61439.0, 61440.0, 1e9]), "e5m2").tolist() == [0x7B, 0x7B, 0x7B]


@pytest.mark.slow
@pytest.mark.parametrize("f", ["e4m3", "e5m2"])
def test_encode_exhaustive_2p32(f, fp8_host_cast, tmp_path):
    """All 2^32 FP32 bit patterns (non-NaN) vs cuda_fp8.hpp host SATFINITE cast."""
    fo = tmp_path / "sweep.u8"
    subprocess.run([fp8_host_cast, "sweep", f, str(fo)], check=True)
    ref = np.memmap(fo, dtype=np.uint8, mode="r")
    step = 1 << 26
    for base in range(0, 1 << 32, step):
        bits = np.arange(base, base + step, dtype=np.uint64).astype(np.uint32)
        v = bits.view(np.float32)
        ok = ~np.isnan(v)
        ours = fp8.encode(v[ok].astype(np.float64), f)
        assert np.array_equal(ours, np.asarray(ref[base:base + step])[ok]), hex(base)
