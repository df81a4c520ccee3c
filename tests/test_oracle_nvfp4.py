"""Pins for oracle/nvfp4.py (D35-D38).

* E2M1 encode vs the CUDA toolkit's host cast (cuda_fp4.hpp __nv_cvt_float_to_fp4, E2M1,
  round-to-nearest) on every code, every midpoint and its FP32 neighbours, random bit patterns,
  log-uniform values and specials (exhaustive 2^32 sweep with LOKA_SLOW=1); decode pinned by
  encode(decode(c)) == c through that library cast.
* Quantize vs an independent per-element re-derivation in float32 IEEE arithmetic with the
  library casts (cuda_fp8.hpp for the E4M3 block scale, cuda_fp4.hpp for the codes).
* A hand-worked example, zero and underflowing blocks, the error bound, packing order.
"""
import subprocess

import numpy as np
import pytest
import torch

from oracle import nvfp4

STEPS = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])


def _host4(helper, v, tmp_path, tag="x"):
    fi, fo = tmp_path / f"{tag}.f32", tmp_path / f"{tag}.u8"
    np.asarray(v, np.float32).tofile(fi)
    subprocess.run([helper, str(fi), str(fo)], check=True)
    return np.fromfile(fo, dtype=np.uint8)


def _host8(helper, v, tmp_path, tag="y"):
    fi, fo = tmp_path / f"{tag}.f32", tmp_path / f"{tag}.u8"
    np.asarray(v, np.float32).tofile(fi)
    subprocess.run([helper, "e4m3", str(fi), str(fo)], check=True)
    return np.fromfile(fo, dtype=np.uint8)


def _stratified(seed=0, n=200000):
    rng = np.random.default_rng(seed)
    pos = STEPS.astype(np.float32)
    mids = ((pos[:-1] + pos[1:]) / 2).astype(np.float32)
    vals = [pos, mids, np.nextafter(mids, np.float32(np.inf)), np.nextafter(mids, np.float32(0)),
            np.array([6.0001, 7.0, 1e30, np.inf, 1e-45, 1e-30, 0.25, 0.2499999], np.float32)]
    bits = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32).view(np.float32)
    vals.append(bits[np.isfinite(bits)])
    vals.append(np.exp2(rng.uniform(-6, 4, n)).astype(np.float32))
    v = np.concatenate([np.asarray(a, np.float32).reshape(-1) for a in vals])
    return np.concatenate([v, -v])


def test_e2m1_decode_via_library_encode(fp4_host_cast, tmp_path):
    """Every code's decoded value is encoded back to the same code by cuda_fp4.hpp (-0 -> 8)."""
    vals = nvfp4.E2M1_TABLE.copy()
    vals[8] = -0.0
    assert np.array_equal(_host4(fp4_host_cast, vals, tmp_path), np.arange(16, dtype=np.uint8))
    assert nvfp4.E2M1_TABLE.max() == 6.0 and nvfp4.E2M1_TABLE[1] == 0.5  # max finite, min subnormal


def test_e2m1_encode_matches_cuda_fp4_host(fp4_host_cast, tmp_path):
    v = _stratified()
    ref = _host4(fp4_host_cast, v, tmp_path)
    ours = nvfp4.e2m1_encode(v.astype(np.float64))
    bad = np.nonzero(ref != ours)[0]
    assert bad.size == 0, [(float(v[i]), int(ref[i]), int(ours[i])) for i in bad[:10]]


@pytest.mark.slow
def test_e2m1_encode_exhaustive_2p32(fp4_host_cast, tmp_path):
    fo = tmp_path / "sweep4.u8"
    subprocess.run([fp4_host_cast, "sweep", str(fo)], check=True)
    ref = np.memmap(fo, dtype=np.uint8, mode="r")
    step = 1 << 26
    for base in range(0, 1 << 32, step):
        v = np.arange(base, base + step, dtype=np.uint64).astype(np.uint32).view(np.float32)
        ok = ~np.isnan(v)
        assert np.array_equal(nvfp4.e2m1_encode(v[ok].astype(np.float64)), np.asarray(ref[base:base + step])[ok]), \
            hex(base)


def test_pack_order():
    c = np.array([[1, 2, 3, 15]], np.uint8)
    p = nvfp4.pack(c)
    assert p.tolist() == [[0x21, 0xF3]]  # element 2j in the low nibble
    assert np.array_equal(nvfp4.unpack(p), c)


def _brute(x, fp8_helper, fp4_helper, tmp_path):
    """Independent re-derivation: float32 IEEE numpy ops + the toolkit's host casts."""
    x = np.asarray(x, np.float32)
    rows, cols = x.shape
    A = np.float32(np.abs(x).max())
    if A == 0:
        s_t = r_t = np.float32(1)
    else:
        with np.errstate(over="ignore"):
            s_t, r_t = A / np.float32(2688), np.float32(2688) / A
        if np.isinf(r_t):  # DESIGN.md D1b: an overflowing reciprocal is FLT_MAX
            r_t = np.finfo(np.float32).max
    a_b = np.abs(x.reshape(rows, cols // 16, 16)).max(axis=2).astype(np.float32)
    u = (a_b * r_t).astype(np.float32)
    sbv = (u / np.float32(6)).astype(np.float32)
    sf = _host8(fp8_helper, sbv.reshape(-1), tmp_path, "sf").reshape(rows, cols // 16)
    d = torch.from_numpy(sf.copy()).view(torch.float8_e4m3fn).float().numpy()
    codes = np.zeros((rows, cols), np.uint8)
    for i in range(rows):
        for b in range(cols // 16):
            blk = x[i, 16 * b:16 * b + 16]
            if d[i, b] == 0:
                v = np.copysign(np.float32(0), blk)
            else:
                with np.errstate(over="ignore"):
                    rb = np.float32(r_t / np.float32(d[i, b]))
                if np.isinf(rb):
                    rb = np.finfo(np.float32).max
                v = (blk * rb).astype(np.float32)
            codes[i, 16 * b:16 * b + 16] = _host4(fp4_helper, v, tmp_path, "c")
    packed = (codes[:, 0::2] | (codes[:, 1::2] << 4)).astype(np.uint8)
    return packed, sf, np.float32(s_t)


@pytest.mark.parametrize("kind", ["gauss", "heavy", "tiny_blocks", "tiny_tensor"])
def test_quantize_matches_bruteforce(kind, fp8_host_cast, fp4_host_cast, tmp_path):
    rng = np.random.default_rng({"gauss": 0, "heavy": 1, "tiny_blocks": 2, "tiny_tensor": 3}[kind])
    rows, cols = 6, 96
    x = rng.standard_normal((rows, cols)).astype(np.float32)
    if kind == "heavy":
        x *= np.exp(rng.standard_normal((rows, 1)) * 3).astype(np.float32)
    if kind == "tiny_blocks":  # blocks far below the tensor max: block scales underflow / subnormal
        x[:, 16:48] *= np.float32(1e-6)
        x[0, 0] = 1e4
        x[2, 64:80] = 0
    if kind == "tiny_tensor":  # D1b: A < 2688 / FLT_MAX, the tensor reciprocal overflows FP32
        x *= np.float32(1e-37)
        x[1, 0:16] *= np.float32(1e-3)
    p, sf, st = nvfp4.quantize(x.astype(np.float64))
    bp, bsf, bst = _brute(x, fp8_host_cast, fp4_host_cast, tmp_path)
    assert np.array_equal(sf, bsf)
    assert np.array_equal(p, bp)
    assert st.view(np.uint32)[0] == np.float32(bst).view(np.uint32)


def test_worked_example():
    """Row 0: block 0 = [6, 3, 1.5, 0.75, -6, 0, ...] sets A = 6: s_t = fl32(6/2688), r_t = 448,
    block scale = E4M3(fl32(6*448)/6) = 448 (0x7E), r_b = 1, codes = E2M1(x): 6 -> 7, 3 -> 5,
    1.5 -> 3, 0.75 -> 2 (tie between 0.5 and 1 goes to the even code, 1.0), -6 -> 15.
    Block 1 = [0.3, 0.15, 0, ...]: u = fl32(0.3f*448), u/6 -> 22.4 -> E4M3 22 (0x5B = 1.375 * 2^4),
    r_b = fl32(448/22) = 20.363636, 0.3f*r_b = 6.109 -> saturates to 6 (7); 0.15 -> 3.05 -> 3 (5)."""
    x = np.zeros((1, 32))
    x[0, :5] = [6, 3, 1.5, 0.75, -6]
    x[0, 16:18] = [np.float32(0.3), np.float32(0.15)]
    p, sf, st = nvfp4.quantize(x)
    c = nvfp4.unpack(p)[0]
    assert c[:5].tolist() == [7, 5, 3, 2, 15] and not c[5:16].any()
    assert sf[0, 0] == 0x7E
    from oracle import fp8
    assert sf[0, 1] == 0x5B and fp8.decode(sf[0, 1:2], "e4m3")[0] == 22.0
    assert c[16:18].tolist() == [7, 5]
    assert st[0] == np.float32(6.0 / 2688.0) and np.float32(2688.0) / np.float32(6.0) == 448.0


def test_zero_tensor_and_zero_block():
    p, sf, st = nvfp4.quantize(np.zeros((2, 32)))
    assert not p.any() and not sf.any() and st[0] == 1.0
    x = np.zeros((1, 32))
    x[0, 0] = 5.0
    x[0, 16] = -1e-30  # block 1: scale underflows E4M3 -> d = 0 -> signed zeros
    p, sf, st = nvfp4.quantize(x)
    c = nvfp4.unpack(p)[0]
    assert sf[0, 1] == 0 and c[16] == 8 and not (c[17:] & 7).any()
    assert np.array_equal(nvfp4.dequantize(p, sf, st)[0, 16:], np.zeros(16))


def test_error_bound():
    """|x * r_b - e2m1(q)| <= half the local E2M1 step, except saturation (|x r_b| > 6)."""
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((8, 128)) * np.exp(rng.standard_normal((8, 1)))).astype(np.float32).astype(np.float64)
    p, sf, st = nvfp4.quantize(x)
    xh = nvfp4.dequantize(p, sf, st)
    from oracle import fp8
    d = np.repeat(fp8.decode(sf, "e4m3"), 16, axis=1) * float(st[0])
    rel = np.abs(x - xh) / d  # in units of the block's code grid
    scaled = np.abs(x) / d
    half_step = np.where(scaled < 2.0, 0.25, np.where(scaled < 4.0, 0.5, 1.0))
    ok = (rel <= half_step * (1 + 1e-5)) | (scaled > 6.0)
    assert ok.all()
    assert np.abs(x - xh).max() <= 0.35 * np.abs(x).max()


def test_linear_vs_float64_matmul():
    rng = np.random.default_rng(7)
    a = rng.standard_normal((16, 64))
    b = rng.standard_normal((8, 64))
    ap, asf, ast = nvfp4.quantize(a)
    bp, bsf, bst = nvfp4.quantize(b)
    y = nvfp4.linear_norm(ap, asf, ast, bp, bsf, bst)
    ah, bh = nvfp4.dequantize(ap, asf, ast), nvfp4.dequantize(bp, bsf, bst)
    brute = np.array([[sum(ah[i, k] * bh[j, k] for k in range(64)) for j in range(8)] for i in range(16)])
    assert np.allclose(y, brute, rtol=1e-12, atol=1e-12)
    yl = nvfp4.linear_norm(ap, asf, ast, bp, bsf, bst, norm="layer")
    t = torch.nn.functional.layer_norm(torch.from_numpy(brute), (8,), eps=1e-5).numpy()
    assert np.allclose(yl, t, rtol=1e-10, atol=1e-10)
