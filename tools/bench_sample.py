"""NEXT-3 timings: the weight tracker update, the jittered Cholesky and the
sampling calls on the GPU, next to the same arithmetic composed from torch ops (torch.linalg /
cuSOLVER + cuBLAS FP32, TF32 off).  CUDA events, warm-up first, median of the timed repeats."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2605_10886_b200 as lk  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
dev = torch.device("cuda")


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def torch_weight_update(st, w):
    """The same update composed from torch ops."""
    mean, u, v, m, er = st
    mm, nn = w.shape
    eu = er * torch.trace(u) / mm
    ev = er * torch.trace(v) / nn
    wc = w - mean
    l_v = torch.linalg.cholesky(v + ev * torch.eye(nn, device=dev))
    wt = torch.linalg.solve_triangular(l_v, wc.T, upper=False)
    u1 = wt.T @ wt / nn
    l_u = torch.linalg.cholesky(u + eu * torch.eye(mm, device=dev))
    wh = torch.linalg.solve_triangular(l_u, wc, upper=False)
    v1 = wh.T @ wh / mm
    u2 = m * u + (1 - m) * u1
    v2 = m * v + (1 - m) * v1
    un = (u2 + u2.T) / 2 + eu * torch.eye(mm, device=dev)
    vn = (v2 + v2.T) / 2 + ev * torch.eye(nn, device=dev)
    s = torch.trace(un) / mm
    return (m * mean + (1 - m) * w, un / s, vn * s, m, er)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = {"what": "NEXT-3 weight tracker / Cholesky / sampling, FP32, B200, CUDA events (median)", "rows": []}
    for (m, n) in [(1024, 1024), (4096, 1024), (4096, 4096)]:
        g = torch.Generator(device=dev).manual_seed(m + n)
        w = torch.randn(m, n, device=dev, generator=g) / n ** 0.5
        tr = lk.WeightTracker(w, momentum=0.95)
        ws = [torch.randn(m, n, device=dev, generator=g) / n ** 0.5 for _ in range(4)]
        it = [0]

        def ours():
            tr.update(ws[it[0] % 4])
            it[0] += 1
        t_ours = timed(ours)
        st = [tr.mean.clone(), tr.U.clone(), tr.V.clone(), 0.95, 1e-6]

        def ref():
            st[:] = torch_weight_update(tuple(st), ws[it[0] % 4])
            it[0] += 1
        t_ref = timed(ref)
        flops = (m ** 3 + n ** 3) / 3 + (m * n * n + n * m * m) + (m * m * n + n * n * m)  # 2 chol + 2 trsm + 2 grams (FMA = 2)
        res["rows"].append({"op": "weight_update", "M": m, "N": n, "ms": round(t_ours, 3), "torch_ms": round(t_ref, 3),
                            "speedup_vs_torch": round(t_ref / t_ours, 2), "tflops": round(2 * flops / t_ours / 1e9, 2)})
        print(res["rows"][-1], flush=True)
    for k in (1024, 4096):
        g = torch.Generator(device=dev).manual_seed(k)
        a = torch.randn(k, k, device=dev, generator=g)
        a = a @ a.T / k + torch.eye(k, device=dev)
        t_ours = timed(lambda: lk.cholesky_jittered(a, 1e-6), reps=5)
        t_ref = timed(lambda: torch.linalg.cholesky(a + 1e-6 * torch.eye(k, device=dev)), reps=5)
        res["rows"].append({"op": "cholesky_jittered (synchronous: trace + status read-back)", "n": k,
                            "ms": round(t_ours, 3), "torch_ms": round(t_ref, 3), "speedup_vs_torch": round(t_ref / t_ours, 2)})
        print(res["rows"][-1], flush=True)
        l, _ = lk.cholesky_jittered(a, 1e-6)
        mu = torch.zeros(k, device=dev)
        b = 32768
        out = torch.empty(b, k, dtype=torch.bfloat16, device=dev)
        t_s = timed(lambda: lk.sample_input(mu, l, b, 1, 0, out=out))

        def ref_s():
            z = torch.randn(b, k, device=dev)
            torch.addmm(mu, z, l.T).to(torch.bfloat16)
        t_rs = timed(ref_s)
        res["rows"].append({"op": "sample_input (bf16 out)", "B": b, "K": k, "ms": round(t_s, 3), "torch_ms": round(t_rs, 3),
                            "speedup_vs_torch": round(t_rs / t_s, 2),
                            "tflops_effective": round(b * k * k / t_s / 1e9, 2)})  # triangular: half of 2 B K^2
        print(res["rows"][-1], flush=True)
    n = 1 << 28
    buf = torch.empty(n, device=dev)
    t = timed(lambda: lk.philox_normal(n, 1, 0, out=buf))
    res["rows"].append({"op": "philox_normal", "n": n, "ms": round(t, 3), "gb_s_written": round(4 * n / t / 1e6, 1),
                        "torch_randn_ms": round(timed(lambda: torch.randn(n, device=dev, out=buf)), 3)})
    print(res["rows"][-1], flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
