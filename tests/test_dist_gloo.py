"""a9 multi-rank protocol on CPU (gloo, world_size 2 and 3): row sharding, the split-phase
tensorwise quantize with an all_reduce(MAX) between the phases, and per-rank probe-statistics
reduction.  The device kernels are replaced by oracle functions here (no GPU); the GPU path of
the same protocol is tests/test_gpu_dist.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2605_10886_b200 import dist as ldist

pytestmark = pytest.mark.dist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_amax(x, fmt):
    return torch.tensor([float(np.abs(x.double().numpy()).max())], dtype=torch.float32)


def _oracle_cast(x, fmt, amax, scale_fmt):
    q, s = oracle.quantize.quantize(x.double().numpy(), fmt, "tensor", scale_fmt, amax=np.array([float(amax[0])]))
    return torch.from_numpy(q), torch.from_numpy(s)


def _worker(rank, world, port, total, cols, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r0, r1 = ldist.shard_rows(total, world, rank)
    x = synth.heavy(r1 - r0, cols, 3, row0=r0, total_rows=total)
    q, s, amax = ldist.quantize_tensorwise_sharded(x, "e4m3", amax_fn=_oracle_amax, cast_fn=_oracle_cast)
    # probe statistics of the shard (oracle), then the cross-rank reduction
    ref = x.double().numpy()
    out = oracle.quantize.dequantize(q.numpy(), s.numpy(), "e4m3", "tensor")
    # (the injected probe is the oracle; the merge is libloka's host loka_probe_merge)
    def probe_fn(prs, fr, gsum):
        return [oracle.probe.mere_stats(o, r, fr, None if gsum is None else fr * float(gsum[i, 0]) / float(gsum[i, 1]))
                for i, (o, r) in enumerate(prs)]
    st = ldist.probe_error_sharded([(out, ref)], probe_fn=probe_fn)[0]
    np.save(os.path.join(out_dir, f"q{rank}.npy"), q.numpy())
    np.save(os.path.join(out_dir, f"s{rank}.npy"), s.numpy())
    if rank == 0:
        np.save(os.path.join(out_dir, "probe.npy"), np.array([st["mere"], st["max_rel"], st["count"], st["n_floored"],
                                                              st["sum_abs_ref"]]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 300), (3, 257)])
def test_sharded_tensorwise_equals_single_device(world, total, tmp_path):
    cols = 96
    mp.spawn(_worker, args=(world, _free_port(), total, cols, str(tmp_path)), nprocs=world, join=True)
    x = synth.heavy(total, cols, 3)
    # the shard generator reproduces the global tensor's rows exactly
    parts = [synth.heavy(r1 - r0, cols, 3, row0=r0, total_rows=total)
             for r0, r1 in (ldist.shard_rows(total, world, r) for r in range(world))]
    assert torch.equal(torch.cat(parts), x)
    qg, sg = oracle.quantize.quantize(x.double().numpy(), "e4m3", "tensor")
    qs = np.concatenate([np.load(tmp_path / f"q{r}.npy") for r in range(world)])
    for r in range(world):
        assert np.load(tmp_path / f"s{r}.npy").view(np.uint32)[0] == sg.view(np.uint32)[0]
    assert np.array_equal(qs, qg)  # bit-identical to the single-device quantization
    # the reduced probe statistics equal the statistics of the whole tensor
    st = oracle.probe.mere_stats(oracle.quantize.dequantize(qg, sg, "e4m3", "tensor"), x.double().numpy())
    pr = np.load(tmp_path / "probe.npy")
    assert int(pr[2]) == st["count"] and abs(pr[1] - st["max_rel"]) <= 1e-12 * st["max_rel"]
    # exact two-pass protocol (global floor, then the merge): MERE, floored count and sum |ref| of
    # the concatenated tensor (per-shard floors made the combination approximate)
    assert abs(pr[0] - st["mere"]) <= 1e-12 * st["mere"]
    assert int(pr[3]) == st["n_floored"] and abs(pr[4] - st["sum_abs_ref"]) <= 1e-12 * st["sum_abs_ref"]


def test_shard_rows_partition():
    for total in (0, 1, 7, 4096, 262144):
        for world in (1, 2, 3, 4, 8):
            spans = [ldist.shard_rows(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def _grad_worker(rank, world, port, rows, cols, out_dir):
    """NEXT-4 quantized gradient reduce-scatter, NCCL-transport protocol over gloo (CPU), with the
    device steps replaced by oracle functions."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    holder = {}

    def quant(g):
        q, s = oracle.quantize.quantize(g.double().numpy(), "e5m2", "row")
        holder["r"].codes.copy_(torch.from_numpy(q))
        holder["r"].scales.copy_(torch.from_numpy(s))

    def reduce(codes, scales, out):
        r = oracle.gradcomm.reduce_dequantized([c.numpy() for c in codes], [s.numpy() for s in scales], "e5m2")
        out.copy_(torch.from_numpy(r))
        return out

    red = ldist.QuantizedGradReducer(rows, cols, "e5m2", transport="nccl", device=torch.device("cpu"),
                                     quant_fn=quant, reduce_fn=reduce)
    holder["r"] = red
    out = red.reduce_scatter(synth.grad(rows, cols, 100 + rank))
    np.save(os.path.join(out_dir, f"g{rank}.npy"), out.double().numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,rows", [(2, 64), (3, 50)])
def test_quantized_grad_reduce_scatter_protocol(world, rows, tmp_path):
    cols = 32
    mp.spawn(_grad_worker, args=(world, _free_port(), rows, cols, str(tmp_path)), nprocs=world, join=True)
    grads = [synth.grad(rows, cols, 100 + p).double().numpy() for p in range(world)]
    ref, _, _ = oracle.gradcomm.quantized_allreduce(grads, "e5m2")
    got = np.concatenate([np.load(tmp_path / f"g{r}.npy") for r in range(world)])
    assert np.allclose(got, ref, rtol=2.0 ** -23, atol=0)  # each rank holds its rows of the sum (FP32 out)


def _dispatch_worker(rank, world, port, out_dir):
    """Every rank measures its own (rank-dependent) timings; the plan must be rank 0's."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tables = {}
    for layer in range(6):
        for d in ("fwd", "dgrad", "wgrad"):
            base = 100.0
            # rank 0 sees FP8 rowwise fastest; the other ranks see the blockwise candidate fastest
            cands = [("fp8_tw", 0.25, 60.0), ("fp8_rw", 0.05 + 0.01 * layer, 70.0 if rank == 0 else 90.0),
                     ("fp8_bw", 0.04, 85.0 if rank == 0 else 50.0), ("nvfp4", 0.15, 96.0)]
            tables[(layer, d)] = (base, cands)
    plan = ldist.dispatch_plan_sharded(tables)
    import pickle
    with open(os.path.join(out_dir, f"plan{rank}.pkl"), "wb") as f:
        pickle.dump((plan, tables), f)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dispatch_plan_broadcast_from_rank0(world, tmp_path):
    """the dispatch plan is rank 0's decision on every rank (a per-rank decision would
    pick different recipes here), and it equals the oracle's select on rank 0's table."""
    import pickle
    mp.spawn(_dispatch_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [pickle.load(open(tmp_path / f"plan{r}.pkl", "rb")) for r in range(world)]
    plan0, tables0 = res[0]
    for plan, _ in res[1:]:
        assert plan == plan0
    for key, (base, cands) in tables0.items():
        i = oracle.dispatch.select([(c[0], c[1], c[2]) for c in cands], base, 0.2, 1.05)
        assert plan0[key] == (cands[i][0] if i >= 0 else None)
    assert set(plan0.values()) == {"fp8_rw"}
    local1 = ldist.dispatch_plan_sharded(res[1][1])  # what rank 1 alone would have chosen
    assert set(local1.values()) == {"fp8_bw"}


def _col_worker(rank, world, port, total, cols, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r0, r1 = ldist.shard_rows(total, world, rank)
    x = synth.heavy(total, cols, 7)[r0:r1]

    def amax_fn(xl, fmt):
        return torch.from_numpy(oracle.quantize.granule_amax(xl.double().numpy(), "col").astype(np.float32).reshape(-1))

    def cast_fn(xl, fmt, amax, scale_fmt, transpose):
        q, s = oracle.quantize.quantize(xl.double().numpy(), fmt, "col", scale_fmt, amax=amax.double().numpy())
        return torch.from_numpy(q), torch.from_numpy(s)

    q, s, amax = ldist.quantize_colwise_sharded(x, "e5m2", amax_fn=amax_fn, cast_fn=cast_fn)
    np.save(os.path.join(out_dir, f"c{rank}.npy"), q.numpy())
    np.save(os.path.join(out_dir, f"s{rank}.npy"), s.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 300), (3, 257)])
def test_sharded_colwise_equals_single_device(world, total, tmp_path):
    """COL granules under M sharding: the all-reduced column amax vector makes every
    rank's codes the rows of the single-device COL quantization, and every rank's scales equal it."""
    cols = 96
    mp.spawn(_col_worker, args=(world, _free_port(), total, cols, str(tmp_path)), nprocs=world, join=True)
    oq, os_ = oracle.quantize.quantize(synth.heavy(total, cols, 7).double().numpy(), "e5m2", "col")
    got = np.concatenate([np.load(tmp_path / f"c{r}.npy") for r in range(world)])
    assert np.array_equal(got, oq)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"s{r}.npy").view(np.uint32), np.asarray(os_, np.float32).view(np.uint32))
