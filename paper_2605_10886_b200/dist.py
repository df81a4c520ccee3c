"""Data-parallel plumbing for the LoKA hot path (a9) — host glue only.

The batch dimension M is sharded over ranks (one process per GPU, torch.distributed over NCCL).
Rowwise / 1x128 / 128x128 granules never cross a shard, so they need no
communication.  Tensorwise scaling is the one real exchange step (BASELINE.json north_star
"NCCL over NVLink is used only for ... the tensorwise amax all-reduce"):

    loka_quantize(PHASE_AMAX_ONLY)  -> local amax (device float, libloka kernel)
    all_reduce(amax, op=MAX)        -> global amax (4 bytes over NVLink / NVSwitch)
    loka_quantize(PHASE_CAST)       -> codes with the global scale (libloka kernel)

MAX is exact and order-independent, so every rank's codes equal the single-GPU codes of the
concatenated tensor (D20).  The amax / cast steps are injectable only so the protocol
can be exercised by CPU gloo tests; the default is libloka on the current CUDA stream.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(total_rows: int, world: int, rank: int):
    """Rows [r0, r1) of rank `rank` when `total_rows` are split over `world` ranks as evenly as
    possible (the first total % world ranks get one extra row)."""
    base, extra = divmod(total_rows, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def _lk():
    import paper_2605_10886_b200 as lk  # the CUDA library; raises if it is missing
    return lk


def _default_amax(x, fmt):
    lk = _lk()
    amax = torch.empty(1, dtype=torch.float32, device=x.device)
    lk.loka_quantize(x, fmt, "tensor", phase="amax", amax=amax, want_q=False)
    return amax


def _default_cast(x, fmt, amax, scale_fmt):
    lk = _lk()
    return lk.loka_quantize(x, fmt, "tensor", scale_fmt, phase="cast", amax=amax)


def quantize_tensorwise_sharded(x_local: torch.Tensor, fmt: str = "e4m3", scale_fmt: str = "f32", group=None,
                                amax_fn=None, cast_fn=None):
    """Tensorwise quantization of a row-sharded tensor with a global scale.

    Returns (codes_local, scale[1], global_amax[1]).  With world_size 1 (or no initialised
    process group) this is exactly loka_quantize(..., "tensor")."""
    amax = (amax_fn or _default_amax)(x_local, fmt)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(amax, op=dist.ReduceOp.MAX, group=group)
    q, s = (cast_fn or _default_cast)(x_local, fmt, amax, scale_fmt)
    return q, s, amax


def _default_col_amax(x, fmt):
    lk = _lk()
    amax = torch.empty(x.shape[1], dtype=torch.float32, device=x.device)
    lk.loka_quantize(x, fmt, "col", phase="amax", amax=amax, want_q=False)
    return amax


def _default_col_cast(x, fmt, amax, scale_fmt, transpose=False):
    lk = _lk()
    return lk.loka_quantize(x, fmt, "col", scale_fmt, phase="cast", amax=amax, transpose=transpose)


def quantize_colwise_sharded(x_local: torch.Tensor, fmt: str = "e4m3", scale_fmt: str = "f32", group=None,
                             transpose: bool = False, amax_fn=None, cast_fn=None):
    """COL-granule quantization (one scale per column over ALL rows) of a row-sharded tensor — the
    rowwise recipe's wgrad operands dY^T / X^T: the per-column amax vector
    (loka_quantize COL AMAX_ONLY, cols floats) is all-reduced with MAX, then each rank casts its rows
    with the global column scales (CAST_WITH_AMAX), so the codes and scales are bit-identical to the
    single-device quantization of the concatenated tensor.  Returns the cast's outputs (+ the
    transposed copy when transpose) and the global amax vector."""
    amax = (amax_fn or _default_col_amax)(x_local, fmt)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(amax, op=dist.ReduceOp.MAX, group=group)
    res = (cast_fn or _default_col_cast)(x_local, fmt, amax, scale_fmt, transpose)
    return (*res, amax)


def dispatch_plan_sharded(tables, mere_budget: float = 0.2, min_speedup: float = 1.05, group=None,
                          select_fn=None):
    """LoKA Dispatch under data parallelism (SURVEY.md §8(e) "the dispatch plan is computed on rank 0 and
    broadcast so every rank runs the same recipe"; the selection rule is PAPER.md:541/547, one decision
    per (layer, direction)).  Per-rank timings differ (clocks, neighbours), and ranks that chose
    different recipes would compute different numerics for the same layer; so rank 0 decides from its
    own table with loka_dispatch_select (host C) and the plan is broadcast.

    tables: {(layer, direction): (baseline_time_us, [(candidate_id, mere, time_us), ...])} — the MERE
    values are the rank-merged ones (probe_error_sharded), identical on every rank.
    Returns {(layer, direction): candidate_id or None (the BF16 baseline)}."""
    if select_fn is None:
        def select_fn(cands, direction, base):
            return _lk().loka_dispatch_select([(c[0], direction, c[1], c[2]) for c in cands], base, mere_budget,
                                              min_speedup)
    multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    plan = None
    if not multi or dist.get_rank(group) == 0:
        plan = {}
        for key in sorted(tables):
            base, cands = tables[key]
            i = select_fn(list(cands), key[1], base)
            plan[key] = cands[i][0] if i >= 0 else None
    if multi:
        obj = [plan]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        plan = obj[0]
    return plan


def probe_error_sharded(pairs, floor_rel: float = 1e-6, group=None, stream=None, probe_fn=None, merge_fn=None):
    """LoKA Probe (a7) over row-sharded layers ("probe sums and max values can be
    all-reduced"), equal to the single-device statistic of the concatenated tensors:

      pass 1  every rank: loka_probe_error on its shards -> per layer (sum |ref|, count);
      reduce  all_reduce(SUM) of the [L, 2] (sum |ref|, count) array: the layer's global floor
              f = floor_rel * sum / count (D10 applied to the whole tensor, not the shard);
      pass 2  every rank: loka_probe_error_global with that floor;
      merge   all_gather of the per-rank stats, combined by libloka's loka_probe_merge (host C).

    Returns a list of dicts (probe_stats_to_dicts).  probe_fn(pairs, floor_rel, gsum_or_None) -> list
    of dicts and merge_fn(list of per-rank lists) -> list of dicts are injectable so the protocol runs
    under CPU gloo tests; the defaults are libloka on the current CUDA stream."""
    lk = _lk()
    if probe_fn is None:
        def probe_fn(prs, fr, gsum):
            return lk.probe_stats_to_dicts(lk.loka_probe_error(prs, fr, stream=stream, global_sum_count=gsum))
    if merge_fn is None:
        merge_fn = lk.probe_merge
    local = probe_fn(pairs, floor_rel, None)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return local
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    gsum = torch.tensor([[st["sum_abs_ref"], float(st["count"])] for st in local], dtype=torch.float64, device=dev)
    dist.all_reduce(gsum, op=dist.ReduceOp.SUM, group=group)
    mine = probe_fn(pairs, floor_rel, gsum)
    world = dist.get_world_size(group)
    gathered = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    return merge_fn(gathered)


class QuantizedGradReducer:
    """NEXT-4 (SURVEY.md §8(f) "quantized (FP8) DP gradient communication"; D39): the data-
    parallel gradient reduce-scatter with FP8 payloads.  Every rank quantizes its gradient G [rows,
    cols] rowwise (loka_quantize, e5m2 by default: D5) into a registered buffer; rank r owns rows
    shard_rows(rows, P, r) and reduces the P ranks' codes of those rows with loka_dequant_reduce.

    transport "p2p": the buffer is torch symmetric memory (every rank's buffer mapped into every
      GPU over NVLink / NVSwitch); the reduction kernel reads the peers' codes directly — the kernel
      is the collective's data path (1 byte + 4/cols bytes per element per peer instead of 4) — and
      two device-side barriers (no host sync) order the peers' quantize before the reads and the
      reads before the next quantize.
    transport "nccl": all_to_all of the code / scale row shards, then the same kernel on the local
      copies (the baseline).
    The quantize / reduce steps are injectable only so the protocol can be exercised by CPU gloo
    tests; the default is libloka on the current CUDA stream."""

    def __init__(self, rows: int, cols: int, fmt: str = "e5m2", group=None, transport: str = "p2p", device=None,
                 quant_fn=None, reduce_fn=None):
        self.rows, self.cols, self.fmt, self.group = rows, cols, fmt, group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        self.r0, self.r1 = shard_rows(rows, self.world, self.rank)
        self.transport = transport if self.world > 1 else "local"
        dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                                 if torch.cuda.is_available() else torch.device("cpu"))
        self.ld = (cols + 15) // 16 * 16
        self.off_s = (rows * self.ld + 255) // 256 * 256  # scales after the codes, 256-B aligned
        nbytes = self.off_s + 4 * rows
        self.hdl = None
        if self.transport == "p2p":
            import torch.distributed._symmetric_memory as symm_mem
            self.buf = symm_mem.empty(nbytes, dtype=torch.uint8, device=dev)
            self.hdl = symm_mem.rendezvous(self.buf, (group or dist.group.WORLD).group_name)
            self.peer_base = [self.hdl.get_buffer(p, (nbytes,), torch.uint8, 0).data_ptr() if p != self.rank
                              else self.buf.data_ptr() for p in range(self.world)]
        else:
            self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        self.codes = self.buf[:rows * self.ld].view(rows, self.ld)[:, :cols]
        self.scales = self.buf[self.off_s:self.off_s + 4 * rows].view(torch.float32)
        self.quant_fn = quant_fn or self._lk_quant
        self.reduce_fn = reduce_fn or self._lk_reduce

    def _lk_quant(self, g):
        import paper_2605_10886_b200 as lk
        lk.loka_quantize(g, self.fmt, "row", out=self.codes, scales=self.scales)

    def _lk_reduce(self, codes, scales, out):
        import paper_2605_10886_b200 as lk
        return lk.loka_dequant_reduce(codes, scales, self.fmt, out=out)

    def reduce_scatter(self, grad: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Returns this rank's reduced rows [r1 - r0, cols] (FP32), stream-ordered on the current stream."""
        n = self.r1 - self.r0
        if out is None:
            out = torch.empty(n, self.cols, dtype=torch.float32, device=self.codes.device)
        self.quant_fn(grad)
        if self.transport == "local":
            return self.reduce_fn([self.codes], [self.scales], out)
        if self.transport == "p2p":
            self.hdl.barrier(channel=0)  # every rank's codes are written (device-side)
            cp = [b + self.r0 * self.ld for b in self.peer_base]
            sp = [b + self.off_s + self.r0 * 4 for b in self.peer_base]
            self.reduce_fn(cp, sp, out)
            self.hdl.barrier(channel=1)  # every rank finished reading before anyone's next quantize
            return out
        # nccl: all_to_all of the row shards of the codes and scales
        if self.cols % 16:
            raise ValueError("cols % 16 != 0")
        bounds = [shard_rows(self.rows, self.world, p) for p in range(self.world)]
        in_split = [(b - a) * self.cols for a, b in bounds]
        recv_c = torch.empty(self.world * n * self.cols, dtype=torch.uint8, device=self.codes.device)
        send_c = self.codes.contiguous().view(-1)
        dist.all_to_all_single(recv_c, send_c, [n * self.cols] * self.world, in_split, group=self.group)
        recv_s = torch.empty(self.world * n, dtype=torch.float32, device=self.codes.device)
        dist.all_to_all_single(recv_s, self.scales.contiguous(), [n] * self.world, [b - a for a, b in bounds],
                               group=self.group)
        rc = recv_c.view(self.world, n, self.cols)
        rs = recv_s.view(self.world, n)
        return self.reduce_fn([rc[p] for p in range(self.world)], [rs[p] for p in range(self.world)], out)
