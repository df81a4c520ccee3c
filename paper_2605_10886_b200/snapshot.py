"""LoKA Probe cadence and snapshots (host side of NEXT-2/3).

"LoKA Probe activates every 100 training iterations and asynchronously saves statistical
parameters every 10,000 iterations".  ``ProbeSchedule`` holds the cadence;
``snapshot`` copies a tracker's device statistics to host memory (the copy is the immutable value
the asynchronous save works on), ``save_async`` writes it from a background thread
while training continues, ``load`` / ``restore`` bring it back.

File format (version 1, little-endian): b"LOKASNAP", uint32 version, uint32 header length,
a UTF-8 JSON header {kind, scalars, arrays: [[name, shape, byte offset]]}, the arrays as row-major
float32, then a CRC-32 (zlib) of every preceding byte.  A round trip is bit-exact.
"""
from __future__ import annotations

import json
import struct
import threading
import zlib
from concurrent.futures import Future

import numpy as np

MAGIC = b"LOKASNAP"
VERSION = 1


class SnapshotError(ValueError):
    pass


class FormatVersionMismatch(SnapshotError):
    pass


class CorruptSnapshot(SnapshotError):
    pass


class ProbeSchedule:
    """Cadence of PAPER.md:366: track every `activate_every` iterations, snapshot every
    `snapshot_every` (a multiple of `activate_every`)."""

    def __init__(self, activate_every: int = 100, snapshot_every: int = 10_000):
        if activate_every <= 0 or snapshot_every <= 0 or snapshot_every % activate_every:
            raise ValueError("snapshot_every must be a positive multiple of activate_every")
        self.activate_every = activate_every
        self.snapshot_every = snapshot_every

    def should_track(self, it: int) -> bool:
        return it % self.activate_every == 0

    def should_snapshot(self, it: int) -> bool:
        return it > 0 and it % self.snapshot_every == 0


def snapshot(tracker) -> dict:
    """Host copy of an InputTracker / WeightTracker's statistics (synchronous device-to-host copy)."""
    if hasattr(tracker, "scatter"):
        return {"kind": "input", "scalars": {"n": int(tracker.n), "K": int(tracker.mean.numel())},
                "arrays": {"mean": tracker.mean.detach().cpu().numpy().copy(),
                           "scatter": tracker.scatter.detach().cpu().numpy().copy()}}
    st = tracker.state
    return {"kind": "weight",
            "scalars": {"M": int(st.M), "N": int(st.N), "count": int(st.count), "momentum": float(st.momentum),
                        "eps_rel": float(st.eps_rel)},
            "arrays": {"mean": tracker.mean.detach().cpu().numpy().copy(), "U": tracker.U.detach().cpu().numpy().copy(),
                       "V": tracker.V.detach().cpu().numpy().copy()}}


def dumps(snap: dict) -> bytes:
    arrays = []
    blobs = []
    off = 0
    for name, a in snap["arrays"].items():
        a = np.ascontiguousarray(a, dtype="<f4")
        arrays.append([name, list(a.shape), off])
        blobs.append(a.tobytes())
        off += a.nbytes
    header = json.dumps({"kind": snap["kind"], "scalars": snap["scalars"], "arrays": arrays},
                        sort_keys=True).encode()
    body = MAGIC + struct.pack("<II", VERSION, len(header)) + header + b"".join(blobs)
    return body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)


def loads(data: bytes) -> dict:
    if len(data) < len(MAGIC) + 12 or data[:len(MAGIC)] != MAGIC:
        raise CorruptSnapshot("not a LoKA snapshot")
    version, hlen = struct.unpack_from("<II", data, len(MAGIC))
    if version != VERSION:
        raise FormatVersionMismatch(f"snapshot version {version}, expected {VERSION}")
    body, crc = data[:-4], struct.unpack_from("<I", data, len(data) - 4)[0]
    if zlib.crc32(body) & 0xFFFFFFFF != crc:
        raise CorruptSnapshot("checksum mismatch (truncated or altered file)")
    h0 = len(MAGIC) + 8
    try:
        header = json.loads(data[h0:h0 + hlen].decode())
    except (UnicodeDecodeError, json.JSONDecodeError) as e:
        raise CorruptSnapshot(f"bad header: {e}") from e
    base = h0 + hlen
    arrays = {}
    for name, shape, off in header["arrays"]:
        n = int(np.prod(shape)) if shape else 1
        start = base + off
        if start + 4 * n > len(body):
            raise CorruptSnapshot("array past the end of the file")
        arrays[name] = np.frombuffer(body, dtype="<f4", count=n, offset=start).reshape(shape).copy()
    return {"kind": header["kind"], "scalars": header["scalars"], "arrays": arrays}


def save(path: str, snap: dict) -> None:
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(dumps(snap))
    import os
    os.replace(tmp, path)


def save_async(path: str, tracker) -> Future:
    """Copy the statistics now (the immutable snapshot), write the file on a background thread."""
    snap = snapshot(tracker)
    fut: Future = Future()

    def run():
        try:
            save(path, snap)
            fut.set_result(path)
        except BaseException as e:  # surfaced through the future
            fut.set_exception(e)
    threading.Thread(target=run, daemon=True).start()
    return fut


def load(path: str) -> dict:
    with open(path, "rb") as f:
        return loads(f.read())


def restore(tracker, snap: dict) -> None:
    """Copy a loaded snapshot back into a tracker of the same kind and shape."""
    import torch
    if snap["kind"] == "input":
        if not hasattr(tracker, "scatter") or tracker.mean.numel() != snap["scalars"]["K"]:
            raise SnapshotError("snapshot does not match the tracker")
        tracker.mean.copy_(torch.from_numpy(snap["arrays"]["mean"]))
        tracker.scatter.copy_(torch.from_numpy(snap["arrays"]["scatter"]))
        tracker.state.n = snap["scalars"]["n"]
        return
    st = tracker.state
    if hasattr(tracker, "scatter") or (st.M, st.N) != (snap["scalars"]["M"], snap["scalars"]["N"]):
        raise SnapshotError("snapshot does not match the tracker")
    tracker.mean.copy_(torch.from_numpy(snap["arrays"]["mean"]))
    tracker.U.copy_(torch.from_numpy(snap["arrays"]["U"]))
    tracker.V.copy_(torch.from_numpy(snap["arrays"]["V"]))
    st.count = snap["scalars"]["count"]
    st.momentum = snap["scalars"]["momentum"]
    st.eps_rel = snap["scalars"]["eps_rel"]
