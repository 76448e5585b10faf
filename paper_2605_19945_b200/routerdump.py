"""Binary router dumps: the on-disk format feeding top-k id ingestion.

The reference takes per-step expert *counts* (trace.py:236-337);
a serving engine's router hook produces top-k expert *ids* per token
("Step 1"). This module defines the file such a hook appends to,
and streams it into the K1 histogram kernel through pinned host buffers, so a
trace never has to fit in host memory or leave the device as counts.

File layout (little endian)::

    header, 64 bytes
      0  magic        8s   b"GEMRDMP1"
      8  version      u32  1
     12  id_bytes     u32  2 (int16) or 4 (int32)
     16  num_layers   u32  L
     20  top_k        u32  k
     24  num_experts  u32  E   (ids outside [0, E) are counted as dropped)
     28  tokens_per_step u32 B (GEM-Place step size, cli.py:498 default 1024)
     32  chunk_steps  u32  S   (steps per chunk)
     36  reserved     u32  0
     40  num_tokens   u64  N   (patched by RouterDumpWriter.close())
     48  reserved     16 bytes of zeros
    chunks: c = 0, 1, ...: ids of tokens [c*S*B, min(N, (c+1)*S*B)) of every
      layer, [L][n_c][k] in the router's order (layer-major inside the chunk,
      so each chunk is one contiguous K1 input)

A hook appends one chunk per S steps while serving; a reader can stream a
file that is still being written up to the last complete chunk.
"""

from __future__ import annotations

import os
import struct
import threading
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import ValidationError

MAGIC = b"GEMRDMP1"
VERSION = 1
HEADER = struct.Struct("<8sIIIIIIIIQ16s")
assert HEADER.size == 64


@dataclass(frozen=True)
class DumpHeader:
    id_bytes: int
    num_layers: int
    top_k: int
    num_experts: int
    tokens_per_step: int
    chunk_steps: int
    num_tokens: int

    @property
    def dtype(self) -> np.dtype:
        return np.dtype("<i2") if self.id_bytes == 2 else np.dtype("<i4")

    @property
    def chunk_tokens(self) -> int:
        return self.chunk_steps * self.tokens_per_step

    @property
    def num_steps(self) -> int:
        return -(-self.num_tokens // self.tokens_per_step)

    @property
    def num_chunks(self) -> int:
        return -(-self.num_tokens // self.chunk_tokens)

    def chunk_range(self, c: int) -> tuple[int, int]:
        t0 = c * self.chunk_tokens
        return t0, min(self.num_tokens, t0 + self.chunk_tokens)

    def chunk_offset(self, c: int) -> int:
        """Byte offset of chunk c (every chunk before it is full)."""
        return HEADER.size + c * self.num_layers * self.chunk_tokens * self.top_k * self.id_bytes

    def pack(self) -> bytes:
        return HEADER.pack(MAGIC, VERSION, self.id_bytes, self.num_layers, self.top_k, self.num_experts,
                           self.tokens_per_step, self.chunk_steps, 0, self.num_tokens, bytes(16))

    @staticmethod
    def unpack(raw: bytes) -> "DumpHeader":
        if len(raw) < HEADER.size:
            raise ValidationError("router dump: truncated header")
        magic, version, idb, L, k, E, B, S, _, N, _ = HEADER.unpack(raw[:HEADER.size])
        if magic != MAGIC:
            raise ValidationError("router dump: bad magic (not a GEM router dump)")
        if version != VERSION:
            raise ValidationError(f"router dump: unsupported version {version}")
        h = DumpHeader(idb, L, k, E, B, S, N)
        h.validate()
        return h

    def validate(self) -> None:
        if self.id_bytes not in (2, 4):
            raise ValidationError("router dump: id_bytes must be 2 or 4")
        if min(self.num_layers, self.top_k, self.num_experts, self.tokens_per_step, self.chunk_steps) < 1:
            raise ValidationError("router dump: layers, top_k, experts, tokens_per_step, chunk_steps must be >= 1")
        if self.num_tokens < 0:
            raise ValidationError("router dump: negative token count")
        if self.id_bytes == 2 and self.num_experts > 32767:
            raise ValidationError("router dump: int16 ids cannot address more than 32767 experts")


class RouterDumpWriter:
    """Append-only writer (what a router hook would call once per S steps)."""

    def __init__(self, path, num_layers: int, top_k: int, num_experts: int, tokens_per_step: int = 1024,
                 chunk_steps: int = 64, id_bytes: int = 2):
        self.header = DumpHeader(id_bytes, num_layers, top_k, num_experts, tokens_per_step, chunk_steps, 0)
        self.header.validate()
        self.path = Path(path)
        self._f = open(self.path, "wb")
        self._f.write(self.header.pack())
        self._pending = []  # token blocks of the current chunk
        self._pending_tokens = 0
        self.num_tokens = 0

    def append(self, ids) -> None:
        """ids [L, n, k] (any n; buffered into whole chunks)."""
        h = self.header
        a = np.asarray(ids)
        if a.ndim != 3 or a.shape[0] != h.num_layers or a.shape[2] != h.top_k:
            raise ValidationError(f"router dump: expected ids of shape [{h.num_layers}, n, {h.top_k}], got {a.shape}")
        self._pending.append(np.ascontiguousarray(a, dtype=h.dtype))
        self._pending_tokens += a.shape[1]
        while self._pending_tokens >= h.chunk_tokens:
            block = np.concatenate(self._pending, axis=1)
            self._write_chunk(block[:, :h.chunk_tokens])
            rest = block[:, h.chunk_tokens:]
            self._pending = [rest] if rest.shape[1] else []
            self._pending_tokens = rest.shape[1]

    def _write_chunk(self, block: np.ndarray) -> None:
        self._f.write(np.ascontiguousarray(block).tobytes())
        self.num_tokens += block.shape[1]

    def close(self) -> DumpHeader:
        if self._f is None:
            return self.header
        if self._pending_tokens:
            self._write_chunk(np.concatenate(self._pending, axis=1))
            self._pending, self._pending_tokens = [], 0
        h = self.header
        self.header = DumpHeader(h.id_bytes, h.num_layers, h.top_k, h.num_experts, h.tokens_per_step, h.chunk_steps,
                                 self.num_tokens)
        self._f.seek(0)
        self._f.write(self.header.pack())
        self._f.close()
        self._f = None
        return self.header

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class RouterDump:
    """Reader: header, per-chunk host views (memory-mapped) and raw reads."""

    def __init__(self, path):
        self.path = Path(path)
        with open(self.path, "rb") as f:
            self.header = DumpHeader.unpack(f.read(HEADER.size))
        h = self.header
        need = HEADER.size + h.num_layers * h.num_tokens * h.top_k * h.id_bytes
        if os.path.getsize(self.path) < need:
            raise ValidationError(f"router dump: file holds {os.path.getsize(self.path)} bytes, header needs {need}")

    def chunk(self, c: int) -> np.ndarray:
        """ids [L, n_c, k] of chunk c (a read-only memory map)."""
        h = self.header
        t0, t1 = h.chunk_range(c)
        return np.memmap(self.path, dtype=h.dtype, mode="r", offset=h.chunk_offset(c),
                         shape=(h.num_layers, t1 - t0, h.top_k))

    def read_chunk_into(self, c: int, out: np.ndarray) -> int:
        """Read chunk c into out (flat, >= the chunk's ids); returns the number of ids."""
        h = self.header
        t0, t1 = h.chunk_range(c)
        n = h.num_layers * (t1 - t0) * h.top_k
        view = memoryview(out.reshape(-1).view(np.uint8))[: n * h.id_bytes]
        with open(self.path, "rb", buffering=0) as f:
            f.seek(h.chunk_offset(c))
            got = 0
            while got < len(view):
                k = f.readinto(view[got:])
                if not k:
                    raise ValidationError("router dump: unexpected end of file")
                got += k
        return n

    def all_ids(self) -> np.ndarray:
        """The whole trace as [L, N, k] in host memory (small dumps, tests)."""
        h = self.header
        return np.concatenate([np.asarray(self.chunk(c)) for c in range(h.num_chunks)], axis=1) if h.num_chunks \
            else np.zeros((h.num_layers, 0, h.top_k), dtype=h.dtype)


def stream_histograms(dump: RouterDump | str | os.PathLike, device: int | None = None, buffers: int = 3,
                      check_dropped: bool = True):
    """Stream a router dump into device histograms (K1 per chunk).

    Chunks are read by a host thread into `buffers` pinned buffers, copied
    host->device on a copy stream and ingested by gem_topk_hist_rows on the
    compute stream into one [L, T, E] histogram (rows of chunk c at its step
    offset); colsum/active/heavy/dropped accumulate across chunks. Copy of chunk
    c+1 overlaps the ingestion of chunk c. Returns ingest.Histograms."""
    import torch

    from . import _device, _lib
    from .ingest import Histograms
    from .trace import DeviceStats

    d = dump if isinstance(dump, RouterDump) else RouterDump(dump)
    h = d.header
    if h.num_tokens == 0:
        raise ValidationError("router dump: no tokens")
    if h.chunk_tokens % h.tokens_per_step:
        raise ValidationError("router dump: chunks must hold whole steps")
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    torch_dtype = torch.int16 if h.id_bytes == 2 else torch.int32
    L, T, E, k = h.num_layers, h.num_steps, h.num_experts, h.top_k
    hist = torch.empty((L, T, E), dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        ds = DeviceStats.allocate(L, E, T)
    dropped = torch.zeros((L,), dtype=torch.int64, device=dev)
    nb = max(2, buffers)
    chunk_ids = L * h.chunk_tokens * k
    host = [torch.empty(chunk_ids, dtype=torch_dtype, pin_memory=True) for _ in range(nb)]
    devb = [torch.empty(chunk_ids, dtype=torch_dtype, device=dev) for _ in range(2)]
    compute = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    done_copy = [torch.cuda.Event() for _ in range(2)]
    done_use = [torch.cuda.Event() for _ in range(2)]
    host_free = [threading.Event() for _ in range(nb)]
    host_full = [threading.Event() for _ in range(nb)]
    for e in host_free:
        e.set()
    err = []

    def reader():
        try:
            for c in range(h.num_chunks):
                i = c % nb
                host_free[i].wait()
                host_free[i].clear()
                d.read_chunk_into(c, host[i].numpy())
                host_full[i].set()
        except Exception as ex:  # surfaced on the caller's thread
            err.append(ex)
            for e in host_full:
                e.set()

    th = threading.Thread(target=reader, daemon=True)
    th.start()
    host_done = [None] * nb  # per pinned buffer: the event of its last host->device copy
    for c in range(h.num_chunks):
        i, j = c % nb, c % 2
        host_full[i].wait()
        host_full[i].clear()
        if err:
            raise err[0]
        t0, t1 = h.chunk_range(c)
        n = L * (t1 - t0) * k
        with torch.cuda.stream(copy):
            if c >= 2:
                copy.wait_event(done_use[j])  # device buffer j is free once chunk c-2 is ingested
            devb[j][:n].copy_(host[i][:n], non_blocking=True)
            done_copy[j].record(copy)
        ev = torch.cuda.Event()
        ev.record(copy)
        host_done[i] = ev
        compute.wait_event(done_copy[j])
        s0 = t0 // h.tokens_per_step
        _lib.call("gem_topk_hist_rows", devb[j].data_ptr(), h.id_bytes, L, t1 - t0, k, h.tokens_per_step, E,
                  hist.data_ptr() + s0 * E * 4, T, ds.colsum.data_ptr(), ds.active.data_ptr(), ds.heavy.data_ptr(),
                  dropped.data_ptr(), compute.cuda_stream)
        done_use[j].record(compute)
        # the reader refills pinned buffer i once its copy has finished (chunk
        # c's ingestion and chunk c+1's copy proceed meanwhile)
        host_done[i].synchronize()
        host_free[i].set()
    th.join()
    if err:
        raise err[0]
    out = Histograms(hist, ds, dropped, h.tokens_per_step, k)
    if check_dropped and int(dropped.sum().item()):
        raise ValidationError(f"{int(dropped.sum().item())} expert ids outside [0, {E})")
    return out


def stream_statistics(dump, device: int | None = None, correlation: bool = True, classify: bool = True,
                      check_dropped: bool = True):
    """Router dump -> ingest.TraceStatistics (K1 streamed, then K2/K3/K3b on the device)."""
    from .ingest import statistics_from_histograms

    return statistics_from_histograms(stream_histograms(dump, device, check_dropped=check_dropped),
                                      correlation=correlation, classify=classify)
