"""Whole-field sharding across ranks.

A field is the unit of parallelism: splitting one would restart the Lorenzo
chain and the Huffman stream and change the archive bytes.  Ranks take
contiguous field ranges; the only collective is an all-gather of per-field
compressed sizes, from which every rank derives the byte offsets of all
archives in the batch container (no data-plane collective).

Batch container ("FZB1"): magic, u32 field count, u64 offset per field plus
the total body size (relative to the end of the table), then the archives
back to back.
"""

from __future__ import annotations

import struct

import numpy as np
import torch

MAGIC = b"FZB1"


def shard_range(num_fields: int, world: int, rank: int) -> range:
    """Contiguous, balanced field range of `rank` (first ranks take the remainder)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    base, extra = divmod(int(num_fields), int(world))
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def gather_sizes(local_sizes, num_fields: int, world: int, rank: int, device=None) -> np.ndarray:
    """All-gather of per-field archive sizes -> int64[num_fields] on every rank.

    Uses torch.distributed (nccl on GPUs, gloo on CPU).  Ranks pad their
    slice to the largest shard so a single fixed-size all_gather suffices."""
    import torch.distributed as dist
    per = max(len(shard_range(num_fields, world, r)) for r in range(world))
    buf = torch.full((per,), -1, dtype=torch.int64, device=device)
    if len(local_sizes):
        buf[: len(local_sizes)] = torch.as_tensor(np.asarray(local_sizes, np.int64), device=device)
    parts = [torch.empty_like(buf) for _ in range(world)]
    if world > 1:
        dist.all_gather(parts, buf)
    else:
        parts = [buf]
    out = np.empty(num_fields, np.int64)
    for r, p in enumerate(parts):
        rg = shard_range(num_fields, world, r)
        out[rg.start:rg.stop] = p[: len(rg)].cpu().numpy()
    return out


def container_offsets(sizes: np.ndarray) -> np.ndarray:
    """Exclusive scan of archive sizes = byte offsets inside the container body."""
    sizes = np.asarray(sizes, np.int64)
    if (sizes < 0).any():
        raise ValueError("negative archive size")
    out = np.zeros(sizes.size, np.int64)
    if sizes.size:
        out[1:] = np.cumsum(sizes[:-1])
    return out


def container_head(sizes) -> bytes:
    """FZB1 header + offset table for archives of these sizes (the body follows)."""
    sizes = np.asarray(sizes, np.int64)
    offs = np.append(container_offsets(sizes), sizes.sum())
    return MAGIC + struct.pack("<I", sizes.size) + offs.astype("<u8").tobytes()


def rank_slice(sizes, rg: range) -> tuple:
    """(start, length) of the container-body bytes that rank's fields `rg` own:
    contiguous fields -> one contiguous slice, written with no coordination."""
    sizes = np.asarray(sizes, np.int64)
    start = int(container_offsets(sizes)[rg.start]) if len(rg) else int(sizes[: rg.start].sum())
    return start, int(sizes[rg.start:rg.stop].sum())


def fill_slice(out: np.ndarray, sizes, rg: range, blobs) -> np.ndarray:
    """Write this rank's archives (fields `rg`, in order) into `out`, its slice
    of the container body, at their offsets relative to the slice start."""
    sizes = np.asarray(sizes, np.int64)
    offs = container_offsets(sizes)
    start, length = rank_slice(sizes, rg)
    if out.size < length:
        raise ValueError("slice buffer too small")
    for f, blob in zip(rg, blobs):
        if len(blob) != sizes[f]:
            raise ValueError(f"field {f}: archive size {len(blob)} != gathered size {sizes[f]}")
        o = int(offs[f]) - start
        out[o:o + len(blob)] = np.frombuffer(blob, np.uint8)
    return out[:length]


def pack_container(archives: list) -> bytes:
    sizes = np.array([len(a) for a in archives], np.int64)
    offs = np.append(container_offsets(sizes), sizes.sum())
    head = MAGIC + struct.pack("<I", len(archives)) + offs.astype("<u8").tobytes()
    return head + b"".join(bytes(a) for a in archives)


def unpack_container(blob: bytes) -> list:
    from .errors import BadMagic, Truncated
    if blob[:4] != MAGIC:
        raise BadMagic("not a batch container")
    if len(blob) < 8:
        raise Truncated("container header cut short")
    (nf,) = struct.unpack_from("<I", blob, 4)
    table = 8 + 8 * (nf + 1)
    if len(blob) < table:
        raise Truncated("offset table cut short")
    offs = np.frombuffer(blob[8:table], "<u8").astype(np.int64)
    if (np.diff(offs) < 0).any() or table + int(offs[-1]) != len(blob):
        raise Truncated("inconsistent offsets")
    return [blob[table + int(o): table + int(e)] for o, e in zip(offs[:-1], offs[1:])]
