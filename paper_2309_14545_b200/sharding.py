"""Multi-GPU sharding of the path.

Configurations and edges are independent, so the path partitions with no
data-path exchange: each rank validates a contiguous slice with the robot
module and environment replicated, and the only collective is an optional
all-gather of the packed verdict words (N/8 bytes: 128 KiB per 1M configs)
when a caller wants the global result on every rank.  Bench runs report weak
scaling (every rank validates its own full batch).

The host logic here is what the gloo CPU tests exercise (world_size 2);
``local_fn`` does the per-rank device work.
"""

from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int, align: int = 32) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of n items for ``rank``; boundaries are
    multiples of ``align`` so packed 32-bit verdict words never straddle ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    units = (n + align - 1) // align
    lo_u = units * rank // world
    hi_u = units * (rank + 1) // world
    return min(lo_u * align, n), min(hi_u * align, n)


def gather_verdict_words(local_words, n: int, rank: int, world: int, group=None, align: int = 32):
    """All-gather per-rank packed words (torch int32 tensors) into the global
    ceil(n/32)-word vector, identical on every rank."""
    import torch
    import torch.distributed as dist

    words_total = (n + 31) // 32
    sizes = []
    for r in range(world):
        lo, hi = shard_range(n, r, world, align)
        sizes.append((hi - lo + 31) // 32)
    cap = max(max(sizes), 1)
    buf = torch.zeros(cap, dtype=torch.int32, device=local_words.device)
    buf[: local_words.numel()] = local_words[: sizes[rank]]
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = torch.cat([p[:s] for p, s in zip(parts, sizes)])
    assert out.numel() == words_total
    return out


def validate_sharded(local_fn, items: np.ndarray, rank: int, world: int, group=None,
                     gather: bool = True):
    """Run ``local_fn(slice) -> packed int32 words`` on this rank's slice of
    ``items`` (first axis = item axis), then optionally all-gather."""
    n = items.shape[0]
    lo, hi = shard_range(n, rank, world)
    words = local_fn(items[lo:hi])
    if not gather:
        return words, (lo, hi)
    return gather_verdict_words(words, n, rank, world, group), (lo, hi)
