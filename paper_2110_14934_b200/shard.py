"""Work partitioning across GPUs (one process per GPU).

Pixels are independent (segmenter.cpp:80-96) and fusion is per pixel
(fusion.cpp:29-44), so a box shards the path with no data-path exchange:

* by camera stream (config 4): rank g owns a contiguous block of streams,
  with their banks and fusion state;
* by row tile of one large frame (config 5): rank g owns a contiguous block
  of rows of every plane -- the reference's own row split
  (parallel_for_rows, engine.cpp:14-37: `base = h / workers`, the first
  `h % workers` ranges get one extra row) with GPUs in place of threads.

Either way the result is bit-identical for every world size, the analogue
of the reference's worker-count invariance (test_segmenter.cpp:103-130).
"""
from __future__ import annotations


def contiguous_split(total: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of `total` items for `rank` of `world`, engine.cpp:20-29."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def stream_shard(streams: int, rank: int, world: int) -> tuple[int, int]:
    return contiguous_split(streams, rank, world)


def row_shard(height: int, rank: int, world: int) -> tuple[int, int]:
    return contiguous_split(height, rank, world)
