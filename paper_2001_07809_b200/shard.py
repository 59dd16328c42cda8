"""Frame sharding across GPUs (one process per GPU, launched by torchrun).

The per-frame path has no cross-frame state and no collective
(pipeline.cpp:50-151 is pure), so a stereo video shards by frame index:
frame f goes to rank f % world.  torch.distributed only carries control:
the barrier around timed regions, the max-over-ranks of device time, and
(optionally) gathering per-frame results back to rank 0 in frame order.
NVLink carries no frame data.
"""
from __future__ import annotations

from typing import Callable, Dict, Iterable, List, Optional


def shard_frames(n_frames: int, rank: int, world: int) -> List[int]:
    """Frame indices owned by `rank`: f = rank, rank + world, ..."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    return list(range(rank, n_frames, world))


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (e.g. elapsed device ms) over the job."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ShardedVideo:
    """Run `process(frame_index)` over this rank's share of a video."""

    def __init__(self, n_frames: int, rank: int = 0, world: int = 1):
        self.n_frames = n_frames
        self.rank = rank
        self.world = world
        self.frames = shard_frames(n_frames, rank, world)

    def run(self, process: Callable[[int], object]) -> Dict[int, object]:
        return {f: process(f) for f in self.frames}

    def gather(self, results: Dict[int, object], dist=None) -> Optional[List[object]]:
        """All ranks' results in frame order on rank 0 (None elsewhere)."""
        if dist is None or not dist.is_initialized() or self.world == 1:
            return [results[f] for f in range(self.n_frames)]
        parts: Optional[list] = [None] * self.world if self.rank == 0 else None
        dist.gather_object(results, parts, dst=0)
        if self.rank != 0:
            return None
        merged: Dict[int, object] = {}
        for p in parts:
            overlap = set(merged) & set(p)
            if overlap:
                raise RuntimeError(f"frames {sorted(overlap)} processed twice")
            merged.update(p)
        missing = set(range(self.n_frames)) - set(merged)
        if missing:
            raise RuntimeError(f"frames {sorted(missing)} never processed")
        return [merged[f] for f in range(self.n_frames)]


def frame_seeds(frames: Iterable[int], base: int = 2001) -> List[int]:
    """G2 synthetic frame seeds (seed = 2001 + frame)."""
    return [base + f for f in frames]
