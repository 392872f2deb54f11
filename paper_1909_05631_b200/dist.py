"""Multi-GPU plumbing: one process per GPU (torchrun), rows sharded.

The reference's data-parallel mode (engine.py:237-251) gives each worker a
contiguous row tile with the full weight stack and stitches results in row
order; there is no per-layer exchange.  The B200 layout is the same with one
GPU per worker: each rank owns rows [r0, r1) and a weight replica, runs all
layers alone, and the only collectives are the final category gather and
the max-over-ranks of the timed region.  torch.distributed is plumbing here
(NCCL on GPUs, gloo on CPU for the tests).
"""

from __future__ import annotations

import os

import numpy as np


def shard(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row block of `rank` (tile = ceil(batch / world), engine.py:240)."""
    per = -(-batch // world) if world > 0 else batch
    r0 = min(batch, rank * per)
    return r0, min(batch, r0 + per)


class RankGroup:
    """torch.distributed wrapper; a single process is a group of one."""

    def __init__(self, backend: str | None = None):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.td = None
        if self.world > 1:
            import torch
            import torch.distributed as td

            if backend is None:
                backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            if not td.is_initialized():
                td.init_process_group(backend)
            self.td = td
            self.torch = torch
            self.backend = backend

    def _t(self, x: float):
        dev = f"cuda:{self.local}" if self.backend == "nccl" else "cpu"
        return self.torch.tensor([float(x)], dtype=self.torch.float64, device=dev)

    def barrier(self) -> None:
        if self.td is not None:
            self.td.barrier()

    def max(self, x: float) -> float:
        """Max over ranks (the timed region is the slowest rank's)."""
        if self.td is None:
            return float(x)
        t = self._t(x)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def max_array(self, x):
        """Elementwise max over ranks of a small float array."""
        import numpy as np

        x = np.asarray(x, dtype=np.float64)
        if self.td is None:
            return x
        dev = f"cuda:{self.local}" if self.backend == "nccl" else "cpu"
        t = self.torch.tensor(x, dtype=self.torch.float64, device=dev)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return t.cpu().numpy()

    def broadcast_layers(self, net, first: int, count: int) -> None:
        """Replicate layers [first, first + count) of a DeviceNetwork from
        rank 0 to every rank, device to device (NCCL over NVLink/NVSwitch):
        rank 0 generated them, the others appended uninitialised layers of
        the same shape (DeviceNetwork.add_layers_uninit)."""
        if self.td is None:
            return
        for l in range(first, first + count):
            idx, val = net.layer_tensors(l)
            self.td.broadcast(idx, src=0)
            self.td.broadcast(val, src=0)
        self.torch.cuda.synchronize(net.device)

    def sum(self, x: float) -> float:
        if self.td is None:
            return float(x)
        t = self._t(x)
        self.td.all_reduce(t)
        return float(t.item())

    def gather_categories(self, local_rows: np.ndarray, row0: int) -> np.ndarray:
        """1-based global category list from each rank's local 1-based list
        (the only data exchange): shift by the rank's first row, gather,
        merge in ascending order."""
        shifted = np.asarray(local_rows, np.int64) + int(row0)
        if self.td is None:
            return shifted
        out = [None] * self.world
        self.td.all_gather_object(out, shifted.tolist())
        return np.asarray(sorted(c for part in out for c in part), np.int64)

    def close(self) -> None:
        if self.td is not None and self.td.is_initialized():
            self.td.destroy_process_group()
