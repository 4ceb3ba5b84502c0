"""Multi-GPU plumbing: one process per GPU, torch.distributed (NCCL) for the two
real exchanges of the serving path:

  * broadcast of the query ciphertext bytes from rank 0 (a1), and of the
    exported evaluation keys once at setup;
  * gather of the per-rank score ciphertexts to rank 0 (a9).

The database is sharded by aggregate: rank r owns aggregates
[floor(r A / P), floor((r + 1) A / P)) and enrolls only their rows; no
collective touches the diagonals.  These helpers move opaque byte tensors
(device tensors under NCCL, CPU tensors under gloo) and hold no arithmetic.

`StepExchange` is the per-query exchange bench.py's timed step runs: every buffer is
allocated once at setup and sized from the static shard map, so a step issues one
broadcast and one gather and nothing else -- no size exchange, no host synchronisation
(`.item()`), no allocation.  The ciphertext export / import calls are passed in (the
C-ABI calls on a GPU; the gloo tests pass byte copies of oracle ciphertexts), so the
tests drive exactly the code the bench runs.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(num_aggregates: int, rank: int, world: int):
    """Contiguous aggregate range of `rank` (sizes differ by at most one)."""
    return (num_aggregates * rank) // world, (num_aggregates * (rank + 1)) // world


def shard_sizes(num_aggregates: int, world: int):
    return [shard_range(num_aggregates, r, world)[1] - shard_range(num_aggregates, r, world)[0]
            for r in range(world)]


def baby_slice(n1: int, rank: int, world: int):
    """Split baby steps (hd_baby_steps): rank r computes r[i] for i in [i0, i1) into its chunk of
    ceil(n1 / world) slots; an all-gather of the equal-size chunks lays r out in order (the
    padding slots past n1 are ignored).  Returns (chunk, i0, i1)."""
    chunk = -(-n1 // world)
    return chunk, min(n1, rank * chunk), min(n1, (rank + 1) * chunk)


def rows_of_aggregates(agg_begin: int, agg_end: int, per_aggregate: int, num_vectors: int):
    return min(agg_begin * per_aggregate, num_vectors), min(agg_end * per_aggregate, num_vectors)


def broadcast_bytes(buf: torch.Tensor | None, nbytes: int, device, src: int = 0) -> torch.Tensor:
    """Broadcast a uint8 tensor of known size from `src` (setup only); returns it on every rank."""
    if dist.get_rank() != src or buf is None:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
    dist.broadcast(buf, src=src)
    return buf


class StepExchange:
    """The per-step collectives of the sharded scan, on buffers allocated once.

    query_bytes: bytes of the exported query ciphertext(s) broadcast from `src` each step.
    per_rank:    result ciphertexts per rank (list of world ints, from the static shard map;
                 1 per rank for the membership partial sum).
    out_bytes:   bytes of one exported result ciphertext (1-limb export, R24).
    """

    def __init__(self, query_bytes: int, per_rank, out_bytes: int, device, src: int = 0):
        self.world, self.rank, self.src = dist.get_world_size(), dist.get_rank(), src
        self.per_rank = list(per_rank)
        self.out_bytes = out_bytes
        self.slots = max(self.per_rank)  # equal-size slabs: gather needs no size exchange
        self.qbuf = torch.empty(query_bytes, dtype=torch.uint8, device=device)
        self.send = torch.empty(self.slots * out_bytes, dtype=torch.uint8, device=device)
        self.recv = ([torch.empty(self.slots * out_bytes, dtype=torch.uint8, device=device)
                      for _ in range(self.world)] if self.rank == src else None)

    def broadcast_query(self):
        """a1: rank src's qbuf (filled by the caller) to every rank."""
        dist.broadcast(self.qbuf, src=self.src)
        return self.qbuf

    def gather(self, results, export_into):
        """a9: export_into(ct, ptr, cap) writes each local result into the send slab (stream-ordered,
        device destination); one gather to src.  Returns, on src, a list over ranks of the
        per-result byte views [(ptr, nbytes), ...] inside the persistent receive slabs."""
        ob = self.out_bytes
        base = self.send.data_ptr()
        for i, ct in enumerate(results):
            export_into(ct, base + i * ob, ob)
        if self.rank == self.src:
            dist.gather(self.send, gather_list=self.recv, dst=self.src)
            return [[(self.recv[r].data_ptr() + i * ob, ob) for i in range(self.per_rank[r])]
                    for r in range(self.world)]
        dist.gather(self.send, dst=self.src)
        return None


def gather_bytes(local: torch.Tensor, max_bytes: int, dst: int = 0):
    """Gather variable-size uint8 tensors (padded to max_bytes) to `dst` -- setup / tests only
    (it exchanges sizes and synchronises the host); the timed step uses StepExchange.

    Returns the list of per-rank tensors (trimmed) on dst, None elsewhere."""
    world = dist.get_world_size()
    n = torch.tensor([local.numel()], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    padded = torch.zeros(max_bytes, dtype=torch.uint8, device=local.device)
    padded[: local.numel()] = local
    if dist.get_rank() == dst:
        bufs = [torch.empty(max_bytes, dtype=torch.uint8, device=local.device) for _ in range(world)]
        dist.gather(padded, gather_list=bufs, dst=dst)
        return [b[: int(s.item())] for b, s in zip(bufs, sizes)]
    dist.gather(padded, dst=dst)
    return None


def max_over_ranks(x: float, device) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
