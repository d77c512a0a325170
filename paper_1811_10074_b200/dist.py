"""Multi-GPU plumbing: sequence shards with halos and the seed-table bucket exchange.

One process per GPU (torchrun), `torch.distributed` over NCCL for the two collectives the
path really has (BASELINE.json C5):
  * all_reduce(SUM) of the per-bucket counts  -> global pointer table
  * all_to_all of (fingerprint, position) entries grouped by bucket owner.
Extraction itself needs no collective: rank g owns the windows [a_g, a_{g+1}) and reads
bases [a_g - 1, a_{g+1} + k + w - 2) (R25; the extra left base lets the change
rule see window a_g - 1).  Concatenating rank outputs in rank order equals the 1-GPU output.

The local phases are injected (`Phases`): the product uses the CUDA library
(`CudaPhases`); the CPU multi-process tests inject oracle-backed phases so that the
planner and the exchange logic run under `gloo` without a GPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


# ---------------------------------------------------------------- shard / halo planner
@dataclass(frozen=True)
class Shard:
    rank: int
    win_a: int      # first owned window (global)
    win_b: int      # one past the last owned window (global)
    base_lo: int    # first base read (global) = max(0, a - 1)
    base_hi: int    # one past the last base read = min(n, b + k + w - 2)
    win_lo: int     # owned windows, local to the bases read
    win_hi: int


def plan_shards(n: int, k: int, w: int, nranks: int, align: int = 32) -> list[Shard]:
    """Contiguous window ranges, starts rounded down to `align` windows (packed-word aligned)."""
    span = k + w - 1
    nwin = max(0, n - span + 1)
    cuts = [0] + [(nwin * g // nranks) // align * align for g in range(1, nranks)] + [nwin]
    out = []
    for g in range(nranks):
        a, b = cuts[g], max(cuts[g], cuts[g + 1])
        lo = max(0, a - 1)
        hi = min(n, b + span - 1) if b > a else lo
        out.append(Shard(g, a, b, lo, hi, a - lo, b - lo))
    return out


def plan_reads(read_off, nranks: int) -> list[tuple[int, int]]:
    """Contiguous read ranges [r0, r1) balanced by cumulative bases (C4); no halo needed."""
    import numpy as np
    ro = np.asarray(read_off, dtype=np.int64)
    total = int(ro[-1])
    cuts = [0] + [int(np.searchsorted(ro, total * g // nranks, side="left")) for g in range(1, nranks)] + [len(ro) - 1]
    return [(cuts[g], max(cuts[g], cuts[g + 1])) for g in range(nranks)]


# ---------------------------------------------------------------- local phases
class Phases:
    """Local seed-table phases on one rank (see include/mzslsum.h)."""

    def count(self, hash_, m, k, bits):  # -> int32[2^bits] (uint32 bits)
        raise NotImplementedError

    def partition(self, hash_, pos, m, k, bits, nranks):  # -> (fp int32[m], pos int64[m], counts list[int])
        raise NotImplementedError

    def finalize(self, recv_fp, recv_pos, m_recv, global_counts, bits, rank, nranks):
        raise NotImplementedError  # -> (offsets_local int64[nbl+1], pos int64[m_recv], fp int32[m_recv])


class CudaPhases(Phases):
    """The product: every phase is a libmzslsum call on the current stream."""

    def __init__(self):
        from . import _lib as L
        self.L = L

    def count(self, hash_, m, k, bits):
        return self.L.seedtable_count(hash_, k, bits, m=m).view(torch.int32)

    def partition(self, hash_, pos, m, k, bits, nranks):
        fp, p, c = self.L.seedtable_partition(hash_, pos, k, bits, nranks, m=m)
        counts = [int(x) for x in c.view(torch.int64).cpu().tolist()]
        return fp[:m].view(torch.int32), p[:m].view(torch.int64), counts

    def finalize(self, recv_fp, recv_pos, m_recv, global_counts, bits, rank, nranks):
        off, p, fp = self.L.seedtable_finalize(recv_fp.view(torch.uint32), recv_pos.view(torch.uint64), m_recv,
                                               global_counts.view(torch.uint32), bits, rank, nranks)
        return off.view(torch.int64), p[:m_recv].view(torch.int64), fp[:m_recv].view(torch.int32)


# ---------------------------------------------------------------- the exchange
def exchange_seedtable(hash_, pos, m: int, k: int, bits: int, phases: Phases, group=None):
    """C5: global seed table from per-rank minimizer lists (ranks hold contiguous,
    ascending position ranges, rank order = position order).

    Returns (offsets_local, pos_local, fp_local, base) where base is the global index of the
    rank's first entry; rank r owns buckets [r*2^bits/G, (r+1)*2^bits/G)."""
    rank = dist.get_rank(group)
    G = dist.get_world_size(group)
    if G & (G - 1):
        raise ValueError("world size must be a power of two (bucket ownership by top bits)")
    counts = phases.count(hash_, m, k, bits)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)        # uint32 sums as int32 bits
    send_fp, send_pos, send_counts = phases.partition(hash_, pos, m, k, bits, G)
    dev = send_pos.device
    sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(x) for x in rc.cpu().tolist()]
    m_recv = sum(recv_counts)
    recv_fp = torch.empty(max(1, m_recv), dtype=torch.int32, device=dev)
    recv_pos = torch.empty(max(1, m_recv), dtype=torch.int64, device=dev)
    dist.all_to_all_single(recv_fp[:m_recv], send_fp, output_split_sizes=recv_counts,
                           input_split_sizes=send_counts, group=group)
    dist.all_to_all_single(recv_pos[:m_recv], send_pos, output_split_sizes=recv_counts,
                           input_split_sizes=send_counts, group=group)
    off, pl, fl = phases.finalize(recv_fp, recv_pos, m_recv, counts, bits, rank, G)
    nbl = (1 << bits) // G
    base = int((counts.to(torch.int64) & 0xFFFFFFFF)[: rank * nbl].sum().item())
    return off, pl, fl, base
