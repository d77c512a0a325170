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


def plan_slsum(n: int, w: int, nranks: int, align: int = 4) -> list[tuple[int, int, int, int]]:
    """C2 sliding sums across ranks: rank g owns outputs [o_a, o_b) of the
    n - w + 1 and reads inputs [o_a, o_b + w - 1) -- a w-1 element halo, no collective.
    Cuts are rounded down to `align` elements (16-byte vectors for 4-byte types).  Returns
    [(o_a, o_b, in_lo, in_hi)] per rank; concatenating the ranks' outputs gives y."""
    nout = max(0, n - w + 1)
    cuts = [0] + [(nout * g // nranks) // align * align for g in range(1, nranks)] + [nout]
    out = []
    for g in range(nranks):
        a, b = cuts[g], max(cuts[g], cuts[g + 1])
        out.append((a, b, a, b + w - 1 if b > a else a))
    return out


# ---------------------------------------------------------------- local phases
class Phases:
    """Local seed-table phases on one rank (see include/mzslsum.h)."""

    def count(self, hash_, m, k, bits):  # -> int32[2^bits] (uint32 bits)
        raise NotImplementedError

    def partition(self, hash_, pos, m, k, bits, nranks):  # -> (fp int32[m], pos int64[m], counts list[int])
        raise NotImplementedError

    def finalize(self, recv_fp, recv_pos, m_recv, global_counts, bits, rank, nranks):
        raise NotImplementedError  # -> (offsets_local int64[nbl+1], pos int64[m_recv], fp int32[m_recv])

    def partition_p2p(self, hash_, pos, m, k, bits, peer_fp, peer_pos, peer_base):  # -> status code
        raise NotImplementedError


class CudaPhases(Phases):
    """The product: every phase is a libmzslsum call on the current stream.  `d_m` (optional,
    a device uint64 count with m as its upper bound) keeps the record count on the device."""

    def __init__(self, d_m=None, items=None):
        from . import _lib as L
        self.L = L
        self.d_m = d_m
        self.items = items    # mz_extract_ex's packed items: the fused partition reads 8 B per entry

    def count(self, hash_, m, k, bits):
        return self.L.seedtable_count(hash_, k, bits, m=m, d_m=self.d_m).view(torch.int32)

    def partition(self, hash_, pos, m, k, bits, nranks):
        fp, p, c = self.L.seedtable_partition(hash_, pos, k, bits, nranks, m=m)
        counts = [int(x) for x in c.view(torch.int64).cpu().tolist()]
        return fp[:m].view(torch.int32), p[:m].view(torch.int64), counts

    def finalize(self, recv_fp, recv_pos, m_recv, global_counts, bits, rank, nranks):
        off, p, fp = self.L.seedtable_finalize(recv_fp.view(torch.uint32), recv_pos.view(torch.uint64), m_recv,
                                               global_counts.view(torch.uint32), bits, rank, nranks)
        return off.view(torch.int64), p[:m_recv].view(torch.int64), fp[:m_recv].view(torch.int32)

    def partition_p2p(self, hash_, pos, m, k, bits, peer_fp, peer_pos, peer_base):
        return self.L.seedtable_partition_p2p(hash_.view(torch.uint64), pos.view(torch.uint64), k, bits,
                                              peer_fp, peer_pos, peer_base, m=m, d_m=self.d_m, items=self.items)


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
    d_m = getattr(phases, "d_m", None)
    if d_m is not None:                              # all_to_all needs host split sizes anyway
        m = min(m, int(d_m.view(torch.int64).item()))
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


# ---------------------------------------------------------------- the fused exchange (peer memory)
def p2p_plan(owner_counts, span_ok):
    """Host logic of the fused exchange, identical on every rank (it sees the same gathered
    matrix).  owner_counts[s][o] = entries sender s holds for owner o; span_ok[s] = sender s's
    positions span < 2^32 (the narrow-item precondition of seedtable_partition_p2p).
    Returns (use_p2p, peer_base[s][o] = where sender s starts writing in owner o's buffer,
    recv[o] = entries owner o receives, cap = the common symmetric-buffer capacity)."""
    G = len(owner_counts)
    recv = [sum(owner_counts[s][o] for s in range(G)) for o in range(G)]
    base = [[sum(owner_counts[t][o] for t in range(s)) for o in range(G)] for s in range(G)]
    cap = max(1, max(recv) if recv else 1)
    return all(bool(x) for x in span_ok), base, recv, cap


class SymmPeerMem:
    """The product's peer memory: one torch symmetric-memory buffer per (group, device), cap u64
    positions then cap u32 fingerprints, mapped into every peer over NVLink.  Grow-only with
    1/8 headroom; every rank takes the same decision (cap is agreed).

    Two steps, so that a rank that cannot allocate never leaves the others waiting inside the
    collective mapping: prepare() allocates locally (no collective) and returns whether it
    could; the caller agrees on the result (all_reduce MIN) and only then calls get(), whose
    rendezvous is collective.  get() returns (c, local recv_pos int64[c], local recv_fp
    int32[c], fp pointers[G], pos pointers[G])."""

    def __init__(self):
        self._ent = {}
        self._new = {}

    def prepare(self, cap: int, dev, group) -> bool:
        key = (id(group), dev.index)
        ent = self._ent.get(key)
        if ent is not None and ent[0] >= cap:
            return True
        try:
            import torch.distributed._symmetric_memory as symm_mem
            c = cap + cap // 8 + 1024
            self._new[key] = (c, symm_mem.empty(c + (c + 1) // 2, dtype=torch.uint64, device=dev))
            return True
        except Exception:                          # no symmetric memory on this box / out of memory
            self._new.pop(key, None)
            return False

    def get(self, cap: int, dev, group):
        key = (id(group), dev.index)
        ent = self._ent.get(key)
        if key not in self._new and (ent is None or ent[0] < cap) and not self.prepare(cap, dev, group):
            raise RuntimeError("symmetric memory allocation failed")   # (callers agree on prepare() first)
        if key in self._new:
            import torch.distributed._symmetric_memory as symm_mem
            c, buf = self._new.pop(key)
            hdl = symm_mem.rendezvous(buf, group if group is not None else dist.group.WORLD)
            G = dist.get_world_size(group)
            ptrs = [hdl.get_buffer(o, (1,), torch.uint8, 0).data_ptr() for o in range(G)]
            self._ent[key] = (c, buf, hdl, ptrs)
        c, buf, _, ptrs = self._ent[key]
        return (c, buf[:c].view(torch.int64), buf[c:].view(torch.uint32)[:c].view(torch.int32),
                [p + 8 * c for p in ptrs], list(ptrs))


_PEER_MEM = SymmPeerMem()


def exchange_seedtable_p2p(hash_, pos, m: int, k: int, bits: int, phases: Phases, group=None, peer_mem=None):
    """C5 with the partition fused into the all-to-all: each sender's last radix pass writes
    its (fingerprint, position) entries straight into the owners' symmetric buffers over
    NVLink (include/mzslsum.h seedtable_partition_p2p), so no send buffer and no NCCL
    all_to_all exist.  Collectives left: all_reduce of the bucket counts and one all_gather of
    G x G owner counts (to place each sender's run), plus two barriers around the writes.
    Same result as exchange_seedtable; falls back to it when a rank's positions span >= 2^32
    (decided uniformly from the gathered flags).  `peer_mem` is injectable for the CPU tests."""
    rank = dist.get_rank(group)
    G = dist.get_world_size(group)
    if G & (G - 1) or G < 2:
        raise ValueError("fused exchange needs a power-of-two world size >= 2")
    peer_mem = peer_mem or _PEER_MEM
    dev = hash_.device
    d_m = getattr(phases, "d_m", None)             # device record count (CudaPhases), if any
    counts = phases.count(hash_, m, k, bits)
    nbl = (1 << bits) // G
    own = (counts.to(torch.int64) & 0xFFFFFFFF).view(G, nbl).sum(1)
    # the narrow-item precondition (positions span < 2^32), decided on the device
    if m > 0:
        last = (d_m.view(torch.int64).clamp(1, m) - 1) if d_m is not None else torch.tensor([m - 1], device=dev)
        ends = torch.cat([pos[:1].view(torch.int64), pos.view(torch.int64).index_select(0, last)])
        span = (ends[1] - ends[0]).view(1)
        span_ok = ((span >= 0) & (span < (1 << 32))).to(torch.int64)
    else:
        span_ok = torch.ones(1, dtype=torch.int64, device=dev)
    row = torch.cat([own, span_ok])
    rows = [torch.empty_like(row) for _ in range(G)]
    dist.all_gather(rows, row, group=group)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    mat = torch.stack(rows).cpu().tolist()         # the one host read: every sender's owner counts
    use, base, recv, cap = p2p_plan([r[:G] for r in mat], [r[G] for r in mat])
    if not use:
        return exchange_seedtable(hash_, pos, m, k, bits, phases, group)

    def agree(ok: bool) -> bool:
        flag = torch.tensor([1 if ok else 0], dtype=torch.int64, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        return bool(int(flag.item()))

    # local allocation first, agreed on by every rank, then the collective mapping
    if not agree(peer_mem.prepare(cap, dev, group)):
        return exchange_seedtable(hash_, pos, m, k, bits, phases, group)
    c, recv_pos, recv_fp, fp_ptrs, pos_ptrs = peer_mem.get(cap, dev, group)
    dist.barrier(group=group)                      # every owner is done with its previous contents
    rc = phases.partition_p2p(hash_, pos, m, k, bits, fp_ptrs, pos_ptrs, base[rank])
    # a sender whose input broke the narrow precondition (unsorted positions) has written wrong
    # entries into the owners' buffers: every rank then discards them and takes the NCCL path
    if not agree(rc == 0):
        return exchange_seedtable(hash_, pos, m, k, bits, phases, group)
    off, pl, fl = phases.finalize(recv_fp, recv_pos, recv[rank], counts, bits, rank, G)
    b0 = int((counts.to(torch.int64) & 0xFFFFFFFF)[: rank * nbl].sum().item())
    return off, pl, fl, b0
