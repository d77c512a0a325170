"""CPU multi-process tests of the multi-GPU path (world_size 2 and 4, gloo backend).

The planner (paper_1811_10074_b200.dist.plan_shards) and the C5 exchange logic
(exchange_seedtable: all_reduce of counts, all_to_all of split sizes and entries,
per-rank base offsets) run exactly as on the GPUs; only the local phases are replaced by
oracle-backed ones (test-only), so no GPU is needed.  Every rank's slice must equal the
matching slice of the single-process oracle table, and the shard outputs must
concatenate to the single-process minimizer list (R25)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from synthgen import host as H

K, W, BITS = 16, 10, 12   # 2k = 32: the fingerprint is the key itself (oracle helpers stay exact)
N = 400_000


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OraclePhases:
    """Test-only local phases built from the oracle + numpy (never used by the product)."""

    def count(self, hash_, m, k, bits):
        key = hash_[:m].numpy().view(np.uint64)
        off, _, _ = O.seedtable(key, np.zeros(m, np.uint64), k, bits)
        return torch.from_numpy(np.diff(off.astype(np.int64)).astype(np.int32))

    def partition(self, hash_, pos, m, k, bits, nranks):
        key = hash_[:m].numpy().view(np.uint64)
        fp = np.array([O.fingerprint(int(x), k) for x in key], dtype=np.uint32)
        g = nranks.bit_length() - 1
        owner = (fp >> (32 - g)) if g else np.zeros(m, np.uint32)
        order = np.argsort(owner, kind="stable")
        counts = np.bincount(owner, minlength=nranks).tolist()
        return (torch.from_numpy(fp[order].view(np.int32).copy()),
                torch.from_numpy(pos[:m].numpy()[order].copy()), counts)

    def finalize(self, recv_fp, recv_pos, m_recv, global_counts, bits, rank, nranks):
        fp = recv_fp[:m_recv].numpy().view(np.uint32).astype(np.uint64)
        ps = recv_pos[:m_recv].numpy().view(np.uint64)
        off, fpo, po = O.seedtable(fp, ps, 16, bits)          # 2k = 32: key = fingerprint
        nbl = (1 << bits) // nranks
        loc = off[rank * nbl: (rank + 1) * nbl + 1].astype(np.int64)
        return (torch.from_numpy(loc - loc[0]), torch.from_numpy(po.view(np.int64).copy()),
                torch.from_numpy(fpo.view(np.int32).copy()))


    def partition_p2p(self, hash_, pos, m, k, bits, peer_fp, peer_pos, peer_base):
        """Writes each owner's run at peer_base[o] of that owner's (file-backed) buffers,
        in position order, as the kernel does over NVLink."""
        fp, ps, counts = self.partition(hash_, pos, m, k, bits, len(peer_fp))
        a = 0
        for o, n in enumerate(counts):
            f = np.memmap(peer_fp[o], dtype=np.int32, mode="r+")
            p = np.memmap(peer_pos[o], dtype=np.int64, mode="r+")
            f[peer_base[o]: peer_base[o] + n] = fp.numpy()[a: a + n]
            p[peer_base[o]: peer_base[o] + n] = ps.numpy()[a: a + n]
            f.flush()
            p.flush()
            a += n
        return 0


class FilePeerMem:
    """Test-only stand-in for the symmetric buffers: one shared file pair per rank; the
    'pointers' handed to partition_p2p are the peers' file paths."""

    def __init__(self, root, rank, world, fail_prepare=False):
        self.root, self.rank, self.world = root, rank, world
        self.fail_prepare = fail_prepare

    def _paths(self, o):
        return os.path.join(self.root, f"fp{o}"), os.path.join(self.root, f"pos{o}")

    def prepare(self, cap, dev, group):
        """Local allocation (no collective), as SymmPeerMem.prepare."""
        if self.fail_prepare:
            return False
        c = cap + 7
        fpp, psp = self._paths(self.rank)
        np.memmap(fpp, dtype=np.int32, mode="w+", shape=(c,)).flush()
        np.memmap(psp, dtype=np.int64, mode="w+", shape=(c,)).flush()
        return True

    def get(self, cap, dev, group):
        c = cap + 7
        fpp, psp = self._paths(self.rank)
        dist.barrier(group=group)
        self.local = (np.memmap(fpp, dtype=np.int32, mode="r"), np.memmap(psp, dtype=np.int64, mode="r"))
        return (c, _LazyFile(psp, np.int64), _LazyFile(fpp, np.int32),
                [self._paths(o)[0] for o in range(self.world)], [self._paths(o)[1] for o in range(self.world)])


class _LazyFile:
    """Reads the file when finalize slices it (after the second barrier)."""

    def __init__(self, path, dt):
        self.path, self.dt = path, dt

    def __getitem__(self, sl):
        return torch.from_numpy(np.array(np.memmap(self.path, dtype=self.dt, mode="r"))[sl])


class BadInputPhases(OraclePhases):
    """Test-only: the fused write reports a broken precondition on rank 1 (as the kernel does
    for unsorted positions), after writing garbage into the owners' buffers."""

    def __init__(self, rank):
        self.rank = rank

    def partition_p2p(self, hash_, pos, m, k, bits, peer_fp, peer_pos, peer_base):
        rc = super().partition_p2p(hash_, pos, m, k, bits, peer_fp, peer_pos, peer_base)
        if self.rank != 1:
            return rc
        for o in range(len(peer_fp)):
            f = np.memmap(peer_fp[o], dtype=np.int32, mode="r+")
            f[:] = -1
            f.flush()
        return -2


def _worker(rank, world, port, q, p2p_root=None, mode="ok"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1811_10074_b200 import dist as D
        c3 = H.C3(n=N)
        seq = c3.ascii()
        sh = D.plan_shards(N, K, W, world)[rank]
        sub = seq[sh.base_lo: sh.base_hi]
        key, pos = O.mz(sub, K, W, pos_base=sh.base_lo, win_lo=sh.win_lo, win_hi=sh.win_hi)
        m = len(key)
        phases = BadInputPhases(rank) if mode == "bad_input" else OraclePhases()
        args = (torch.from_numpy(key.view(np.int64).copy()), torch.from_numpy(pos.view(np.int64).copy()),
                m, K, BITS, phases)
        if p2p_root is None:
            off, pl, fl, base = D.exchange_seedtable(*args)
        else:
            pm = FilePeerMem(p2p_root, rank, world, fail_prepare=(mode == "no_peer_mem" and rank == world - 1))
            off, pl, fl, base = D.exchange_seedtable_p2p(*args, peer_mem=pm)
        q.put((rank, key, pos, off.numpy(), pl.numpy(), fl.numpy(), base))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,p2p,mode", [(2, False, "ok"), (4, False, "ok"), (8, False, "ok"), (2, True, "ok"),
                                           (4, True, "ok"), (8, True, "ok"), (4, True, "no_peer_mem"),
                                           (2, True, "bad_input")])
def test_sharded_extraction_and_exchange(world, p2p, mode, tmp_path):
    """p2p=True runs exchange_seedtable_p2p (the fused partition-to-peers path) with
    file-backed peer buffers in place of NVLink-mapped symmetric memory.  no_peer_mem: one
    rank cannot allocate its buffer, so every rank takes the NCCL exchange (no rank is left in
    the collective mapping).  bad_input: one sender's fused write reports a broken precondition
    after writing garbage; every rank discards the buffers and takes the NCCL exchange."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    root = str(tmp_path) if p2p else None
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, root, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    seq = H.C3(n=N).ascii()
    wk, wp = O.mz(seq, K, W)
    # shard outputs concatenate to the single-process list
    assert np.array_equal(np.concatenate([r[1] for r in res]), wk)
    assert np.array_equal(np.concatenate([r[2] for r in res]), wp)
    # the ranks' table slices concatenate to the single-process table
    wo, wf, wpos = O.seedtable(wk, wp, K, BITS)
    nbl = (1 << BITS) // world
    for rank, _, _, off, pl, fl, base in res:
        assert np.array_equal(off.astype(np.uint64) + np.uint64(base), wo[rank * nbl: (rank + 1) * nbl + 1])
    assert np.array_equal(np.concatenate([r[4] for r in res]).view(np.uint64), wpos)
    assert np.array_equal(np.concatenate([r[5] for r in res]).view(np.uint32), wf)


def test_plan_shards_covers_windows():
    from paper_1811_10074_b200 import dist as D
    for n, k, w, G in [(10_000, 19, 10, 8), (100, 15, 10, 4), (24, 15, 10, 2), (3_100_000_000, 19, 10, 8)]:
        sh = D.plan_shards(n, k, w, G)
        nwin = max(0, n - (k + w - 1) + 1)
        assert sh[0].win_a == 0 and sh[-1].win_b == nwin
        for a, b in zip(sh, sh[1:]):
            assert a.win_b == b.win_a
        for s in sh:
            if s.win_b > s.win_a:
                assert s.base_lo == max(0, s.win_a - 1) and s.base_hi == s.win_b + k + w - 2
                assert s.win_hi - s.win_lo == s.win_b - s.win_a


def test_p2p_plan():
    from paper_1811_10074_b200 import dist as D
    oc = [[3, 0, 5], [1, 2, 0], [4, 4, 4]]          # [sender][owner]
    use, base, recv, cap = D.p2p_plan(oc, [1, 1, 1])
    assert use and recv == [8, 6, 9] and cap == 9
    assert base == [[0, 0, 0], [3, 0, 5], [4, 2, 5]]
    assert not D.p2p_plan(oc, [1, 0, 1])[0]
    assert D.p2p_plan([[0, 0], [0, 0]], [1, 1])[3] == 1


def test_plan_reads_balanced():
    from paper_1811_10074_b200 import dist as D
    c4 = H.C4(nreads=10_000)
    parts = D.plan_reads(c4.read_off, 8)
    assert parts[0][0] == 0 and parts[-1][1] == 10_000
    sizes = [int(c4.read_off[b] - c4.read_off[a]) for a, b in parts]
    assert max(sizes) < 1.2 * (c4.n / 8)


def test_plan_slsum_shards_concatenate():
    """C2 sharding: every rank's slice, summed by the oracle on its own input
    range (halo w-1), concatenates to the single-process result."""
    from paper_1811_10074_b200 import dist as D
    rng = np.random.default_rng(8)
    for n, w, G in [(10_000, 4, 8), (10_000, 1000, 4), (5000, 17, 3), (64, 64, 2), (100, 3, 8)]:
        x = rng.integers(0, 2 ** 32, size=n, dtype=np.uint64).astype(np.uint32)
        want = O.slsum(O.MIN_U32, w, x)
        parts = []
        for a, b, lo, hi in D.plan_slsum(n, w, G):
            assert a % 4 == 0 or a == 0
            ys = O.slsum(O.MIN_U32, w, x[lo:hi]) if hi > lo else np.zeros(0, np.uint32)
            assert len(ys) == b - a
            parts.append(ys)
        assert np.array_equal(np.concatenate(parts), want)
