"""GPU, two or more devices: the real multi-GPU path -- one process per GPU over NCCL, the
minimizer shards of the C3 recipe (R25), and the seed-table exchange both through
NCCL (exchange_seedtable) and fused into the partition over symmetric memory
(exchange_seedtable_p2p), with the CUDA phases reading the device record counts and the packed
items, as bench.py runs them.  Every rank's slice must equal its slice of the oracle table and
the shard records must concatenate to the oracle's list.  Skipped when fewer than two GPUs are
visible (the round's boxes have one; tests/test_dist_gloo.py covers the exchange logic on CPU
at world sizes 2, 4 and 8)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle as O
from synthgen import host as G

pytestmark = pytest.mark.gpu

N = 6_000_000
K, W, BITS = 19, 10, 24


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, exchange):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        import paper_1811_10074_b200 as P
        from paper_1811_10074_b200 import dist as D
        c3 = G.C3(n=N, mean_run=5_000.0, n_frac=0.02)
        sh = D.plan_shards(N, K, W, world)[rank]
        seq = torch.from_numpy(c3.ascii(sh.base_lo, sh.base_hi - sh.base_lo)).to(dev)
        n = seq.numel()
        cap = int(0.25 * n) + 1024
        items = torch.empty(cap, dtype=torch.uint64, device=dev)
        words, inval = P.mz_encode(seq)
        h, p, c = P.mz_extract_ex(words, K, W, n=n, kind=P.MZ_IN_PACKED2, invalid=inval, pos_base=sh.base_lo,
                                  win_lo=sh.win_lo, win_hi=sh.win_hi, capacity=cap, out_items=items)
        xchg = D.exchange_seedtable_p2p if exchange == "p2p" else D.exchange_seedtable
        off, pl, fl, base = xchg(h, p, cap, K, BITS, D.CudaPhases(d_m=c, items=items))
        torch.cuda.synchronize()
        m = int(c.item())
        q.put((rank, h[:m].cpu().numpy(), p[:m].cpu().numpy(), off.cpu().numpy(), pl.cpu().numpy(),
               fl.cpu().numpy(), base))
    finally:
        dist.destroy_process_group()


def _run(world, exchange):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, exchange)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    seq = G.C3(n=N, mean_run=5_000.0, n_frac=0.02).ascii()
    wk, wp = O.mz(seq, K, W)
    assert np.array_equal(np.concatenate([r[1] for r in res]), wk)
    assert np.array_equal(np.concatenate([r[2] for r in res]), wp)
    wo, wf, wpos = O.seedtable(wk, wp, K, BITS)
    nbl = (1 << BITS) // world
    for rank, _, _, off, pl, fl, base in res:
        assert np.array_equal(off.astype(np.uint64) + np.uint64(base), wo[rank * nbl: (rank + 1) * nbl + 1])
    assert np.array_equal(np.concatenate([r[4] for r in res]).view(np.uint64), wpos)
    assert np.array_equal(np.concatenate([r[5] for r in res]).view(np.uint32), wf)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two or more GPUs")
@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
def test_multi_rank_exchange_vs_oracle(exchange):
    _run(2 if torch.cuda.device_count() < 4 else 4, exchange)


def test_one_rank_nccl_exchange_vs_oracle():
    """The same worker as one NCCL rank on one GPU: the exchange's collectives are trivial, but
    the CUDA phases run with the device record count (capacity-sized arrays + d_count)."""
    _run(1, "nccl")
