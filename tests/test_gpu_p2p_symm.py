"""GPU: the product's peer memory (dist.SymmPeerMem, torch symmetric memory) with the fused
partition kernel writing into it.  One GPU is available, so the group has one rank; owner 0's
buffer is the symmetric one (reached through its mapped pointer), owner 1's a plain device
buffer.  Checks the pointer layout (positions, then fingerprints at +8c) and that the local
views finalize to the oracle's slice.  The G >= 2 exchange logic runs under gloo
(tests/test_dist_gloo.py); the per-sender kernel with all owners on one device in
tests/test_gpu_seedtable.py::test_partition_p2p_emulated."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle as O
from synthgen import host as G

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_1811_10074_b200")


def test_symm_buffers_receive_partition():
    from paper_1811_10074_b200 import dist as D
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        k, bits, nr = 19, 24, 2
        key, pos = O.mz(G.C3(n=1_000_000).ascii(), k, 10)
        m = len(key)
        kt = torch.from_numpy(key).cuda()
        pt = torch.from_numpy(pos).cuda()
        cnt = P.seedtable_count(kt, k, bits)
        gc = cnt.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        nbl = (1 << bits) // nr
        own = gc.view(nr, nbl).sum(1).tolist()
        pm = D.SymmPeerMem()
        c, rpos, rfp, fps, poss = pm.get(own[0], torch.device("cuda:0"), None)
        assert c >= own[0] and rpos.data_ptr() == poss[0] and rfp.data_ptr() == fps[0]
        other_fp = torch.empty(own[1], dtype=torch.uint32, device="cuda")
        other_pos = torch.empty(own[1], dtype=torch.uint64, device="cuda")
        rc = P.seedtable_partition_p2p(kt, pt, k, bits, [fps[0], other_fp.data_ptr()],
                                       [poss[0], other_pos.data_ptr()], [0, 0])
        assert rc == P.SLSUM_OK
        wo, wf, wp = O.seedtable(key, pos, k, bits)
        off, po, fp = P.seedtable_finalize(rfp.view(torch.uint32), rpos.view(torch.uint64), own[0],
                                           cnt, bits, 0, nr)
        assert np.array_equal(off.cpu().numpy(), wo[: nbl + 1])
        assert np.array_equal(po[: own[0]].cpu().numpy(), wp[: own[0]])
        assert np.array_equal(fp[: own[0]].cpu().numpy(), wf[: own[0]])
        # a second call with a larger capacity re-rendezvouses and still aliases correctly
        c2, rpos2, _, _, poss2 = pm.get(c * 2, torch.device("cuda:0"), None)
        assert c2 >= 2 * c and rpos2.data_ptr() == poss2[0]
    finally:
        dist.destroy_process_group()
