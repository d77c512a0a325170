import os, sys, torch
sys.path.insert(0, '/root/repo')
import paper_1811_10074_b200 as P
from synthgen import device as SD
from synthgen import host as H
k, w, bits = 19, 10, 24
c3 = H.C3(); n = c3.n
seq = SD.c3_ascii(c3)
nw = (n + 31) // 32
words = torch.empty(nw + 1, dtype=torch.uint64, device="cuda"); inval = torch.empty(nw + 1, dtype=torch.uint32, device="cuda")
P.mz_encode(seq, words, inval); del seq
cap = int(0.25 * (n - k - w + 2)) + 1024
items = torch.empty(cap, dtype=torch.uint64, device="cuda")
hb = torch.empty(cap, dtype=torch.uint64, device="cuda"); pb = torch.empty(cap, dtype=torch.uint64, device="cuda")
dc = torch.zeros(1, dtype=torch.uint64, device="cuda")
ws = torch.empty(P.mz_workspace_bytes(n, k, w, P.MZ_IN_PACKED2), dtype=torch.uint8, device="cuda")
hist = torch.empty(P.seedtable_hist_words(cap, bits), dtype=torch.uint32, device="cuda")
for fused in [int(x) for x in os.environ.get("AB", "0,1,0,1").split(",")]:
    def run():
        P.mz_extract_ex(words, k, w, n=n, kind=P.MZ_IN_PACKED2, invalid=inval, capacity=cap, out_hash=hb, out_pos=pb,
                        d_count=dc, ws=ws, out_items=items, out_hist=hist if fused else None, hist_bits=bits)
    for _ in range(3): run()
    torch.cuda.synchronize(); ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(f"mz fused_hist={fused}: median {sorted(ts)[5]:.3f} ms", flush=True)
