"""The README's Python API example, as a script (run from the repo root: PYTHONPATH=. python tools/readme_example.py)."""
import torch, paper_1811_10074_b200 as P

seq = torch.frombuffer(bytearray(b"ACGT" * 1000), dtype=torch.uint8).cuda()  # ASCII DNA
h, pos = P.mz_extract(seq, 15, 10)                      # minimizers: hashes and positions
off, tab_pos, tab_fp = P.seedtable_build(h, pos, 15, 24)  # CSR seed table, 2^24 buckets
hit_off, hit_pos, total = P.seedtable_lookup(h[:100], 15, 24, off, tab_fp, tab_pos)
x = torch.randint(0, 2**31, (1 << 20,), dtype=torch.int64).to(torch.uint32).cuda()
y = P.slsum_run(P.SLSUM_MIN_U32, 10, x)                 # sliding-window min, Alg. 2 path
y2 = P.slsum_run(P.SLSUM_MIN_U32, 10, x, path=P.SLSUM_PATH_COMMUTATIVE)  # O(log w) doubling

print('readme example ok', int(total.view(torch.int64).item()), y.shape, bool((y == y2).all()))
