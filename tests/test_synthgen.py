"""Checks of the shared input generators (synthgen/host.py) -- CPU only.

Statistical shape of the synthetic stand-ins for the paper's workloads
(hashed 15-mers of GRCh38; BASELINE.json configs C1-C4), and the
counter-based property that sub-ranges reproduce the full stream.
"""
import numpy as np

from synthgen import host as G


def test_mix64_known_values():
    # SplitMix64 reference outputs for seed 0 (first three draws of the published generator)
    v = G.mix64(0, np.arange(3, dtype=np.uint64))
    assert [hex(int(x)) for x in v] == ["0xe220a8397b1dcdaf", "0x6e789e6aa1b965f4", "0x6c45d188009454f"]


def test_subrange_reproduces():
    a = G.c1_ascii(10_000)
    assert np.array_equal(a[1234:5678], G.c1_ascii(5678 - 1234, lo=1234))
    c3 = G.C3(n=3_000_000)
    full = c3.ascii()
    assert np.array_equal(full[2_000_000:2_100_000], c3.ascii(2_000_000, 100_000))


def test_c1_uniform():
    a = G.c1_ascii(1_000_000)
    cnt = np.array([np.sum(a == ord(c)) for c in "ACGT"]) / len(a)
    assert np.all(np.abs(cnt - 0.25) < 0.003)


def test_c3_shape():
    c3 = G.C3()                                    # full 3.1 Gbp layout (intervals only)
    iv = c3.intervals
    frac = (iv[:, 1] - iv[:, 0]).sum() / c3.n
    assert 0.008 < frac < 0.012
    assert 2500 < len(iv) < 3800
    assert np.all(iv[1:, 0] > iv[:-1, 1])          # sorted, disjoint, separated by a gap
    s = c3.ascii(0, 2_000_000)
    valid = s != ord("N")
    gc = np.isin(s[valid], np.frombuffer(b"CG", np.uint8)).mean()
    assert abs(gc - 0.41) < 0.003


def test_c4_shape():
    c4 = G.C4()
    assert c4.nreads == 1_000_000
    assert abs(c4.lengths.mean() - 10_000) < 100
    assert abs(c4.lengths.std() - 8_000) < 300
    assert c4.lengths.min() >= 24                  # k + w - 1 for k=15, w=10 (sample property)
    assert np.all(c4.starts + c4.lengths <= c4.tlen)
    r = c4.read_ascii(17)
    tmpl = G.codes_to_ascii(G.uniform_codes(G.SEED_C4_TEMPLATE, int(c4.starts[17]), len(r)))
    diff = (r != tmpl).mean()
    assert 0.07 < diff < 0.13                      # 10 % substitution


def test_c2_streams():
    u = G.c2_u32(1 << 16)
    r = G.mix64(G.SEED_C2_U32, np.arange(1 << 15, dtype=np.uint64))
    assert np.array_equal(u.view(np.uint64), r)    # little-endian halves
    f = G.c2_f32(1 << 18)
    assert abs(f.mean()) < 0.01 and abs(f.std() - 1) < 0.01
    assert np.array_equal(G.c2_f32(100, lo=500), f[500:600])
