"""GPU parity: slsum_run_ex (GENERIC and COMMUTATIVE paths) vs the oracle's strict left
fold (Eq. 2).  Integer ops bit-exact; f32 add within the BASELINE
tolerance |g - o| <= 1e-5 |o| + 1e-6 w."""
import numpy as np
import pytest
import torch

import oracle as O
from synthgen import host as G

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1811_10074_b200")

OPS = [(P.SLSUM_MIN_U32, O.MIN_U32), (P.SLSUM_MAX_U32, O.MAX_U32), (P.SLSUM_ADD_U32, O.ADD_U32),
       (P.SLSUM_ADD_F32, O.ADD_F32), (P.SLSUM_AFFINE_U32X2, O.AFFINE_U32X2), (P.SLSUM_MIN_U64, O.MIN_U64),
       (P.SLSUM_CONCAT_U32X2, O.CONCAT_U32X2)]
PAIR_OPS = (P.SLSUM_AFFINE_U32X2, P.SLSUM_CONCAT_U32X2)    # (n, 2) uint32, not commutative
WS = [1, 2, 3, 4, 5, 6, 7, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 20, 22, 24, 26, 28, 30, 31, 32, 33, 64, 100, 255, 256, 1000, 1024]


def _input(op, n, rng):
    if op == P.SLSUM_ADD_F32:
        return rng.standard_normal(n).astype(np.float32)
    if op == P.SLSUM_AFFINE_U32X2:
        return rng.integers(0, 2 ** 32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    if op == P.SLSUM_MIN_U64:
        return rng.integers(0, 2 ** 63, size=n, dtype=np.uint64)
    if op == P.SLSUM_CONCAT_U32X2:     # symbols of a sigma-letter alphabet (L67), else any pairs
        sigma = int(rng.choice([4, 20, 256, 0]))
        if sigma == 0:
            return rng.integers(0, 2 ** 32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
        b = rng.integers(0, sigma, size=n, dtype=np.uint64).astype(np.uint32)
        return np.stack([b, np.full(n, sigma, np.uint32)], axis=1)
    hi = 2 ** 32 if rng.random() < 0.7 else 5  # small alphabets force ties
    return rng.integers(0, hi, size=n, dtype=np.uint64).astype(np.uint32)


def _check(op, w, x, got):
    want = O.slsum(dict(OPS)[op], w, x)
    assert got.shape == want.shape
    if op == P.SLSUM_ADD_F32:
        tol = 1e-5 * np.abs(want.astype(np.float64)) + 1e-6 * w
        err = np.abs(got.astype(np.float64) - want.astype(np.float64))
        assert np.all(err <= tol), (w, float((err / tol).max()))
    else:
        assert np.array_equal(got, want), (op, w)


def _run(op, w, x, path):
    xt = torch.from_numpy(x).cuda()
    y = P.slsum_run(op, w, xt, path=path)
    torch.cuda.synchronize()
    return y.cpu().numpy()  # uint32/uint64 tensors only move bytes here (no torch arithmetic)


@pytest.mark.parametrize("op", [o for o, _ in OPS])
@pytest.mark.parametrize("w", WS)
def test_generic_vs_oracle(op, w):
    rng = np.random.default_rng(op * 10000 + w)
    for n in sorted({w, w + 1, 2 * w + 3, 5000, 70_001}):
        x = _input(op, n, rng)
        _check(op, w, x, _run(op, w, x, P.SLSUM_PATH_GENERIC))


@pytest.mark.parametrize("op", [o for o, _ in OPS if o not in PAIR_OPS])
@pytest.mark.parametrize("w", WS)
def test_commutative_vs_oracle(op, w):
    rng = np.random.default_rng(op * 777 + w)
    for n in sorted({w, w + 5, 9000, 50_003}):
        x = _input(op, n, rng)
        _check(op, w, x, _run(op, w, x, P.SLSUM_PATH_COMMUTATIVE))


@pytest.mark.parametrize("w", WS + [4095, 4096, 4097, 8000])
def test_recurrent_vs_oracle(w):
    """RECURRENT path (Conclusion): prefix differences for the invertible u32 add,
    bit-exact vs the strict left fold, across several tiles and a ragged tail."""
    rng = np.random.default_rng(4242 + w)
    for n in sorted({w, w + 1, 2 * w + 3, 5000, 70_001, 3 * 4096 + 17}):
        if n < w:
            continue
        x = rng.integers(0, 2 ** 32, size=n, dtype=np.uint64).astype(np.uint32)
        _check(P.SLSUM_ADD_U32, w, x, _run(P.SLSUM_ADD_U32, w, x, P.SLSUM_PATH_RECURRENT))
    # unaligned output and input views take the scalar loads / stores
    x = rng.integers(0, 2 ** 32, size=20_000, dtype=np.uint64).astype(np.uint32)
    xt = torch.from_numpy(np.concatenate([[0], x]).astype(np.uint32)).cuda()[1:]
    yb = torch.empty(20_000 - w + 2, dtype=torch.uint32, device="cuda")
    if w <= 20_000:
        y = P.slsum_run(P.SLSUM_ADD_U32, w, xt, y=yb[1:], path=P.SLSUM_PATH_RECURRENT)
        assert np.array_equal(y.cpu().numpy(), O.slsum(O.ADD_U32, w, x))


@pytest.mark.parametrize("op", [o for o, _ in OPS])
@pytest.mark.parametrize("w", WS)
def test_scalar_alg1_bit_exact(op, w):
    """SCALAR path = Algorithm 1: every window is the strict left fold, so the
    result equals the oracle's bit for bit for every op -- f32 add included (no tolerance)."""
    rng = np.random.default_rng(op * 31337 + w)
    for n in sorted({w, w + 1, 2 * w + 3, 5000, 70_001}):
        x = _input(op, n, rng)
        got = _run(op, w, x, P.SLSUM_PATH_SCALAR)
        want = O.slsum(dict(OPS)[op], w, x)
        if op == P.SLSUM_ADD_F32:
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), w
        else:
            assert np.array_equal(got, want), (op, w)


def test_scalar_rejects_w_over_1024():
    x = torch.zeros(5000, dtype=torch.uint32, device="cuda")
    with pytest.raises(P.SlsumError) as e:
        P.slsum_run(P.SLSUM_MIN_U32, 1025, x, path=P.SLSUM_PATH_SCALAR)
    assert e.value.rc == P.SLSUM_EUNSUPPORTED


@pytest.mark.parametrize("op", [o for o, _ in OPS if o != P.SLSUM_ADD_U32])
def test_recurrent_rejects_non_invertible(op):
    x = torch.zeros((100, 2) if op in PAIR_OPS else (100,),
                    dtype={P.SLSUM_ADD_F32: torch.float32, P.SLSUM_MIN_U64: torch.uint64}.get(op, torch.uint32),
                    device="cuda")
    with pytest.raises(P.SlsumError) as e:
        P.slsum_run(op, 4, x, path=P.SLSUM_PATH_RECURRENT)
    assert e.value.rc == P.SLSUM_EUNSUPPORTED


@pytest.mark.parametrize("w", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024])
@pytest.mark.parametrize("path", ["generic", "commutative"])
def test_unaligned_and_ragged_views(w, path):
    """The warp- and CTA-tiled kernels fall back to scalar loads/stores for views 4 or 8 bytes
    off a 16-byte boundary, and handle ragged tails; bit-exact vs the oracle (u32 / u64)."""
    pth = P.SLSUM_PATH_GENERIC if path == "generic" else P.SLSUM_PATH_COMMUTATIVE
    rng = np.random.default_rng(w * 3 + len(path))
    for op, dt in ((P.SLSUM_MIN_U32, np.uint32), (P.SLSUM_ADD_U32, np.uint32), (P.SLSUM_MIN_U64, np.uint64)):
        for n in (w, w + 3, 3 * 512 + 7, 40_003):
            x = rng.integers(0, 2 ** 32 if dt == np.uint32 else 2 ** 63, size=n, dtype=np.uint64).astype(dt)
            xt = torch.from_numpy(np.concatenate([np.zeros(1, dt), x])).cuda()[1:]
            yb = torch.empty(n - w + 2, dtype=xt.dtype, device="cuda")
            y = P.slsum_run(op, w, xt, y=yb[1:], path=pth)
            assert np.array_equal(y.cpu().numpy(), O.slsum(dict(OPS)[op], w, x)), (op, n)


@pytest.mark.parametrize("op", PAIR_OPS)
def test_pair_ops_rejected_by_commutative_path(op):
    x = torch.zeros((100, 2), dtype=torch.uint32, device="cuda")
    with pytest.raises(P.SlsumError) as e:
        P.slsum_run(op, 4, x, path=P.SLSUM_PATH_COMMUTATIVE)
    assert e.value.rc == P.SLSUM_EUNSUPPORTED


@pytest.mark.parametrize("path", [P.SLSUM_PATH_GENERIC, P.SLSUM_PATH_SCALAR])
def test_concat_kmer_codes_any_alphabet(path):
    """k-mers as a sliding sum under concatenation (L67) for alphabets that are not 2-bit
    packable: a 20-letter (protein) alphabet with k = 7 (20^7 < 2^32, exact codes) and DNA
    with k = 16 (= the 2-bit k-mer codes); checked against Python big-integer numerals."""
    rng = np.random.default_rng(67)
    for sigma, k in ((20, 7), (4, 16), (256, 4)):
        n = 50_001
        b = rng.integers(0, sigma, size=n, dtype=np.uint64).astype(np.uint32)
        x = np.stack([b, np.full(n, sigma, np.uint32)], axis=1)
        y = _run(P.SLSUM_CONCAT_U32X2, k, x, path)
        assert np.all(y[:, 1] == np.uint32(sigma ** k % 2 ** 32))
        pw = np.array([sigma ** (k - 1 - t) for t in range(k)], dtype=np.uint64)
        want = (np.lib.stride_tricks.sliding_window_view(b.astype(np.uint64), k) * pw).sum(axis=1)
        assert np.array_equal(y[:, 0].astype(np.uint64), want)       # exact: sigma^k <= 2^32


def test_degenerate():
    x = torch.from_numpy(np.arange(10, dtype=np.uint32)).cuda()
    assert P.slsum_run(P.SLSUM_ADD_U32, 11, x).numel() == 0
    y = P.slsum_run(P.SLSUM_ADD_U32, 10, x)
    assert y.cpu().numpy().tolist() == [45]
    assert np.array_equal(P.slsum_run(P.SLSUM_MIN_U32, 1, x).cpu().numpy(), np.arange(10, dtype=np.uint32))
    with pytest.raises(P.SlsumError):
        P.slsum_run(P.SLSUM_ADD_U32, 0, x)
    e = torch.zeros(0, dtype=torch.uint32, device="cuda")
    assert P.slsum_run(P.SLSUM_MIN_U32, 3, e).numel() == 0


@pytest.mark.parametrize("w", [4, 16, 64, 256, 1024])
def test_c2_full_size_sampled(w):
    """C2 at full size (2^28 elements) in bench.py's launch configuration: sampled outputs vs
    the oracle computed one by one, plus the exact u32-add closed form at every position."""
    n = 1 << 28
    from synthgen import device as D
    xu = D.c2_u32(n)
    rng = np.random.default_rng(w)
    idx = np.concatenate([[0, n - w], rng.integers(0, n - w + 1, size=200)])
    it = torch.from_numpy(idx).cuda()
    for op in (P.SLSUM_MIN_U32, P.SLSUM_ADD_U32):
        paths = (P.SLSUM_PATH_GENERIC, P.SLSUM_PATH_COMMUTATIVE) + ((P.SLSUM_PATH_RECURRENT,) if op == P.SLSUM_ADD_U32 else ())
        for path in paths:
            y = P.slsum_run(op, w, xu, path=path)
            ys = y.view(torch.int32)[it].cpu().numpy().view(np.uint32)
            for j, i in enumerate(idx):
                xs = G.c2_u32(w, lo=int(i))
                assert ys[j] == O.slsum(dict(OPS)[op], w, xs)[0], (op, path, i)
            if op == P.SLSUM_ADD_U32:
                # exact closed form at every position: prefix differences mod 2^32 (torch.cumsum)
                x64 = xu.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
                ps = torch.cumsum(x64, 0)  # < 2^60, exact
                del x64
                ref = ps[w - 1:].clone()
                ref[1:] -= ps[: n - w]
                del ps
                got = y.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
                assert torch.equal(ref & 0xFFFFFFFF, got)
                del ref, got
            del y
    xf = D.c2_f32(n)
    for path in (P.SLSUM_PATH_GENERIC, P.SLSUM_PATH_COMMUTATIVE, P.SLSUM_PATH_SCALAR):
        y = P.slsum_run(P.SLSUM_ADD_F32, w, xf, path=path)
        ys = y[it].cpu().numpy()
        for j, i in enumerate(idx):
            o = O.slsum(O.ADD_F32, w, G.c2_f32(w, lo=int(i)))[0]
            if path == P.SLSUM_PATH_SCALAR:      # Alg. 1 is the strict left fold: bit-exact
                assert np.float32(ys[j]).view(np.uint32) == np.float32(o).view(np.uint32)
            else:
                assert abs(float(ys[j]) - float(o)) <= 1e-5 * abs(float(o)) + 1e-6 * w
        del y


@pytest.mark.parametrize("op", [P.SLSUM_MIN_U32, P.SLSUM_ADD_F32, P.SLSUM_AFFINE_U32X2, P.SLSUM_MIN_U64])
@pytest.mark.parametrize("m_lanes", [16, 32, 64, 128])
def test_generic_large_blocks(op, m_lanes):
    """GENERIC for w = M*E (M = 16..128 lanes of E elements per block): the team kernel (a team
    of warps per block of 256*NWT, streaming over a range of blocks, carrying the suffix folds)
    and the one-shot CTA kernel (8-byte w = 128): inputs that are an exact multiple of the
    block and tile sizes, ragged ones, many blocks per team, and a misaligned view."""
    e = 8 if op in (P.SLSUM_AFFINE_U32X2, P.SLSUM_MIN_U64) else 16
    w = m_lanes * e
    L = 256 * e
    rng = np.random.default_rng(op * 100 + m_lanes)
    for n in (3 * L, 7 * L + 5, 1_500 * L, 1_500 * L + L - 1):
        x = _input(op, n, rng)
        _check(op, w, x, _run(op, w, x, P.SLSUM_PATH_GENERIC))
    x = _input(op, 40 * L + 3, rng)
    xt = torch.from_numpy(np.concatenate([x[:1], x])).cuda()[1:]      # 4/8-byte aligned, not 16
    y = P.slsum_run(op, w, xt, path=P.SLSUM_PATH_GENERIC)
    torch.cuda.synchronize()
    _check(op, w, x, y.cpu().numpy())


@pytest.mark.parametrize("op,w", [(P.SLSUM_MIN_U32, 128), (P.SLSUM_MIN_U32, 1024), (P.SLSUM_ADD_U32, 256),
                                  (P.SLSUM_ADD_U32, 4096), (P.SLSUM_ADD_F32, 512), (P.SLSUM_MAX_U32, 300),
                                  (P.SLSUM_MAX_U32, 2049), (P.SLSUM_MIN_U64, 64), (P.SLSUM_MIN_U64, 777),
                                  (P.SLSUM_MIN_U64, 256), (P.SLSUM_ADD_F32, 2048), (P.SLSUM_ADD_U32, 1024)])
def test_commutative_register_start(op, w):
    """The COMMUTATIVE kernel for w >= 8E (first rounds in registers on overlapping warp spans,
    the rest in shared memory): power-of-two w for any commutative op, other w for idempotent
    ones; several tiles, a ragged end, and a misaligned view.  Power-of-two w with log2(w) - 2
    register-or-more rounds finish with the 4-way combine of t_{m-2} (MIN_U32 1024, ADD_U32
    1024 / 4096, ADD_F32 512 / 2048, MIN_U64 256)."""
    rng = np.random.default_rng(op * 31 + w)
    for n in (w + 16 * 1024, 200_003, 1 << 20):
        x = _input(op, n, rng)
        _check(op, w, x, _run(op, w, x, P.SLSUM_PATH_COMMUTATIVE))
    x = _input(op, 100_001, rng)
    xt = torch.from_numpy(np.concatenate([x[:1], x])).cuda()[1:]
    y = P.slsum_run(op, w, xt, path=P.SLSUM_PATH_COMMUTATIVE)
    torch.cuda.synchronize()
    _check(op, w, x, y.cpu().numpy())


@pytest.mark.parametrize("op", [P.SLSUM_MIN_U32, P.SLSUM_ADD_F32, P.SLSUM_AFFINE_U32X2, P.SLSUM_MIN_U64])
@pytest.mark.parametrize("w", [257, 300, 400, 511, 513, 700, 777, 1025, 1500, 1700, 2047])
def test_generic_team_runtime_w(op, w):
    """GENERIC for any w in (256, 2048] outside the powers of two: the team kernel with a
    runtime block length (slots past w hold the identity; blocks start at b*w, so most are not
    16-byte aligned).  Operand order is kept (AFFINE is not commutative), many blocks per team,
    a ragged end and a misaligned view; bit-exact vs the oracle (f32 within the BASELINE bound)."""
    rng = np.random.default_rng(op * 1000 + w)
    for n in (w, w + 1, 5 * w + 3, 300_001):
        x = _input(op, n, rng)
        _check(op, w, x, _run(op, w, x, P.SLSUM_PATH_GENERIC))
    x = _input(op, 100_003, rng)
    xt = torch.from_numpy(np.concatenate([x[:1], x])).cuda()[1:]
    y = P.slsum_run(op, w, xt, path=P.SLSUM_PATH_GENERIC)
    torch.cuda.synchronize()
    _check(op, w, x, y.cpu().numpy())
