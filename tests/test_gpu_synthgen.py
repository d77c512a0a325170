"""The device generators (synthgen/device.py) reproduce the host generators bit for bit."""
import numpy as np
import pytest
import torch

from synthgen import host as H

pytestmark = pytest.mark.gpu


def test_device_matches_host():
    from synthgen import device as D
    assert np.array_equal(D.c1_ascii(100_000).cpu().numpy(), H.c1_ascii(100_000))
    assert np.array_equal(D.c1_ascii(5000, lo=12345).cpu().numpy(), H.c1_ascii(5000, lo=12345))
    c3 = H.C3(n=5_000_000)
    assert np.array_equal(D.c3_ascii(c3).cpu().numpy(), c3.ascii())
    assert np.array_equal(D.c3_ascii(c3, lo=86_000, n=300_000).cpu().numpy(), c3.ascii(86_000, 300_000))
    c4 = H.C4(nreads=500)
    assert np.array_equal(D.c4_ascii(c4).cpu().numpy(), c4.ascii_range(0, c4.n))
    assert np.array_equal(D.c2_u32(10_001, lo=3).cpu().numpy(), H.c2_u32(10_001, lo=3))
    assert np.array_equal(D.c2_f32(10_001, lo=5).cpu().numpy(), H.c2_f32(10_001, lo=5))
