"""Device PCG64 + ziggurat vs numpy (the reference's random_signals, signals.py:16-37)."""
import numpy as np
import pytest

from oracle import csc_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,seed,sd", [(7, 3, 5, None), (1000, 40, 0, None), (20000, 40, 3, 80),
                                         (300001, 13, 11, 26), (2_000_000, 4, 7, None)])
def test_device_signals_match_numpy(cuda_ok, n, d, seed, sd):
    from paper_1706_03591_b200.signals import device_signals
    blk = device_signals(n, d, seed, scale_dim=sd, mode="device")
    got = blk[:, :d].cpu().numpy()
    ref = O.random_signals(n, d, seed, scale_dim=sd)
    diff = got != ref
    # bit-identical except possibly the last ulp of tail draws (device log1p/exp)
    assert diff.mean() <= 1e-4, diff.sum()
    if diff.any():
        rel = np.abs(got[diff] - ref[diff]) / np.abs(ref[diff])
        assert rel.max() <= 4.5e-16
        z = np.abs(ref[diff]) * np.sqrt(sd or d)   # back to the standard-normal scale
        assert np.all(z > 3.6)
    # padding columns stay zero
    assert np.all(blk[:, d:].cpu().numpy() == 0.0)


def test_device_signals_spawn_order(cuda_ok):
    """The caller's SeedSequence advances exactly like the reference's spawn(d)."""
    from paper_1706_03591_b200.signals import device_signals
    a = np.random.SeedSequence(9)
    b = np.random.SeedSequence(9)
    device_signals(100, 6, a, mode="device")
    b.spawn(6)
    assert a.spawn(1)[0].spawn_key == b.spawn(1)[0].spawn_key
