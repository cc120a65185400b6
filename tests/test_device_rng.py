"""Device PCG64 + ziggurat vs numpy (the reference's random_signals, signals.py:16-37)."""
import numpy as np
import pytest

from oracle import csc_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,seed,sd", [(7, 3, 5, None), (1000, 40, 0, None), (20000, 40, 3, 80),
                                         (300001, 13, 11, 26), (2_000_000, 4, 7, None),
                                         (2_000_000, 16, 21, 64)])
def test_device_signals_match_numpy(cuda_ok, n, d, seed, sd):
    """Bit-identical to numpy, tail draws included (glibc log1p restated on the
    device, rng.cu); no column needed the host redraw."""
    from paper_1706_03591_b200 import signals as S
    before = S.RNG_STATS["redrawn_columns"]
    blk = S.device_signals(n, d, seed, scale_dim=sd, mode="device")
    got = blk[:, :d].cpu().numpy()
    ref = O.random_signals(n, d, seed, scale_dim=sd)
    z = np.abs(ref) * np.sqrt(sd or d)
    print(f"tail draws (|z| > 3.65): {int((z > 3.6541528853610088).sum())}")
    assert np.array_equal(got, ref), int((got != ref).sum())
    assert S.RNG_STATS["redrawn_columns"] == before
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
