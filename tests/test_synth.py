"""The shared input generator: numpy and torch implementations agree bit for bit."""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("kind", synth.KINDS)
def test_numpy_torch_identical(kind):
    a = synth.fp16_np((3, 7, 128), 1234, kind, scale=0.8)
    b = synth.fp16_torch((3, 7, 128), 1234, kind, scale=0.8, device="cpu", chunk=999).numpy()
    assert np.array_equal(a.view(np.uint16), b.view(np.uint16))


def test_determinism_and_seed_sensitivity():
    a = synth.fp16_np((64, 128), 5)
    assert np.array_equal(a.view(np.uint16), synth.fp16_np((64, 128), 5).view(np.uint16))
    assert not np.array_equal(a.view(np.uint16), synth.fp16_np((64, 128), 6).view(np.uint16))


def test_normal_moments():
    x = synth.fp16_np((1000, 64), 9).astype(np.float64)
    assert abs(x.mean()) < 0.02 and abs(x.std() - 1.0) < 0.02
    assert np.isfinite(x).all()


def test_lattice_is_exact_and_tie_heavy():
    x = synth.fp16_np((100, 128), 3, "lattice").astype(np.float64)
    assert np.array_equal(x * 4, np.round(x * 4)) and len(np.unique(np.abs(x))) <= 17
