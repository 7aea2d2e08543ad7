"""Synthetic config builders without a GPU: C2-np's normal tilt is bounded,
unit-length and seeded; every config builds and carries the radio counts §8.0 names."""
import numpy as np
import pytest

from paper_2402_13747_b200 import scenes


def test_c2np_tilt_bounded_and_seeded():
    base, _ = scenes.build_scene("C2")
    a, _ = scenes.build_scene("C2np")
    b, _ = scenes.build_scene("C2np")
    assert np.array_equal(a.normal, b.normal)
    assert np.array_equal(a.position, base.position) and np.array_equal(a.label, base.label)
    assert np.abs(np.linalg.norm(a.normal, axis=1) - 1.0).max() < 1e-12
    cosang = np.clip((a.normal * base.normal).sum(1), -1.0, 1.0)
    ang = np.degrees(np.arccos(cosang))
    assert ang.max() <= 1.0 + 1e-9 and ang.mean() > 0.3


@pytest.mark.parametrize("name,tx,rx", [("C1", 1, 1), ("C2", 1, 64)])
def test_small_configs_radios(name, tx, rx):
    s, cfg = scenes.build_scene(name)
    assert len(s.tx) == tx and len(s.rx) == rx
    assert set(cfg.run) >= {"max_interactions", "max_diffractions"}
