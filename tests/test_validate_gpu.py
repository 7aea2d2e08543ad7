"""validate_scene on the device (SURVEY §8f "next" #1), rule by rule against the
reference (proj/src/scene.cpp:31-91): the pipeline's "validate: <rule> (<detail>)" error
(pipeline.cpp:106-110) names the FIRST violation in the reference's report order —
points in index order (position before normal at the same index), then edges in order
(zero length stops that edge's checks; then normal_a unit, normal_b unit, normal_a
perpendicular, normal_b perpendicular, wedge defined, label disjoint), then TX and RX
radios (finite, unique id), then has_transmitter, has_receiver, carrier frequency.
Each scene below violates several rules; the message must be the reference's."""
import dataclasses

import numpy as np
import pytest

from fixtures import add_wall, make_scene
from paper_2402_13747_b200 import abi, pcray

pytestmark = pytest.mark.gpu

NAN, INF = float("nan"), float("inf")
RUN = dict(max_interactions=1, max_diffractions=0)


def _base():
    pts = []
    add_wall(pts, (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), 3, 0.1)
    return make_scene(pts, tx=[(0.5, 0.5, 1.0)], rx=[(0.2, 0.3, 0.8)],
                      edges=[((0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), 1000),
                             ((0, 1, 0), (1, 1, 0), (0, -1, 0), (0, 0, 1), 1001)])


def _edit(**kw):
    s = _base()
    arrays = {k: np.array(getattr(s, k), copy=True) for k in ["position", "normal", "label", "edges", "edge_label",
                                                               "tx", "tx_id", "rx", "rx_id"]}
    extra = {}
    for k, f in kw.items():
        if callable(f):
            arrays[k] = f(arrays[k])
        else:
            extra[k] = f
    return dataclasses.replace(s, **arrays, **extra)


def _set(idx, val):
    def f(a):
        a = a.astype(float) if a.dtype.kind == "f" else a
        a[idx] = val
        return a
    return f


CASES = {
    # points: the lowest index wins; at one index the position rule comes first
    "normal_then_position": dict(normal=_set(5, [0, 0, 2]), position=_set(9, [NAN, 0, 0])),
    "position_then_normal": dict(position=_set(3, [0, INF, 0]), normal=_set(7, [0, 0.5, 0])),
    "both_at_one_point": dict(position=_set(4, [NAN, NAN, NAN]), normal=_set(4, [2, 0, 0])),
    "normal_nan_is_not_a_violation_but_next_is": dict(normal=lambda a: _set(6, [1, 0, 0.5])(_set(2, [NAN, 0, 0])(a))),
    "point_before_edge": dict(normal=_set(40, [0, 0, 1.01]), edges=_set((0, slice(3, 6)), [0, 0, 0])),
    # edges, report order within and across edges
    "zero_length_edge_skips_its_checks": dict(edges=_set((0, slice(0, 12)), [1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0])),
    "normal_a_unit_before_perpendicular": dict(edges=_set((1, slice(6, 9)), [1.0, 0.2, 0.0])),
    "normal_b_unit": dict(edges=_set((0, slice(9, 12)), [0, 0, 3])),
    "normal_a_perpendicular": dict(edges=_set((0, slice(6, 9)), [0.6, 0.8, 0.0])),
    "normal_b_perpendicular": dict(edges=_set((1, slice(9, 12)), [0.8, 0.0, 0.6])),
    "wedge_undefined": dict(edges=_set((0, slice(9, 12)), [0, 1, 0])),
    "label_collides": dict(edge_label=_set(1, 3)),
    "first_edge_wins": dict(edge_label=_set(1, 3), edges=_set((0, slice(9, 12)), [0, 1, 0])),
    # radios and scene-level rules
    "tx_not_finite": dict(tx=_set(0, [NAN, 0, 0])),
    "rx_duplicate_id": dict(rx=lambda a: np.vstack([a, [[0.4, 0.4, 0.4]]]), rx_id=lambda a: np.array([7, 7], np.uint32)),
    "tx_duplicate_before_rx": dict(tx=lambda a: np.vstack([a, a]), tx_id=lambda a: np.array([1, 1], np.uint32),
                                   rx=_set(0, [INF, 0, 0])),
    "no_transmitter": dict(tx=lambda a: np.zeros((0, 3)), tx_id=lambda a: np.zeros(0, np.uint32)),
    "no_receiver": dict(rx=lambda a: np.zeros((0, 3)), rx_id=lambda a: np.zeros(0, np.uint32)),
    "no_radios_at_all": dict(tx=lambda a: np.zeros((0, 3)), tx_id=lambda a: np.zeros(0, np.uint32),
                             rx=lambda a: np.zeros((0, 3)), rx_id=lambda a: np.zeros(0, np.uint32)),
    "frequency_zero": dict(carrier_frequency_hz=0.0),
    "frequency_nan": dict(carrier_frequency_hz=NAN),
    "edge_before_radios": dict(edges=_set((1, slice(6, 9)), [0, -2, 0]), tx=_set(0, [NAN, 0, 0])),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_validate_first_violation_matches_reference(oracle, gpu, name):
    scene = _edit(**CASES[name])
    ref_err = got_err = None
    try:
        ref = oracle.run_pipeline_on_scene(oracle.RefScene(scene), oracle.default_run_config(**RUN))
    except oracle.RefError as e:
        ref_err = str(e)
    try:
        got = pcray.run_pipeline_on_scene(scene, abi.default_run_config(**RUN))
    except pcray.PcrError as e:
        got_err = str(e)
    assert got_err == ref_err
    if ref_err is None:  # a scene the reference accepts runs through, same counts
        for k in ["ie_count", "coarse_paths", "refined_paths", "exact_paths"]:
            assert got[k] == ref[k], k
    else:
        assert ref_err.startswith("validate: "), ref_err


def test_validate_report_order_is_the_references(oracle):
    """The cases above hit the rule the test name says (checked on the oracle), so the
    device comparison covers every rule and every ordering decision."""
    want = {"normal_then_position": "point_normal_unit", "position_then_normal": "point_position_finite",
            "both_at_one_point": "point_position_finite", "normal_nan_is_not_a_violation_but_next_is":
            "point_normal_unit", "point_before_edge": "point_normal_unit",
            "zero_length_edge_skips_its_checks": "edge_nondegenerate",
            "normal_a_unit_before_perpendicular": "edge_normal_a_unit", "normal_b_unit": "edge_normal_b_unit",
            "normal_a_perpendicular": "edge_normal_a_perpendicular",
            "normal_b_perpendicular": "edge_normal_b_perpendicular", "wedge_undefined": "edge_wedge_defined",
            "label_collides": "edge_label_disjoint", "first_edge_wins": "edge_wedge_defined",
            "tx_not_finite": "tx_position_finite", "rx_duplicate_id": "rx_id_unique",
            "tx_duplicate_before_rx": "tx_id_unique", "no_transmitter": "has_transmitter",
            "no_receiver": "has_receiver", "no_radios_at_all": "has_transmitter",
            "frequency_zero": "carrier_frequency_positive", "frequency_nan": "carrier_frequency_positive",
            "edge_before_radios": "edge_normal_a_unit"}
    assert set(want) == set(CASES)
    for name, rule in want.items():
        with pytest.raises(oracle.RefError, match="^validate: " + rule + " "):
            oracle.run_pipeline_on_scene(oracle.RefScene(_edit(**CASES[name])), oracle.default_run_config(**RUN))
