"""Oracle pins for the file-level rows (load_edges, run_pipeline): the restated
wrapper (oracle/ref_capi.cpp over the unmodified reference) against the known answers
of the reference's own tests (proj/tests/test_io.cpp:206-238) and the load/write
stage prefixes of proj/src/pipeline.cpp:214-247. CPU only."""
import numpy as np
import pytest


def _msg(fn):
    try:
        fn()
    except Exception as e:  # RefError carries the reference's runtime_error text
        return str(e)
    return None


def test_edges_known_answers(oracle, tmp_path):
    f = tmp_path / "edges.txt"
    f.write_text("# start xyz, end xyz, normal_a xyz, normal_b xyz, label\n"
                 "0 0 0 1 0 0 0 0 2 0 -3 0 7\n")
    e = oracle.load_edges(str(f))
    assert len(e["label"]) == 1
    assert e["start"][0].tolist() == [0, 0, 0] and e["end"][0].tolist() == [1, 0, 0]
    assert e["normal_a"][0].tolist() == [0, 0, 1]  # normalised on load
    assert e["normal_b"][0].tolist() == [0, -1, 0]
    assert e["label"][0] == 7


@pytest.mark.parametrize("text,needle", [
    ("0 0 0 0 0 0 0 0 1 0 -1 0 7\n", "edge record 0: degenerate edge"),
    ("0 0 0 1 0 0 0 0 1 0 -1 0\n", "expected 13 values"),
    ("0 0 0 1 0 0 1 0 0 0 -1 0 7\n", "not perpendicular"),
    ("0 0 0 1 0 0 0 0 0 0 -1 0 7\n", "edge record 0: zero normal"),
])
def test_edges_error_texts(oracle, tmp_path, text, needle):
    f = tmp_path / "bad.txt"
    f.write_text(text)
    assert needle in _msg(lambda: oracle.load_edges(str(f)))


def test_edges_empty_and_missing(oracle, tmp_path):
    f = tmp_path / "empty.txt"
    f.write_text("# nothing here\n")
    assert len(oracle.load_edges(str(f))["label"]) == 0
    assert _msg(lambda: oracle.load_edges(str(tmp_path / "nope.txt"))) == \
        "cannot open edges file: " + str(tmp_path / "nope.txt")


def test_run_pipeline_stage_prefixes(oracle, tmp_path):
    cfg = oracle.default_run_config()
    missing = str(tmp_path / "nope.ply")
    assert _msg(lambda: oracle.run_pipeline(missing)) == "load: cannot open point cloud file: " + missing
    bad = tmp_path / "bad.txt"
    bad.write_text("0 0 0 0 0 0 0 0 1 0 -1 0 7\n")
    assert _msg(lambda: oracle.run_pipeline("", str(bad), config=cfg)) == "load: edge record 0: degenerate edge"
    # nothing loaded at all: the pipeline's own validate stage speaks
    m = _msg(lambda: oracle.run_pipeline(config=cfg))
    assert m is not None and m.startswith("validate: ")


def test_run_pipeline_timings_and_jsonl(oracle, tmp_path):
    from paper_2402_13747_b200 import scenes

    scene, _ = scenes.build_scene("C1")
    ply = str(tmp_path / "c1.ply")
    oracle.save_point_cloud(ply, oracle.RefScene(scene), True)
    out = str(tmp_path / "paths.jsonl")
    s = oracle.run_pipeline(ply, "", out, scene.tx, scene.rx, oracle.default_run_config(max_interactions=1))
    stages = [t[0] for t in s["timings"]]
    assert stages[0] == "load" and stages[-1] == "write"
    lines = open(out, "rb").read().splitlines()
    assert len(lines) == s["exact_paths"] + 1
    assert np.all(s["paths"]["tx_id"] < len(scene.tx))
