"""The data formats either side of the hot path against the
reference's own io.cpp: PLY point clouds loaded straight into HBM (binary and ascii,
unknown properties, every header/data error text) and the paths JSONL artifact
(byte-identical files)."""
import os
import struct

import numpy as np
import pytest

from fixtures import box_room, make_scene
from paper_2402_13747_b200 import abi, pcray, scenes

pytestmark = pytest.mark.gpu


def _same_points(got: dict, ref: dict):
    for k in ["position", "normal", "label"]:
        a, b = np.ascontiguousarray(got[k]), np.ascontiguousarray(ref[k])
        assert a.shape == b.shape, k
        if a.dtype == np.float64:
            a, b = a.view(np.uint64), b.view(np.uint64)
        assert np.array_equal(a, b), k


@pytest.mark.parametrize("binary", [True, False])
def test_ply_roundtrip_c1(oracle, gpu, tmp_path, binary):
    scene, cfg = scenes.build_scene("C1")
    path = str(tmp_path / "c1.ply")
    oracle.save_point_cloud(path, oracle.RefScene(scene), binary)
    ref = oracle.load_point_cloud(path)
    ds = pcray.DeviceScene.from_ply(path, scene)
    _same_points(ds.points(), ref)
    assert ds.scene.n_points == scene.n_points


def _write_ply(path, header_props, rows, binary=True, count=None, extra_header=()):
    """header_props: [(type, name, struct code)], rows: list of tuples in that order."""
    with open(path, "wb") as f:
        f.write(b"ply\n")
        f.write(b"format binary_little_endian 1.0\n" if binary else b"format ascii 1.0\n")
        f.write(b"comment made by the test\n")
        for line in extra_header:
            f.write(line.encode() + b"\n")
        f.write(f"element vertex {len(rows) if count is None else count}\n".encode())
        for t, n, _ in header_props:
            f.write(f"property {t} {n}\n".encode())
        f.write(b"element face 0\nproperty list uchar int vertex_indices\nend_header\n")
        for r in rows:
            if binary:
                f.write(b"".join(struct.pack("<" + c, v) for (_, _, c), v in zip(header_props, r)))
            else:
                f.write((" ".join(repr(v) for v in r) + "\n").encode())


@pytest.mark.parametrize("binary", [True, False])
def test_ply_unknown_properties_any_order(oracle, gpu, tmp_path, binary):
    rng = np.random.default_rng(3)
    props = [("uchar", "red", "B"), ("float", "nz", "f"), ("double", "quality", "d"), ("float", "x", "f"),
             ("uint", "label", "I"), ("float", "y", "f"), ("short", "s", "h"), ("float", "z", "f"),
             ("float", "nx", "f"), ("float", "ny", "f"), ("int", "extra", "i")]
    rows = []
    for i in range(2000):
        v = rng.normal(size=6).astype(np.float32)
        rows.append((int(i % 256), float(v[5]), float(rng.normal()), float(v[0]), int(rng.integers(0, 2**32 - 1)),
                     float(v[1]), int(rng.integers(-1000, 1000)), float(v[2]), float(v[3]), float(v[4]),
                     int(rng.integers(-5, 5))))
    path = str(tmp_path / "odd.ply")
    _write_ply(path, props, rows, binary)
    ref = oracle.load_point_cloud(path)
    _same_points(pcray.DeviceScene.from_ply(path).points(), ref)


def _errors(oracle, path):
    try:
        oracle.load_point_cloud(path)
        ref = None
    except oracle.RefError as e:
        ref = str(e)
    try:
        pcray.DeviceScene.from_ply(path)
        got = None
    except pcray.PcrError as e:
        got = str(e)
    return got, ref


XYZ = [("float", "x", "f"), ("float", "y", "f"), ("float", "z", "f"), ("float", "nx", "f"), ("float", "ny", "f"),
       ("float", "nz", "f"), ("uint", "label", "I")]


@pytest.mark.parametrize("case", ["missing_file", "bad_magic", "bad_format", "missing_field", "wrong_type",
                                  "label_type", "truncated_bin", "truncated_ascii", "malformed_ascii",
                                  "list_prop", "unknown_keyword", "unknown_type", "no_vertex", "eof_header"])
def test_ply_error_texts(oracle, gpu, tmp_path, case):
    path = str(tmp_path / f"{case}.ply")
    rows = [(1.0, 2.0, 3.0, 0.0, 0.0, 1.0, 7)] * 5
    if case == "missing_file":
        path = str(tmp_path / "nope.ply")
    elif case == "bad_magic":
        open(path, "wb").write(b"plx\nformat ascii 1.0\n")
    elif case == "bad_format":
        open(path, "wb").write(b"ply\nformat binary_big_endian 1.0\nend_header\n")
    elif case == "missing_field":
        _write_ply(path, [p for p in XYZ if p[1] != "ny"], [r[:4] + r[5:] for r in rows])
    elif case == "wrong_type":
        _write_ply(path, [("double", "x", "d")] + XYZ[1:], rows)
    elif case == "label_type":
        _write_ply(path, XYZ[:6] + [("int", "label", "i")], rows)
    elif case == "truncated_bin":
        _write_ply(path, XYZ, rows, count=9)
    elif case == "truncated_ascii":
        _write_ply(path, XYZ, rows, binary=False, count=9)
    elif case == "malformed_ascii":
        _write_ply(path, XYZ, [r[:5] for r in rows], binary=False)
    elif case == "list_prop":
        open(path, "wb").write(b"ply\nformat ascii 1.0\nelement vertex 1\nproperty list uchar int idx\nend_header\n")
    elif case == "unknown_keyword":
        _write_ply(path, XYZ, rows, extra_header=["bogus line"])
    elif case == "unknown_type":
        open(path, "wb").write(b"ply\nformat ascii 1.0\nelement vertex 1\nproperty half x\nend_header\n")
    elif case == "no_vertex":
        open(path, "wb").write(b"ply\nformat ascii 1.0\nelement face 0\nend_header\n")
    elif case == "eof_header":
        open(path, "wb").write(b"ply\nformat ascii 1.0\nelement vertex 1\n")
    got, ref = _errors(oracle, path)
    assert ref is not None, "the reference accepted the file"
    assert got == ref


def test_pipeline_from_ply_equals_in_memory(oracle, gpu, tmp_path):
    sc = make_scene(box_room((2, 2, 2), 0.05), tx=[(0.6, 0.7, 0.9)], rx=[(1.3, 1.2, 1.1)])
    path = str(tmp_path / "box.ply")
    oracle.save_point_cloud(path, oracle.RefScene(sc), True)
    pts = oracle.load_point_cloud(path)  # float32-rounded points, as the reference pipeline reads them
    mem = abi.Scene(pts["position"], pts["normal"], pts["label"], sc.edges, sc.edge_label, sc.tx, sc.tx_id, sc.rx,
                    sc.rx_id, sc.carrier_frequency_hz)
    cfg = abi.default_run_config(max_interactions=2)
    ref = oracle.run_pipeline_on_scene(oracle.RefScene(mem), oracle.default_run_config(max_interactions=2))
    got = pcray.run_pipeline_device(pcray.DeviceScene.from_ply(path, sc), cfg)
    assert got["exact_paths"] == ref["exact_paths"] > 0
    for k in ["position", "length", "delay"]:
        a, b = got["paths"][k], ref["paths"][k]
        assert np.array_equal(np.ascontiguousarray(a).view(np.uint64), np.ascontiguousarray(b).view(np.uint64)), k


@pytest.mark.parametrize("name,mi,md", [("C1", 2, 0), ("C2", 2, 1)])
def test_paths_jsonl_byte_identical(oracle, gpu, tmp_path, name, mi, md):
    scene, _ = scenes.build_scene(name)
    kw = dict(max_interactions=mi, max_diffractions=md)
    ref = oracle.run_pipeline_on_scene(oracle.RefScene(scene), oracle.default_run_config(**kw))
    got = pcray.run_pipeline_on_scene(scene, abi.default_run_config(**kw))
    a, b = str(tmp_path / "gpu.jsonl"), str(tmp_path / "ref.jsonl")
    pcray.write_paths(a, got["paths"], got["hash"])
    oracle.write_paths(b, ref["paths"], ref["hash"])
    da, db = open(a, "rb").read(), open(b, "rb").read()
    assert da.count(b"\n") == ref["exact_paths"] + 1
    assert da == db
    # the writer alone, fed the reference's own paths
    c = str(tmp_path / "gpu_writer_ref_paths.jsonl")
    pcray.write_paths(c, ref["paths"], ref["hash"])
    assert open(c, "rb").read() == db


def test_write_paths_error(gpu, tmp_path):
    with pytest.raises(pcray.PcrError, match="cannot write paths file"):
        pcray.write_paths(str(tmp_path / "no_such_dir" / "x.jsonl"), {"n": 0, "stride": 1}, 0)


# ---- edges file + file-level run_pipeline (io.cpp:191-229, pipeline.cpp:214-247) -------------------
def _save_edges(path, scene):
    with open(path, "w") as f:
        f.write("# start_xyz end_xyz normal_a_xyz normal_b_xyz label\n")
        for g, lab in zip(np.asarray(scene.edges).reshape(-1, 12), scene.edge_label):
            f.write(" ".join(repr(float(v)) for v in g) + f" {int(lab)}\n")


def _edges_equal(got, ref):
    for k in ["start", "end", "normal_a", "normal_b", "label"]:
        a, b = np.ascontiguousarray(got[k]), np.ascontiguousarray(ref[k])
        assert a.shape == b.shape, k
        if a.dtype == np.float64:
            a, b = a.view(np.uint64), b.view(np.uint64)
        assert np.array_equal(a, b), k


def test_load_edges_parity(oracle, gpu, tmp_path):
    f = tmp_path / "edges.txt"
    f.write_text("# header comment\n"
                 "\n"
                 "   \t\n"
                 "0 0 0 1 0 0 0 0 2 0 -3 0 7   # trailing comment\n"
                 "-2e0 0 1 +2 0 1 0 -1.5 0 0 0 3e-1 7.9\n"
                 "0.1 0.2 0.3 0.1 0.2 3.3 1 1e-5 0 -0.70710678118654757 0.7071067811865476 0 4294967295\n"
                 "not-a-number line is skipped like a blank one\n"
                 "1 2 3 1 2 4 0.6 0.8 0 0 1e300 0 12 extra tokens ignored\n")
    ref = oracle.load_edges(str(f))
    got = pcray.load_edges(str(f))
    assert len(ref["label"]) == 4
    _edges_equal(got, ref)
    # C2's own edges through a file
    scene, _ = scenes.build_scene("C2")
    g = str(tmp_path / "c2_edges.txt")
    _save_edges(g, scene)
    _edges_equal(pcray.load_edges(g), oracle.load_edges(g))


@pytest.mark.parametrize("text", [
    "0 0 0 0 0 0 0 0 1 0 -1 0 7\n",
    "0 0 0 1 0 0 0 0 1 0 -1 0\n",
    "0 0 0 1 0 0 1 0 0 0 -1 0 7\n",
    "0 0 0 1 0 0 0 0 0 0 -1 0 7\n",
    "0 0 0 1 0 0 0 0 1 0 -1 0 7\n0 0 0 1 0 0 0 0 1 0 -1 x 7\n",
    "0 0 0 1 0 0 0 0 1 0 1e-12 0 7\n# c\n0 0 0 1 0 0 0 0 1 0.002 1 0 3\n",
    "0 0 0 1 0 0 0 0 1 0 -1 0 7\n0 0 0 1e-13 0 0 0 0 1 0 -1 0 7\n",
])
def test_load_edges_error_texts(oracle, gpu, tmp_path, text):
    f = tmp_path / "bad.txt"
    f.write_text(text)
    with pytest.raises(oracle.RefError) as r:
        oracle.load_edges(str(f))
    with pytest.raises(pcray.PcrError) as g:
        pcray.load_edges(str(f))
    assert str(g.value) == str(r.value)
    missing = str(tmp_path / "nope.txt")
    with pytest.raises(pcray.PcrError, match="cannot open edges file: " + missing):
        pcray.load_edges(missing)


@pytest.mark.parametrize("binary", [True, False])
def test_run_pipeline_files_c2(oracle, gpu, tmp_path, binary):
    scene, _ = scenes.build_scene("C2")
    ply, edges = str(tmp_path / "c2.ply"), str(tmp_path / "c2_edges.txt")
    oracle.save_point_cloud(ply, oracle.RefScene(scene), binary)
    _save_edges(edges, scene)
    kw = dict(max_interactions=2, max_diffractions=1)
    a, b = str(tmp_path / "gpu.jsonl"), str(tmp_path / "ref.jsonl")
    ref = oracle.run_pipeline(ply, edges, b, scene.tx, scene.rx, oracle.default_run_config(**kw))
    got = pcray.run_pipeline(ply, edges, a, scene.tx, scene.rx, abi.default_run_config(**kw))
    for k in ["point_count", "edge_count", "ie_count", "coarse_paths", "refined_paths", "exact_paths", "hash"]:
        assert got[k] == ref[k], k
    assert list(got["rejected"]) == list(ref["rejected"])
    assert [t[0] for t in got["timings"]] == [t[0] for t in ref["timings"]]
    assert got["timings"][0][0] == "load" and got["timings"][-1][0] == "write"
    assert got["exact_paths"] > 0
    assert open(a, "rb").read() == open(b, "rb").read()


def test_run_pipeline_files_error_texts(oracle, gpu, tmp_path):
    scene, _ = scenes.build_scene("C1")
    ply = str(tmp_path / "c1.ply")
    oracle.save_point_cloud(ply, oracle.RefScene(scene), True)
    bad_edges = tmp_path / "bad.txt"
    bad_edges.write_text("0 0 0 1 0 0 1 0 0 0 -1 0 7\n")
    cases = [
        dict(scene_path=str(tmp_path / "nope.ply")),
        dict(scene_path=str(tmp_path / "nope.ply"), edges_path=str(bad_edges)),  # points fail first
        dict(scene_path=ply, edges_path=str(bad_edges)),
        dict(scene_path=ply, edges_path=str(tmp_path / "nope.txt")),
        dict(scene_path=ply, output_path=str(tmp_path / "no_dir" / "p.jsonl"), transmitters=scene.tx,
             receivers=scene.rx),
        dict(),  # nothing at all: validate
        dict(scene_path=ply),  # no radios: validate
    ]
    cfg = dict(max_interactions=1)
    for kw in cases:
        with pytest.raises(oracle.RefError) as r:
            oracle.run_pipeline(config=oracle.default_run_config(**cfg), **kw)
        with pytest.raises(pcray.PcrError) as g:
            pcray.run_pipeline(config=abi.default_run_config(**cfg), **kw)
        assert str(g.value) == str(r.value), kw
