"""Canonical digests of candidate / outcome / path tables (test infrastructure).

Full-size contract runs (C2 at 4 / 1 and at depth 3) produce ~10^5-10^6 rows, too
many to commit as raw fixtures, so `tests/golden/make_contract_golden.py` stores a
SHA-256 per field plus a digest per block of rows, computed by the functions below
from the oracle's output; the GPU parity tests recompute them from the CUDA path's
output on the same scene. Interaction slots past `n_inter` are zeroed and the slot
axis is cut / padded to the config's max_interactions, so the digest depends only on
the used slots (not on either side's buffer stride). Bitwise by construction: float
fields are hashed as their IEEE bit patterns.
"""
from __future__ import annotations

import hashlib

import numpy as np

BLOCK = 8192

CAND_FIELDS = ["tx_id", "rx_id", "tx_position", "rx_position", "length", "n_inter",
               "kind", "label", "ie_index", "edge_index", "position", "normal"]
OUTCOME_FIELDS = ["reason", "has_path", "n_inter", "kind", "label", "position", "length"]
PATH_FIELDS = ["tx_id", "rx_id", "tx_position", "rx_position", "length", "delay", "converged", "gradient_norm",
               "n_inter", "kind", "label", "ie_index", "edge_index", "position", "normal"]
SLOT_FIELDS = {"kind", "label", "ie_index", "edge_index", "position", "normal"}


def normalize(d: dict, fields, slots: int, rows_mask=None) -> dict:
    """Row-aligned arrays: interaction fields cut/padded to `slots`, unused slots zeroed;
    rows outside rows_mask (e.g. has_path == 0 for geometry fields) zeroed."""
    n = int(d["n"])
    n_inter = np.asarray(d["n_inter"], np.int64).reshape(n) if n else np.zeros(0, np.int64)
    out = {}
    for f in fields:
        a = np.asarray(d[f])
        if f in SLOT_FIELDS:
            shape = (n, slots) + a.shape[2:]
            b = np.zeros(shape, a.dtype)
            k = min(slots, a.shape[1]) if a.ndim >= 2 else 0
            if n and k:
                b[:, :k] = a[:n, :k]
            used = np.arange(slots)[None, :] < n_inter[:, None]
            b[~used] = 0
            a = b
        else:
            a = np.ascontiguousarray(a[:n])
        if rows_mask is not None and f not in ("reason", "has_path"):
            a = a.copy()
            a[~rows_mask] = 0
        out[f] = np.ascontiguousarray(a)
    return out


def _h(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def digest(d: dict, fields, slots: int, geometry_only_where=None) -> dict:
    """{"n", "fields": {f: sha}, "blocks": [sha of rows [i*BLOCK, (i+1)*BLOCK) over all fields]}"""
    n = int(d["n"])
    mask = None
    if geometry_only_where is not None:
        mask = np.asarray(d[geometry_only_where]).reshape(n).astype(bool) if n else np.zeros(0, bool)
    a = normalize(d, fields, slots, mask)
    blocks = [_h(*(a[f][i:i + BLOCK] for f in fields)) for i in range(0, n, BLOCK)]
    return {"n": n, "fields": {f: _h(a[f]) for f in fields}, "blocks": blocks}


def candidates_digest(c: dict, slots: int) -> dict:
    return digest(c, CAND_FIELDS, slots)


def outcomes_digest(o: dict, slots: int) -> dict:
    return digest(o, OUTCOME_FIELDS, slots, geometry_only_where="has_path")


def paths_digest(p: dict, slots: int) -> dict:
    return digest(p, PATH_FIELDS, slots)


def compare(got: dict, want: dict, what: str) -> None:
    """Assert two digests are equal; name the differing fields and the first block."""
    assert got["n"] == want["n"], f"{what}: {got['n']} rows vs {want['n']} (oracle)"
    bad = [f for f in want["fields"] if got["fields"].get(f) != want["fields"][f]]
    if bad:
        first = next((i for i, (a, b) in enumerate(zip(got["blocks"], want["blocks"])) if a != b), None)
        raise AssertionError(f"{what}: fields {bad} differ from the oracle; first differing block {first} "
                             f"(rows {first * BLOCK if first is not None else '?'}..)")
