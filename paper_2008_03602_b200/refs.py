"""Stored fp64 oracle reference points for the in-loop correctness gate (a10).

Reads the data files ``refs/<catalog>_cfg<config>.npz`` that
``tools/make_refs.py`` writes from ``oracle/`` (see refs/README.md); this
module executes no oracle code.  ``load(catalog, config)`` returns, per layer,
(check_idx, check_ref) for ``tp.tune*``'s ``check_idx`` / ``check_ref``: the
indices are regenerated with ``datagen.sample_points`` and verified against
the stored count and checksum, so a stale file fails loudly.
"""
from __future__ import annotations

import json
import os

import numpy as np

from . import datagen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "refs")


def path(catalog: str, config: int) -> str:
    return os.path.join(REF_DIR, f"{catalog}_cfg{config}.npz")


def point_seed(layer: int) -> int:
    return 11 + layer


def load(catalog: str, config: int, layers: list[dict] | None = None) -> list[tuple[np.ndarray, np.ndarray]]:
    """[(idx int64, ref float64)] per layer of the catalog."""
    z = np.load(path(catalog, config))
    meta = json.loads(bytes(z["meta"]).decode())
    if meta["catalog"] != catalog or meta["config"] != config:
        raise ValueError(f"reference file {path(catalog, config)} is for {meta['catalog']} config {meta['config']}")
    out = []
    for li, m in enumerate(meta["layers"]):
        if layers is not None and layers[li]["name"] != m["name"]:
            raise ValueError(f"reference layer {li} is {m['name']}, expected {layers[li]['name']}")
        idx = datagen.sample_points(m["total"], meta["points"], point_seed(li))
        if idx.shape[0] != m["n_points"] or int(idx.sum()) != m["idx_sum"]:
            raise ValueError(f"reference points of {m['name']} do not match datagen.sample_points")
        out.append((idx, np.asarray(z[f"ref_{li}"], dtype=np.float64)))
    return out
