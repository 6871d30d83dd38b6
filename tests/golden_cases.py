"""Loader for the reference-generated fixtures (see tests/golden/gen_golden.py)."""

from __future__ import annotations

import json
import os
from functools import lru_cache

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@lru_cache(maxsize=1)
def _load():
    meta = json.load(open(os.path.join(HERE, "cases.json")))
    arrays = dict(np.load(os.path.join(HERE, "cases.npz")))
    return meta, arrays


def meta_dumps() -> dict:
    return _load()[0]["meta"]


def cases():
    """Yield (name, dag_bytes, shapes{int: tuple}, expected{int: ndarray}, rounds, batch)."""
    meta, arrays = _load()
    for c in meta["cases"]:
        name = c["name"]
        shapes = {int(k): tuple(v) for k, v in c["shapes"].items()}
        expected = {a: arrays[f"{name}__a{a}"] for a in c["arrays"]}
        rounds = {int(k): v for k, v in c["rounds"].items()}
        yield name, arrays[f"{name}__dag"].tobytes(), shapes, expected, rounds, c["batch"]


def case_names():
    return [c["name"] for c in _load()[0]["cases"]]


def get_case(name):
    for c in cases():
        if c[0] == name:
            return c
    raise KeyError(name)
