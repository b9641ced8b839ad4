"""Shared test plumbing: markers, paths, golden-fixture loaders."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the native path")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


class SmallCase:
    """One reference-generated tick with every intermediate (make_golden.py)."""

    def __init__(self, name, arrays, meta):
        self.name = name
        self.meta = meta
        self.a = {k.split("__", 1)[1]: arrays[k] for k in arrays.files if k.startswith(name + "__")}

    def __getattr__(self, item):
        try:
            return self.__dict__["a"][item]
        except KeyError as e:
            raise AttributeError(item) from e

    @property
    def th_quad(self):
        return self.meta["th_quad"]

    @property
    def l_max(self):
        return self.meta["l_max"]

    @property
    def covering(self):
        return self.meta["covering"]

    def inputs(self):
        r = self.rects
        return (self.ids, self.xs, self.ys, self.qids, r[:, 0].copy(), r[:, 1].copy(),
                r[:, 2].copy(), r[:, 3].copy())


def load_small_cases():
    arrays = np.load(os.path.join(GOLDEN, "small_cases.npz"))
    with open(os.path.join(GOLDEN, "small_cases.json")) as fp:
        meta = json.load(fp)
    return [SmallCase(n, arrays, m) for n, m in sorted(meta["cases"].items())]


def load_digests():
    with open(os.path.join(GOLDEN, "digests.json")) as fp:
        return json.load(fp)["runs"]


def workload_from_json(w):
    from paper_1411_3212_b200.workload import WorkloadConfig

    kw = dict(w)
    if isinstance(kw.get("query_side"), list):
        kw["query_side"] = tuple(kw["query_side"])
    return WorkloadConfig(**kw)


@pytest.fixture(scope="session")
def small_cases():
    return load_small_cases()


@pytest.fixture(scope="session")
def digests():
    return load_digests()
