"""Loader for tests/golden/reference_golden.npz (made by
tests/golden/make_golden.py from the reference library itself)."""

import os

import numpy as np

from oracle import Csr

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")
_data = None


def data():
    global _data
    if _data is None:
        _data = dict(np.load(PATH))
    return _data


def n_random():
    return sum(1 for k in data() if k.endswith("_modularity") and k.startswith("rnd"))


def n_planted():
    return sum(1 for k in data() if k.endswith("_seq_modularity"))


def graph(prefix):
    d = data()
    return Csr(d[prefix + "offsets"], d[prefix + "targets"], d[prefix + "weights"], float(d[prefix + "total_weight"]))


def field(prefix, name):
    return data()[prefix + name]
