"""Helpers to read the golden fixtures written by tests/golden/make_golden.py."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def items(buf, off):
    b = bytes(buf)
    return [b[off[i] : off[i + 1]] for i in range(len(off) - 1)]
