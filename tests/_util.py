"""Shared helpers for the parity tests."""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name: str):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        return None
    return np.load(path)


def normwise(a, ref, axis=-1):
    """max_i |a - ref| / max_i |ref| per row (SURVEY.md §8(c) recommended metric)."""
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    a = a.reshape(a.shape[0], -1)
    ref = ref.reshape(ref.shape[0], -1)
    scale = np.abs(ref).max(axis=1)
    scale = np.where(scale == 0, 1.0, scale)
    return np.abs(a - ref).max(axis=1) / scale


def rel(a, ref):
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return np.abs(a - ref) / np.where(ref == 0, 1.0, np.abs(ref))
