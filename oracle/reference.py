"""Loader for the real reference package (pivgen) built into oracle/_ref.

TEST INFRASTRUCTURE. oracle/build_ref.sh compiles /root/reference/pkg
(Cython native splat kernel, -O3) into oracle/_ref with an empty h5py stub
(flowfield.py:15 imports h5py at module scope; only load_hdf5 uses it).
oracle/_ref is git-ignored but travels to the GPU box with the snapshot.
"""

from __future__ import annotations

import importlib
import os
import sys

REF_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "pivgen"))


def load(pure_python: bool = False):
    """Import and return the reference ``pivgen`` package (native backend
    unless ``pure_python``)."""
    if not available():
        raise ImportError(f"reference not built: run oracle/build_ref.sh ({REF_DIR})")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    if pure_python:
        os.environ["PIVGEN_PURE_PYTHON"] = "1"
    mod = importlib.import_module("pivgen")
    return mod
