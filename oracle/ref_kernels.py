"""Loader for oracle/_ref/_kernels*.so -- the reference's Cython kernels
(``pkg/src/ringsim/_kernels.pyx:15-102``) compiled by ``oracle/Makefile``.
Test / CPU-baseline infrastructure only."""

import glob
import importlib.util
import os

_HERE = os.path.dirname(os.path.abspath(__file__))


def load():
    paths = glob.glob(os.path.join(_HERE, "_ref", "_kernels*.so"))
    if not paths:
        return None
    spec = importlib.util.spec_from_file_location("_kernels", paths[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod
