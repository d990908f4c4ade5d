"""Loaders for the test oracles (TEST INFRASTRUCTURE).

- reference(): oracle/_ref/libsfref.so — the unmodified reference sources compiled with the
  Eigen/doctest shims plus a C-ABI wrapper (oracle/ref_capi.cpp); symbols ``sfref_*``.
- port():      oracle/liboracle.so — the plain-C restatement (oracle/sf_oracle.c); symbols
  ``sfo_*``.
Both expose the signatures of include/sf_gpu.h, so the same Python API drives them.
"""
import os
import subprocess

from paper_1311_7194_b200 import _abi as A
from paper_1311_7194_b200.api import Backend

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libsfref.so")
PORT_SO = os.path.join(ROOT, "oracle", "liboracle.so")

_cache = {}


def _try_build(target):
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), target], check=False,
                       stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)


def reference():
    if "ref" not in _cache:
        if not os.path.exists(REF_SO):
            _try_build("ref")
        _cache["ref"] = Backend(A.Lib(REF_SO, "sfref", {**A.REF_ONLY, **A.MESH}), "reference") if os.path.exists(REF_SO) else None
    return _cache["ref"]


def port():
    if "port" not in _cache:
        if not os.path.exists(PORT_SO):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "port"], check=False,
                           stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        _cache["port"] = Backend(A.Lib(PORT_SO, "sfo", {}), "port") if os.path.exists(PORT_SO) else None
    return _cache["port"]
