"""Synthetic corpus generator (libpjg_synth.so): baseline JPEGs of the
BASELINE.json shapes for the benchmark (csrc/synth.cpp).

``synth_ref_batch`` produces the SURVEY.md §8(d) corpus: files byte-identical
to the reference's ``oracle_encode(make_test_image(...))`` (checked against
oracle/_ref by tests/test_synth.py), generated natively so that nothing under
oracle/ runs on the benchmark path.  ``synth_batch`` is an independent fast
float encoder (restart-interval twin tests)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SYNTH_PATH = os.path.join(HERE, "libpjg_synth.so")
SAMPLING = {"444": 0, "422": 1, "420": 2, "gray": 3}
_lib = None


def _L():
    global _lib
    if _lib is None:
        if not os.path.exists(SYNTH_PATH):
            raise RuntimeError(f"{SYNTH_PATH} missing: run `make -C paper_2111_09219_b200/csrc`")
        _lib = C.CDLL(SYNTH_PATH)
        _lib.pjg_synth_batch.restype = C.c_uint64
        _lib.pjg_synth_ref_batch.restype = C.c_uint64
    return _lib


def synth_batch(n, w, h, seed0, quality, sampling="420", restart_interval=0, threads=None, out=None):
    """Returns (blob uint8 array, offsets int64[n], sizes int64[n]).  ``out`` may
    supply the destination (e.g. a pinned buffer); it is used if big enough."""
    threads = threads or os.cpu_count() or 1
    offs = np.zeros(n, np.uint64)
    sizes = np.zeros(n, np.uint64)
    need = C.c_uint64()
    cap = 0 if out is None else out.size
    ptr = None if out is None else out.ctypes.data_as(C.POINTER(C.c_uint8))
    args = (C.c_uint32(n), C.c_uint32(w), C.c_uint32(h), C.c_uint32(seed0), C.c_int(quality),
            C.c_int(SAMPLING[sampling]), C.c_int(restart_interval), C.c_uint(threads))
    tot = _L().pjg_synth_batch(*args, ptr, C.c_uint64(cap), offs.ctypes.data_as(C.POINTER(C.c_uint64)),
                               sizes.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(need))
    if tot == 0:
        blob = np.empty(need.value, np.uint8)
        tot = _L().pjg_synth_batch(*args, blob.ctypes.data_as(C.POINTER(C.c_uint8)), C.c_uint64(blob.size),
                                   offs.ctypes.data_as(C.POINTER(C.c_uint64)),
                                   sizes.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(need))
    else:
        blob = out
    return blob[:tot], offs.astype(np.int64), sizes.astype(np.int64)


def synth_ref_batch(n, w, h, seed0, quality, sampling="420", restart_interval=0, channels=0, threads=None,
                    out=None):
    """n files oracle_encode(make_test_image(w, h, seed0 + i, channels), quality,
    sampling) [+ DRI/RSTn every ``restart_interval`` MCUs]; channels 0 = 1 for
    gray, else 3.  Returns (blob, offsets, sizes) like :func:`synth_batch`."""
    threads = threads or os.cpu_count() or 1
    offs = np.zeros(n, np.uint64)
    sizes = np.zeros(n, np.uint64)
    need = C.c_uint64()
    args = (C.c_uint32(n), C.c_uint32(w), C.c_uint32(h), C.c_uint32(seed0), C.c_int(quality),
            C.c_int(SAMPLING[sampling]), C.c_int(restart_interval), C.c_uint(channels), C.c_uint(threads))
    cap = 0 if out is None else out.size
    ptr = None if out is None else out.ctypes.data_as(C.POINTER(C.c_uint8))
    tot = _L().pjg_synth_ref_batch(*args, ptr, C.c_uint64(cap), offs.ctypes.data_as(C.POINTER(C.c_uint64)),
                                   sizes.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(need))
    if tot == 0:
        blob = np.empty(need.value, np.uint8)
        tot = _L().pjg_synth_ref_batch(*args, blob.ctypes.data_as(C.POINTER(C.c_uint8)), C.c_uint64(blob.size),
                                       offs.ctypes.data_as(C.POINTER(C.c_uint64)),
                                       sizes.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(need))
    else:
        blob = out
    return blob[:tot], offs.astype(np.int64), sizes.astype(np.int64)
