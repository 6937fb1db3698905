"""Contexts are independent (include/pjg.h: one context per host thread and
GPU, no global mutable state): two host threads, each with its own context,
decode concurrently on the same GPU — a latency-bound batch (replayed as a
CUDA graph with programmatic dependent launch) next to a large one (plain
stream launches) — and every output equals the reference's."""
import threading

import numpy as np
import pytest

from oracle.oracle import Ref
from tests.corpus import ref_jpeg

pj = pytest.importorskip("paper_2111_09219_b200")
pytestmark = pytest.mark.gpu


def _work(files, reps, out, key, errors):
    try:
        dec = pj.Decoder(0)
        for r in range(reps):
            with dec.batch(files, pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
                st = b.run()
                out[(key, r)] = (st.copy(), [o.copy() for o in b.download()], list(b.infos))
        dec.close()
    except Exception as e:  # reported by the main thread
        errors.append(repr(e))


def test_two_threads_two_contexts_one_gpu():
    small = [ref_jpeg(64 + 8 * k, 48, 800 + k, 80, ["420", "444"][k % 2]) for k in range(3)]
    large = [ref_jpeg(500, 375, 900 + k, 75, "420") for k in range(160)]
    out, errors = {}, []
    ts = [threading.Thread(target=_work, args=(small, 6, out, "small", errors)),
          threading.Thread(target=_work, args=(large, 3, out, "large", errors))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for key, files, reps in (("small", small, 6), ("large", large, 3)):
        want = [Ref.decode(f, rgb=True).data for f in files]
        for r in range(reps):
            st, outs, infos = out[(key, r)]
            assert (st == 0).all(), (key, r, st)
            for i, w in enumerate(want):
                assert np.array_equal(outs[i][: w.size], w.reshape(-1)), (key, r, i)
