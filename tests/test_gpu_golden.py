"""GPU: the product against the committed golden vectors that the reference
generated (tests/golden/make_golden.py) — runs without /root/reference."""
import os

import numpy as np
import pytest

pj = pytest.importorskip("paper_2111_09219_b200")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_corpus.npz")


@pytest.fixture(scope="module")
def corpus():
    return np.load(GOLD)


@pytest.mark.parametrize("sb", [128, 1024])
def test_golden_corpus_coefficients_states_planes(decoder, corpus, sb):
    names = [n for n in corpus["names"] if f"{n}.ents{sb}" in corpus]
    files = [corpus[f"{n}.jpg"].tobytes() for n in names]
    with decoder.batch(files, pj.DecodeConfig(subsequence_bits=sb), pj.OutputColorspace.YCbCrPlanes) as b:
        st = b.run()
        assert (st == 0).all()
        outs = b.download()
        for i, n in enumerate(names):
            assert np.array_equal(b.coefficients(i, True), corpus[f"{n}.coeffs"]), n
            ents = corpus[f"{n}.ents{sb}"]
            got = b.sync_states(i).astype(np.int64)
            assert got.shape == ents.shape, n
            assert np.array_equal(got[:, 1], ents[:, 1]), n  # trimmed n: exact
            tr, valid = corpus[f"{n}.trace{sb}"], corpus[f"{n}.valid{sb}"]
            for k in range(len(valid)):
                if valid[k]:
                    assert (got[k, 0], got[k, 2], got[k, 3]) == (tr[k, 0], tr[k, 2], tr[k, 3]), (n, k)
            pl = corpus[f"{n}.planes"]
            assert np.array_equal(outs[i][: pl.size], pl), n


def test_golden_corpus_rgb(decoder, corpus):
    names = list(corpus["names"])
    files = [corpus[f"{n}.jpg"].tobytes() for n in names]
    with decoder.batch(files, pj.DecodeConfig(), pj.OutputColorspace.RGBInterleaved) as b:
        assert (b.run() == 0).all()
        outs = b.download()
        for i, n in enumerate(names):
            rgb = corpus[f"{n}.rgb"]
            assert np.array_equal(outs[i][: rgb.size], rgb), n


def test_worked_example_through_the_gpu(decoder):
    from oracle.oracle import example_jpeg
    with decoder.batch([example_jpeg()], pj.DecodeConfig(subsequence_bits=32), pj.OutputColorspace.YCbCrPlanes) as b:
        assert b.run()[0] == 0
        c = b.coefficients(0, True)
        want = np.zeros(64, np.int16)
        want[[0, 1, 2, 3, 5, 6, 8]] = [-2, -3, 2, -1, -1, 1, 1]
        assert np.array_equal(c, want)
        s = b.sync_states(0)
        assert list(s[0][[0, 1, 2, 3]]) == [32, 64, 0, 0]
