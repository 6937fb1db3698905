"""Test corpus: synthetic baseline JPEGs encoded by the REFERENCE encoder
(oracle_encode over make_test_image, reference oracle.hpp:272-478 and
tests/helpers.hpp:107-135) through oracle/_ref — the same generator the
reference's own acceptance corpus uses (acceptance.cpp:76-102)."""
import functools

from oracle.oracle import Ref


@functools.lru_cache(maxsize=None)
def ref_jpeg(w, h, seed, quality, sampling):
    return Ref.encode_test_image(w, h, seed, quality, sampling)


# acceptance.cpp:76-102: dims x q x sampling, plus two larger files
ACCEPTANCE = [(w, h, q, s) for (w, h) in [(48, 48), (64, 48), (96, 96), (160, 120)]
              for q in (92, 75, 50, 20) for s in ("444", "422", "420", "gray")]
ACCEPTANCE += [(320, 240, 85, "420"), (640, 400, 70, "422")]


def acceptance_corpus():
    out = []
    for k, (w, h, q, s) in enumerate(ACCEPTANCE):
        out.append(((w, h, q, s), ref_jpeg(w, h, 1000 + k, q, s)))
    return out
