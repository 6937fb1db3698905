"""Corrupt-stream parity: mutated files through the GPU decoder must give the
reference's outcome exactly — the same Errc (decode_single with the default
worker_count = 1, pipeline.hpp:36-41, so the reference's first failing
subsequence is deterministic), or success with the same RGB.

Corpora:
  * the reference's parser fuzz recipe (test_parser.cpp:146-162): 300
    mutations (1-8 random byte edits, every third one truncated) of
    oracle_encode(make_test_image(32, 24, 7), 70, 4:2:0);
  * scan-only mutations of a larger file, at the default partition (one
    sequence: intra-sequence semantics) and at sb = 128, b = 4 (many
    sequences: inter-sequence passes, parallel_decode.hpp:227-285).

The reference runs in forked workers with a timeout: for some corrupt scans
its inter-sequence loop never terminates (a stuck boundary whose start is
divergent keeps `progressed` true while another flag is set,
parallel_decode.hpp:277-283); those files have no reference outcome and are
excluded (counted in the assertion message)."""
import multiprocessing as mp

import numpy as np
import pytest

from oracle.oracle import Ref
from tests.corpus import ref_jpeg

pj = pytest.importorskip("paper_2111_09219_b200")
pytestmark = pytest.mark.gpu


def _mutants(base, n, seed, scan_only):
    rng = np.random.default_rng(seed)
    sos = base.index(b"\xff\xda")
    scan0 = sos + 2 + ((base[sos + 2] << 8) | base[sos + 3])
    lo = scan0 if scan_only else 0
    out = []
    for trial in range(n):
        m = bytearray(base)
        for _ in range(int(rng.integers(1, 9))):
            m[int(rng.integers(lo, len(base)))] = int(rng.integers(0, 256))
        if trial % 3 == 0:
            m = m[: int(rng.integers(lo, len(m))) + 1]
        out.append(bytes(m))
    return out


def _ref_child(conn, f, sb, b):
    r = Ref.decode(f, rgb=True, sb=sb, b=b, workers=1)
    conn.send((r.status, r.data.tobytes() if r.status == 0 else b""))
    conn.close()


def _ref_outcomes(files, sb, b, timeout=20.0, par=16):
    """The reference's outcome per file, one forked child each (a child that
    does not finish within `timeout` is killed: outcome None)."""
    import time
    ctx = mp.get_context("fork")
    out = [None] * len(files)
    live = {}  # index -> (process, conn, deadline)
    nxt = 0
    while nxt < len(files) or live:
        while nxt < len(files) and len(live) < par:
            rd, wr = ctx.Pipe(duplex=False)
            p = ctx.Process(target=_ref_child, args=(wr, files[nxt], sb, b), daemon=True)
            p.start()
            wr.close()
            live[nxt] = (p, rd, time.monotonic() + timeout)
            nxt += 1
        time.sleep(0.002)
        for i, (p, rd, dl) in list(live.items()):
            if rd.poll():
                try:
                    out[i] = rd.recv()
                except EOFError:
                    out[i] = None
                p.join()
                del live[i]
            elif not p.is_alive() or time.monotonic() > dl:
                p.kill()
                p.join()
                del live[i]
    return out


CORPORA = {
    "parser_recipe": (lambda: _mutants(ref_jpeg(32, 24, 7, 70, "420"), 300, 13, False), 1024, 256),
    "scan_intra": (lambda: _mutants(ref_jpeg(256, 192, 8, 75, "420"), 200, 14, True), 1024, 256),
    "scan_inter": (lambda: _mutants(ref_jpeg(256, 192, 9, 75, "420"), 200, 15, True), 128, 4),
    "header_and_scan_444": (lambda: _mutants(ref_jpeg(120, 72, 10, 90, "444"), 200, 16, False), 256, 2),
}


@pytest.mark.parametrize("name", list(CORPORA))
def test_mutated_files_match_reference_outcome(decoder, name):
    make, sb, b = CORPORA[name]
    files = make()
    ref = _ref_outcomes(files, sb, b)
    cfg = pj.DecodeConfig(subsequence_bits=sb, sequence_length_b=b)
    with decoder.batch(files, cfg, pj.OutputColorspace.RGBInterleaved) as bt:
        st = bt.run()
        outs = bt.download()
    hung = sum(r is None for r in ref)
    bad = []
    for i, r in enumerate(ref):
        if r is None:
            continue
        rs, rgb = r
        if int(st[i]) != rs:
            bad.append((i, int(st[i]), rs))
        elif rs == 0 and outs[i][: len(rgb)].tobytes() != rgb:
            bad.append((i, "rgb", 0))
    assert not bad, f"{len(bad)} of {len(files) - hung} outcomes differ ({hung} reference hangs): {bad[:12]}"
    assert hung < len(files) // 4
