"""GPU: the emit kernel's chunked item scan on large blocks (4K-wide frames:
hundreds of words per block, several segments per 256-item chunk).  A chunk
that holds no events but holds a segment's first item must still rebase that
segment's offset (regression: the rebase sat after the empty-chunk skip, so
the segment's events landed shifted by the events of earlier chunks)."""
import numpy as np
import pytest

from helpers import assert_same_events, concat, run_oracle_stream
from paper_2209_04634_b200 import SimulatorConfig, Simulator
from paper_2209_04634_b200.abi import Method, make_config

pytestmark = pytest.mark.gpu


def _block_words(w, h):
    # EventEngine::geometry(fine = false): ~8 blocks of 256 threads per SM on 148 SMs
    wpr = (w + 31) // 32
    n_words = h * wpr
    per = -(-n_words // (148 * 8))
    per = max(8, -(-per // 8) * 8)
    return wpr, per


@pytest.mark.parametrize("method", [Method.difference_only, Method.sparse])
def test_empty_chunk_holding_a_segment_start(oracle, method):
    w, h = 3840, 1904
    wpr, wpb = _block_words(w, h)
    assert wpb >= 200  # segments of one block span most of a 256-item chunk

    def region(word_lo, word_hi):  # pixel mask of words [lo, hi) of block 1
        m = np.zeros(h * wpr * 32, bool)
        for wd in range(wpb + word_lo, wpb + word_hi):
            row, col = divmod(wd, wpr)
            m[row * wpr * 32 + col * 32: row * wpr * 32 + col * 32 + 32] = True
        m = m.reshape(h, wpr * 32)[:, :w]
        return m

    f0 = np.full((h, w), 100, np.uint8)
    f1 = f0.copy()
    f1[region(0, 32)] = 160          # pair 0: events in words 0..31 of block 1
    f2 = f0.copy()                   # pair 1: back, events in words 0..31 again
    f3 = f2.copy()
    # pair 2: events only in the words of block 1 that fall into the third
    # 256-item chunk (segment s occupies items [s * wpb, (s + 1) * wpb)), so
    # the second chunk holds pair 2's first item but no event at all
    lo = 512 - 2 * wpb + 8
    assert 0 < lo < wpb - 16
    f3[region(lo, wpb - 4)] = 30
    frames = np.stack([f0, f1, f2, f3])
    ts = np.array([0, 1000, 2000, 3000], np.int64)
    cfg = make_config(method, n_interp=0 if method == Method.difference_only else 2)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    got = sim.push_frames(frames, ts).events
    assert len(exp) > 0
    assert_same_events(got, exp, what=f"{method.name} {w}x{h}")
