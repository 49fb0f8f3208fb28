"""GPU: the tile-staged dense chain (chain_dense_tile_kernel)
against the oracle.  EVSIM_CHAIN_QUAD=tile forces the tile geometry on small
frames (any even width whose word count per row is a multiple of 4); the
setting is read when a simulator is created.  Covered: both contrast modes,
every batch size of the interior links (8, 10, 5, 4 and ragged remainders),
no-endpoint chains, tile rows hanging over the frame, widths that are not a
multiple of 32, frame borders (clamped samples), noise frames whose flow is
large and irregular (regions that do not fit fall back to the gathers),
colliding sub-interval timestamps (the general emit over 4-word blocks), row
bands, sub-batched long pushes, and both resident-block settings."""
import numpy as np
import pytest

from helpers import assert_same_events, concat, run_oracle_stream
from paper_2209_04634_b200 import SimulatorConfig, Simulator, scenes
from paper_2209_04634_b200.abi import Method, make_config

pytestmark = pytest.mark.gpu


def _run(oracle, cfg, frames, ts, cuts, what):
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    got, a = [], 0
    for b in cuts:
        got.append(sim.push_frames(frames[a:b], ts[a:b]).events)
        a = b
    assert_same_events(concat(got), exp, what=what)
    return len(exp)


@pytest.mark.parametrize("mode", [1, 0])
@pytest.mark.parametrize("N,incl", [(8, 1), (10, 1), (5, 1), (4, 0), (7, 1), (32, 1), (16, 0), (1, 1)])
def test_tile_chain_matches_oracle(oracle, mode, N, incl, monkeypatch):
    monkeypatch.setenv("EVSIM_CHAIN_QUAD", "tile")
    frames, ts = scenes.generate("c2", n_frames=6, width=256, height=44)
    cfg = make_config(Method.dense, n_interp=N, contrast_mode=mode, c_pos_log=0.1, c_neg_log=-0.1,
                      include_endpoints=incl)
    n = _run(oracle, cfg, frames, ts, (1, 3, 6), f"tile mode={mode} N={N} incl={incl}")
    assert n > 0


@pytest.mark.parametrize("blocks", ["3", "4"])
@pytest.mark.parametrize("w,h", [(384, 17), (250, 33), (128, 8), (640, 61)])
def test_tile_chain_sizes(oracle, w, h, blocks, monkeypatch):
    monkeypatch.setenv("EVSIM_CHAIN_QUAD", "tile")
    monkeypatch.setenv("EVSIM_TILE_BLOCKS", blocks)
    frames, ts = scenes.generate("c4", n_frames=5, width=w, height=h)
    for mode in (1, 0):
        cfg = make_config(Method.dense, n_interp=16, contrast_mode=mode, c_pos_log=0.2, c_neg_log=-0.2)
        _run(oracle, cfg, frames, ts, (2, 5), f"tile {w}x{h} mode={mode} blocks={blocks}")


@pytest.mark.parametrize("seed", range(6))
def test_tile_chain_noise_flow(oracle, seed, monkeypatch):
    """Unblurred noise with a fast pan (c5's generator): the LK field is large
    and irregular, so sample regions vary per tile and some do not fit."""
    monkeypatch.setenv("EVSIM_CHAIN_QUAD", "tile")
    rng = np.random.default_rng(300 + seed)
    w, h = int(rng.choice([256, 384, 512])), int(rng.choice([24, 50, 64]))
    frames, ts = scenes.generate("c5", n_frames=4, width=w, height=h)
    mode = seed & 1
    cfg = make_config(Method.dense, n_interp=int(rng.choice([8, 32])), contrast_mode=mode, c_pos_log=0.1,
                      c_neg_log=-0.1, flow_preset=int(rng.integers(0, 2)))
    _run(oracle, cfg, frames, ts, (1, 4), f"tile noise seed={seed} {w}x{h} mode={mode}")


def test_tile_chain_colliding_timestamps(oracle, monkeypatch):
    monkeypatch.setenv("EVSIM_CHAIN_QUAD", "tile")
    frames, ts = scenes.generate("c2", n_frames=6, width=256, height=30)
    ts = np.cumsum([5, 3, 1000, 2, 33333, 7]).astype(np.int64)  # dt < K: equal sub-interval stamps
    for mode in (1, 0):
        cfg = make_config(Method.dense, n_interp=10, contrast_mode=mode, c_pos_log=0.1, c_neg_log=-0.1)
        _run(oracle, cfg, frames, ts, (6,), f"tile collisions mode={mode}")


def test_tile_chain_long_push_and_bands(oracle, monkeypatch):
    monkeypatch.setenv("EVSIM_CHAIN_QUAD", "tile")
    frames, ts = scenes.generate("c2", n_frames=41, width=256, height=40)
    cfg = make_config(Method.dense, n_interp=10, contrast_mode=1, c_pos_log=0.1, c_neg_log=-0.1)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    got = concat([sim.push_frames(frames[a:b], ts[a:b]).events for a, b in ((0, 1), (1, 41))])
    assert_same_events(got, exp, what="tile long push (sub-batches)")
    # two row bands, merged per timestamp by (y, x): band rows 0..19 and 20..39
    parts = []
    for y0, y1 in ((0, 20), (20, 40)):
        s = Simulator(SimulatorConfig.from_c(cfg))
        s.set_row_band(y0, y1)
        parts.append(concat([s.push_frames(frames[a:b], ts[a:b]).events for a, b in ((0, 1), (1, 41))]))
    allp = np.concatenate(parts)
    order = np.lexsort((allp["x"], allp["y"], allp["t"]))
    # (within one timestamp the reference orders by (y, x); polarity ties cannot occur in single mode)
    assert_same_events(allp[order], exp, what="tile bands")


def test_tile_chain_on_a_4k_wide_strip(oracle, monkeypatch):
    """c5's width (30 tile columns, 60 tile rows) through the tile kernel."""
    monkeypatch.setenv("EVSIM_CHAIN_QUAD", "tile")
    frames, ts = scenes.generate("c5", n_frames=3, width=3840, height=480)
    cfg = make_config(Method.dense, n_interp=8, contrast_mode=1, c_pos_log=0.1, c_neg_log=-0.1)
    _run(oracle, cfg, frames, ts, (3,), "tile 3840x480")
