"""GPU: the dense chain's three gather images (EVSIM_CHAIN_QUAD = u8 quads,
fp32 lerp quads, bf16 lerp quads) give the same bit-exact
events as the oracle — pipelined pushes of a c2-like sequence (sub-batches,
flow / chain overlap), both contrast modes, magnitude and no-endpoint chains.
The setting is read when a simulator is created."""
import os

import numpy as np
import pytest

from helpers import assert_same_events, concat, run_oracle_stream
from paper_2209_04634_b200 import SimulatorConfig, Simulator, scenes
from paper_2209_04634_b200.abi import EventsPerCrossing, Method, make_config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["u8", "f4", "bf16"])
@pytest.mark.parametrize("mode,mag,incl", [(1, 0, 1), (0, 0, 1), (1, 1, 1), (0, 0, 0)])
def test_quad_kinds_match_oracle(oracle, kind, mode, mag, incl, monkeypatch):
    monkeypatch.setenv("EVSIM_CHAIN_QUAD", kind)
    frames, ts = scenes.generate("c2", n_frames=34, width=131, height=77)
    cfg = make_config(Method.dense, n_interp=10, contrast_mode=mode, c_pos_log=0.1, c_neg_log=-0.1,
                      events_per_crossing=int(EventsPerCrossing.magnitude) if mag else 0, include_endpoints=incl)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    got = concat([sim.push_frames(frames[a:b], ts[a:b]).events for a, b in ((0, 1), (1, 34))])
    assert_same_events(got, exp, what=f"{kind} mode={mode} mag={mag} incl={incl}")


@pytest.mark.parametrize("width", [32768, 32770])
def test_fp32_quads_at_their_width_bound(oracle, width):
    """The fp32 quads hold tap-relative constants (a00 - x*dx, dy - x*dxy) that
    are exact integers below 2^24 up to 32768 columns (kernels.h
    kLerpQuadMaxW); wider frames take the bf16 quads.  Strong contrast in the
    last columns (|dx| = 255, |dxy| = 510) with motion there, on both sides
    of the bound."""
    rng = np.random.default_rng(width)
    h, n = 24, 4
    base = rng.integers(0, 2, size=(h, width + 8)).astype(np.uint8) * 255  # checker-like extremes
    frames = np.stack([np.ascontiguousarray(base[:, k:k + width]) for k in range(n)])
    ts = np.arange(n, dtype=np.int64) * 33333
    cfg = make_config(Method.dense, n_interp=4, contrast_mode=0, c_pos=2, c_neg=-2)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    got = concat([sim.push_frames(frames[a:b], ts[a:b]).events for a, b in ((0, 1), (1, n))])
    assert_same_events(got, exp, what=f"width {width}")
