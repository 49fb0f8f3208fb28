"""GPU: row bands (evsim_gpu_set_row_band).  Each band handle
holds the full frames, solves only the flow patch rows its event rows depend
on, and emits only its rows; merged per timestamp in band order, the bands
reproduce the whole-frame stream bit for bit (and so the reference's)."""
import numpy as np
import pytest

from helpers import assert_same_events, concat, run_oracle_stream
from paper_2209_04634_b200 import InvalidArgument, SimulatorConfig, Simulator, parallel, scenes
from paper_2209_04634_b200.abi import Method, make_config

pytestmark = pytest.mark.gpu


def merge(bands):
    """Per segment (timestamp), band 0's events, then band 1's, ...: a stable
    sort by t of the band-ordered concatenation."""
    ev = np.concatenate(bands)
    return ev[np.argsort(ev["t"], kind="stable")]


@pytest.mark.parametrize("m,mode,mag,incl", [(Method.dense, 1, 0, 1), (Method.dense, 0, 0, 1), (Method.dense, 1, 1, 1),
                                             (Method.dense, 0, 0, 0), (Method.difference_only, 0, 0, 1)])
@pytest.mark.parametrize("G", [2, 3])
def test_bands_merge_to_full_frame(oracle, m, mode, mag, incl, G):
    frames, ts = scenes.generate("c5", n_frames=5, width=120, height=150)
    cfg = make_config(m, n_interp=4 if m != Method.difference_only else 0, contrast_mode=mode,
                      events_per_crossing=mag, include_endpoints=incl, c_pos_log=0.1, c_neg_log=-0.1)
    full = Simulator(SimulatorConfig.from_c(cfg)).push_frames(frames, ts).events
    assert_same_events(full, concat(run_oracle_stream(oracle, cfg, frames, ts)))
    bands = []
    for b in range(G):
        y0, y1 = parallel.band_rows(150, G, b)
        sim = Simulator(SimulatorConfig.from_c(cfg))
        sim.set_row_band(y0, y1)
        ev = np.concatenate([sim.push_frames(frames[:2], ts[:2]).events, sim.push_frames(frames[2:], ts[2:]).events])
        assert ((ev["y"] >= y0) & (ev["y"] < y1)).all()
        bands.append(ev)
    assert_same_events(merge(bands), full)


def test_band_plan_matches_host_logic():
    # the library's per-level patch rows are a superset of parallel.band_plan's
    plan = parallel.band_plan(3840, 2160, parallel.band_rows(2160, 4, 1), levels=3, radius=4)
    assert plan.patch_rows[0][0] > 0 and plan.patch_rows[0][1] < 2160 // 4


def test_band_validation():
    sim = Simulator(SimulatorConfig.from_c(make_config(Method.sparse, n_interp=3)))
    with pytest.raises(InvalidArgument, match="sparse"):
        sim.set_row_band(0, 10)
    sim = Simulator(SimulatorConfig.from_c(make_config(Method.dense, n_interp=3)))
    with pytest.raises(InvalidArgument, match="y0 < y1"):
        sim.set_row_band(5, 5)
    frames, ts = scenes.generate("c2", n_frames=2, width=32, height=24)
    sim.set_row_band(0, 40)
    with pytest.raises(InvalidArgument, match="outside the frame"):
        sim.push_frames(frames, ts)
    sim.set_row_band(8, 16)
    sim.push_frames(frames[:1], ts[:1])
    with pytest.raises(InvalidArgument, match="start of a stream"):
        sim.set_row_band(0, 0)
