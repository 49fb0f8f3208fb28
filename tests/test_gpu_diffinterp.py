"""GPU: the difference_interp method (simulate.cpp:212-285, 334-341; SURVEY.md
§8f item 1) against the oracle restatement (itself pinned to the compiled
reference by tests/test_oracle_vs_ref.py and the diffinterp_* golden fixtures,
which test_gpu_parity also runs on the GPU)."""
import numpy as np
import pytest

from helpers import assert_same_events, concat, run_oracle_stream
from paper_2209_04634_b200 import (Frame, InvalidArgument, SimulatorConfig, Simulator, scenes, simulate_difference)
from paper_2209_04634_b200.abi import Method, make_config, unpack_events

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,mag,incl", [(10, 0, 1), (4, 1, 1), (6, 0, 0), (0, 0, 1), (0, 1, 0), (1, 0, 1),
                                        (40, 0, 1)])
def test_diffinterp_stream_matches_oracle(oracle, n, mag, incl):
    frames, ts = scenes.generate("c3", n_frames=7, width=112, height=80)
    cfg = make_config(Method.difference_interp, n_interp=n, events_per_crossing=mag, include_endpoints=incl,
                      c_pos=12, c_neg=-12)
    exp = run_oracle_stream(oracle, cfg, frames, ts)
    sim = Simulator(SimulatorConfig.from_c(cfg))
    for k in range(len(frames)):
        got = sim.push_frame(Frame.from_array(frames[k], ts[k])).events
        assert_same_events(got, exp[k], what=f"frame {k}")
    assert len(exp[0]) == 0 and len(exp[1]) == 0  # two frames buffered before the first events


@pytest.mark.parametrize("batch", [1, 2, 3, 8])
def test_diffinterp_batches_and_reset(oracle, batch):
    frames, ts = scenes.generate("c2", n_frames=9, width=96, height=64)
    cfg = make_config(Method.difference_interp, n_interp=5, c_pos=8, c_neg=-8)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    got = [sim.push_frames(frames[a:a + batch], ts[a:a + batch]).events for a in range(0, len(frames), batch)]
    assert_same_events(concat(got), exp)
    sim.reset()
    again = sim.push_frames(frames, ts).events
    assert_same_events(again, exp)
    sim.reset()
    p, t, o = sim.push_frames_streamed(frames, ts, chunk=2)
    assert_same_events(unpack_events(p, t, o), exp)


def test_diffinterp_collision_timestamps(oracle):
    frames, _ = scenes.generate("c1", n_frames=5, width=48, height=40)
    ts = np.array([0, 4, 9, 12, 20], np.int64)  # dt < K: equal sub-interval stamps with the d2 link
    cfg = make_config(Method.difference_interp, n_interp=10, c_pos=5, c_neg=-5)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    assert_same_events(sim.push_frames(frames, ts).events, exp)


def test_simulate_difference_free_function(oracle):
    frames, ts = scenes.generate("c3", n_frames=3, width=64, height=48)
    cfg = SimulatorConfig.defaults(Method.difference_interp)
    got = simulate_difference(*[Frame.from_array(frames[k], ts[k]) for k in range(3)], cfg).events
    exp = run_oracle_stream(oracle, cfg.to_c(), frames, ts)[2]
    assert_same_events(got, exp)
    with pytest.raises(InvalidArgument, match="strictly increasing"):
        simulate_difference(Frame.from_array(frames[0], 5), Frame.from_array(frames[1], 5),
                            Frame.from_array(frames[2], 9), cfg)


def test_diffinterp_rejects_log_mode():
    with pytest.raises(InvalidArgument, match="no log contrast mode"):
        Simulator(SimulatorConfig.from_c(make_config(Method.difference_interp, contrast_mode=1)))
