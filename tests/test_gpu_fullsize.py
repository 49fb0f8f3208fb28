"""GPU: BASELINE.json configs at FULL size — bit-exact against the oracle on
the first frame pairs, plus size-independent properties of the whole output
(ordering, bounds, determinism, count consistency)."""
import numpy as np
import pytest

from helpers import assert_same_events, run_oracle_stream
from paper_2209_04634_b200 import Frame, Method, SimulatorConfig, Simulator, scenes
from paper_2209_04634_b200.abi import make_config

pytestmark = pytest.mark.gpu


def cfg_for(name, mode):
    c = scenes.CONFIGS[name]
    cp, cn = scenes.LINEAR_THRESHOLDS[c.method]
    return make_config(Method[c.method], n_interp=c.n_interp, c_pos=cp, c_neg=cn, contrast_mode=mode,
                       c_pos_log=c.contrast, c_neg_log=-c.contrast)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
@pytest.mark.parametrize("mode", [1, 0])
def test_fullsize_vs_oracle(oracle, name, mode):
    n = 3 if name != "c5" else 2
    frames, ts = scenes.generate(name, n_frames=n)
    cfg = cfg_for(name, mode)
    exp = run_oracle_stream(oracle, cfg, frames, ts)
    sim = Simulator(SimulatorConfig.from_c(cfg))
    for k in range(n):
        got = sim.push_frame(Frame.from_array(frames[k], ts[k])).events
        assert_same_events(got, exp[k], f"{name} frame {k}")


@pytest.mark.parametrize("name", ["c2", "c5"])
def test_fullsize_properties(name):
    """Ordering (t, y, x, p), bounds, per-interval timestamps, determinism."""
    c = scenes.CONFIGS[name]
    frames, ts = scenes.generate(name, n_frames=4)
    cfg = SimulatorConfig.from_c(cfg_for(name, 1))
    outs = []
    for _ in range(2):
        sim = Simulator(cfg)
        outs.append([sim.push_frame(Frame.from_array(frames[k], ts[k])).events for k in range(4)])
    for k in range(1, 4):
        e = outs[0][k]
        assert_same_events(e, outs[1][k])
        assert len(e) > 0
        assert np.all((e["t"] > ts[k - 1]) & (e["t"] <= ts[k]))
        assert np.all(e["x"] < c.width) and np.all(e["y"] < c.height)
        assert len(np.unique(e["t"])) == c.n_interp + 1
        key = (e["t"].astype(np.int64) * c.height + e["y"]) * c.width + e["x"]
        assert np.all(np.diff(key) > 0)  # single mode: strictly increasing (t, y, x)
