"""GPU: the reference test suite's behavioural cases (tests/test_simulate.cpp,
test_flow.cpp) restated against the B200 Simulator API, plus error / state
semantics of the C-ABI."""
import numpy as np
import pytest

from helpers import assert_same_events
from paper_2209_04634_b200 import (DenseFlowEstimator, FlowField, FlowPreset, Frame, InvalidArgument, Method,
                                   SimulatorConfig, Simulator, dense_events_with_flow, estimate_dense_flow,
                                   estimate_sparse_flow, interpolate_frames, simulate_dense)

pytestmark = pytest.mark.gpu

ALL = [Method.difference_only, Method.dense, Method.sparse]


def textured(w, h, seed):
    rng = np.random.default_rng(seed)
    from scipy.ndimage import uniform_filter
    a = rng.integers(0, 256, (h, w)).astype(float)
    a = uniform_filter(uniform_filter(a, 3, mode="nearest"), 3, mode="nearest")
    return np.clip(np.rint(a), 0, 255).astype(np.uint8)


@pytest.mark.parametrize("m", ALL)
def test_first_frame_is_warm_up(m):
    # test_simulate.cpp:30-39
    sim = Simulator(SimulatorConfig.defaults(m))
    out = sim.push_frame(Frame.from_array(textured(16, 16, 3), 0))
    assert len(out) == 0 and out.width == 16 and out.height == 16


@pytest.mark.parametrize("m", ALL)
def test_identical_frames_no_events(m):
    # test_simulate.cpp:41-49
    base = textured(24, 18, 77)
    sim = Simulator(SimulatorConfig.defaults(m))
    for k in range(4):
        assert len(sim.push_frame(Frame.from_array(base, 1000 * k))) == 0


def test_rejects_bad_timestamps_and_resolution_changes_state_untouched():
    # test_simulate.cpp:66-74 + simulate.cpp:307-318 messages
    sim = Simulator(SimulatorConfig.defaults(Method.difference_only))
    sim.push_frame(Frame.make(8, 8, 100))
    with pytest.raises(InvalidArgument, match="^push_frame: timestamps must be strictly increasing$"):
        sim.push_frame(Frame.make(8, 8, 100))
    with pytest.raises(InvalidArgument, match="strictly increasing"):
        sim.push_frame(Frame.make(8, 8, 50))
    with pytest.raises(InvalidArgument, match="^push_frame: frame dimensions changed mid-stream$"):
        sim.push_frame(Frame.make(8, 9, 200))
    f = Frame.make(8, 8, 200)
    f.pixels[3, 4] = 50
    out = sim.push_frame(f)  # still usable; prev is still the t=100 frame
    assert len(out) == 1 and out.events["t"][0] == 200


def test_malformed_frame():
    sim = Simulator(SimulatorConfig.defaults(Method.dense))
    with pytest.raises(InvalidArgument, match="^push_frame: malformed frame$"):
        sim.push_frame(Frame(4, 4, 0, np.zeros(15, np.uint8)))


def test_reset_allows_new_resolution():
    sim = Simulator(SimulatorConfig.defaults(Method.dense))
    sim.push_frame(Frame.from_array(textured(32, 24, 1), 0))
    sim.push_frame(Frame.from_array(textured(32, 24, 2), 10))
    sim.reset()
    assert len(sim.push_frame(Frame.from_array(textured(40, 30, 3), 5))) == 0  # warm-up again
    out = sim.push_frame(Frame.from_array(textured(40, 30, 4), 20))
    assert len(out) > 0 and out.width == 40


def test_interpolate_zero_flow_copies_and_stamps():
    # test_simulate.cpp:76-87
    f = textured(20, 20, 5)
    inter = interpolate_frames(Frame.from_array(f, 0), Frame.from_array(f, 1100), FlowField.zeros(20, 20), 3)
    assert [x.timestamp for x in inter] == [275, 550, 825]
    for x in inter:
        assert np.array_equal(x.pixels, f)


def test_interpolate_blend_midpoint():
    # test_simulate.cpp:89-98
    a, b = Frame.make(6, 6, 0, 40), Frame.make(6, 6, 1000, 120)
    inter = interpolate_frames(a, b, FlowField.zeros(6, 6), 3)
    assert inter[1].pixels[3, 3] == 80 and inter[0].pixels[0, 0] == 60 and inter[2].pixels[0, 0] == 100


def test_interpolate_flow_dimension_mismatch():
    # test_simulate.cpp:126-129
    with pytest.raises(InvalidArgument):
        interpolate_frames(Frame.make(8, 8, 0), Frame.make(8, 8, 10), FlowField.zeros(8, 7), 2)


def test_zero_flow_dense_matches_brute_force():
    # test_simulate.cpp:143-156 against oracles.hpp:70-99 restated
    rng = np.random.default_rng(33)
    cfg = SimulatorConfig.defaults(Method.dense)
    cfg.n_interp = 3
    for _ in range(5):
        a = rng.integers(0, 256, (8, 8), dtype=np.uint8)
        b = rng.integers(0, 256, (8, 8), dtype=np.uint8)
        got = dense_events_with_flow(Frame.from_array(a, 0), Frame.from_array(b, 1000), FlowField.zeros(8, 8), cfg)
        exp = []
        for k in range(1, 5):
            t = (k * 1000 + 3) // 4
            for y in range(8):
                for x in range(8):
                    bl = lambda kk: int(np.floor((1.0 - kk / 4) * a[y, x] + (kk / 4) * b[y, x] + 0.5))
                    v = bl(k) - bl(k - 1)
                    if v > 2:
                        exp.append((x, y, t, 1))
                    elif v < -2:
                        exp.append((x, y, t, -1))
        e = got.events
        assert list(zip(e["x"].tolist(), e["y"].tolist(), e["t"].tolist(), e["p"].tolist())) == exp


class ConstantFlow(DenseFlowEstimator):
    """test_simulate.cpp:311-324 stub backend."""

    def __init__(self, du, dv):
        self.du, self.dv = du, dv

    def estimate(self, prev, curr):
        f = FlowField.zeros(prev.width, prev.height)
        f.du[:] = self.du
        f.dv[:] = self.dv
        return f


def test_plugin_backend_equivalence():
    # test_simulate.cpp:328-339
    rng = np.random.default_rng(64)
    a = Frame.from_array(rng.integers(0, 256, (16, 16), dtype=np.uint8), 0)
    b = Frame.from_array(rng.integers(0, 256, (16, 16), dtype=np.uint8), 800)
    cfg = SimulatorConfig.defaults(Method.dense)
    cfg.n_interp = 2
    stub = ConstantFlow(1.5, -0.5)
    via_interface = simulate_dense(a, b, cfg, stub)
    via_field = dense_events_with_flow(a, b, stub.estimate(a, b), cfg)
    assert_same_events(via_interface.events, via_field.events)
    sim = Simulator(cfg, dense_flow=stub)
    sim.push_frame(a)
    assert_same_events(sim.push_frame(b).events, via_field.events)


@pytest.mark.parametrize("m", ALL)
def test_timestamps_in_interval_and_ordered(m):
    # test_simulate.cpp:274-306
    cfg = SimulatorConfig.defaults(m)
    cfg.c_pos, cfg.c_neg = 2, -2
    sim = Simulator(cfg)
    rng = np.random.default_rng(101)
    prev_t = -1
    allev = []
    for k in range(5):
        t = 700 * k
        out = sim.push_frame(Frame.from_array(rng.integers(0, 256, (12, 12), dtype=np.uint8), t))
        e = out.events
        assert np.all(e["t"] > prev_t) and np.all(e["t"] <= t)
        assert np.all(e["x"] < 12) and np.all(e["y"] < 12)
        allev.append(e)
        prev_t = t
    e = np.concatenate(allev)
    key = np.lexsort((e["p"], e["x"], e["y"], e["t"]))
    assert np.array_equal(key, np.arange(len(e)))


@pytest.mark.parametrize("m", ALL)
def test_deterministic_runs(m):
    # test_simulate.cpp:341-355
    from paper_2209_04634_b200 import scenes
    frames, ts = scenes.generate("c3", n_frames=4, width=96, height=72)
    runs = []
    for _ in range(2):
        sim = Simulator(SimulatorConfig.defaults(m))
        runs.append(np.concatenate([sim.push_frame(Frame.from_array(frames[k], ts[k])).events for k in range(4)]))
    assert_same_events(runs[0], runs[1])


def test_dense_flow_identical_frames_exact_zero():
    # test_flow.cpp:25-37
    f = textured(64, 48, 21)
    for p in (FlowPreset(3, 2, 4), FlowPreset(5, 16, 6)):
        fl = estimate_dense_flow(Frame.from_array(f, 0), Frame.from_array(f, 1000), p)
        assert np.max(np.abs(fl.du)) == 0.0 and np.max(np.abs(fl.dv)) == 0.0


def test_dense_flow_translation_recovered():
    # test_flow.cpp:80-97 (median error < 0.5 px)
    base = textured(200, 200, 7)
    for dx, dy in ((1, 0), (0, 2), (2, 1), (3, 0)):
        a = base[50:130, 50:146]
        b = base[50 - dy:130 - dy, 50 - dx:146 - dx]
        for p in (FlowPreset(3, 2, 4), FlowPreset(5, 16, 6)):
            fl = estimate_dense_flow(Frame.from_array(a, 0), Frame.from_array(b, 1), p)
            err = np.sqrt((fl.du - dx) ** 2 + (fl.dv - dy) ** 2)
            assert np.median(err) < 0.5


def test_sparse_flow_lost_and_empty():
    # test_flow.cpp:131-162
    a = Frame.make(32, 32, 0, 128)
    b = Frame.make(32, 32, 10, 128)
    assert estimate_sparse_flow(a, b, [[16, 16]], FlowPreset()).status[0] == 0
    f = Frame.from_array(textured(32, 32, 9), 0)
    empty = estimate_sparse_flow(f, f, np.zeros((0, 2), np.int32), FlowPreset())
    assert len(empty.status) == 0
    with pytest.raises(InvalidArgument, match="point outside frame bounds"):
        estimate_sparse_flow(f, f, [[32, 0]], FlowPreset())


def test_events_are_kernel_output():
    """The push path launches our kernels (no host fallback)."""
    sim = Simulator(SimulatorConfig.defaults(Method.dense))
    sim.push_frame(Frame.from_array(textured(64, 64, 1), 0))
    sim.push_frame(Frame.from_array(textured(64, 64, 2), 33))
    assert sim.kernel_launches >= 6
