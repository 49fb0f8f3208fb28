"""difference_frame / threshold_events (core.hpp:8-19, core.cpp:5-52) on the
GPU against a numpy restatement of the reference's scan (core.cpp:27-45),
at sizes and value ranges the reference's own 8x8 tests do not reach:
full int16 values, magnitude mode with thousands of copies per pixel,
odd shapes, empty results, and the config validation messages."""
import numpy as np
import pytest

from paper_2209_04634_b200 import (DifferenceFrame, EventsPerCrossing, Frame, InvalidArgument, Method,
                                   SimulatorConfig, difference_frame, threshold_events)


def scan(values, c_pos, c_neg, t, magnitude):
    """threshold_events_into, core.cpp:27-45: row-major scan, copies in place."""
    v = values.astype(np.int64).ravel()
    w = values.shape[1]
    cnt = np.where(v > c_pos, (v // c_pos) if magnitude else 1,
                   np.where(v < c_neg, (np.trunc(v / c_neg).astype(np.int64)) if magnitude else 1, 0))
    idx = np.repeat(np.arange(v.size), cnt)
    return idx % w, idx // w, np.where(v[idx] > c_pos, 1, -1)


def cfg(c_pos, c_neg, magnitude=False):
    c = SimulatorConfig.defaults(Method.difference_only)
    c.c_pos, c.c_neg = c_pos, c_neg
    c.events_per_crossing = EventsPerCrossing.magnitude if magnitude else EventsPerCrossing.single
    return c


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1, 1), (7, 13), (480, 640), (1080, 1921)])
@pytest.mark.parametrize("magnitude", [False, True])
def test_threshold_events_match_scan(shape, magnitude):
    rng = np.random.default_rng(shape[0] * 7 + magnitude)
    lim = 32767 if magnitude and shape[0] < 100 else 255
    vals = rng.integers(-lim, lim + 1, size=shape).astype(np.int16)
    for c_pos, c_neg in ((1, -1), (3, -7), (40, -2)):
        d = DifferenceFrame(shape[1], shape[0], 0, 99, vals)
        ev = threshold_events(d, cfg(c_pos, c_neg, magnitude), 99)
        x, y, p = scan(vals, c_pos, c_neg, 99, magnitude)
        assert len(ev) == len(x)
        assert np.array_equal(ev["x"], x) and np.array_equal(ev["y"], y) and np.array_equal(ev["p"], p)
        assert (ev["t"] == 99).all()


@pytest.mark.gpu
def test_difference_frame_and_threshold_equal_difference_only_push():
    """difference_only push == threshold_events(difference_frame) (test_simulate.cpp:52-66), 1080p."""
    from paper_2209_04634_b200 import Simulator
    rng = np.random.default_rng(5)
    a = Frame.from_array(rng.integers(0, 256, (1080, 1920), dtype=np.uint8), 0)
    b = Frame.from_array(rng.integers(0, 256, (1080, 1920), dtype=np.uint8), 40)
    d = difference_frame(a, b)
    assert np.array_equal(d.values, b.pixels.astype(np.int16) - a.pixels.astype(np.int16))
    c = cfg(2, -2)
    ev = threshold_events(d, c, 40)
    sim = Simulator(c)
    sim.push_frame(a)
    got = sim.push_frame(b).events
    assert len(got) == len(ev)
    for f in ("x", "y", "t", "p"):
        assert np.array_equal(got[f], ev[f])


@pytest.mark.gpu
def test_threshold_events_empty_and_invalid():
    d = DifferenceFrame(5, 4, 0, 1, np.zeros((4, 5), np.int16))
    assert len(threshold_events(d, cfg(1, -1), 1)) == 0
    with pytest.raises(InvalidArgument, match="c_pos must be > 0"):
        threshold_events(d, cfg(0, -2), 1)
    with pytest.raises(InvalidArgument, match="c_neg must be < 0"):
        threshold_events(d, cfg(2, 0), 1)


def test_difference_frame_dimension_message():
    """The reference's message (core.cpp:6-11), raised before any device work."""
    a = Frame.from_array(np.zeros((4, 4), np.uint8), 0)
    b = Frame.from_array(np.zeros((5, 4), np.uint8), 1)
    with pytest.raises(InvalidArgument, match=r"difference_frame: incompatible input frames \(4x4 vs 4x5\)"):
        difference_frame(a, b)
