"""The data formats either side of the path: frame ingestion
(io.cpp:41-103), event files (io.cpp:105-170) and event metrics
(metrics.cpp:7-69).

CPU: the byte-level restatement of the .evs / text formats used by the GPU
tests is pinned to the reference's own writers (oracle/_ref), and the golden
fixtures to the reference's functions.  GPU: the device paths against the
golden fixtures and the pinned restatement."""
import os

import numpy as np
import pytest

from helpers import load_golden
from paper_2209_04634_b200 import (Frame, InvalidArgument, SimulatorConfig, Simulator, accumulate, EventStream,
                                   events_per_pixel_second, ingest_frames, scenes)
from paper_2209_04634_b200._lib import EvsimError
from paper_2209_04634_b200.abi import EVENT_DTYPE, Method, make_config


def evs_bytes(events, w, h) -> bytes:
    """write_events_binary (io.cpp:148-170) restated: 'EVS1', u16 w, u16 h,
    u64 count, then 13-byte little-endian records (x, y, t, p)."""
    rec = np.zeros(len(events), np.dtype([("x", "<u2"), ("y", "<u2"), ("t", "<i8"), ("p", "i1")]))
    for k in ("x", "y", "t", "p"):
        rec[k] = events[k]
    return b"EVS1" + np.array([w, h], "<u2").tobytes() + np.array([len(events)], "<u8").tobytes() + rec.tobytes()


def text_bytes(events) -> bytes:
    """write_events_text (io.cpp:105-126) restated."""
    return "".join(f"{int(e['x'])},{int(e['y'])},{int(e['t'])},{'1' if e['p'] > 0 else '-1'}\n"
                   for e in events).encode()


def metrics_events():
    g = load_golden("metrics")
    ev = np.zeros(len(g["ev_x"]), EVENT_DTYPE)
    for k in ("x", "y", "t", "p"):
        ev[k] = g[f"ev_{k}"]
    return g, ev


def test_format_restatement_matches_reference_writers(reference, tmp_path):
    g, ev = metrics_events()
    p1, p2 = str(tmp_path / "a.evs"), str(tmp_path / "a.txt")
    reference.write_events_binary(ev, 64, 48, p1)
    reference.write_events_text(ev, 64, 48, p2)
    assert open(p1, "rb").read() == evs_bytes(ev, 64, 48)
    assert open(p2, "rb").read() == text_bytes(ev)


def test_golden_io_fixtures_match_reference(reference):
    g = load_golden("io_ingest")
    for k in range(len(g["rgb"])):
        assert np.array_equal(reference.luma(g["rgb"][k]).reshape(g["gray"][k].shape), g["gray"][k])
        assert np.array_equal(reference.resize_bilinear(g["gray"][k], 29, 17), g["down"][k])
    g, ev = metrics_events()
    m = reference.events_per_pixel_second(ev, 64, 48, 0.05)
    assert np.array_equal(np.array(m[:3]), g["rate"]) and m[3] == int(g["total"])
    assert np.array_equal(reference.accumulate(ev, 64, 48, *[int(t) for t in g["window"]]), g["classes"])


@pytest.mark.gpu
def test_gpu_ingest_matches_reference():
    g = load_golden("io_ingest")
    assert np.array_equal(ingest_frames(g["rgb"]), g["gray"])
    assert np.array_equal(ingest_frames(g["rgb"], (29, 17)), g["down"])
    assert np.array_equal(ingest_frames(g["gray"], (50, 40)), g["up"])
    assert np.array_equal(ingest_frames(g["gray"], (37, 23)), g["gray"])
    with pytest.raises(InvalidArgument, match="target must be positive"):
        ingest_frames(g["gray"], (-1, 5))


@pytest.mark.gpu
def test_gpu_metrics_match_reference():
    g, ev = metrics_events()
    s = EventStream(64, 48)
    s.events = ev
    st = events_per_pixel_second(s, 0.05)
    assert (st.mean_rate, st.std_rate, st.duration) == tuple(g["rate"]) and st.total_events == int(g["total"])
    assert np.array_equal(accumulate(s, *[int(t) for t in g["window"]]), g["classes"])
    with pytest.raises(InvalidArgument, match="duration must be > 0"):
        events_per_pixel_second(s, 0.0)
    with pytest.raises(InvalidArgument, match="t_start < t_end"):
        accumulate(s, 5, 5)


@pytest.mark.gpu
@pytest.mark.parametrize("m", [Method.dense, Method.sparse, Method.difference_only])
def test_gpu_event_files(tmp_path, m):
    frames, ts = scenes.generate("c2", n_frames=4, width=80, height=60)
    sim = Simulator(SimulatorConfig.from_c(make_config(m, n_interp=3 if m != Method.difference_only else 0)))
    ev = sim.push_frames(frames, ts).events
    p1, p2 = str(tmp_path / "e.evs"), str(tmp_path / "e.txt")
    sim.write_events_binary(p1)
    sim.write_events_text(p2)
    assert open(p1, "rb").read() == evs_bytes(ev, 80, 60)
    assert open(p2, "rb").read() == text_bytes(ev)
    with pytest.raises(EvsimError, match="cannot open for writing"):
        sim.write_events_binary(os.path.join(str(tmp_path), "no", "such", "dir.evs"))
