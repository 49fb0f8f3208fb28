"""Throughput of the data formats either side of the path:
device frame ingestion, .evs record formatting, event metrics.  One JSON line
per measurement; CUDA-event timing is not available through these host-buffer
entry points, so each is timed end to end (host wall clock, H2D + kernel +
D2H), after a warm-up call.

    python tools/bench_formats.py
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2209_04634_b200 import (EventStream, SimulatorConfig, Simulator, accumulate, events_per_pixel_second,  # noqa
                                   ingest_frames, scenes)
from paper_2209_04634_b200.abi import Method, make_config  # noqa: E402


def timed(fn, reps=5):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps


def main():
    rng = np.random.default_rng(0)
    # 1080p RGB -> luma -> 640x480 (DSEC-like ingestion), 32 frames per call
    rgb = rng.integers(0, 256, size=(32, 1080, 1920, 3), dtype=np.uint8)
    dt = timed(lambda: ingest_frames(rgb, (640, 480)))
    print(json.dumps({"what": "ingest_frames 1920x1080 RGB -> 640x480 gray", "frames_per_s": round(32 / dt, 1),
                      "input_GB_per_s": round(rgb.nbytes / dt / 1e9, 2), "timing": "host wall clock, e2e"}))
    # events of one c2 push
    frames, ts = scenes.generate("c2", n_frames=32)
    sim = Simulator(SimulatorConfig.from_c(make_config(Method.dense, n_interp=10, contrast_mode=0)))
    ev = sim.push_frames(frames, ts).events
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "e.evs")
        dt = timed(lambda: sim.write_events_binary(p))
        print(json.dumps({"what": "write_events_binary (device-formatted .evs records)", "events": int(len(ev)),
                          "events_per_s": round(len(ev) / dt, 1), "MB_per_s": round((16 + 13 * len(ev)) / dt / 1e6, 1),
                          "timing": "host wall clock incl. D2H and file write"}))
    s = EventStream(640, 480)
    s.events = ev
    dt = timed(lambda: events_per_pixel_second(s, 1.0))
    print(json.dumps({"what": "events_per_pixel_second", "events": int(len(ev)), "events_per_s": round(len(ev) / dt, 1),
                      "timing": "host wall clock incl. H2D of 24-B events and the fp64 pixel-order reduction"}))
    dt = timed(lambda: accumulate(s, int(ts[0]), int(ts[-1])))
    print(json.dumps({"what": "accumulate", "events": int(len(ev)), "events_per_s": round(len(ev) / dt, 1),
                      "timing": "host wall clock incl. H2D of 24-B events"}))


if __name__ == "__main__":
    main()
