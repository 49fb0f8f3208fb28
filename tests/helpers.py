"""Shared test helpers: golden fixtures, event comparison, GPU stream runner."""
from __future__ import annotations

import glob
import os

import numpy as np

from paper_2209_04634_b200.abi import CConfig

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


NON_STREAM_FIXTURES = {"interp_random_flow", "io_ingest", "metrics"}


def golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def stream_fixtures():
    return [n for n in golden_names() if n not in NON_STREAM_FIXTURES]


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def golden_cfg(g) -> CConfig:
    c = CConfig()
    for f, _ in CConfig._fields_:
        v = g[f"cfg_{f}"].item()
        setattr(c, f, v)
    return c


def cols(ev):
    return ev["x"], ev["y"], ev["t"], ev["p"]


def assert_events_equal(got, exp_x, exp_y, exp_t, exp_p, what=""):
    gx, gy, gt, gp = (np.asarray(a) for a in cols(got))
    assert len(gx) == len(exp_x), f"{what}: {len(gx)} events vs {len(exp_x)} expected"
    for name, a, b in (("x", gx, exp_x), ("y", gy, exp_y), ("t", gt, exp_t), ("p", gp, exp_p)):
        bad = np.nonzero(np.asarray(a).astype(np.int64) != np.asarray(b).astype(np.int64))[0]
        assert bad.size == 0, f"{what}: field {name} differs at {bad.size} events, first at {bad[0]}: " \
                              f"got {a[bad[0]]} want {b[bad[0]]}"


def assert_same_events(got, exp, what=""):
    assert_events_equal(got, *cols(exp), what=what)


def run_oracle_stream(oracle, cfg, frames, ts):
    sim = oracle.simulator(cfg)
    return [sim.push_frame(frames[k], int(ts[k])) for k in range(len(frames))]


def concat(evs):
    from paper_2209_04634_b200.abi import EVENT_DTYPE
    return np.concatenate(evs) if evs else np.zeros(0, EVENT_DTYPE)
