"""CPU: differential test of the C restatement against the compiled reference.

Runs only where oracle/_ref can be built (the source container: the reference
sources at /root/reference are compiled in place, never copied).  Randomised
inputs and configs beyond the committed golden fixtures.
"""
import numpy as np
import pytest

from helpers import assert_same_events
from paper_2209_04634_b200.abi import Method, make_config


def _cfgs():
    out = []
    for m in (Method.difference_only, Method.dense, Method.sparse, Method.difference_interp):
        for mag in (0, 1):
            for incl in (1, 0):
                for q in (0, 1):
                    out.append((m, mag, incl, q))
    return out


@pytest.mark.parametrize("m,mag,incl,q", _cfgs())
def test_stream_linear_random_configs(oracle, reference, m, mag, incl, q):
    rng = np.random.default_rng(int(m) * 100 + mag * 10 + incl * 3 + q)
    frames, ts = reference.panning_texture(53, 37, 4 if m == Method.difference_interp else 3,
                                           int(rng.integers(-3, 4)), int(rng.integers(-2, 3)), 20.0,
                                           int(rng.integers(1, 1000)))
    n = int(rng.integers(0, 7))
    cfg = make_config(m, n_interp=n, events_per_crossing=mag, include_endpoints=incl, flow_preset=q,
                      c_pos=int(rng.integers(1, 6)), c_neg=-int(rng.integers(1, 6)))
    so, sr = oracle.simulator(cfg), reference.simulator(cfg)
    for k in range(len(frames)):
        assert_same_events(so.push_frame(frames[k], ts[k]), sr.push_frame(frames[k], ts[k]), f"frame {k}")


def test_difference_interp_moving_disk(oracle, reference):
    frames, ts = reference.moving_disk(80, 64, 6, 7.0, 4.0, 60.0, 40, 230, 8)
    for n in (0, 1, 5):
        cfg = make_config(Method.difference_interp, n_interp=n, c_pos=10, c_neg=-10)
        so, sr = oracle.simulator(cfg), reference.simulator(cfg)
        for k in range(len(frames)):
            assert_same_events(so.push_frame(frames[k], ts[k]), sr.push_frame(frames[k], ts[k]), f"N={n} frame {k}")


@pytest.mark.parametrize("m", [Method.difference_only, Method.dense, Method.sparse])
@pytest.mark.parametrize("mag", [0, 1])
def test_stream_log_mode(oracle, reference, m, mag):
    frames, ts = reference.moving_disk(90, 70, 4, 8.0, 5.0, 60.0, 60, 200, 21)
    cfg = make_config(m, n_interp=4, contrast_mode=1, c_pos_log=0.1, c_neg_log=-0.12, events_per_crossing=mag)
    so, sr = oracle.simulator(cfg), reference.simulator(cfg)
    for k in range(len(frames)):
        assert_same_events(so.push_frame(frames[k], ts[k]), sr.push_frame(frames[k], ts[k]), f"frame {k}")


@pytest.mark.parametrize("seed", range(6))
def test_dense_flow_random_presets(oracle, reference, seed):
    rng = np.random.default_rng(seed)
    w, h = int(rng.integers(8, 120)), int(rng.integers(8, 90))
    a = reference.textured_frame(w, h, seed + 1)
    b = np.roll(a, (int(rng.integers(-3, 4)), int(rng.integers(-3, 4))), axis=(0, 1))
    lv, it, r = int(rng.integers(1, 6)), int(rng.integers(1, 5)), int(rng.integers(1, 7))
    o = oracle.dense_flow(a, b, lv, it, r)
    f = reference.dense_flow(a, b, lv, it, r)
    assert np.array_equal(o[0].view(np.uint32), f[0].view(np.uint32))
    assert np.array_equal(o[1].view(np.uint32), f[1].view(np.uint32))


def test_sparse_flow_full_grid(oracle, reference):
    frames, _ = reference.panning_texture(64, 64, 2, 2, 1, 20.0, 17)
    pts = np.array([[x, y] for y in range(64) for x in range(64)], np.int32)
    o = oracle.sparse_flow(frames[0], frames[1], pts)
    r = reference.sparse_flow(frames[0], frames[1], pts)
    assert np.array_equal(o[0].view(np.uint32), r[0].view(np.uint32))
    assert np.array_equal(o[1], r[1])


def test_baseline_generator_frames(oracle, reference):
    """The BASELINE c2 generator through both, a few frames at reduced size."""
    from paper_2209_04634_b200 import scenes
    frames, ts = scenes.generate("c2", n_frames=3, width=160, height=120)
    for mode in (0, 1):
        cfg = make_config(Method.dense, contrast_mode=mode)
        so, sr = oracle.simulator(cfg), reference.simulator(cfg)
        for k in range(3):
            assert_same_events(so.push_frame(frames[k], ts[k]), sr.push_frame(frames[k], ts[k]))
