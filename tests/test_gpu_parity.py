"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden
vectors and the CPU oracle — bit-exact on every event (x, y, t, p), order and
count, and bit-exact on flow fields (north_star's 1e-3 px gate is implied).
"""
import numpy as np
import pytest

from helpers import (stream_fixtures, assert_events_equal, assert_same_events, golden_cfg, golden_names, load_golden,
                     run_oracle_stream)
from paper_2209_04634_b200 import (FlowField, FlowPreset, Frame, SimulatorConfig, Simulator, SparseFlow,
                                   dense_events_with_flow, estimate_dense_flow, estimate_sparse_flow,
                                   interpolate_frames, sparse_events_with_flow)
from paper_2209_04634_b200.abi import Method, make_config

pytestmark = pytest.mark.gpu

STREAM_FIXTURES = stream_fixtures()


def gpu_stream(cfg_c, frames, ts):
    sim = Simulator(SimulatorConfig.from_c(cfg_c))
    out = [sim.push_frame(Frame.from_array(frames[k], int(ts[k]))).events for k in range(len(frames))]
    sim.close()
    return out


@pytest.mark.parametrize("name", STREAM_FIXTURES)
def test_gpu_matches_reference_golden(name):
    g = load_golden(name)
    evs = gpu_stream(golden_cfg(g), g["frames"], g["ts"])
    assert [len(e) for e in evs] == list(g["counts"])
    assert_events_equal(np.concatenate(evs), g["ev_x"], g["ev_y"], g["ev_t"], g["ev_p"], what=name)


@pytest.mark.parametrize("name", ["dense_lq_pan", "dense_hq_pan"])
def test_gpu_dense_flow_bit_exact(name):
    g = load_golden(name)
    p = FlowPreset(3, 2, 4) if "lq" in name else FlowPreset(5, 16, 6)
    f = estimate_dense_flow(Frame.from_array(g["frames"][0], 0), Frame.from_array(g["frames"][1], 1), p)
    assert np.max(np.abs(f.du - g["flow_du"])) <= 1e-3  # north_star gate
    assert np.array_equal(f.du.view(np.uint32), g["flow_du"].view(np.uint32))
    assert np.array_equal(f.dv.view(np.uint32), g["flow_dv"].view(np.uint32))


def test_gpu_sparse_flow_bit_exact():
    g = load_golden("sparse_pan")
    f = estimate_sparse_flow(Frame.from_array(g["frames"][0], 0), Frame.from_array(g["frames"][1], 1),
                             g["sf_pts"], FlowPreset(3, 2, 4))
    assert np.array_equal(f.displacements.view(np.uint32), g["sf_disp"].view(np.uint32))
    assert np.array_equal(f.status, g["sf_status"])


def test_gpu_interpolation_and_events_with_flow():
    g = load_golden("interp_random_flow")
    a, b = Frame.from_array(g["a"], 0), Frame.from_array(g["b"], 1100)
    flow = FlowField(40, 30, g["du"], g["dv"])
    inter = interpolate_frames(a, b, flow, 5)
    assert np.array_equal(np.stack([f.pixels for f in inter]), g["inter"])
    assert [f.timestamp for f in inter] == list(g["inter_t"])
    ev = dense_events_with_flow(a, b, flow, SimulatorConfig.from_c(golden_cfg(g)))
    assert_events_equal(ev.events, g["ev_x"], g["ev_y"], g["ev_t"], g["ev_p"])


# ---- randomised differential tests against the oracle -------------------------

SIZES = [(1, 1), (3, 2), (33, 17), (64, 1), (1, 40), (97, 71), (130, 45)]


@pytest.mark.parametrize("w,h", SIZES)
@pytest.mark.parametrize("m", [Method.difference_only, Method.dense, Method.sparse])
@pytest.mark.parametrize("mode", [0, 1])
def test_gpu_vs_oracle_sizes(oracle, w, h, m, mode):
    rng = np.random.default_rng(w * 1000 + h + int(m) * 7 + mode)
    base = rng.integers(0, 256, (h + 8, w + 8), dtype=np.uint8)
    frames = np.stack([np.roll(base, (k, 2 * k), axis=(0, 1))[:h, :w] for k in range(4)])
    frames[2] = np.clip(frames[2].astype(int) + rng.integers(-20, 20, (h, w)), 0, 255).astype(np.uint8)
    ts = np.array([0, 33333, 66667, 100000], np.int64)
    cfg = make_config(m, n_interp=4 if m != Method.difference_only else 0, contrast_mode=mode,
                      c_pos_log=0.1, c_neg_log=-0.1, selection_threshold=5)
    exp = run_oracle_stream(oracle, cfg, frames, ts)
    got = gpu_stream(cfg, frames, ts)
    for k in range(4):
        assert_same_events(got[k], exp[k], f"frame {k}")


def _variants():
    v = []
    for m in (Method.dense, Method.sparse):
        for mag in (0, 1):
            for incl in (1, 0):
                for n in (0, 1, 3, 7):
                    for mode in (0, 1):
                        v.append((m, mag, incl, n, mode))
    return v


@pytest.mark.parametrize("m,mag,incl,n,mode", _variants())
def test_gpu_vs_oracle_config_matrix(oracle, m, mag, incl, n, mode):
    from paper_2209_04634_b200 import scenes
    frames, ts = scenes.generate("c2", n_frames=3, width=96, height=72)
    cfg = make_config(m, n_interp=n, events_per_crossing=mag, include_endpoints=incl, contrast_mode=mode,
                      c_pos_log=0.08, c_neg_log=-0.1)
    exp = run_oracle_stream(oracle, cfg, frames, ts)
    got = gpu_stream(cfg, frames, ts)
    for k in range(3):
        assert_same_events(got[k], exp[k], f"frame {k}")


@pytest.mark.parametrize("preset", [(1, 1, 1), (2, 3, 2), (4, 5, 3), (5, 16, 6), (6, 2, 5)])
def test_gpu_dense_flow_vs_oracle_presets(oracle, preset):
    from paper_2209_04634_b200 import scenes
    frames, _ = scenes.generate("c2", n_frames=2, width=150, height=101)
    lv, it, r = preset
    du, dv = oracle.dense_flow(frames[0], frames[1], lv, it, r)
    f = estimate_dense_flow(Frame.from_array(frames[0], 0), Frame.from_array(frames[1], 1), FlowPreset(lv, it, r))
    assert np.array_equal(f.du.view(np.uint32), du.view(np.uint32))
    assert np.array_equal(f.dv.view(np.uint32), dv.view(np.uint32))


def test_gpu_sparse_flow_vs_oracle_hq(oracle):
    from paper_2209_04634_b200 import scenes
    frames, _ = scenes.generate("c3", n_frames=2, width=160, height=120)
    pts = np.array([[x, y] for y in range(0, 120, 2) for x in range(0, 160, 3)], np.int32)
    for lv, it, r in ((3, 2, 4), (5, 16, 6)):
        disp, st = oracle.sparse_flow(frames[0], frames[1], pts, lv, it, r)
        f = estimate_sparse_flow(Frame.from_array(frames[0], 0), Frame.from_array(frames[1], 1), pts,
                                 FlowPreset(lv, it, r))
        assert np.array_equal(f.displacements.view(np.uint32), disp.view(np.uint32))
        assert np.array_equal(f.status, st)


def test_gpu_sparse_events_with_supplied_flow(oracle):
    g = load_golden("sparse_pan")
    a, b = Frame.from_array(g["frames"][0], int(g["ts"][0])), Frame.from_array(g["frames"][1], int(g["ts"][1]))
    rng = np.random.default_rng(3)
    pts = g["sf_pts"]
    disp = rng.uniform(-5, 5, size=pts.shape).astype(np.float32)
    st = (rng.uniform(size=len(pts)) < 0.8).astype(np.uint8)
    cfg = make_config(Method.sparse, n_interp=6)
    exp = oracle.sparse_events_with_flow(g["frames"][0], g["frames"][1], a.timestamp, b.timestamp, pts, disp, st, cfg)
    got = sparse_events_with_flow(a, b, SparseFlow(pts, disp, st), SimulatorConfig.from_c(cfg))
    assert_same_events(got.events, exp)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
@pytest.mark.parametrize("mode", [0, 1])
def test_gpu_vs_oracle_baseline_configs_reduced(oracle, name, mode):
    """BASELINE configs with their own N / C / method, at 1/4 linear size."""
    from paper_2209_04634_b200 import scenes
    c = scenes.CONFIGS[name]
    frames, ts = scenes.generate(name, n_frames=3, width=c.width // 4, height=c.height // 4)
    m = Method[c.method]
    cp, cn = scenes.LINEAR_THRESHOLDS[c.method]
    cfg = make_config(m, n_interp=c.n_interp, c_pos=cp, c_neg=cn, contrast_mode=mode, c_pos_log=c.contrast,
                      c_neg_log=-c.contrast)
    exp = run_oracle_stream(oracle, cfg, frames, ts)
    got = gpu_stream(cfg, frames, ts)
    for k in range(3):
        assert_same_events(got[k], exp[k], f"{name} frame {k}")
