"""GPU: randomised differential test of the whole push path against the
oracle — random frame sizes (including 1-pixel rows / columns and widths that
are not multiples of 32), methods, contrast modes, thresholds, N, endpoints,
magnitude, flow presets, batch splits and timestamp spacings (including dt < K,
where sub-interval timestamps collide)."""
import numpy as np
import pytest

from helpers import assert_same_events, concat, run_oracle_stream
from paper_2209_04634_b200 import SimulatorConfig, Simulator
from paper_2209_04634_b200.abi import Method, make_config

pytestmark = pytest.mark.gpu


def _frames(rng, n, w, h):
    kind = rng.integers(0, 3)
    if kind == 0:  # noise
        return rng.integers(0, 256, size=(n, h, w), dtype=np.uint8)
    base = rng.integers(0, 256, size=(h + 8, w + 8)).astype(np.float32)
    for _ in range(2):  # blur so the flow has something to track
        base = 0.25 * (np.roll(base, 1, 0) + np.roll(base, -1, 0) + np.roll(base, 1, 1) + np.roll(base, -1, 1))
    out = []
    dx, dy = rng.integers(-2, 3, size=2)
    for k in range(n):
        f = np.roll(base, (int(k * dy), int(k * dx)), axis=(0, 1))[:h, :w]
        if kind == 2:
            f = f * (1.0 + 0.05 * k)
        out.append(np.clip(f, 0, 255).astype(np.uint8))
    return np.stack(out)


@pytest.mark.parametrize("seed", range(96))
def test_random_streams(oracle, seed):
    rng = np.random.default_rng(1000 + seed)
    w = int(rng.choice([1, 2, 7, 31, 32, 33, 64, 95, 130]))
    h = int(rng.choice([1, 3, 16, 17, 40, 71]))
    n = int(rng.integers(2, 7))
    m = Method(int(rng.integers(0, 4)))
    mode = int(rng.integers(0, 2)) if m != Method.difference_interp else 0
    N = int(rng.choice([0, 1, 3, 5, 10, 33]))
    cfg = make_config(m, n_interp=N, contrast_mode=mode, events_per_crossing=int(rng.integers(0, 2)),
                      include_endpoints=int(rng.integers(0, 2)), flow_preset=int(rng.integers(0, 2)),
                      c_pos=int(rng.integers(1, 12)), c_neg=-int(rng.integers(1, 12)),
                      selection_threshold=int(rng.integers(0, 6)),
                      c_pos_log=float(rng.uniform(0.03, 0.4)), c_neg_log=-float(rng.uniform(0.03, 0.4)))
    frames = _frames(rng, n, w, h)
    gaps = rng.choice([1, 3, 17, 1000, 33333], size=n)
    ts = np.cumsum(gaps).astype(np.int64)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    cuts = sorted(set(int(c) for c in rng.integers(1, n, size=int(rng.integers(0, 3))))) + [n]
    got, a = [], 0
    for b in cuts:
        got.append(sim.push_frames(frames[a:b], ts[a:b]).events)
        a = b
    assert_same_events(concat(got), exp, what=f"seed {seed}: {m.name} mode={mode} N={N} {w}x{h} n={n}")


@pytest.mark.parametrize("seed", range(12))
def test_dense_gather_bias_wrap_form(oracle, seed, monkeypatch):
    """The dense chain's gather index with a non-zero Y magic (the form used
    when qshift + P would exceed 2^32; forced here on small frames)."""
    monkeypatch.setenv("EVSIM_TEST_MAGIC_Y", "1")
    rng = np.random.default_rng(5000 + seed)
    w = int(rng.choice([600, 640, 641, 700, 1000]))  # m_y < 2^23 needs w > ~512
    h = int(rng.choice([3, 17, 40]))
    n = int(rng.integers(2, 5))
    mode = int(rng.integers(0, 2))
    N = int(rng.choice([1, 5, 10]))
    cfg = make_config(Method.dense, n_interp=N, contrast_mode=mode, include_endpoints=int(rng.integers(0, 2)),
                      c_pos_log=0.1, c_neg_log=-0.1)
    frames = _frames(rng, n, w, h)
    ts = np.cumsum(rng.choice([1, 1000, 33333], size=n)).astype(np.int64)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    sim = Simulator(SimulatorConfig.from_c(cfg))
    got = sim.push_frames(frames, ts).events
    assert_same_events(got, exp, what=f"seed {seed}: dense mode={mode} N={N} {w}x{h} n={n} (magic_y form)")
