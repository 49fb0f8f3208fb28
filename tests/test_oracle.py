"""CPU: pin the C restatement (oracle/) against the reference's golden vectors.

* golden fixtures generated from the compiled reference (tests/golden/make_golden.py)
* the reference tests' known-answer cases (tests/test_core.cpp, test_simulate.cpp,
  acceptance.cpp), restated on the oracle
"""
import numpy as np
import pytest

from helpers import (stream_fixtures, assert_events_equal, golden_cfg, golden_names, load_golden, run_oracle_stream)
from paper_2209_04634_b200.abi import Method, make_config

STREAM_FIXTURES = stream_fixtures()


@pytest.mark.parametrize("name", STREAM_FIXTURES)
def test_oracle_matches_reference_golden(oracle, name):
    g = load_golden(name)
    evs = run_oracle_stream(oracle, golden_cfg(g), g["frames"], g["ts"])
    assert [len(e) for e in evs] == list(g["counts"])
    got = np.concatenate(evs)
    assert_events_equal(got, g["ev_x"], g["ev_y"], g["ev_t"], g["ev_p"], what=name)


@pytest.mark.parametrize("name", ["dense_lq_pan", "dense_hq_pan"])
def test_oracle_dense_flow_bit_exact(oracle, name):
    g = load_golden(name)
    lv, it, r = (3, 2, 4) if "lq" in name else (5, 16, 6)
    du, dv = oracle.dense_flow(g["frames"][0], g["frames"][1], lv, it, r)
    assert np.array_equal(du.view(np.uint32), g["flow_du"].view(np.uint32))
    assert np.array_equal(dv.view(np.uint32), g["flow_dv"].view(np.uint32))


def test_oracle_sparse_flow_bit_exact(oracle):
    g = load_golden("sparse_pan")
    disp, st = oracle.sparse_flow(g["frames"][0], g["frames"][1], g["sf_pts"], 3, 2, 4)
    assert np.array_equal(disp.view(np.uint32), g["sf_disp"].view(np.uint32))
    assert np.array_equal(st, g["sf_status"])


def test_oracle_interpolation_and_events_with_flow(oracle):
    g = load_golden("interp_random_flow")
    inter, its = oracle.interpolate_frames(g["a"], g["b"], 0, 1100, g["du"], g["dv"], 5)
    assert np.array_equal(inter, g["inter"])
    assert np.array_equal(its, g["inter_t"])
    ev = oracle.dense_events_with_flow(g["a"], g["b"], 0, 1100, g["du"], g["dv"], golden_cfg(g))
    assert_events_equal(ev, g["ev_x"], g["ev_y"], g["ev_t"], g["ev_p"])


# ---- known-answer tests of the reference suite -------------------------------

def test_kat_difference_100_to_103(oracle):
    # test_core.cpp:42-49 + :78-87: +3 with dense defaults -> one positive event
    a = np.full((4, 4), 100, np.uint8)
    b = a.copy()
    b[1, 2] = 103
    sim = oracle.simulator(make_config(Method.difference_only))
    sim.push_frame(a, 0)
    ev = sim.push_frame(b, 10)
    assert len(ev) == 1 and (ev["x"][0], ev["y"][0], ev["t"][0], ev["p"][0]) == (2, 1, 10, 1)


def test_kat_strict_thresholds(oracle):
    # acceptance.cpp:74-93: {-3..3} with C=+/-2 -> one event per polarity
    a = np.full((1, 7), 100, np.uint8)
    b = (100 + np.arange(-3, 4)).astype(np.uint8).reshape(1, 7)
    sim = oracle.simulator(make_config(Method.difference_only))
    sim.push_frame(a, 0)
    ev = sim.push_frame(b, 1000)
    assert sorted(zip(ev["x"].tolist(), ev["p"].tolist())) == [(0, -1), (6, 1)]


def test_kat_magnitude(oracle):
    # test_core.cpp:113-129: 7 -> 3 positive, -5 -> 2 negative, 3 -> 1, 2 -> 0
    a = np.full((1, 4), 100, np.uint8)
    b = (100 + np.array([7, -5, 3, 2])).astype(np.uint8).reshape(1, 4)
    sim = oracle.simulator(make_config(Method.difference_only, events_per_crossing=1))
    sim.push_frame(a, 0)
    ev = sim.push_frame(b, 7)
    assert int((ev["p"] > 0).sum()) == 4 and int((ev["p"] < 0).sum()) == 2


def test_kat_interpolation_timestamps_and_blend(oracle):
    # test_simulate.cpp:76-98: stamps 275/550/825; 40 -> 120 gives 60/80/100
    a = np.full((6, 6), 40, np.uint8)
    b = np.full((6, 6), 120, np.uint8)
    z = np.zeros((6, 6), np.float32)
    inter, ts = oracle.interpolate_frames(a, b, 0, 1100, z, z, 3)
    assert list(ts) == [275, 550, 825]
    inter, ts = oracle.interpolate_frames(a, b, 0, 1000, z, z, 3)
    assert inter[1, 3, 3] == 80 and inter[0, 0, 0] == 60 and inter[2, 0, 0] == 100


def test_kat_zero_flow_brute_force(oracle):
    # test_simulate.cpp:143-156 vs oracles.hpp:70-99 (zero_flow_dense_events)
    rng = np.random.default_rng(33)
    cfg = make_config(Method.dense, n_interp=3)
    for _ in range(10):
        a = rng.integers(0, 256, (8, 8), dtype=np.uint8)
        b = rng.integers(0, 256, (8, 8), dtype=np.uint8)
        z = np.zeros((8, 8), np.float32)
        ev = oracle.dense_events_with_flow(a, b, 0, 1000, z, z, cfg)
        exp = []
        for k in range(1, 5):
            t = (k * 1000 + 3) // 4
            for y in range(8):
                for x in range(8):
                    def blend(kk):
                        al = kk / 4
                        return int(np.floor((1.0 - al) * a[y, x] + al * b[y, x] + 0.5))
                    v = blend(k) - blend(k - 1)
                    if v > 2:
                        exp.append((x, y, t, 1))
                    elif v < -2:
                        exp.append((x, y, t, -1))
        got = list(zip(ev["x"].tolist(), ev["y"].tolist(), ev["t"].tolist(), ev["p"].tolist()))
        assert got == exp


def test_oracle_validation_messages(oracle):
    from oracle import OracleError
    with pytest.raises(OracleError, match="c_pos must be > 0"):
        oracle.simulator(make_config(Method.dense, c_pos=0))
    sim = oracle.simulator(make_config(Method.difference_only))
    sim.push_frame(np.zeros((8, 8), np.uint8), 100)
    with pytest.raises(OracleError, match="strictly increasing"):
        sim.push_frame(np.zeros((8, 8), np.uint8), 100)
    with pytest.raises(OracleError, match="dimensions changed"):
        sim.push_frame(np.zeros((9, 8), np.uint8), 200)
    sim.push_frame(np.zeros((8, 8), np.uint8), 200)  # still usable (test_simulate.cpp:66-74)


def test_log_lut_definition(oracle):
    lut = oracle.log_lut()
    exp = np.log(np.arange(256, dtype=np.float32) / np.float32(255.0) + np.float32(1e-3)).astype(np.float32)
    assert np.max(np.abs(lut - exp)) < 1e-6
