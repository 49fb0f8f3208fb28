"""GPU: the plug-in seam (Simulator(config, dense_flow, sparse_flow),
simulate.hpp:68-77) through the handle (evsim_gpu_push_frame_with_flow /
_with_tracks): the stream's state stays on the device, so log mode works
through the seam (round-1 gap: the stateless entry points are linear-only).
An estimator that returns the library's own flow must reproduce the built-in
simulator's stream bit for bit, in both modes; a constant-flow estimator must
match the stateless dense_events_with_flow frame by frame in linear mode."""
import numpy as np
import pytest

from helpers import assert_same_events, concat
from paper_2209_04634_b200 import (DenseFlowEstimator, FlowField, Frame, InvalidArgument, SimulatorConfig, Simulator,
                                   SparseFlowEstimator, dense_events_with_flow, estimate_dense_flow,
                                   estimate_sparse_flow, flow_preset, scenes)
from paper_2209_04634_b200.abi import ContrastMode, EventsPerCrossing, Method

pytestmark = pytest.mark.gpu


class OwnDense(DenseFlowEstimator):
    def __init__(self, preset):
        self.preset = preset

    def estimate(self, prev, curr):
        return estimate_dense_flow(prev, curr, self.preset)


class OwnSparse(SparseFlowEstimator):
    def __init__(self, preset):
        self.preset = preset

    def estimate(self, prev, curr, points):
        return estimate_sparse_flow(prev, curr, points, self.preset)


def _cfg(method, mode, mag=False, incl=True):
    c = SimulatorConfig.defaults(method)
    c.contrast_mode = ContrastMode.log if mode else ContrastMode.linear
    c.c_pos_log, c.c_neg_log = 0.15, -0.15
    c.events_per_crossing = EventsPerCrossing.magnitude if mag else EventsPerCrossing.single
    c.include_endpoints = incl
    return c


@pytest.mark.parametrize("method", [Method.dense, Method.sparse, Method.difference_only])
@pytest.mark.parametrize("mode,mag,incl", [(1, False, True), (0, False, True), (1, True, True), (1, False, False)])
def test_own_flow_through_the_seam_equals_builtin(method, mode, mag, incl):
    cname = "c3" if method == Method.sparse else "c2"
    frames, ts = scenes.generate(cname, n_frames=7, width=96, height=64)
    cfg = _cfg(method, mode, mag, incl)
    preset = flow_preset(cfg.flow_preset)
    builtin = Simulator(cfg)
    seam = Simulator(cfg, OwnDense(preset), OwnSparse(preset))
    for k in range(len(frames)):
        a = builtin.push_frame(Frame.from_array(frames[k], int(ts[k]))).events
        b = seam.push_frame(Frame.from_array(frames[k], int(ts[k]))).events
        assert_same_events(b, a, what=f"{method} mode={mode} mag={mag} incl={incl} frame {k}")


class ConstantFlow(DenseFlowEstimator):
    def estimate(self, prev, curr):
        return FlowField(prev.width, prev.height, np.full((prev.height, prev.width), 1.5, np.float32),
                         np.full((prev.height, prev.width), -0.5, np.float32))


def test_constant_flow_matches_stateless_linear():
    """test_simulate.cpp:308-339 over a stream: each push equals
    dense_events_with_flow of the same pair (linear mode is stateless)."""
    frames, ts = scenes.generate("c2", n_frames=5, width=40, height=30)
    cfg = _cfg(Method.dense, 0)
    cfg.n_interp = 3
    sim = Simulator(cfg, ConstantFlow(), OwnSparse(flow_preset(cfg.flow_preset)))
    prev = None
    for k in range(len(frames)):
        f = Frame.from_array(frames[k], int(ts[k]))
        got = sim.push_frame(f).events
        if prev is not None:
            exp = dense_events_with_flow(prev, f, ConstantFlow().estimate(prev, f), cfg).events
            assert_same_events(got, exp, what=f"frame {k}")
        prev = f


def test_custom_handle_rejects_builtin_pushes():
    from paper_2209_04634_b200 import _lib
    from paper_2209_04634_b200.abi import CEvents
    import ctypes
    frames, ts = scenes.generate("c2", n_frames=3, width=32, height=24)
    cfg = _cfg(Method.dense, 1)
    sim = Simulator(cfg, ConstantFlow(), OwnSparse(flow_preset(cfg.flow_preset)))
    sim.push_frame(Frame.from_array(frames[0], int(ts[0])))
    px = np.ascontiguousarray(frames[1])
    ev = CEvents()
    rc = sim._lib.evsim_gpu_push_frame(sim._h, px.ctypes.data, 32, 24, int(ts[1]), 0, ctypes.byref(ev))
    assert rc == 1 and b"reset() first" in sim._lib.evsim_gpu_last_error()
    sim.reset()
    rc = sim._lib.evsim_gpu_push_frame(sim._h, px.ctypes.data, 32, 24, int(ts[1]), 0, ctypes.byref(ev))
    assert rc == 0
