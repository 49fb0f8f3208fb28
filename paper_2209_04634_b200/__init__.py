"""B200-native event-camera simulation hot path (arXiv 2209.04634, reference `evsim`).

Drop-in for the reference's ``Simulator::push_frame`` dense / sparse path:
hand-written sm_100a kernels behind the C-ABI of include/evsim_gpu.h, with a
host-side mirror of the reference API in :mod:`.simulator`.
"""
from .abi import EVENT_DTYPE, ContrastMode, EventsPerCrossing, FlowQuality, Method  # noqa: F401
from ._lib import EvsimError, InvalidArgument  # noqa: F401
from .simulator import (EventRateStats, accumulate, events_per_pixel_second, ingest_frames,  # noqa: F401
                        DenseFlowEstimator, EventStream, FlowField, FlowPreset, Frame,  # noqa: F401
                        PyramidalLucasKanade, PyramidalPatchFlow, SimulatorConfig, Simulator, SparseFlow,
                        SparseFlowEstimator, dense_events_with_flow, estimate_dense_flow, estimate_sparse_flow,
                        flow_preset, interpolate_frames, push_frames_batched, simulate_dense, simulate_difference,
                        simulate_sparse,
                        sparse_events_with_flow, DifferenceFrame, difference_frame, threshold_events)

__all__ = [
    "EventRateStats", "accumulate", "events_per_pixel_second", "ingest_frames",
    "EVENT_DTYPE", "ContrastMode", "EventsPerCrossing", "FlowQuality", "Method", "EvsimError", "InvalidArgument",
    "DenseFlowEstimator", "EventStream", "FlowField", "FlowPreset", "Frame", "PyramidalLucasKanade",
    "PyramidalPatchFlow", "SimulatorConfig", "Simulator", "SparseFlow", "SparseFlowEstimator",
    "dense_events_with_flow", "estimate_dense_flow", "estimate_sparse_flow", "flow_preset", "interpolate_frames",
    "push_frames_batched", "simulate_dense", "simulate_difference", "simulate_sparse", "sparse_events_with_flow",
    "DifferenceFrame", "difference_frame", "threshold_events",
]
