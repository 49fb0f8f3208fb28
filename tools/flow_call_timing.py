"""Wall-clock per call of the stateless estimate_dense_flow (the reference's
test_flow.cpp:68-78 comparison), in the test's order, then repeated."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_04634_b200 import Frame, FlowQuality, estimate_dense_flow, flow_preset  # noqa: E402

rng = np.random.default_rng(1)
a = Frame.from_array(rng.integers(0, 256, (48, 64), dtype=np.uint8), 0)
b = Frame.from_array(rng.integers(0, 256, (48, 64), dtype=np.uint8), 1000)
for q in (FlowQuality.low_quality, FlowQuality.high_quality):
    estimate_dense_flow(a, b, flow_preset(q))
a = Frame.from_array(rng.integers(0, 256, (480, 640), dtype=np.uint8), 0)
b = Frame.from_array(rng.integers(0, 256, (480, 640), dtype=np.uint8), 1000)
for rep in range(4):
    out = []
    for q in (FlowQuality.low_quality, FlowQuality.high_quality):
        t0 = time.perf_counter()
        estimate_dense_flow(a, b, flow_preset(q))
        out.append(round(1e3 * (time.perf_counter() - t0), 3))
    print("rep", rep, "lq_ms", out[0], "hq_ms", out[1])
