"""GPU: evsim_gpu_push_frames_batched — several independent camera streams in
one call (c4-style) — gives every stream exactly the events of
its own frame-by-frame reference Simulator, and rejects the whole call (no
stream touched) when one batch is invalid."""
import numpy as np
import pytest

from helpers import assert_same_events, concat, run_oracle_stream
from paper_2209_04634_b200 import InvalidArgument, SimulatorConfig, Simulator, push_frames_batched, scenes
from paper_2209_04634_b200.abi import Method, make_config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,mode", [(Method.dense, 1), (Method.dense, 0), (Method.sparse, 1),
                                    (Method.difference_only, 0)])
def test_batched_streams_match_oracle(oracle, m, mode):
    n_streams, F = 5, 7
    seqs = [scenes.generate("c4", n_frames=F, width=72, height=48, stream=s) for s in range(n_streams)]
    cfg = make_config(m, n_interp=4 if m != Method.difference_only else 0, contrast_mode=mode,
                      c_pos_log=0.1, c_neg_log=-0.1, selection_threshold=4)
    exp = [concat(run_oracle_stream(oracle, cfg, f, t)) for f, t in seqs]
    sims = [Simulator(SimulatorConfig.from_c(cfg)) for _ in range(n_streams)]
    got = [[] for _ in range(n_streams)]
    for a, b in ((0, 3), (3, 4), (4, 7)):  # uneven batches, warm-up inside the first
        outs = push_frames_batched(sims, [f[a:b] for f, _ in seqs], [t[a:b] for _, t in seqs])
        for i, o in enumerate(outs):
            got[i].append(o.events)
    for i in range(n_streams):
        assert_same_events(concat(got[i]), exp[i], what=f"stream {i}")


def test_batched_rejects_atomically(oracle):
    seqs = [scenes.generate("c4", n_frames=4, width=40, height=32, stream=s) for s in range(3)]
    cfg = make_config(Method.dense, n_interp=3)
    sims = [Simulator(SimulatorConfig.from_c(cfg)) for _ in range(3)]
    bad = [t.copy() for _, t in seqs]
    bad[2][1] = bad[2][0]
    with pytest.raises(InvalidArgument, match="strictly increasing"):
        push_frames_batched(sims, [f for f, _ in seqs], bad)
    with pytest.raises(InvalidArgument, match="twice"):
        push_frames_batched([sims[0], sims[0]], [seqs[0][0], seqs[0][0]], [seqs[0][1], seqs[0][1]])
    outs = push_frames_batched(sims, [f for f, _ in seqs], [t for _, t in seqs])
    for (f, t), o in zip(seqs, outs):
        assert_same_events(o.events, concat(run_oracle_stream(oracle, cfg, f, t)))
    assert push_frames_batched([], [], []) == []


@pytest.mark.parametrize("mode", [1, 0])
def test_batched_streams_pipelined_dense(oracle, mode):
    """Several handles pushing >= 16 pairs each: every handle's flow runs in
    sub-batches on its own flow stream, all handles at once."""
    n_streams, F = 3, 21
    seqs = [scenes.generate("c4", n_frames=F, width=72, height=48, stream=s) for s in range(n_streams)]
    cfg = make_config(Method.dense, n_interp=4, contrast_mode=mode, c_pos_log=0.1, c_neg_log=-0.1)
    exp = [concat(run_oracle_stream(oracle, cfg, f, t)) for f, t in seqs]
    sims = [Simulator(SimulatorConfig.from_c(cfg)) for _ in range(n_streams)]
    got = [[] for _ in range(n_streams)]
    for a, b in ((0, 1), (1, F)):
        outs = push_frames_batched(sims, [f[a:b] for f, _ in seqs], [t[a:b] for _, t in seqs])
        for i, o in enumerate(outs):
            got[i].append(o.events)
    for i in range(n_streams):
        assert_same_events(concat(got[i]), exp[i], what=f"stream {i}")
