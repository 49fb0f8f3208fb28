"""GPU: S difference_only streams stacked into one simulator
(parallel.stack_streams / split_stacked, the batched c1 workload) give every
stream exactly the events of its own reference Simulator (oracle), and the
streaming difference_only chain (chain_diff_kernel) equals the oracle on long
pushes in both modes, magnitude excluded (it keeps the generic chain)."""
import numpy as np
import pytest

from helpers import assert_same_events, concat, run_oracle_stream
from paper_2209_04634_b200 import Frame, SimulatorConfig, Simulator, scenes
from paper_2209_04634_b200.abi import Method, make_config, unpack_events
from paper_2209_04634_b200.parallel import split_stacked, stack_streams



def _cfg(mode):
    return make_config(Method.difference_only, contrast_mode=mode, c_pos_log=0.2, c_neg_log=-0.2)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("S,w,h,F", [(4, 45, 17, 9), (7, 96, 33, 40), (64, 346, 26, 12)])
def test_stacked_streams_equal_per_stream_oracle(oracle, mode, S, w, h, F):
    cfg = _cfg(mode)
    seqs = [scenes.generate("c1", n_frames=F, width=w, height=h, stream=s) for s in range(S)]
    ts = seqs[0][1]
    stacked = stack_streams([f for f, _ in seqs])
    sim = Simulator(SimulatorConfig.from_c(cfg))
    parts = [[] for _ in range(S)]
    for a, b in ((0, 1), (1, F // 2), (F // 2, F)):  # warm-up push, then two batches
        packed, seg_t, seg_off = sim.push_frames_streamed(stacked[a:b], ts[a:b])
        for s, (rec, st, so) in enumerate(split_stacked(packed, seg_t, seg_off, S, h)):
            parts[s].append(unpack_events(rec, st, so))
    for s in range(S):
        exp = concat(run_oracle_stream(oracle, cfg, seqs[s][0], ts))
        assert_same_events(concat(parts[s]), exp, what=f"stream {s} of {S}")


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_streaming_difference_chain_long_push(oracle, mode):
    """One push of 200 frames (chain_diff_kernel: prefetched pairs, staged masks
    flushed every 32 links) and frame-by-frame pushes equal the oracle."""
    cfg = _cfg(mode)
    frames, ts = scenes.generate("c1", n_frames=201, width=70, height=23)
    exp = run_oracle_stream(oracle, cfg, frames, ts)
    sim = Simulator(SimulatorConfig.from_c(cfg))
    got = sim.push_frames(frames[:1], ts[:1]).events
    assert len(got) == 0
    got = sim.push_frames(frames[1:], ts[1:]).events
    assert_same_events(got, concat(exp[1:]), what="one push")
    sim.reset()
    for k in range(12):
        ev = sim.push_frame(Frame.from_array(frames[k], int(ts[k]))).events
        assert_same_events(ev, exp[k], what=f"frame {k}")


@pytest.mark.parametrize("mode", [0, 1])
def test_stacking_is_exact_on_the_oracle(oracle, mode):
    """CPU: the C oracle over the stacked frames, split per stream, equals the
    oracle over each stream — the exactness claim of parallel.stack_streams
    for difference_only, independent of the GPU."""
    S, w, h, F = 5, 37, 11, 7
    cfg = _cfg(mode)
    seqs = [scenes.generate("c1", n_frames=F, width=w, height=h, stream=s) for s in range(S)]
    ts = seqs[0][1]
    stacked = stack_streams([f for f, _ in seqs])
    ev = concat(run_oracle_stream(oracle, cfg, stacked, ts))
    # oracle records -> packed form + segment table
    packed = (ev["x"].astype(np.uint32) | (ev["y"].astype(np.uint32) << 16) |
              ((ev["p"] < 0).astype(np.uint32) << 31))
    t = ev["t"]
    starts = np.concatenate([[0], np.nonzero(np.diff(t))[0] + 1]) if len(t) else np.zeros(0, int)
    seg_t = t[starts] if len(t) else np.zeros(0, np.int64)
    seg_off = np.concatenate([starts, [len(t)]]).astype(np.int64)
    for s, (rec, st, so) in enumerate(split_stacked(packed, seg_t, seg_off, S, h)):
        exp = concat(run_oracle_stream(oracle, cfg, seqs[s][0], ts))
        assert_same_events(unpack_events(rec, st, so), exp, what=f"stream {s}")
