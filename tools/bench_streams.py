"""Batched multi-stream throughput on one GPU (BASELINE config c4: independent
1920x1080 camera streams, dense N=16): S simulators, one CUDA stream each,
pushed together through evsim_gpu_push_frames_batched.

    python tools/bench_streams.py --streams 32 --frames 32

One JSON line.  `value`: device-resident frames (all streams' frames in HBM
before timing), host wall clock around `steps` whole-sequence passes with a
device synchronise on both sides (the batched call returns after every
stream's push completed).  `e2e`: the same frames through the public streamed
call (evsim_gpu_push_frames_streamed), one host thread per stream handle, with
the H2D of the frames and the packed events' download inside the timed region.
The per-stream sequence is shortened to --frames (default 32 of the config's
120) to bound host-side generation time; the frames are generated in a
process pool.
"""
import argparse
import ctypes
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _gen(args):
    name, n, s = args
    from paper_2209_04634_b200 import scenes
    return scenes.generate(name, n_frames=n, stream=s)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--streams", type=int, default=32)
    ap.add_argument("--frames", type=int, default=32)
    ap.add_argument("--mode", default="log", choices=["log", "linear"])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    a = ap.parse_args()

    import torch
    from paper_2209_04634_b200 import SimulatorConfig, Simulator, scenes
    from paper_2209_04634_b200 import _lib
    from paper_2209_04634_b200.abi import CEvents, Method, make_config

    c = scenes.CONFIGS[a.config]
    S, n = a.streams, a.frames
    with ProcessPoolExecutor(min(S, os.cpu_count() or 1)) as ex:
        data = list(ex.map(_gen, [(c.name, n, s) for s in range(S)]))
    frames = np.stack([d[0] for d in data])  # (S, n, H, W)
    ts = [d[1] for d in data]
    cp, cn = scenes.LINEAR_THRESHOLDS[c.method]
    cfg = make_config(Method[c.method], n_interp=c.n_interp, c_pos=cp, c_neg=cn,
                      contrast_mode=1 if a.mode == "log" else 0, c_pos_log=c.contrast, c_neg_log=-c.contrast)
    sims = [Simulator(SimulatorConfig.from_c(cfg)) for _ in range(S)]
    W, H = c.width, c.height
    P = W * H
    d_frames = torch.from_numpy(frames).cuda()
    mb = sims[0].max_batch(W, H)
    batch = max(1, min(a.batch or mb, mb, n))
    lib = sims[0]._lib
    hs = (ctypes.c_void_p * S)(*[s._h.value for s in sims])
    outs = (CEvents * S)()

    per_stream = [0] * S

    def device_step():
        for s in sims:
            s.reset()
        ev = 0
        for i in range(S):
            per_stream[i] = 0
        for b in range(0, n, batch):
            nb = min(batch, n - b)
            px = (ctypes.c_void_p * S)(*[d_frames[i].data_ptr() + b * P for i in range(S)])
            tsl = [np.ascontiguousarray(ts[i][b:b + nb]) for i in range(S)]
            tp = (ctypes.c_void_p * S)(*[t.ctypes.data for t in tsl])
            _lib.check(lib.evsim_gpu_push_frames_batched(hs, S, px, nb, W, H, tp, 1, outs))
            for i, o in enumerate(outs):
                per_stream[i] += int(o.n_events)
                ev += int(o.n_events)
        return ev

    for _ in range(max(a.warmup, 1)):
        ev_total = device_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        device_step()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    value = S * n * a.steps / dt

    e2e = None
    caps = [int(e * 1.05) + 4096 for e in per_stream]
    pinned = S * n * P + 4 * sum(caps)
    if not a.no_e2e and pinned > (12 << 30):
        e2e = {"skipped": f"{pinned / 2**30:.1f} GiB of pinned host buffers needed"}
    elif not a.no_e2e:
        # every stream through the public streamed call (pinned host frames
        # in, packed host events out), one host thread per stream handle
        from concurrent.futures import ThreadPoolExecutor
        h_frames = torch.from_numpy(frames).pin_memory()
        h_ev = [torch.empty(cap, dtype=torch.int32).pin_memory() for cap in caps]

        def run_stream(i):
            sims[i].reset()
            d2h = 0
            for b in range(0, n, batch):
                nb = min(batch, n - b)
                r = sims[i].push_frames_streamed_ptr(h_frames[i].data_ptr() + b * P, nb, W, H, ts[i][b:b + nb],
                                                     h_ev[i].data_ptr(), caps[i])
                d2h += 4 * int(r.n_events) + 16 * (int(r.n_segments) + 1)
            return d2h

        with ThreadPoolExecutor(S) as ex:
            list(ex.map(run_stream, range(S)))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(a.steps):
                d2h = sum(ex.map(run_stream, range(S)))
            torch.cuda.synchronize()
            e2e_dt = time.perf_counter() - t0
        e2e = {"value": round(S * n * a.steps / e2e_dt, 3), "unit": "frames/s", "h2d_bytes_per_step": S * n * P,
               "d2h_bytes_per_step": d2h,
               "api": "evsim_gpu_push_frames_streamed per stream handle, one host thread each (pinned host "
                      "frames in, packed host events out)"}

    print(json.dumps({
        "metric": "simulated input frames/sec, all streams", "value": round(value, 3), "unit": "frames/s",
        "events_per_s": round(ev_total * a.steps / dt, 1), "n_gpus": 1, "steps": a.steps, "warmup": a.warmup,
        "timing": "host wall clock, device synchronised both sides; device-resident frames",
        "config": {"workload": f"{c.name}: {S} streams x {n} frames {W}x{H} u8, {c.method} N={c.n_interp}, "
                               f"{a.mode}", "streams": S, "frames_per_stream": n, "frames_per_push": batch},
        "e2e": e2e}), flush=True)
    for s in sims:
        s.close()


if __name__ == "__main__":
    main()
