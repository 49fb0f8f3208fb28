"""Generate tests/golden/*.npz from the compiled reference (oracle/_ref).

Run in the source container (needs /root/reference to build oracle/_ref):

    PYTHONPATH=. python tests/golden/make_golden.py

Every fixture stores its inputs and the reference outputs, so the tests on
the GPU box (where /root/reference does not exist) can pin both the oracle
and the CUDA path to the reference's own results.  Inputs come from the
reference's own scene generators (src/scenes.cpp) and from seeded uniform
noise (tests/helpers.hpp:26-31 style); log-mode fixtures run the reference's
flow / interpolation with the DESIGN.md §3 rule on top (oracle/ref_shim.cpp).
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from oracle import Reference  # noqa: E402
from paper_2209_04634_b200.abi import Method, make_config  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def ev_cols(ev):
    return dict(ev_x=ev["x"].copy(), ev_y=ev["y"].copy(), ev_t=ev["t"].copy(), ev_p=ev["p"].copy())


def run_stream(R, cfg, frames, ts):
    sim = R.simulator(cfg)
    xs, ys, tt, ps, counts = [], [], [], [], []
    for k in range(len(frames)):
        ev = sim.push_frame(frames[k], int(ts[k]))
        xs.append(ev["x"]), ys.append(ev["y"]), tt.append(ev["t"]), ps.append(ev["p"])
        counts.append(len(ev))
    return dict(ev_x=np.concatenate(xs), ev_y=np.concatenate(ys), ev_t=np.concatenate(tt),
                ev_p=np.concatenate(ps), counts=np.array(counts, np.int64))


def cfg_arrays(cfg):
    from paper_2209_04634_b200.abi import config_dict
    d = config_dict(cfg)
    return {f"cfg_{k}": np.array(v) for k, v in d.items()}


def main():
    R = Reference()
    out = {}
    rng = np.random.default_rng(2024)

    # 1. difference_only on random 8x8 pairs (acceptance.cpp:47-71 shape)
    fr = rng.integers(0, 256, size=(2, 8, 8), dtype=np.uint8)
    ts = np.array([0, 1000], np.int64)
    frames = rng.integers(0, 256, size=(51, 8, 8), dtype=np.uint8)
    ts = np.arange(51, dtype=np.int64) * 1000
    cfg = make_config(Method.difference_only)
    out["diff_random8"] = dict(frames=frames, ts=ts, **cfg_arrays(cfg), **run_stream(R, cfg, frames, ts))

    # 2. dense lq/hq on a panning texture (scenes.cpp:88-114), odd size
    frames, ts = R.panning_texture(97, 71, 4, 3, 1, 20.0, 99)
    for q, name in [(0, "dense_lq_pan"), (1, "dense_hq_pan")]:
        cfg = make_config(Method.dense, flow_preset=q)
        out[name] = dict(frames=frames, ts=ts, **cfg_arrays(cfg), **run_stream(R, cfg, frames, ts))
        lv, it, r = (3, 2, 4) if q == 0 else (5, 16, 6)
        du, dv = R.dense_flow(frames[0], frames[1], lv, it, r)
        out[name].update(flow_du=du, flow_dv=dv)

    # 3. dense variants: magnitude, no endpoints, N=3, collision timestamps (dt < K)
    frames, ts = R.panning_texture(64, 48, 3, 2, -1, 20.0, 5)
    cfg = make_config(Method.dense, n_interp=3, events_per_crossing=1)
    out["dense_mag"] = dict(frames=frames, ts=ts, **cfg_arrays(cfg), **run_stream(R, cfg, frames, ts))
    cfg = make_config(Method.dense, n_interp=4, include_endpoints=0)
    out["dense_noend"] = dict(frames=frames, ts=ts, **cfg_arrays(cfg), **run_stream(R, cfg, frames, ts))
    ts_c = np.array([0, 5, 9], np.int64)  # K = 11 links over dt = 5 -> equal stamps
    cfg = make_config(Method.dense, n_interp=10)
    out["dense_collide"] = dict(frames=frames, ts=ts_c, **cfg_arrays(cfg), **run_stream(R, cfg, frames, ts_c))
    cfg = make_config(Method.dense, n_interp=10, events_per_crossing=1)
    out["dense_collide_mag"] = dict(frames=frames, ts=ts_c, **cfg_arrays(cfg), **run_stream(R, cfg, frames, ts_c))

    # 4. sparse on the moving disk (scenes.cpp:116-145) and on a textured pan
    frames, ts = R.moving_disk(128, 96, 4, 6.0, 6.0, 100.0, 70, 235, 0)
    cfg = make_config(Method.sparse)
    out["sparse_disk"] = dict(frames=frames, ts=ts, **cfg_arrays(cfg), **run_stream(R, cfg, frames, ts))
    frames, ts = R.panning_texture(80, 60, 3, 2, 1, 20.0, 17)
    cfg = make_config(Method.sparse, n_interp=5, selection_threshold=3)
    out["sparse_pan"] = dict(frames=frames, ts=ts, **cfg_arrays(cfg), **run_stream(R, cfg, frames, ts))
    pts = np.array([[x, y] for y in range(0, 60, 3) for x in range(0, 80, 4)], np.int32)
    disp, st = R.sparse_flow(frames[0], frames[1], pts, 3, 2, 4)
    out["sparse_pan"].update(sf_pts=pts, sf_disp=disp, sf_status=st)

    # 5. interpolate_frames with a random flow field (simulate.cpp:91-121)
    a = R.textured_frame(40, 30, 5)
    b = R.textured_frame(40, 30, 6)
    du = rng.uniform(-6, 6, size=(30, 40)).astype(np.float32)
    dv = rng.uniform(-6, 6, size=(30, 40)).astype(np.float32)
    inter, its = R.interpolate_frames(a, b, 0, 1100, du, dv, 5)
    cfg = make_config(Method.dense, n_interp=5)
    ev = R.dense_events_with_flow(a, b, 0, 1100, du, dv, cfg)
    out["interp_random_flow"] = dict(a=a, b=b, du=du, dv=dv, inter=inter, inter_t=its, **cfg_arrays(cfg),
                                     **ev_cols(ev))

    # 6. log mode (reference stages + DESIGN.md §3 rule)
    frames, ts = R.panning_texture(72, 56, 4, 2, 1, 30.0, 11)
    for m, name in [(Method.difference_only, "log_diff"), (Method.dense, "log_dense"),
                    (Method.sparse, "log_sparse")]:
        cfg = make_config(m, contrast_mode=1, c_pos_log=0.15, c_neg_log=-0.15)
        out[name] = dict(frames=frames, ts=ts, **cfg_arrays(cfg), **run_stream(R, cfg, frames, ts))
    cfg = make_config(Method.dense, n_interp=6, contrast_mode=1, c_pos_log=0.05, c_neg_log=-0.07,
                      events_per_crossing=1)
    out["log_dense_mag"] = dict(frames=frames, ts=ts, **cfg_arrays(cfg), **run_stream(R, cfg, frames, ts))

    # 7. difference_interp (simulate.cpp:212-285, 334-341): sparse LK on the
    # magnitude of consecutive difference frames, signed splats, thresholded
    frames, ts = R.moving_disk(96, 72, 6, 6.0, 5.0, 100.0, 60, 220, 3)
    cfg = make_config(Method.difference_interp)
    out["diffinterp_disk"] = dict(frames=frames, ts=ts, **cfg_arrays(cfg), **run_stream(R, cfg, frames, ts))
    cfg = make_config(Method.difference_interp, n_interp=4, c_pos=6, c_neg=-6, events_per_crossing=1)
    out["diffinterp_disk_mag"] = dict(frames=frames, ts=ts, **cfg_arrays(cfg), **run_stream(R, cfg, frames, ts))
    frames, ts = R.panning_texture(70, 52, 5, 2, -1, 20.0, 23)
    cfg = make_config(Method.difference_interp, n_interp=6, c_pos=8, c_neg=-8, include_endpoints=0)
    out["diffinterp_pan_noend"] = dict(frames=frames, ts=ts, **cfg_arrays(cfg), **run_stream(R, cfg, frames, ts))

    # 8. data formats either side of the path (io.cpp, metrics.cpp)
    rgb = rng.integers(0, 256, size=(3, 23, 37, 3), dtype=np.uint8)
    gray = np.stack([R.luma(f).reshape(23, 37) for f in rgb])
    out["io_ingest"] = dict(rgb=rgb, gray=gray,
                            down=np.stack([R.resize_bilinear(g, 29, 17) for g in gray]),
                            up=np.stack([R.resize_bilinear(g, 50, 40) for g in gray]))
    frames, ts = R.moving_disk(64, 48, 4, 7.0, 5.0, 60.0, 40, 230, 9)
    cfg = make_config(Method.dense, n_interp=4)
    sim = R.simulator(cfg)
    evs = np.concatenate([sim.push_frame(frames[k], int(ts[k])) for k in range(len(frames))])
    m = R.events_per_pixel_second(evs, 64, 48, 0.05)
    t0, t1 = int(ts[1]), int(ts[3])
    out["metrics"] = dict(ev_x=evs["x"].copy(), ev_y=evs["y"].copy(), ev_t=evs["t"].copy(), ev_p=evs["p"].copy(),
                          rate=np.array(m[:3], np.float64), total=np.array(m[3], np.int64),
                          window=np.array([t0, t1], np.int64), classes=R.accumulate(evs, 64, 48, t0, t1))

    only = sys.argv[1] if len(sys.argv) > 1 else ""
    for name, d in out.items():
        if not name.startswith(only):
            continue
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
        print(name, {k: v.shape for k, v in d.items() if hasattr(v, "shape") and v.ndim > 0 and v.size > 1})


if __name__ == "__main__":
    main()
