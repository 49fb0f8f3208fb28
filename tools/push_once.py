"""Minimal driver for ncu: `pushes` device pushes of `frames` frames of a
BASELINE config (stream 0), after one untimed push (warm-up + allocation).

    ncu ... python tools/push_once.py c5 log 8 2
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2209_04634_b200 import Simulator, SimulatorConfig, scenes
    from paper_2209_04634_b200.abi import Method, make_config
    name, mode = sys.argv[1], sys.argv[2]
    F = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    pushes = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    c = scenes.CONFIGS[name]
    cp, cn = scenes.LINEAR_THRESHOLDS[c.method]
    cfg = make_config(Method[c.method], n_interp=c.n_interp, c_pos=cp, c_neg=cn,
                      contrast_mode=1 if mode == "log" else 0, c_pos_log=c.contrast, c_neg_log=-c.contrast)
    frames, ts = scenes.generate(c, n_frames=F * (pushes + 1) + 1)
    sim = Simulator(SimulatorConfig.from_c(cfg))
    d = torch.from_numpy(frames).cuda()
    P = c.width * c.height
    sim.push_frames_device(d.data_ptr(), 1, c.width, c.height, ts[:1])
    for j in range(pushes + 1):
        a = 1 + j * F
        ev = sim.push_frames_device(d.data_ptr() + a * P, F, c.width, c.height, ts[a:a + F])
    torch.cuda.synchronize()
    print("events of the last push:", int(ev.n_events))


if __name__ == "__main__":
    main()
