"""Per-frame event counts + checksums of whole BASELINE sequences, from the
compiled reference (oracle/_ref).  TEST INFRASTRUCTURE.

    PYTHONPATH=. python tests/golden/make_sequences.py [c2:log c5:linear c2:log:hq ...]

For every (config, mode) the sequence of scenes.generate(config) (stream 0) is
pushed frame by frame through the reference's own Simulator::push_frame
(src/simulate.cpp:306-347; log mode = the reference's flow + interpolation
with the DESIGN.md §3 rule, oracle/ref_shim.cpp), and each frame's events are
reduced to (count, seqhash.frame_hash_np).  Results go to
tests/golden/sequences.json, which the -m gpu sequence tests and bench.py's
parity check compare against — the GPU box has no /root/reference.
"""
from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "sequences.json")

# (config, stream) of each pinned sequence; c4 pins its stream 0
JOBS = [(c, m) for c in ("c1", "c2", "c3", "c5", "c4") for m in ("log", "linear")]
# the high-quality flow preset (types.hpp:93) on c2: keys "c2:<mode>:hq"
JOBS += [("c2", "log", "hq"), ("c2", "linear", "hq")]


def sequence_config(name: str, mode: str, preset: str = "lq"):
    from paper_2209_04634_b200 import scenes
    from paper_2209_04634_b200.abi import Method, make_config
    c = scenes.CONFIGS[name]
    cp, cn = scenes.LINEAR_THRESHOLDS[c.method]
    return c, make_config(Method[c.method], n_interp=c.n_interp, c_pos=cp, c_neg=cn,
                          contrast_mode=1 if mode == "log" else 0, c_pos_log=c.contrast, c_neg_log=-c.contrast,
                          flow_preset=1 if preset == "hq" else 0)


def seq_key(name: str, mode: str, preset: str = "lq") -> str:
    return f"{name}:{mode}" + ("" if preset == "lq" else f":{preset}")


def run(job):
    name, mode, preset = (tuple(job) + ("lq",))[:3]
    import numpy as np

    from oracle import Reference
    from paper_2209_04634_b200 import scenes
    from paper_2209_04634_b200.seqhash import frame_hash_np
    c, cfg = sequence_config(name, mode, preset)
    frames, ts = scenes.generate(c, stream=0)
    sim = Reference().simulator(cfg)
    counts, hashes = [], []
    t0 = time.time()
    for k in range(len(frames)):
        ev = sim.push_frame(frames[k], int(ts[k]))
        counts.append(int(len(ev)))
        hashes.append(f"{frame_hash_np(ev['x'], ev['y'], ev['t'], ev['p'], int(ts[k - 1]) if k else 0):016x}")
        del ev
    sim.close()
    fr_bytes = np.ascontiguousarray(frames).tobytes()
    import hashlib
    rec = {"config": name, "mode": mode, "preset": preset, "stream": 0, "n_frames": len(frames), "width": c.width,
           "height": c.height, "n_interp": c.n_interp, "method": c.method,
           "frames_sha256": hashlib.sha256(fr_bytes).hexdigest(),
           "timestamps": [int(t) for t in ts], "counts": counts, "hashes": hashes,
           "ref_seconds": round(time.time() - t0, 1)}
    path = os.path.join(ROOT, "tests", "golden", f".seq_{name}_{mode}_{preset}.json")
    json.dump(rec, open(path, "w"))
    print(f"{name} {mode} {preset}: {sum(counts)} events, {rec['ref_seconds']} s", flush=True)
    return path


def main():
    jobs = JOBS
    if len(sys.argv) > 1:
        jobs = [tuple(a.split(":")) for a in sys.argv[1:]]
    with mp.get_context("spawn").Pool(min(len(jobs), os.cpu_count() or 1)) as pool:
        paths = pool.map(run, jobs, chunksize=1)
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for p in paths:
        rec = json.load(open(p))
        data[seq_key(rec["config"], rec["mode"], rec.get("preset", "lq"))] = rec
        os.remove(p)
    json.dump(data, open(OUT, "w"), indent=0, sort_keys=True)
    print(OUT)


if __name__ == "__main__":
    main()
