"""One-off randomized differential campaign on the GPU (beyond the committed
seeds of tests/test_gpu_random.py): random sizes / methods / modes / N /
thresholds / batch cuts / timestamp gaps against the C oracle, optionally with
library switches (e.g. EVSIM_CHAIN_QUAD=tile on tile-compatible widths).

    python tools/stress_random.py 2000 [tile]      # prints mismatching seeds, exits 1 on any
    EVSIM_STRESS_BASE=910000 python tools/stress_random.py 2000   # other seeds
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def frames_for(rng, n, w, h):
    kind = rng.integers(0, 3)
    if kind == 0:
        return rng.integers(0, 256, size=(n, h, w), dtype=np.uint8)
    base = rng.integers(0, 256, size=(h + 16, w + 16)).astype(np.float32)
    for _ in range(int(rng.integers(1, 4))):
        base = 0.25 * (np.roll(base, 1, 0) + np.roll(base, -1, 0) + np.roll(base, 1, 1) + np.roll(base, -1, 1))
    out = []
    dx, dy = rng.integers(-5, 6, size=2)
    for k in range(n):
        f = np.roll(base, (int(k * dy), int(k * dx)), axis=(0, 1))[:h, :w]
        if kind == 2:
            f = f * (1.0 + 0.05 * k)
        out.append(np.clip(f, 0, 255).astype(np.uint8))
    return np.stack(out)


def main():
    n_seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    tile = len(sys.argv) > 2 and sys.argv[2] == "tile"
    if tile:
        os.environ["EVSIM_CHAIN_QUAD"] = "tile"
    from helpers import concat
    from oracle import Oracle
    from paper_2209_04634_b200 import Simulator, SimulatorConfig
    from paper_2209_04634_b200.abi import Method, make_config
    oracle = Oracle()
    bad = []
    total_ev = 0
    base = int(os.environ.get("EVSIM_STRESS_BASE", "770000"))  # a new base = seeds no earlier campaign used
    for seed in range(n_seeds):
        rng = np.random.default_rng(base + seed + (10 ** 6 if tile else 0))
        if tile:
            os.environ["EVSIM_TILE_BLOCKS"] = str(int(rng.choice([3, 4])))
            w = int(rng.choice([128, 250, 256, 384, 512, 640]))
            h = int(rng.integers(1, 70))
            m = Method.dense
            N = int(rng.choice([1, 2, 3, 4, 5, 7, 8, 10, 16, 20, 32, 40]))
        else:
            w = int(rng.choice([1, 2, 7, 31, 32, 33, 64, 95, 130, 256, 346]))
            h = int(rng.choice([1, 3, 16, 17, 40, 71, 130]))
            m = Method(int(rng.integers(0, 4)))
            N = int(rng.choice([0, 1, 3, 5, 8, 10, 16, 33]))
        n = int(rng.integers(2, 8))
        mode = int(rng.integers(0, 2)) if m != Method.difference_interp else 0
        cfg = make_config(m, n_interp=N, contrast_mode=mode,
                          events_per_crossing=0 if tile else int(rng.integers(0, 2)),
                          include_endpoints=int(rng.integers(0, 2)), flow_preset=int(rng.integers(0, 2)),
                          c_pos=int(rng.integers(1, 12)), c_neg=-int(rng.integers(1, 12)),
                          selection_threshold=int(rng.integers(0, 6)),
                          c_pos_log=float(rng.uniform(0.03, 0.4)), c_neg_log=-float(rng.uniform(0.03, 0.4)))
        frames = frames_for(rng, n, w, h)
        ts = np.cumsum(rng.choice([1, 3, 17, 1000, 33333], size=n)).astype(np.int64)
        osim = oracle.simulator(cfg)
        exp = concat([osim.push_frame(frames[k], int(ts[k])) for k in range(n)])
        sim = Simulator(SimulatorConfig.from_c(cfg))
        cuts = sorted(set(int(c) for c in rng.integers(1, n, size=int(rng.integers(0, 3))))) + [n]
        got, a = [], 0
        for b in cuts:
            got.append(sim.push_frames(frames[a:b], ts[a:b]).events)
            a = b
        got = concat(got)
        ok = len(got) == len(exp) and all(np.array_equal(got[f], exp[f]) for f in ("x", "y", "t", "p"))
        total_ev += len(exp)
        if not ok:
            bad.append(seed)
            print(f"MISMATCH seed {seed}: {m.name} mode={mode} N={N} {w}x{h} n={n} got {len(got)} want {len(exp)}",
                  flush=True)
    print(f"{'tile' if tile else 'default'}: {n_seeds} seeds, {total_ev} events compared, {len(bad)} mismatches {bad[:20]}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
