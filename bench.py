"""Benchmark of the B200 event-simulation hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c5] [--mode log|linear] [--split auto|streams|bands]

Workload (default): BASELINE.json's largest single-GPU configuration, the one
its metric ("per B200 (1/2/4/8 GPU)") is quoted on — c5: one 3840x2160 u8
stream of 60 frames (seeded synthetic sequence, paper_2209_04634_b200/
scenes.py: unblurred U[0,255] texture, 16 px/frame pan, 20 % flicker), dense
pyramidal LK (lq preset), N = 32 interpolated frames, log intensity C = 0.1.
One STEP = one pass of Simulator::push_frame over the whole sequence (reset
+ every frame; the reference's bench_method protocol, src/bench.cpp:53-64).
Metric: simulated input frames/s, counting the frames that close an interval
(n - 1 per step: the warm-up frame produces no events), events/s beside it.

* value: frames already resident in HBM, device-timed with CUDA events on the
  simulator's stream, L2 flushed (256 MiB memset) before every step.
* parity: an untimed pass with the timed pass's batches, each push's events
  reduced on the device to per-frame (count, checksum)
  (paper_2209_04634_b200/seqhash.py) and compared with the compiled
  reference's (tests/golden/sequences.json, tests/golden/make_sequences.py);
  the last timed push is checked the same way.
* e2e: the same metric through the C-ABI with HOST buffers
  (evsim_gpu_push_frames_streamed: pinned host frames in, events out to pinned
  host memory, upload / compute / download overlapped), host wall clock.
* roofline: the event stage (chain -> offsets -> emit) against the measured
  HBM peak, algorithmic bytes per frame B_alg = 2P + 4E.
* cpu_baseline / --impl reference: the reference compiled from its own sources
  (oracle/_ref) run by evsim_ref_run_sequence on the host's threads (output
  identical to one streaming Simulator, checked against the same checksums),
  on a bounded sample of the sequence; also a 1-thread sample.

Multi-GPU (torchrun), one process per GPU, no data-path collective:
* --split bands (default for single-stream configs, c5): rank r emits the
  events of its row band, solving only the flow patch rows they depend on
  (exact); NCCL all-gathers per-(band, link) counts — the merged stream's
  offsets — and the per-band partial checksums.  Strong scaling.
* --split streams (default for c4: 32 streams): rank r owns a contiguous block
  of the config's streams (shard_streams), pushed concurrently; weak per
  stream, the total is fixed: "strong".
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_FLUSH_BYTES = 256 << 20
CHAIN_KERNEL = {"dense": "chain_dense_kernel", "sparse": "chain_sparse_kernel", "difference_only": "chain_diff_kernel",
                "difference_interp": "chain_diffinterp_kernel"}
METRIC = "simulated input frames/sec and events/sec per B200, % of HBM roofline"
GOLDEN = os.path.join(ROOT, "tests", "golden", "sequences.json")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c5")
    p.add_argument("--mode", default="log", choices=["log", "linear"])
    p.add_argument("--preset", default="lq", choices=["lq", "hq"], help="flow preset (types.hpp:93: lq default)")
    p.add_argument("--frames", type=int, default=0, help="override sequence length")
    p.add_argument("--streams", type=int, default=0, help="total camera streams (0 = the config's)")
    p.add_argument("--split", default="auto", choices=["auto", "streams", "bands"])
    p.add_argument("--batch", type=int, default=0,
                   help="frames per push_frames call (0 = the simulator's maximum; 1 = frame-by-frame)")
    p.add_argument("--chunk", type=int, default=0, help="e2e: frames per streamed chunk (0 = library default)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-e2e-extra", action="store_true", help="skip the one-step e2e lines of the other formats")
    p.add_argument("--e2e-format", default="auto", choices=["auto", "wire", "packed", "event24"],
                   help="host event format of e2e (auto: wire when it is smaller than packed records)")
    p.add_argument("--no-parity", action="store_true")
    p.add_argument("--force-band", action="store_true", help=argparse.SUPPRESS)
    p.add_argument("--no-stack", action="store_true",
                   help="difference_only streams: one simulator per stream instead of one stacked simulator")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ----------------------------------------------------------------------------- workload

def make_cfg(c, args):
    from paper_2209_04634_b200 import scenes
    from paper_2209_04634_b200.abi import Method, make_config
    cp, cn = scenes.LINEAR_THRESHOLDS[c.method]
    return make_config(Method[c.method], n_interp=c.n_interp, c_pos=cp, c_neg=cn,
                       contrast_mode=1 if args.mode == "log" else 0, c_pos_log=c.contrast, c_neg_log=-c.contrast,
                       flow_preset=1 if args.preset == "hq" else 0)


def _gen(job):
    name, n, stream = job
    from paper_2209_04634_b200 import scenes
    return scenes.generate(scenes.CONFIGS[name], n_frames=n, stream=stream)


def generate_streams(c, n, streams):
    """Frames of several streams, generated in a process pool (c4: ~26 s each)."""
    streams = list(streams)
    if len(streams) == 1:
        return [_gen((c.name, n, streams[0]))]
    import multiprocessing as mp
    with mp.get_context("spawn").Pool(min(len(streams), os.cpu_count() or 1)) as pool:
        return pool.map(_gen, [(c.name, n, s) for s in streams], chunksize=1)


def config_json(c, args, n_frames, split, ws, n_streams):
    par = f"row bands x{ws}" if split == "bands" else f"streams: {n_streams} over {ws} GPU(s)"
    return {
        "workload": f"{c.name}: {n_streams} x {c.width}x{c.height} u8 stream(s), {c.method} (LK {args.preset}) "
                    f"N={c.n_interp}, {args.mode} C={c.contrast if args.mode == 'log' else 'int Table I'}, "
                    f"{n_frames}-frame seeded synthetic sequence",
        "width": c.width, "height": c.height, "streams": n_streams, "frames_per_stream": n_frames,
        "n_interp": c.n_interp, "method": c.method, "mode": args.mode,
        "flow_preset": "high_quality" if args.preset == "hq" else "low_quality",
        "l2": "flushed before every step (256 MiB memset); device-resident inputs",
        "parallelism": par,
    }


def golden_entry(c, args, n_frames, stream=0):
    """The committed reference checksums of this sequence, if pinned."""
    if stream != 0:
        return None
    try:
        key = f"{c.name}:{args.mode}" + ("" if args.preset == "lq" else f":{args.preset}")
        g = json.load(open(GOLDEN)).get(key)
    except Exception:
        return None
    if not g or g["n_frames"] < n_frames:
        return None
    return g


# ----------------------------------------------------------------------------- CPU arms

def cpu_sample(c, cfg, frames, ts, threads, pairs):
    """The reference (oracle/_ref via evsim_ref_run_sequence; the C port when it
    is absent) over frames[0 .. pairs]: (pairs, seconds, kind, counts, hashes)."""
    import oracle
    pairs = max(1, min(pairs, len(frames) - 1))
    sub = np.ascontiguousarray(frames[:pairs + 1])
    if os.path.exists(oracle.REF_SO):
        R = oracle.Reference()
        t0 = time.perf_counter()
        counts, hashes = R.run_sequence(cfg, sub, ts[:pairs + 1], threads)
        return pairs, time.perf_counter() - t0, "reference", counts, hashes
    # fallback: the C restatement, one streaming simulator (1 thread)
    from paper_2209_04634_b200.seqhash import frame_hash_np
    sim = oracle.Oracle().simulator(cfg)
    counts, hashes = [], []
    t0 = time.perf_counter()
    for k in range(pairs + 1):
        ev = sim.push_frame(sub[k], int(ts[k]))
        counts.append(len(ev))
        hashes.append(frame_hash_np(ev["x"], ev["y"], ev["t"], ev["p"], int(ts[k - 1]) if k else 0))
    return pairs, time.perf_counter() - t0, "port", np.array(counts), np.array(hashes, np.uint64)


def sample_parity(g, counts, hashes):
    if g is None:
        return "unpinned"
    n = len(counts)
    ok = list(map(int, counts[1:])) == g["counts"][1:n] and \
        [f"{int(h):016x}" for h in hashes[1:]] == g["hashes"][1:n]
    return "match" if ok else "MISMATCH"


def cpu_pairs_for(c, threads):
    # log mode pipelines one pair per thread; bound the sample to ~10-30 s
    return min(threads, 8 if c.pixels >= 4_000_000 else 64)


def run_reference(args):
    ws, rank, _ = dist_env()
    if ws > 1 and rank != 0:
        return 0
    from paper_2209_04634_b200 import scenes
    c = scenes.CONFIGS[args.config]
    n = args.frames or c.n_frames
    cfg = make_cfg(c, args)
    threads = os.cpu_count() or 1
    n_streams = args.streams or c.streams
    split = "streams" if n_streams > 1 else "bands"
    if n_streams > 1:
        # one reference thread per stream (independent instances), up to nproc
        use = list(range(min(threads, n_streams)))
        nf = 3 if c.pixels >= 1_000_000 else n
        data = generate_streams(c, nf, use)
        vals = []
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            with cf.ThreadPoolExecutor(len(use)) as ex:
                res = list(ex.map(lambda d: cpu_sample(c, cfg, d[0], d[1], 1, nf - 1), data))
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                vals.append(sum(r[0] for r in res) / dt)
        kind = res[0][2]
        parity = sample_parity(golden_entry(c, args, nf), res[0][3], res[0][4])
        sample = (f"{len(use)} of the {n_streams} {c.name} streams, frames 0-{nf - 1} each, one reference thread "
                  f"per stream")
        evs = sum(int(r[3].sum()) for r in res) / sum(r[0] for r in res)
        cores = len(use)
        sample_pairs = sum(r[0] for r in res)
    else:
        frames, ts = _gen((c.name, n, 0))
        pairs = cpu_pairs_for(c, threads)
        g = golden_entry(c, args, pairs + 1)
        vals = []
        for i in range(args.warmup + args.steps):
            p, dt, kind, counts, hashes = cpu_sample(c, cfg, frames, ts, threads, pairs)
            if i >= args.warmup:
                vals.append(p / dt)
        parity = sample_parity(g, counts, hashes)
        sample = (f"{c.name} frames 0-{p} ({p} intervals) of the {n}-frame sequence, {threads} host threads "
                  f"(evsim_ref_run_sequence: {'pairs in parallel + the log rule over row bands' if args.mode == 'log' else 'contiguous chunks, one Simulator each'}; output = one streaming Simulator)")
        evs = float(counts.sum()) / p
        cores = threads
        sample_pairs = p
    v = statistics.mean(vals)
    out = {
        "metric": METRIC, "impl": "reference", "value": round(v, 4), "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * sample_pairs / v, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8/f32/f64",
        "data": "synthetic", "config": config_json(c, args, n, split, 1, n_streams),
        "events_per_s": round(v * evs, 1), "parity": parity,
        "cpu_baseline": {"value": round(v, 4), "unit": "frames/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": round(v, 4), "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


# ----------------------------------------------------------------------------- clocks

class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region (NVML
    polling thread, ~2 ms; nvidia-smi when NVML is unavailable)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.nvml = None
        self.rows = []
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def _sample(self):
        import pynvml
        h = self.handle
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        try:
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.rows.append((float(sm), float(mx), [n for n, bit in self.REASONS.items() if r & bit]))

    def _poll(self):
        while not self.stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self.stop.wait(0.002)

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self._nvml_index())
            self.nvml = pynvml
            self._sample()
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def _nvml_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            if self.device < len(ids) and ids[self.device].isdigit():
                return int(ids[self.device])
        return self.device

    def __exit__(self, *a):
        if self.nvml:
            self.stop.set()
            self.thread.join(timeout=2)
            try:
                self._sample()
            except Exception:
                pass
            return
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        rows = self.rows
        src = "nvml"
        if not self.nvml:
            src = "nvidia-smi"
            if not self.proc:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
            rows = []
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
                    rows.append((float(parts[1]), float(parts[2]),
                                 [names[i] for i in range(4) if parts[5 + i].lower().startswith("active")]))
                except ValueError:
                    continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        reasons = sorted({n for _, _, r in rows for n in r})
        return {"sm_mhz": statistics.median(s for s, _, _ in rows), "sm_max_mhz": max(m for _, m, _ in rows),
                "reasons": reasons, "samples": len(rows), "source": src}


# ----------------------------------------------------------------------------- ours

class Arm:
    """This rank's simulators (one per stream; one row band for bands) with
    their frames resident in HBM."""

    def __init__(self, c, cfg, args, ws, rank, device, split):
        import torch

        from paper_2209_04634_b200 import Simulator, SimulatorConfig
        from paper_2209_04634_b200.parallel import band_rows, shard_streams, stack_streams
        self.c, self.args, self.ws, self.rank, self.device, self.split = c, args, ws, rank, device, split
        self.n = args.frames or c.n_frames
        total = args.streams or c.streams
        # difference_only streams stacked into one simulator (parallel.stack_streams:
        # exact, every pixel its own chain) — S streams in one launch sequence
        self.stacked = split == "streams" and c.method == "difference_only" and total > 1 and not args.no_stack
        if self.stacked:
            self.streams = list(shard_streams(total, ws, rank))
            self.band = None
            data = generate_streams(c, self.n, self.streams)
            self.frames = [stack_streams([d[0] for d in data])]
            self.cpu_frames = data[0][0]  # stream 0 alone (the CPU baseline's sample)
            self.ts = data[0][1]
            self.H = len(self.streams) * c.height
            self.sims = [Simulator(SimulatorConfig.from_c(cfg), device=device)]
            self.P = c.width * self.H
            self.d_frames = [torch.from_numpy(self.frames[0]).to(f"cuda:{device}")]
            self.batch = max(1, min(args.batch or self.sims[0].max_batch(c.width, self.H), self.n))
            self.torch_stream = torch.cuda.ExternalStream(self.sims[0].stream, device=device)
            self.other_streams = []
            return
        self.H = c.height
        if split == "bands":
            self.streams = [0]
            # (--force-band: the band path at N = 1 — one band = the frame — to
            # exercise the placement / merged-output check on one GPU)
            self.band = band_rows(c.height, ws, rank) if (ws > 1 or args.force_band) else None
        else:
            self.streams = list(shard_streams(total, ws, rank)) if total > 1 else [rank]
            self.band = None
        data = generate_streams(c, self.n, self.streams)
        self.frames = [d[0] for d in data]
        self.cpu_frames = self.frames[0]
        self.ts = data[0][1]
        self.sims = []
        for _ in self.streams:
            s = Simulator(SimulatorConfig.from_c(cfg), device=device)
            if self.band:
                s.set_row_band(*self.band)
            self.sims.append(s)
        self.P = c.width * c.height
        self.d_frames = [torch.from_numpy(f).to(f"cuda:{device}") for f in self.frames]
        mb = self.sims[0].max_batch(c.width, c.height)
        if len(self.sims) > 1:
            mb = min(mb, 8)  # many resident streams: bound each handle's event buffers
        self.batch = max(1, min(args.batch or mb, mb, self.n))
        self.torch_stream = torch.cuda.ExternalStream(self.sims[0].stream, device=device)
        self.other_streams = [torch.cuda.ExternalStream(s.stream, device=device) for s in self.sims[1:]]

    def merged_buffer(self, ws, need):
        """Rank 0's merged-output buffer (every band's events, placed by
        each rank) as a device address in this process: allocated once at the
        push's upper bound (every link-pixel an event) and mapped into the
        other ranks with CUDA IPC."""
        import torch
        if getattr(self, "_merged", None) is None:
            cap = (self.c.n_interp + 1) * self.P * self.batch
            handle = [None]
            if self.rank == 0:
                self._merged_t = torch.empty(cap, dtype=torch.int32, device=f"cuda:{self.device}")
                self._merged = self._merged_t.data_ptr()
                if ws > 1:
                    from paper_2209_04634_b200.parallel import share_buffer
                    handle = [share_buffer(self._merged)]
            if ws > 1:
                torch.distributed.broadcast_object_list(handle, src=0)
                if self.rank != 0:
                    from paper_2209_04634_b200.parallel import open_shared
                    self._merged = open_shared(handle[0], self.device)
            self._merged_cap = cap
        if need > self._merged_cap:
            raise RuntimeError("merged output larger than its bound")
        return self._merged

    def pushes(self):
        return [(a, min(self.batch, self.n - a)) for a in range(0, self.n, self.batch)]

    def push(self, a, nb, sync):
        from paper_2209_04634_b200.simulator import push_frames_batched_device
        c = self.c
        if len(self.sims) == 1:
            return [self.sims[0].push_frames_device(self.d_frames[0].data_ptr() + a * self.P, nb, c.width, self.H,
                                                    self.ts[a:a + nb], on_device=True, sync=sync)]
        return push_frames_batched_device(self.sims, [d.data_ptr() + a * self.P for d in self.d_frames], nb,
                                          c.width, c.height, [self.ts[a:a + nb]] * len(self.sims))

    def enqueue_step(self):
        for s in self.sims:
            s.reset()
        for a, nb in self.pushes():
            self.push(a, nb, sync=False)

    def sync(self):
        for s in self.sims:
            s.sync()


def push_checksums(arm, a, nb, outs, timeline_counts=None):
    """Per-frame (count, checksum) of one push for this rank's stream 0 (bands:
    the band's partial checksums with global frame indices)."""
    from paper_2209_04634_b200.seqhash import push_frame_hashes
    ev = outs[0]
    S = int(ev.n_segments)
    seg_t = np.ctypeslib.as_array(ev.seg_t, shape=(S,)).copy() if S else np.zeros(0, np.int64)
    seg_off = np.ctypeslib.as_array(ev.seg_offset, shape=(S + 1,)).copy() if S else np.zeros(1, np.int64)
    f0 = max(a, 1)
    frame_ts = arm.ts[f0 - 1:a + nb]
    if timeline_counts is None:
        return seg_t, seg_off, push_frame_hashes(int(ev.d_packed), seg_t, seg_off, frame_ts, arm.device)
    timeline, jbase = timeline_counts
    return seg_t, seg_off, push_frame_hashes(int(ev.d_packed), seg_t, seg_off, frame_ts, arm.device, timeline, jbase)


def stacked_stream0_checksums(arm, a, nb, ev):
    """Per-frame (count, checksum) of stream 0 of a stacked push: its events
    are the rows [0, h) of every segment (parallel.split_stacked)."""
    from paper_2209_04634_b200.parallel import split_stacked
    from paper_2209_04634_b200.seqhash import device_int32, frame_hash_packed_np
    n = int(ev.n_events)
    S = int(ev.n_segments)
    seg_t = np.ctypeslib.as_array(ev.seg_t, shape=(S,)).copy() if S else np.zeros(0, np.int64)
    seg_off = np.ctypeslib.as_array(ev.seg_offset, shape=(S + 1,)).copy() if S else np.zeros(1, np.int64)
    packed = device_int32(int(ev.d_packed), n, arm.device).cpu().numpy().view(np.uint32) if n else np.zeros(0, np.uint32)
    rec, st, so = split_stacked(packed, seg_t, seg_off, len(arm.streams), arm.c.height)[0]
    out = []
    for k in range(max(a, 1), a + nb):  # frames that close an interval
        t0, t1 = int(arm.ts[k - 1]), int(arm.ts[k])
        sel = (st > t0) & (st <= t1)
        idx = np.nonzero(sel)[0]
        if len(idx):
            r = rec[so[idx[0]]:so[idx[-1] + 1]]
            out.append((len(r), frame_hash_packed_np(r, st[idx], so[idx[0]:idx[-1] + 2] - so[idx[0]], t0)))
        else:
            out.append((0, frame_hash_packed_np(np.zeros(0, np.uint32), np.zeros(0), np.zeros(1, np.int64), t0)))
    return out


def parity_pass(arm, g, ws):
    """Untimed pass with the timed pass's batches; per-frame checksums of
    stream 0 compared with the reference's.  Returns (status, events total of
    this rank, per-frame (count, hash) list)."""
    import torch
    from paper_2209_04634_b200.parallel import gather_counts, link_timeline, segment_dst_offsets, timeline_counts
    from paper_2209_04634_b200.seqhash import push_frame_hashes
    for s in arm.sims:
        s.reset()
    frames_out = []
    ev_total = 0
    for a, nb in arm.pushes():
        outs = arm.push(a, nb, sync=True)
        ev_total += sum(int(o.n_events) for o in outs)
        if arm.stacked:
            frames_out += stacked_stream0_checksums(arm, a, nb, outs[0])
            continue
        if arm.band is None:
            frames_out += push_checksums(arm, a, nb, outs)[2]
            continue
        # row bands: counts per (band, link) over the push's full link
        # timeline, all-gathered over NCCL (the merged stream's offsets);
        # every rank places its events into rank 0's buffer (CUDA IPC over
        # NVLink, evsim_gpu_place_events); rank 0 checks the merged stream
        f0 = max(a, 1)
        timeline = link_timeline(arm.ts[f0 - 1:a + nb], arm.c.n_interp)
        ev = outs[0]
        S = int(ev.n_segments)
        seg_t = np.ctypeslib.as_array(ev.seg_t, shape=(S,)).copy() if S else np.zeros(0, np.int64)
        seg_off = np.ctypeslib.as_array(ev.seg_offset, shape=(S + 1,)).copy()
        local = timeline_counts(seg_t, seg_off, timeline)
        allc = gather_counts(local, device=torch.device("cuda", arm.device)) if ws > 1 else local[None]
        merged_ptr = arm.merged_buffer(ws, int(allc.sum()))
        arm.sims[0].place_events(merged_ptr, segment_dst_offsets(allc, arm.rank, timeline, seg_t))
        arm.sims[0].sync()
        if ws > 1:
            torch.distributed.barrier()
        if arm.rank == 0:
            tot = allc.sum(axis=0)
            m_off = np.concatenate([[0], np.cumsum(tot)]).astype(np.int64)
            keep = tot > 0
            frames_out += push_frame_hashes(merged_ptr, timeline[keep],
                                            np.concatenate([m_off[:-1][keep], [m_off[-1]]]),
                                            arm.ts[f0 - 1:a + nb], arm.device)
        if ws > 1:
            torch.distributed.barrier()
    status = "unpinned"
    if g is not None and (arm.streams[0] == 0):
        got_c = [cnt for cnt, _ in frames_out]
        got_h = [f"{h:016x}" for _, h in frames_out]
        n = len(got_c) + 1
        status = "match" if (got_c == g["counts"][1:n] and got_h == g["hashes"][1:n]) else "MISMATCH"
    return status, ev_total, frames_out


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = local if ws > 1 else 0
    torch.cuda.set_device(device)
    from paper_2209_04634_b200 import scenes
    c = scenes.CONFIGS[args.config]
    split = args.split
    if split == "auto":
        split = "streams" if (args.streams or c.streams) > 1 else "bands"
    cfg = make_cfg(c, args)
    arm = Arm(c, cfg, args, ws, rank, device, split)
    n, P = arm.n, arm.P
    # streams simulated per step over all ranks (a single-stream config split
    # by streams runs one replica per rank)
    if split == "bands":
        n_streams = 1
    elif (args.streams or c.streams) > 1:
        n_streams = args.streams or c.streams
    else:
        n_streams = ws
    scaling = "weak" if (split == "streams" and (args.streams or c.streams) == 1) else "strong"
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=f"cuda:{device}")
    torch.cuda.synchronize()

    for _ in range(max(args.warmup, 1)):
        arm.enqueue_step()
        arm.sync()
    g = golden_entry(c, args, n)
    parity, ev_total, frames_out = ("skipped", 0, [])
    if not args.no_parity:
        parity, ev_total, frames_out = parity_pass(arm, g, ws)
    else:
        for s in arm.sims:
            s.reset()
        for a, nb in arm.pushes():
            ev_total += sum(int(o.n_events) for o in arm.push(a, nb, sync=True))
    torch.cuda.synchronize()

    # ---- timed region: device-resident, L2 flushed before each step -------------
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = sum(s.kernel_launches for s in arm.sims)
    times = []
    with Clocks(device) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(arm.torch_stream):
                flush.fill_(1)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(arm.torch_stream)
            # every handle's stream waits for the flush + start event
            for st in arm.other_streams:
                st.wait_event(e0)
            arm.enqueue_step()
            for s in arm.sims[1:]:
                s.sync()
            e1.record(arm.torch_stream)
            arm.sims[0].sync()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    launches = sum(s.kernel_launches for s in arm.sims) - launches0
    # the last timed push, checked against the parity pass (same frames)
    timed_check = "skipped"
    if frames_out and arm.band is None and not arm.stacked:
        a, nb = arm.pushes()[-1]
        ev = arm.sims[0].sync()
        part = push_checksums(arm, a, nb, [ev])[2]
        timed_check = "match" if part == frames_out[-len(part):] else "MISMATCH"

    # stage split: the same steps with per-stage CUDA events (stage timing
    # serialises the flow / chain overlap, so it runs outside the timed region)
    for s in arm.sims:
        s.set_profiling(True)
    for _ in range(max(1, min(args.steps, 3))):
        with torch.cuda.stream(arm.torch_stream):
            flush.fill_(1)
        arm.enqueue_step()
        arm.sync()
    torch.cuda.synchronize()
    stages, timed_pushes = arm.sims[0].stage_times()
    for s in arm.sims:
        s.set_profiling(False)
    prof_steps = max(1, min(args.steps, 3))

    total_ms = sum(times)
    t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{device}")
    evs = torch.tensor([ev_total], dtype=torch.int64, device=f"cuda:{device}")
    if ws > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(evs, op=dist.ReduceOp.SUM)
    max_ms = float(t.item())
    ev_all = int(evs.item())
    frames_per_step = (n - 1) * n_streams  # intervals closed per step, all streams / the whole frame
    value = frames_per_step * args.steps / (max_ms / 1e3)
    events_per_s = ev_all * args.steps / (max_ms / 1e3)

    # ---- roofline of the event stage (chain -> offsets -> emit) -----------------
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6.65 TB/s (B200_PROFILING.md)"
    E_frame = ev_all / max(frames_per_step, 1)
    b_alg = 2 * P + 4 * E_frame  # read 2 u8 frames, write 4 B per event
    # stream 0's handle: its pushes (launches of the event stage) over its pairs
    pairs_prof = prof_steps * (n - 1)
    launches_ev = max(timed_pushes, 1)
    ev_stage_ms = stages["chain"] + stages["scan"] + stages["emit"]
    E_band = (ev_total / max(len(arm.sims), 1)) / max(n - 1, 1)  # this rank's (band's / stack's) events per pair
    P_band = c.width * (arm.band[1] - arm.band[0]) if arm.band else arm.P  # rows of stream 0's handle
    b_alg_band = 2 * P_band + 4 * E_band
    bytes_per_launch = b_alg_band * pairs_prof / launches_ev
    ms_per_launch = ev_stage_ms / launches_ev
    achieved = bytes_per_launch / (ms_per_launch / 1e3) / 1e9 if ms_per_launch > 0 else 0.0
    e2e_frac = b_alg * (value / ws) / 1e9 / hbm
    roofline = {"bound": "hbm", "achieved": round(achieved, 2), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4),
                "traffic": traffic_for(c.name, args.mode, pairs_prof / launches_ev) if ws == 1 else None,
                "kernel": f"event stage = {CHAIN_KERNEL[c.method]} + offsets_kernel + segbase_kernel + emit kernel "
                          "(one push_frames call)",
                "algorithmic_bytes_per_frame": round(b_alg_band), "frames_per_launch": round(pairs_prof / launches_ev, 2),
                "algorithmic_bytes_per_launch": round(bytes_per_launch), "avg_launch_ms": round(ms_per_launch, 5),
                "peak_source": peak_src, "end_to_end_frac": round(e2e_frac, 5),
                "stage_us_per_frame": {k: round(1e3 * v / pairs_prof, 3) for k, v in stages.items()},
                "issue_roofline": issue_roofline(c.name, args.mode, args.preset, pairs_prof / launches_ev,
                                                 stages["chain"] / launches_ev) if ws == 1 else None}

    # ---- e2e through the C-ABI with host buffers ---------------------------------
    e2e = None
    e2e_other = {}
    if not args.no_e2e:
        fmt = args.e2e_format
        if fmt == "auto":
            fmt = "wire" if wire_is_smaller(c, E_frame) else "packed"
        e2e = run_e2e(arm, args, ws, n_streams, fmt, args.steps, events_per_frame=E_frame)
        # the other host formats, one step each (bounded: the 24-byte records
        # of c5 are 1.6-3.8 GB per frame)
        for other in ("packed", "wire", "event24"):
            if other != fmt and not args.no_e2e_extra:
                r = run_e2e(arm, args, ws, n_streams, other, 1, max_calls=1 if other == "event24" else None,
                            events_per_frame=E_frame)
                e2e_other[other] = {k: r[k] for k in ("value", "unit", "d2h_bytes_per_step")}

    cpu = cpu1 = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        pairs = cpu_pairs_for(c, threads)
        p, dt, kind, cc, hh = cpu_sample(c, cfg, arm.cpu_frames, arm.ts, threads, pairs)
        cpu = {"value": round(p / dt, 4), "unit": "frames/s", "cores": threads, "kind": kind,
               "sample": f"{c.name} stream 0, frames 0-{p} ({p} intervals), {threads} host threads "
                         f"(evsim_ref_run_sequence, output = one streaming Simulator), {dt:.1f} s",
               "parity": sample_parity(golden_entry(c, args, p + 1), cc, hh)}
        p1 = 2 if c.pixels >= 2_000_000 else 8
        p, dt, kind, cc, hh = cpu_sample(c, cfg, arm.cpu_frames, arm.ts, 1, p1)
        cpu1 = {"value": round(p / dt, 4), "unit": "frames/s", "cores": 1, "kind": kind,
                "sample": f"{c.name} stream 0, frames 0-{p}, one reference Simulator (single thread), {dt:.1f} s"}

    if rank == 0:
        clocks = clk.summary()
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "frames/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(max_ms / args.steps, 4), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "u8/f32/f64", "data": "synthetic",
            "config": {**config_json(c, args, n, split, ws, n_streams), "frames_per_push": arm.batch,
                       **({"stacked_streams": f"{len(arm.streams)} streams stacked into one {c.width}x{arm.H} "
                                              "simulator per rank (parallel.stack_streams, exact for difference_only)"}
                          if arm.stacked else {})},
            "parity": parity, "timed_output_check": timed_check,
            "parity_ref": "tests/golden/sequences.json (compiled reference, per-frame count + checksum)",
            "events_per_s": round(events_per_s, 1), "events_per_frame": round(E_frame, 1),
            "roofline": roofline, "cpu_baseline": cpu, "cpu_baseline_1thread": cpu1, "e2e": e2e,
            "e2e_other_formats": e2e_other,
            "gpu_launches": int(launches), "clocks": clocks,
            "flow_gsamples_per_s": flow_rate(c, args, stages, pairs_prof),
        }
        print(json.dumps(out), flush=True)
    for s in arm.sims:
        s.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def run_e2e(arm, args, ws, n_streams, fmt, steps, max_calls=None, events_per_frame=0.0):
    """Steps through the public C-ABI with pinned host frames in and the
    events on the host (one host thread per handle), host wall clock:
      wire    evsim_gpu_push_frames_wire: planes + polarity bits (lossless,
              evsim_gpu_wire_unpack gives the reference's stream)
      packed  evsim_gpu_push_frames_streamed: packed 4-byte records
      event24 evsim_gpu_push_frames + evsim_gpu_copy_events format 1: the
              reference's 24-byte evsim::Event records
    The sequence goes in calls of at most max_batch frames whose events land
    in one reused host buffer (a consumer that takes each call's events
    before the next call); max_calls bounds the sample."""
    import torch

    from paper_2209_04634_b200.simulator import WireBuffer
    c, n, P = arm.c, arm.n, arm.P
    h_frames = [torch.from_numpy(f).pin_memory() for f in arm.frames]
    H = arm.H
    rows = (arm.band[1] - arm.band[0]) if arm.band else H
    # a streamed / device call holds <= max_batch frames; a wire call's launches
    # are chunks of <= max_batch pairs, so one call can take the sequence
    per_call = n if fmt == "wire" else min(n, arm.sims[0].max_batch(c.width, H))
    # many resident handles (c4: 32 streams): every handle's call buffers
    # (device chunks, host planes / records) scale with its frames per call;
    # keep calls at the device pushes' batch and size the packed host records
    # from the events the device pass produced instead of the every-link-pixel
    # bound
    multi = len(arm.sims) > 1
    if multi:
        per_call = min(per_call, arm.batch)
    chunk = args.chunk or (arm.batch if multi else 0)
    calls = [(a, min(per_call, n - a)) for a in range(0, n, per_call)][:max_calls]
    pairs_per_step = sum(nb for _, nb in calls) - 1
    cap = (c.n_interp + 1) * c.width * rows * per_call
    if multi and events_per_frame:
        cap = min(cap, int(3 * events_per_frame * per_call) + (1 << 20))
    bufs = []
    for s in arm.sims:
        if fmt == "wire":
            bufs.append(WireBuffer.for_call(s, per_call, c.width, H, rows=rows))
        elif fmt == "packed":
            bufs.append(torch.empty(cap, dtype=torch.int32).pin_memory())
        else:
            bufs.append(None)

    def one(i):
        s = arm.sims[i]
        s.reset()
        d2h = 0
        for a, nb in calls:
            ptr = h_frames[i].data_ptr() + a * P
            if fmt == "wire":
                bufs[i].run(s, ptr, nb, c.width, H, arm.ts[a:a + nb], chunk=chunk)
                d2h += bufs[i].bytes
            elif fmt == "packed":
                e = s.push_frames_streamed_ptr(ptr, nb, c.width, H, arm.ts[a:a + nb], bufs[i].data_ptr(),
                                               cap, chunk=chunk)
                d2h += 4 * int(e.n_events) + 16 * (int(e.n_segments) + 1)
            else:
                e = s.push_frames_device(ptr, nb, c.width, H, arm.ts[a:a + nb], on_device=False, sync=True)
                ev = np.empty(max(int(e.n_events), 1), dtype=[("b", "V24")])
                s.copy_events(ev.ctypes.data, int(e.n_events), 1)
                d2h += 24 * int(e.n_events) + 16 * (int(e.n_segments) + 1)
        return d2h

    def step():
        if len(arm.sims) == 1:
            return one(0)
        with cf.ThreadPoolExecutor(len(arm.sims)) as ex:
            return sum(ex.map(one, range(len(arm.sims))))

    step()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d2h = 0
    for _ in range(steps):
        d2h = step()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{arm.device}")
    if ws > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    frames_total = pairs_per_step * n_streams * steps
    api = {"wire": "evsim_gpu_push_frames_wire (pinned host frames in; event planes + polarity bits out, lossless: "
                   "evsim_gpu_wire_unpack reproduces the reference stream)",
           "packed": "evsim_gpu_push_frames_streamed (pinned host frames in, packed 4-byte host events out)",
           "event24": "evsim_gpu_push_frames + evsim_gpu_copy_events(format 1): 24-byte evsim::Event records"}[fmt]
    return {"value": round(frames_total / float(te.item()), 3), "unit": "frames/s",
            "h2d_bytes_per_step": sum(nb for _, nb in calls) * P * len(arm.sims), "d2h_bytes_per_step": int(d2h),
            "format": fmt, "api": f"{api}; {len(calls)} call(s) of <= {per_call} frames per stream per step, "
                                  "H2D / compute / D2H overlapped, host wall clock"}


def wire_is_smaller(c, events_per_frame):
    """Wire bytes (1 bit per pixel-link + 1 per event) below packed (4 B per event)?"""
    links = c.n_interp + 1
    return links * c.width * c.height / 8 + events_per_frame / 8 < 4 * events_per_frame


def flow_rate(c, args, stages, pairs):
    """Flow-stage template samples per second."""
    S = {("c1", "lq"): 1.74e6, ("c2", "lq"): 6.00e6, ("c3", "lq"): 18.16e6, ("c4", "lq"): 41.03e6,
         ("c5", "lq"): 164.7e6, ("c2", "hq"): 31.82e6, ("c5", "hq"): 876.2e6}
    s = S.get((c.name, args.preset))
    ms = stages.get("flow", 0.0)
    if s is None or ms <= 0 or c.method != "dense":
        return None
    return round(s * pairs / (ms / 1e3) / 1e9, 2)


def issue_roofline(config: str, mode: str, preset: str, pairs_per_launch: float, chain_ms_per_launch: float):
    """The chain kernel against the SM issue peak: warp-instructions per launch
    from the committed ncu capture of the same workload (lq preset, the same
    pairs per launch) over the chain's average launch time in this run;
    peak = 148 SMs x 4 schedulers x the SM clock (profiles/r02/peaks.json)."""
    if preset != "lq" or chain_ms_per_launch <= 0:
        return None
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "r02", f"traffic_{config}_{mode}.json")))
        pk = json.load(open(os.path.join(ROOT, "profiles", "r02", "peaks.json")))
    except Exception:
        return None
    if abs(pairs_per_launch - t.get("pairs_per_launch", -1)) >= 0.5:
        return None
    instr = sum(v for k, v in t.get("per_kernel_warp_instr", {}).items() if k.startswith("chain_"))
    if not instr:
        return None
    instr = int(instr * pairs_per_launch / t["pairs_per_launch"])  # per pair x this run's pairs per launch
    achieved = instr / (chain_ms_per_launch / 1e3) / 1e9
    peak = float(pk["issue_peak_G_per_s_theoretical"])
    return {"bound": "issue", "kernel": "chain kernel", "warp_instr_per_launch": instr,
            "achieved": round(achieved, 1), "peak": peak, "unit": "G warp-instr/s", "frac": round(achieved / peak, 4),
            "source": f"profiles/r02/traffic_{config}_{mode}.json (ncu instruction count) + this run's chain time"}


def traffic_for(config: str, mode: str, pairs_per_launch: float):
    """DRAM bytes (read + write) per launch of the event stage, from the
    committed ncu --set full capture of the same workload
    (profiles/r02/traffic_<config>_<mode>.json), or None."""
    for r in ("r02", "r01"):
        try:
            t = json.load(open(os.path.join(ROOT, "profiles", r, f"traffic_{config}_{mode}.json")))
        except Exception:
            continue
        if abs(pairs_per_launch - t.get("pairs_per_launch", -1)) < 0.5:
            return t["event_stage_dram_bytes_per_launch"]
    return None


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
