"""Benchmark of the B200 event-simulation hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2] [--mode log|linear]

Workload (BASELINE.json configs[1], the metric's headline config): c2 —
640x480 u8 frames, 128-frame seeded synthetic sequence (paper_2209_04634_b200/
scenes.py), dense pyramidal LK (lq preset), N = 10 interpolated frames, log
intensity with C = 0.2.  One STEP = one pass of Simulator::push_frame over
the whole 128-frame sequence (reset + 128 pushes; the reference's
bench_method protocol, src/bench.cpp:53-64).  Metric: input frames/s (events/s
reported beside it).

* value: frames already resident in HBM, device-timed with CUDA events on the
  simulator's stream, L2 flushed (256 MiB memset) before every step.
* e2e: the same metric through the C-ABI with HOST buffers: per frame a pinned
  H2D upload inside evsim_gpu_push_frame and a D2H of the packed events
  (4 B/event) + segment table; host wall clock around the step.
* roofline: event stage (chain -> scan -> emit) against measured HBM peak;
  algorithmic bytes per frame B_alg = 2P + 4E.
* cpu_baseline / --impl reference: the reference compiled from /root/reference
  (oracle/_ref; the oracle C port when absent), one independent simulator per
  host thread over contiguous chunks of the same sequence.

Multi-GPU (torchrun): each rank simulates its own independent stream (per-rank
seed) — stream sharding with no data-path collective ("weak" scaling); NCCL
only all-reduces the timing and gathers event counts.
"""
from __future__ import annotations

import argparse
import ctypes
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


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2")
    p.add_argument("--mode", default="log", choices=["log", "linear"])
    p.add_argument("--preset", default="lq", choices=["lq", "hq"], help="flow preset (types.hpp:93: lq default)")
    p.add_argument("--frames", type=int, default=0, help="override sequence length")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--chunk", type=int, default=0, help="e2e: frames per streamed chunk (0 = the library default, 64)")
    p.add_argument("--split", default="streams", choices=["streams", "bands"],
                   help="N>1: one camera stream per rank (weak scaling) or row bands of one stream (strong, c5)")
    p.add_argument("--batch", type=int, default=0,
                   help="frames per push_frames call (0 = the simulator's maximum; 1 = frame-by-frame)")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload(args, stream=0):
    from paper_2209_04634_b200 import scenes
    from paper_2209_04634_b200.abi import Method, make_config
    c = scenes.CONFIGS[args.config]
    n = args.frames or c.n_frames
    frames, ts = scenes.generate(c, n_frames=n, stream=stream)
    cp, cn = scenes.LINEAR_THRESHOLDS[c.method]
    cfg = make_config(Method[c.method], n_interp=c.n_interp, c_pos=cp, c_neg=cn,
                      contrast_mode=1 if args.mode == "log" else 0, c_pos_log=c.contrast, c_neg_log=-c.contrast,
                      flow_preset=1 if getattr(args, "preset", "lq") == "hq" else 0)
    return c, cfg, frames, ts


def config_json(c, args, n_frames):
    return {
        "workload": f"{c.name}: {c.width}x{c.height} u8, {c.method} (LK {args.preset}) N={c.n_interp}, "
                    f"{args.mode} C={c.contrast if args.mode == 'log' else 'int Table I'}, "
                    f"{n_frames}-frame seeded synthetic sequence",
        "width": c.width, "height": c.height, "frames_per_step": n_frames, "n_interp": c.n_interp,
        "method": c.method, "mode": args.mode,
        "flow_preset": "high_quality" if args.preset == "hq" else "low_quality",
        "l2": "flushed before every step (256 MiB memset); device-resident inputs",
    }


# ----------------------------------------------------------------------------- CPU arms

def cpu_run(cfg, frames, ts, threads, prefer_reference=True):
    """Time the reference (or the oracle port) over the sequence split into
    contiguous chunks, one independent simulator per host thread.  Returns
    (useful frames, seconds, kind, events)."""
    import oracle
    kind = "reference" if (prefer_reference and os.path.exists(oracle.REF_SO)) else "port"
    lib = oracle.Reference() if kind == "reference" else oracle.Oracle()
    n = len(frames)
    bounds = np.linspace(0, n - 1, threads + 1).astype(int)
    counts = [0] * threads
    useful = [0] * threads

    def work(i):
        lo, hi = int(bounds[i]), int(bounds[i + 1])
        sim = lib.simulator(cfg)
        ev = 0
        for k in range(lo, hi + 1):
            ev += len(sim.push_frame(frames[k], int(ts[k])))
        counts[i] = ev
        useful[i] = hi - lo
        sim.close()

    t0 = time.perf_counter()
    th = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    dt = time.perf_counter() - t0
    return sum(useful), dt, kind, sum(counts)


def run_reference(args):
    ws, rank, _ = dist_env()
    if ws > 1 and rank != 0:
        return 0
    c, cfg, frames, ts = workload(args)
    threads = os.cpu_count() or 1
    vals = []
    evs = 0
    kind = "port"
    for i in range(args.warmup + args.steps):
        f, dt, kind, evs = cpu_run(cfg, frames, ts, threads)
        if i >= args.warmup:
            vals.append(f / dt)
    v = statistics.mean(vals)
    out = {
        "metric": "simulated input frames/sec (events/sec beside it), % of HBM roofline",
        "impl": "reference", "value": round(v, 3), "unit": "frames/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * len(frames) / v, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8/f32/f64", "data": "synthetic",
        "config": config_json(c, args, len(frames)),
        "events_per_s": round(v * evs / max(len(frames) - threads, 1), 1),
        "cpu_baseline": {"value": round(v, 3), "unit": "frames/s", "cores": threads, "kind": kind,
                         "sample": f"{c.name} {len(frames)}-frame sequence, {args.mode} mode, split into "
                                   f"{threads} contiguous chunks (one simulator per host thread)"},
        "e2e": {"value": round(v, 3), "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


# ----------------------------------------------------------------------------- clocks

class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region: an NVML
    polling thread (every ~2 ms, so even a 20-ms region gets samples; one
    sample is taken on entry and one on exit), or nvidia-smi when NVML is
    unavailable."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
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
            import threading
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
        # CUDA_VISIBLE_DEVICES remaps CUDA ordinals; NVML sees all GPUs
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

def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = local if ws > 1 else 0
    torch.cuda.set_device(device)

    from paper_2209_04634_b200 import SimulatorConfig, Simulator
    from paper_2209_04634_b200._lib import load
    bands = args.split == "bands" and ws > 1
    c, cfg, frames, ts = workload(args, stream=0 if bands else rank)
    n = len(frames)
    P = c.width * c.height
    sim = Simulator(SimulatorConfig.from_c(cfg), device=device)
    if bands:
        # every rank holds the whole frames and emits its own rows
        from paper_2209_04634_b200.parallel import band_rows
        sim.set_row_band(*band_rows(c.height, ws, rank))
    stream_ptr = sim.stream
    torch_stream = torch.cuda.ExternalStream(stream_ptr, device=device)

    d_frames = torch.from_numpy(frames).to(f"cuda:{device}")
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=f"cuda:{device}")
    base = d_frames.data_ptr()
    torch.cuda.synchronize()

    mb = sim.max_batch(c.width, c.height)
    batch = args.batch or mb
    batch = max(1, min(batch, mb, n))

    def enqueue_step():
        # reset + the whole sequence in batches of `batch` frames (one launch
        # sequence per batch); the first frame is the warm-up frame
        sim.reset()
        for a in range(0, n, batch):
            nb = min(batch, n - a)
            sim.push_frames_device(base + a * P, nb, c.width, c.height, ts[a:a + nb], on_device=True, sync=False)

    # warm-up, then an untimed synchronous pass that counts the events
    for _ in range(max(args.warmup, 1)):
        enqueue_step()
        sim.sync()
    ev_total = 0
    sim.reset()
    for a in range(0, n, batch):
        nb = min(batch, n - a)
        e = sim.push_frames_device(base + a * P, nb, c.width, c.height, ts[a:a + nb], on_device=True, sync=True)
        ev_total += e.n_events
    torch.cuda.synchronize()

    # ---- timed region: device-resident, L2 flushed before each step -------------
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = sim.kernel_launches
    times = []
    with Clocks(device) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(torch_stream):
                flush.fill_(1)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(torch_stream)
            enqueue_step()
            e1.record(torch_stream)
            sim.sync()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    launches = sim.kernel_launches - launches0
    # stage split: the same steps again with per-stage CUDA events (stage
    # timing serialises the library's flow / chain overlap, so it is measured
    # outside the timed region)
    sim.set_profiling(True)
    for _ in range(args.steps):
        with torch.cuda.stream(torch_stream):
            flush.fill_(1)
        enqueue_step()
        sim.sync()
    torch.cuda.synchronize()
    stages, timed_pushes = sim.stage_times()
    sim.set_profiling(False)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    total_ms = sum(times)
    t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{device}")
    evs = torch.tensor([ev_total], dtype=torch.int64, device=f"cuda:{device}")
    if ws > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        gathered = [torch.zeros_like(evs) for _ in range(ws)]
        dist.all_gather(gathered, evs)  # per-stream event counts (merged-output offsets)
        ev_all = int(sum(int(g.item()) for g in gathered))
    else:
        ev_all = ev_total
    max_ms = float(t.item())
    frames_total = (1 if bands else ws) * n * args.steps
    value = frames_total / (max_ms / 1e3)
    events_per_s = ev_all * args.steps / (max_ms / 1e3)

    # ---- roofline of the event stage (chain -> scan -> emit) ---------------------
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6.65 TB/s (B200_PROFILING.md)"
    E_frame = ev_total / max(n - 1, 1)
    b_alg = 2 * P + 4 * E_frame  # read 2 u8 frames, write 4 B per event
    # the event stage (chain_kernel -> offsets_kernel -> segbase+emit_kernel)
    # runs once per push_frames call, over all of the call's frame pairs
    launches_ev = max(timed_pushes, 1)
    pairs_timed = args.steps * (n - 1)
    ev_stage_ms = stages["chain"] + stages["scan"] + stages["emit"]
    bytes_per_launch = b_alg * pairs_timed / launches_ev
    ms_per_launch = ev_stage_ms / launches_ev
    achieved = bytes_per_launch / (ms_per_launch / 1e3) / 1e9 if ms_per_launch > 0 else 0.0
    e2e_frac = b_alg * (value / ws) / 1e9 / hbm
    frames_timed = args.steps * n
    roofline = {"bound": "hbm", "achieved": round(achieved, 2), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": traffic_for(c.name, args.mode, pairs_timed / launches_ev),
                "kernel": "event stage = chain_dense_kernel + offsets_kernel + segbase_kernel + emit_kernel (one push_frames call)",
                "algorithmic_bytes_per_frame": round(b_alg), "frames_per_launch": round(pairs_timed / launches_ev, 2),
                "algorithmic_bytes_per_launch": round(bytes_per_launch), "avg_launch_ms": round(ms_per_launch, 5),
                "peak_source": peak_src, "end_to_end_frac": round(e2e_frac, 5),
                "stage_us_per_frame": {k: round(1e3 * v / frames_timed, 3) for k, v in stages.items()}}

    # ---- e2e through the C-ABI with host buffers ---------------------------------
    e2e = None
    if not args.no_e2e:
        h_frames = torch.from_numpy(frames).pin_memory()
        hbase = h_frames.data_ptr()
        cap = (c.n_interp + 1) * P * batch
        h_events = torch.empty(cap, dtype=torch.int32).pin_memory()
        hev = h_events.data_ptr()

        def e2e_step():
            # evsim_gpu_push_frames_streamed: pinned host frames in, packed
            # host events out; chunk j+1's H2D and chunk j-1's D2H overlap
            # chunk j's compute
            sim.reset()
            d2h = 0
            for a in range(0, n, batch):
                nb = min(batch, n - a)
                e = sim.push_frames_streamed_ptr(hbase + a * P, nb, c.width, c.height, ts[a:a + nb], hev, cap,
                                                 chunk=args.chunk)
                d2h += 4 * e.n_events + 16 * (e.n_segments + 1)
            return d2h

        e2e_step()
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d2h = 0
        for _ in range(args.steps):
            d2h = e2e_step()
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        te = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{device}")
        if ws > 1:
            import torch.distributed as dist
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(frames_total / float(te.item()), 3), "unit": "frames/s",
               "h2d_bytes_per_step": n * P, "d2h_bytes_per_step": int(d2h),
               "api": f"evsim_gpu_push_frames_streamed (pinned host frames in, packed host events out, "
                      f"chunks of ~{args.chunk or 64} frames: H2D / compute / D2H overlapped)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        f, dt, kind, _ = cpu_run(cfg, frames, ts, os.cpu_count() or 1)
        cpu = {"value": round(f / dt, 3), "unit": "frames/s", "cores": os.cpu_count() or 1, "kind": kind,
               "sample": f"{c.name} {n}-frame sequence, {args.mode} mode, split into {os.cpu_count()} contiguous "
                         f"chunks (one simulator per host thread), {dt:.1f} s"}

    if rank == 0:
        out = {
            "metric": "simulated input frames/sec (events/sec beside it), % of HBM roofline",
            "value": round(value, 3), "unit": "frames/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(max_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong" if bands else "weak", "vs_baseline": None, "dtype": "u8/f32/f64",
            "data": "synthetic",
            "config": {**config_json(c, args, n), "parallelism": f"row bands x{ws}" if bands else f"streams x{ws}",
                       "frames_per_push": batch},
            "events_per_s": round(events_per_s, 1), "events_per_frame": round(E_frame, 1),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "issue_roofline": issue_roofline(c.name, args.mode, pairs_timed / launches_ev, stages, launches_ev,
                                             clk.summary().get("sm_mhz")),
        }
        print(json.dumps(out), flush=True)
    sim.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def issue_roofline(config: str, mode: str, pairs_per_launch: float, stages_ms: dict, launches: int,
                   sm_mhz):
    """SM-issue roofline of the two dominant kernels (both are issue / L1
    bound, not HBM bound): warp instructions per launch from the committed
    ncu --set full capture of this workload, over the live CUDA-event time of
    the stage, against 148 SMs x 4 issue slots x the measured SM clock."""
    if not (config == "c2" and mode == "log" and abs(pairs_per_launch - 127) < 0.5 and launches > 0):
        return None
    try:
        rows = json.load(open(os.path.join(ROOT, "profiles", "r01", "ncu_full_summary.json")))
    except Exception:
        return None
    clock = float(sm_mhz or 1965.0) * 1e6
    peak = 148 * 4 * clock
    out = {"unit": "warp-instructions/s", "peak": peak, "peak_source": "148 SMs x 4 schedulers x measured SM clock",
           "instructions_source": "profiles/r01/ncu_full_summary.json (smsp__inst_executed.sum, every launch of one push)"}
    fam = {"chain": "chain_dense_kernel", "flow": "dense_lk_warp_kernel"}
    for stage, name in fam.items():
        ks = [r for r in rows if name in r["kernel"]]
        if not ks:
            continue
        instr = sum(r["warp_instr"] for r in ks)  # the capture holds every launch of one push
        t = stages_ms[stage] / launches / 1e3
        if t > 0:
            out[stage] = {"kernel": name, "warp_instr_per_launch": instr, "achieved": round(instr / t, 1),
                          "frac": round(instr / t / peak, 4)}
    return out


def traffic_for(config: str, mode: str, pairs_per_launch: float):
    """DRAM bytes (read + write) per launch of the event stage, from the
    committed ncu --set full capture of the same workload
    (profiles/r01/traffic_<config>_<mode>.json), or None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "r01", f"traffic_{config}_{mode}.json")))
    except Exception:
        return None
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
