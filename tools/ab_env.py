"""A/B of library switches (environment variables read by libevsim_gpu.so)
on one workload: bench.py's device-resident line per setting, per-stage
us/frame from its profiled pass.

    python tools/ab_env.py c5 log EVSIM_EMIT_LANES=0 EVSIM_EMIT_LANES=33 ...
(a setting "-" = the defaults; several VAR=val joined with ',')"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg, mode = sys.argv[1], sys.argv[2]
for setting in sys.argv[3:] or ["-"]:
    env = dict(os.environ)
    if setting != "-":
        for kv in setting.split(","):
            k, v = kv.split("=")
            env[k] = v
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--mode", mode, "--steps",
                          "3", "--warmup", "2", "--no-e2e", "--no-cpu-baseline"], env=env, capture_output=True,
                         text=True)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")]
    if not line:
        print(json.dumps({"setting": setting, "error": out.stderr[-1500:]}))
        continue
    d = json.loads(line[-1])
    print(json.dumps({"setting": setting, "config": cfg, "mode": mode, "value": d["value"], "parity": d["parity"],
                      "stages": d["roofline"]["stage_us_per_frame"], "frac": d["roofline"]["frac"]}), flush=True)
