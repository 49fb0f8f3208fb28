"""Summarise an ncu --set full report into profiles/<round>/ncu_full_summary.json
and the event-stage DRAM traffic into traffic_c2_log.json (read by bench.py).

    python tools/ncu_summary.py gpurun_out/prof_all.ncu-rep profiles/r02 [config:mode:pairs_per_launch]
"""
import csv
import io
import json
import os
import subprocess
import sys

WANT = {"dur_ms": "gpu__time_duration.sum", "dram_rd_MB": "dram__bytes_read.sum",
        "dram_wr_MB": "dram__bytes_write.sum", "warp_instr": "smsp__inst_executed.sum",
        "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "regs": "launch__registers_per_thread", "l1tex_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "alu_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "fma_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "grid": "launch__grid_size", "block": "launch__block_size"}
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "second": 1e3, "s": 1e3}


def main(rep, outdir, *_):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:80]}
        for k, m in WANT.items():
            if m not in hdr:
                continue
            v, u = r[hdr.index(m)], units[hdr.index(m)]
            try:
                v = float(v.replace(",", ""))
                if k.endswith("_MB") or k == "dur_ms":
                    v *= SCALE.get(u, 1.0)
            except ValueError:
                pass
            d[k] = v
        for st in ("long_scoreboard", "short_scoreboard", "wait", "barrier", "math_pipe_throttle", "not_selected",
                   "mio_throttle"):
            m = f"smsp__average_warps_issue_stalled_{st}_per_issue_active.ratio"
            if m in hdr:
                d["stall_" + st] = float(r[hdr.index(m)])
        out.append(d)
    os.makedirs(outdir, exist_ok=True)
    json.dump(out, open(os.path.join(outdir, "ncu_full_summary.json"), "w"), indent=1)

    # the capture holds one whole push: sum each event-stage kernel over it
    # (the chain may run as several pipelined sub-batch launches)
    tag = sys.argv[3] if len(sys.argv) > 3 else "c2:log:127"
    config, mode, ppl = tag.split(":")
    stage = ("chain_", "offsets", "segbase_kernel", "emit")
    xs = [x for x in out if any(k in x["kernel"] for k in stage) and "dram_rd_MB" in x]
    if xs:
        # one launch of each event-stage kernel per push here (no sub-batches
        # below 16 pairs): the last launch of each, i.e. the capture's last push
        per, instr = {}, {}
        for x in xs:
            name = x["kernel"].split("(")[0].replace("void ", "")
            per[name] = int((x["dram_rd_MB"] + x["dram_wr_MB"]) * 1e6)
            instr[name] = int(x.get("warp_instr", 0))
        json.dump({"source": f"{outdir}/ncu_full_summary.json (ncu --set full --clock-control none, every "
                             "event-stage launch of one push)",
                   "workload": f"{config} {mode}, one push of {ppl} frame pairs (tools/push_once.py)",
                   "pairs_per_launch": float(ppl),
                   "event_stage_dram_bytes_per_launch": sum(per.values()), "per_kernel_dram_bytes": per,
                   "per_kernel_warp_instr": instr},
                  open(os.path.join(outdir, f"traffic_{config}_{mode}.json"), "w"), indent=1)
    for x in out:
        print(f"{x['kernel'][:44]:44s} {x.get('dur_ms', 0):8.3f} ms  issue {x.get('issue_active_pct', 0):5.1f}%  "
              f"instr {x.get('warp_instr', 0):.3g}")


if __name__ == "__main__":
    main(*sys.argv[1:])
