"""Markdown table of bench lines from the evidence pass.

    python tools/results_table.py gpurun_out/ev_default.json gpurun_out/ev_matrix.jsonl \
        --ref gpurun_out/ev_reference_c5.json gpurun_out/ev_reference.jsonl
"""
import argparse
import json


def lines(paths):
    out = []
    for p in paths:
        for ln in open(p):
            ln = ln.strip()
            if ln.startswith("{"):
                out.append(json.loads(ln))
    return out


def key(d):
    c = d.get("config", {})
    return (c.get("workload", "").split(":")[0], c.get("mode"), c.get("streams"), c.get("flow_preset"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("ours", nargs="+")
    ap.add_argument("--ref", nargs="*", default=[])
    a = ap.parse_args()
    ours = [d for d in lines(a.ours) if d.get("impl") != "reference" and "value" in d]
    refs = {key(d): d for d in lines(a.ref) if "value" in d}
    print("| Config | mode | streams | frames/s | e2e frames/s (format) | events/frame | chain | flow | emit "
          "| event-stage HBM frac | parity | reference (CPU) frames/s | CPU threads | x ref (e2e) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for d in ours:
        k = key(d)
        st = d["roofline"].get("stage_us_per_frame", {})
        r = refs.get(k)
        rv = r["value"] if r else (d.get("cpu_baseline") or {}).get("value")
        rc = r["cpu_baseline"]["cores"] if r else (d.get("cpu_baseline") or {}).get("cores")
        e2e = d.get("e2e") or {}
        ratio = f"{e2e['value'] / rv:,.0f}" if (rv and e2e.get("value")) else "–"
        name = k[0] + (" hq" if k[3] == "high_quality" else "")
        print(f"| {name} | {k[1]} | {k[2]} | {d['value']:,.1f} | {e2e.get('value', 0):,.1f} ({e2e.get('format', '-')}) "
              f"| {d.get('events_per_frame', 0):,.0f} | {st.get('chain', 0):.2f} | {st.get('flow', 0):.2f} "
              f"| {st.get('emit', 0):.2f} | {100 * d['roofline']['frac']:.2f} % | {d.get('parity')} "
              f"| {rv if rv is not None else '–'} | {rc if rc is not None else '–'} | {ratio} |")


if __name__ == "__main__":
    main()
