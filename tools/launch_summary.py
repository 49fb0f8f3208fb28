"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py gpurun_out/launches.csv "header line" > profiles/r01/ncu_launches_<tag>.txt
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path, header=""):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            agg[r[ki][:72]].append(float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0))
    tot = sum(sum(v) for v in agg.values())
    if header:
        print("# " + header)
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:72s} n={len(v):4d} mean={sum(v) / len(v):10.2f}us share={100 * sum(v) / tot:5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
