"""Hottest source lines of one kernel in an ncu report (--page source, cuda view).

    python tools/ncu_source_hot.py rep.ncu-rep "dense_lk_warp_kernel<(int)4, (bool)1>" [N]
"""
import csv
import io
import subprocess
import sys


def main(rep, fn, n=25):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] in ("File Path", "File Name"):
            cur = {"file": r[1], "rows": []}
            blocks.append(cur)
        elif r and r[0] == "Function Name" and cur is not None:
            cur["fn"] = r[1]
        elif r and r[0] == "Line No" and cur is not None:
            cur["hdr"] = r
        elif cur is not None and "hdr" in cur:
            cur["rows"].append(r)
    lines = []
    for b in blocks:
        if fn not in b.get("fn", ""):
            continue
        h = b["hdr"]
        ii, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
        f = b["file"].split("/")[-1]
        for r in b["rows"]:
            if len(r) > max(ii, si) and r[0]:
                try:
                    iv = int(r[ii]) if r[ii] not in ("-", "") else 0
                    sv = int(r[si]) if r[si] not in ("-", "") else 0
                except ValueError:  # source text with quotes breaks ncu's CSV quoting
                    continue
                if iv or sv:
                    lines.append((f"{f}:{r[0]}", r[1].strip()[:90], iv, sv))
    ti = sum(x[2] for x in lines) or 1
    ts = sum(x[3] for x in lines) or 1
    print(f"{fn}: {ti:.4g} warp instructions, {ts} stall samples")
    for x in sorted(lines, key=lambda x: -x[2])[:int(n)]:
        print(f"{x[0]:>26} instr {100 * x[2] / ti:5.1f}%  stall {100 * x[3] / ts:5.1f}%  {x[1]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
