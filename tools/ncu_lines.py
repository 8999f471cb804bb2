"""Per-source-line stall samples and instruction counts from an ncu report.

  python tools/ncu_lines.py REPORT.ncu-rep [top=40]

Runs `ncu -i REPORT --page source --csv --print-source cuda,sass` and sums the
source-line rows (warp stall samples, executed warp instructions, top stall
reasons) across files, sorted by samples."""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True, check=True).stdout
    fname, hdr = "?", None
    lines = []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0] or len(r) < 8:
            continue
        try:
            s = int(r[4])
            n = int(r[7])
        except ValueError:
            continue
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    v = int(r[i])
                except ValueError:
                    continue
                if v:
                    stalls[h[6:]] = v
        lines.append((s, n, f"{fname}:{r[0]}", r[1].strip()[:90], stalls))
    tot = sum(x[0] for x in lines)
    print(f"total samples {tot}, warp instructions {sum(x[1] for x in lines)}")
    for s, n, loc, src, st in sorted(lines, reverse=True)[:top]:
        top3 = ", ".join(f"{k} {v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
        print(f"{s:6d} {100 * s / tot:5.1f}% {n:9d}  {loc:22s} {src}\n{'':40s}[{top3}]")


if __name__ == "__main__":
    main()
