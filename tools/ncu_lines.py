"""Aggregate ncu source-page warp-stall samples per CUDA source line.

  python tools/ncu_lines.py gpurun_out/prof.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = []
    fname = ""
    hdr = None
    for line in out.splitlines():
        if line.startswith('"File Path"'):
            fname = line.split(",", 1)[1].strip('"').split("/")[-1]
            continue
        if line.startswith('"Function Name"'):
            continue
        if line.startswith('"Line No"'):
            hdr = next(csv.reader(io.StringIO(line)))
            continue
        if hdr is None:
            continue
        r = next(csv.reader(io.StringIO(line)))
        if r and r[0] not in ("", "-"):
            d = dict(zip(hdr, r))
            try:
                s = int(d["Warp Stall Sampling (All Samples)"])
            except (ValueError, KeyError):
                continue
            stalls = {k: int(v) for k, v in zip(hdr[31:48], r[31:48]) if v.isdigit() and int(v)}
            rows.append((s, fname, r[0], r[1].strip()[:90], stalls))
    tot = sum(x[0] for x in rows) or 1
    rows.sort(key=lambda x: -x[0])
    for s, f, ln, src, st in rows[:top]:
        big = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        bs = " ".join(f"{k.replace('stall_', '')}={v * 100 // max(s, 1)}%" for k, v in big)
        print(f"{100 * s / tot:5.1f}% {f}:{ln:>5} {src:90s} | {bs}")


if __name__ == "__main__":
    main()
