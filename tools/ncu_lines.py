"""Per-source-line instruction and stall-sample shares of an ncu --set full capture
(--import-source on, -lineinfo build): the hot lines of a kernel.

    python tools/ncu_lines.py <file.ncu-rep> [TOP]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, data = "?", []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
        elif r and r[0].isdigit() and len(r) > 7:
            try:
                data.append((int(r[7] or 0), int(r[4] or 0), f"{fname}:{r[0]}", r[1].strip()[:90]))
            except ValueError:
                pass
    ti = sum(d[0] for d in data) or 1
    ts = sum(d[1] for d in data) or 1
    print(f"# {rep}: {ti} warp instructions, {ts} stall samples")
    for ie, st, loc, src in sorted(data, reverse=True)[:top]:
        print(f"{100 * ie / ti:5.1f}% inst {100 * st / ts:5.1f}% samples  {loc:18s} {src}")


if __name__ == "__main__":
    main()
