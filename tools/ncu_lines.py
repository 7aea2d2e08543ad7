"""Aggregate an ncu report's source page per CUDA source line: warp-stall samples and
executed instructions, hottest first (development aid for reading --set full captures).
Usage: ncu_lines.py report.ncu-rep [top_n]"""
import csv
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True, check=True).stdout.splitlines()
    rows, fname, hdr = [], None, None
    for l in out:
        r = next(csv.reader([l]))
        if not r:
            continue
        if r[0] == "File Path":
            fname, hdr = r[1].rsplit("/", 1)[-1], None
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "":
            continue  # SASS rows under a source line
        d = dict(zip(hdr[:4] + hdr[4:], r))
        try:
            samples = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            inst = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        rows.append((samples, inst, fname, r[0], r[1].strip()[:90]))
    tot_s = sum(x[0] for x in rows) or 1
    tot_i = sum(x[1] for x in rows) or 1
    print(f"{'stall%':>7s} {'inst%':>7s}  location")
    for s, i, f, ln, src in sorted(rows, reverse=True)[:top]:
        print(f"{100 * s / tot_s:7.2f} {100 * i / tot_i:7.2f}  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
