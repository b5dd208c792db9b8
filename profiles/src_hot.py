"""Aggregate an ncu `--page source --csv --print-source sass,cuda` export per CUDA line.

usage: python profiles/src_hot.py export.csv [top_n]
Prints the top lines by warp-stall samples with their share, executed instructions and
average active threads, so traversal hot spots map back to device_scene.cuh / kernels.cu.
"""
import csv
import sys


def main(path, top=40):
    rows = []
    fname = None
    header = None
    with open(path, newline="") as f:
        for rec in csv.reader(f):
            if not rec:
                continue
            if rec[0] == "File Path":
                fname = rec[1].rsplit("/", 1)[-1]
                continue
            if rec[0] == "Line No":
                header = rec
                continue
            if header is None or rec[0] in ("Function Name",) or not rec[0].isdigit():
                continue
            d = dict(zip(header, rec))
            try:
                samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
                inst = int(d.get("Instructions Executed", "0") or 0)
                thr = float(d.get("Avg. Threads Executed", "0") or 0)
            except ValueError:
                continue
            rows.append((samp, inst, thr, fname, int(rec[0]), rec[1][:70]))
    total = sum(r[0] for r in rows) or 1
    rows.sort(reverse=True)
    print(f"total samples {total}")
    for s, i, t, fn, ln, src in rows[:top]:
        print(f"{100.0 * s / total:5.1f}%  inst={i:>10}  thr={t:5.1f}  {fn}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
