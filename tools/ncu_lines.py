"""Aggregate ncu warp-stall samples per CUDA source line.

    ncu -i rep.ncu-rep --page source --csv --print-source=cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [topN]
"""
import csv
import sys


def main(path, top=25):
    rows = []
    cur_file = "?"
    with open(path) as f:
        for row in csv.reader(f):
            if len(row) >= 2 and row[0] in ("File Path", "File Name"):
                cur_file = row[1].split("/")[-1]
                continue
            if len(row) > 6 and row[0] not in ("", "Line No"):
                try:
                    s = int(row[4])
                except ValueError:
                    continue
                if s:
                    rows.append((s, cur_file, row[0], row[1].strip()[:100]))
    tot = sum(r[0] for r in rows) or 1
    rows.sort(reverse=True)
    print(f"total samples {tot}")
    for s, fn, ln, src in rows[:top]:
        print(f"{100.0 * s / tot:5.1f}%  {fn}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
