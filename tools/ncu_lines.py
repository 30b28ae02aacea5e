"""Top source lines by warp-stall samples from an ncu report's mixed source/SASS CSV export:
ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X.csv; python tools/ncu_lines.py X.csv [N]"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    cur, hdr, out = None, None, []
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) >= 2 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 5 or r[0] == "" or r[2] != "-":
            continue
        try:
            out.append((float(r[4]), cur, r[0], r[1].strip()[:96]))
        except ValueError:
            pass
    tot = sum(o[0] for o in out)
    out.sort(key=lambda x: -x[0])
    print(f"total samples {tot:.0f}")
    for o in out[:n]:
        print(f"{o[0] / tot * 100:5.1f}% {o[1]}:{o[2]} {o[3]}")


if __name__ == "__main__":
    main()
