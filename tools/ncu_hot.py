"""Top SASS instructions of an .ncu-rep by warp-stall samples (with the dominant stall reasons)."""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ix = {n: i for i, n in enumerate(h)}
    stalls = [n for n in h if n.startswith("stall_")]
    body = [r for r in rows[2:] if len(r) == len(h)]
    tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
    print("total samples", tot)
    seq = {r[0]: i for i, r in enumerate(body)}
    for r in sorted(body, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:top]:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        st = sorted(((int(float(r[ix[n]] or 0)), n[6:]) for n in stalls), reverse=True)[:3]
        print(f"{seq[r[0]]:5d} {s:6d} {100*s/tot:5.1f}%  {r[1].strip()[:60]:60s} {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
