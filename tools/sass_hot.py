"""Top SASS instructions by warp-stall samples from an ncu report:
    python tools/sass_hot.py report.ncu-rep [N]"""
import csv
import subprocess
import sys


def main(path, n=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    h = rows[0]
    ia, isrc, ismp = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[1:] if len(r) == len(h)]
    tot = sum(float(r[ismp] or 0) for r in data)
    print(f"total samples {tot:.0f}, {len(data)} instructions")
    idx = sorted(range(len(data)), key=lambda i: -float(data[i][ismp] or 0))[:n]
    for i in idx:
        r = data[i]
        print(f"{100 * float(r[ismp]) / tot:5.1f}%  {r[ia]}  {r[isrc][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
