"""Executed-instruction mix by SASS opcode from an ncu report:
    python tools/sass_mix.py report.ncu-rep [N]"""
import collections
import csv
import subprocess
import sys


def main(path, n=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    h = rows[0]
    isrc, iex, ismp = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    cnt, smp = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if len(r) != len(h):
            continue
        toks = r[isrc].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        cnt[op] += float(r[iex] or 0)
        smp[op] += float(r[ismp] or 0)
    tot, ts = sum(cnt.values()), sum(smp.values())
    print(f"total warp-instructions {tot:.3e}")
    for op, c in cnt.most_common(n):
        print(f"{op:28s} {c:12.0f} {100 * c / tot:5.1f}%  stall-samples {100 * smp[op] / max(ts, 1):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
