"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel for the
last step (kernels after the last embed_norm launch):
    python tools/launch_summary.py gpurun_out/launch_mixed.csv [label]"""
import collections
import csv
import sys


def summarise(path, label=None, marker="embed_norm"):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    starts = [i for i, d in enumerate(data) if marker in d["Kernel Name"]]
    start = starts[-1] if starts else 0
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for d in data[start:]:
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        name = name.split("<")[0].strip()
        tot[name] += float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1.0)
        cnt[name] += 1
    s = sum(tot.values())
    out = [f"== {label or path}: one step, {sum(cnt.values())} launches, {s / 1e3:.3f} ms "
           f"(ncu, serialised, cold caches: compare shares)"]
    for k, v in sorted(tot.items(), key=lambda t: -t[1]):
        out.append(f"  {k:34s} {cnt[k]:5d} launches {v / 1e3:8.3f} ms {100 * v / s:5.1f}%")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None))
