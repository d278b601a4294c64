"""Kernel time shares from an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file F`)."""
import collections
import csv
import json
import sys


def share(path, skip_until=None):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0][:90]
        v = float(r["Metric Value"]) * (1e3 if r.get("Metric Unit") == "us" else 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [{"kernel": k, "launches": v[0], "ms": v[1] / 1e6, "share": v[1] / tot}
           for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    return {"total_ms": tot / 1e6, "launches": sum(v[0] for v in agg.values()), "kernels": out}


if __name__ == "__main__":
    s = share(sys.argv[1])
    print("total %.1f ms over %d launches" % (s["total_ms"], s["launches"]))
    for k in s["kernels"][:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
        print("%5d %10.3f ms %5.1f%%  %s" % (k["launches"], k["ms"], 100 * k["share"], k["kernel"]))
