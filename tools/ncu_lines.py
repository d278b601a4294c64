"""Top source lines by warp-stall samples from `ncu -i rep --page source --csv --print-source cuda,sass`."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur = None
    agg = {}
    total = 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or r[0] == "":
            continue
        try:
            ln = int(r[0])
            samp = int(r[4]) if r[4] not in ("-", "") else 0
        except (ValueError, IndexError):
            continue
        agg[(cur, ln)] = (agg.get((cur, ln), (0, r[1]))[0] + samp, r[1])
        total += samp
    items = sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]
    print("total samples", total)
    for (f, ln), (s, src) in items:
        print("%6d %5.1f%%  %s:%d  %s" % (s, 100.0 * s / max(total, 1), f, ln, src.strip()[:90]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)


def stalls(path, keys):
    """Stall-reason breakdown for (file, line) keys, e.g. ["engine.cuh:558"]."""
    rows = list(csv.reader(open(path)))
    hdr = None
    cur = None
    out = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if r[0] in ("Function Name", ""):
            continue
        k = "%s:%s" % (cur, r[0])
        if k in keys:
            d = out.setdefault(k, {})
            for i in range(32, 49):
                try:
                    d[hdr[i]] = d.get(hdr[i], 0) + int(r[i])
                except (ValueError, IndexError):
                    pass
    for k, d in out.items():
        tops = sorted(d.items(), key=lambda kv: -kv[1])[:5]
        print(k, ", ".join("%s=%d" % kv for kv in tops))
