"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel count, time, share."""
import collections
import csv
import re
import sys


def kname(s):
    s = s.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    s = re.sub(r"^void ", "", s)
    base = s.split("(")[0]
    m = re.match(r"([A-Za-z_0-9]+)(<[^>]*>)?", base)
    return (m.group(1) + (m.group(2) or "")) if m else base


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale[r[ui]]
        n = kname(r[ki])
        tot[n] += v
        cnt[n] += 1
    T = sum(tot.values())
    out = ["total %.1f us over %d launches" % (T, sum(cnt.values()))]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append("%-34s %6d launches %11.1f us %6.2f%%" % (k, cnt[k], v, 100 * v / T))
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
