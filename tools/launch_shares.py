"""Per-kernel time shares from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def main(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.OrderedDict(), collections.Counter()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        tot[r[ki]] = tot.get(r[ki], 0.0) + v
        cnt[r[ki]] += 1
    T = sum(tot.values())
    print("launch list %s: %d launches, %.1f ms total (cold-cache, serialised by ncu)" % (path, sum(cnt.values()), T))
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print("%10.2f ms %6.2f%%  x%-4d %s" % (v, 100 * v / T, cnt[k], k))


if __name__ == "__main__":
    main(sys.argv[1])
