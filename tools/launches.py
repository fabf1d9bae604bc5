"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys


def summarise(path, per=1):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("fs::<unnamed>::", "").replace("void ", "")[-48:]
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
        v *= scale.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':48s} {'launches':>8s} {'total_us':>11s} {'share':>6s} {'avg_us':>9s} {'per_view_us':>11s}"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k:48s} {c:8d} {t:11.1f} {100 * t / tot:5.1f}% {t / c:9.1f} {t / per:11.1f}")
    lines.append(f"{'TOTAL':48s} {'':8s} {tot:11.1f}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1))
