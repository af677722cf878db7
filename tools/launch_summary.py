"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)
into a per-kernel markdown table: python tools/launch_summary.py launches.csv"""
import csv
import collections
import sys


def main(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    head = rows[0]
    ki, mi, vi = head.index("Kernel Name"), head.index("Metric Name"), head.index("Metric Value")
    idi = head.index("ID")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    seen = set()
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        key = (r[idi], r[ki])
        if key in seen:
            continue
        seen.add(key)
        v = float(r[vi].replace(",", ""))
        unit = r[head.index("Metric Unit")]
        us = v * {"nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        tot[r[ki]] += us
        cnt[r[ki]] += 1
    allus = sum(tot.values())
    print("| kernel | launches | total us | share | avg us |")
    print("|---|---|---|---|---|")
    for k, us in sorted(tot.items(), key=lambda kv: -kv[1]):
        if us / allus < 0.005:
            continue
        name = k.replace("(anonymous namespace)::", "").replace("unnamed>::", "").split("(")[0]
        print(f"| {name} | {cnt[k]} | {us:.0f} | {100 * us / allus:.1f}% | {us / cnt[k]:.1f} |")
    print(f"\ntotal {allus:.0f} us, {sum(cnt.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
