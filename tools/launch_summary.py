"""Summarise an ncu launch-list CSV (gpu__time_duration per launch) by kernel."""
import collections
import csv
import sys


def summarize(path, out=sys.stdout):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    data = rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in data:
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    s = sum(tot.values())
    print(f"# {path}: {len(data)} launches, {s / 1e6:.3f} ms total (cold-cache, serialised)", file=out)
    print(f"{'ms':>9} {'share':>6} {'n':>4}  kernel", file=out)
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v / 1e6:9.3f} {100 * v / s:5.1f}% {cnt[k]:4d}  {k}", file=out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summarize(p)
