"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel name, total device time, launch count and share.  Serialised,
cold-cache times -- compare shares, not absolutes.

    python tools/launch_shares.py gpurun_out/launches.csv [--seq]

--seq also prints every launch in order (name, us).
"""
import csv
import sys
from collections import OrderedDict


def rows(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        us = v / 1e3 if unit.startswith("n") else (v if unit.startswith("u") else v * 1e3)
        yield r["Kernel Name"], us


def main():
    path = sys.argv[1]
    seq = list(rows(path))
    tot = OrderedDict()
    for name, us in seq:
        t, c = tot.get(name, (0.0, 0))
        tot[name] = (t + us, c + 1)
    all_us = sum(t for t, _ in tot.values())
    print(f"# {path}: {len(seq)} launches, {all_us:.1f} us total")
    for name, (t, c) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
        print(f"{t:10.1f} us {c:5d}x {100 * t / all_us:5.1f}%  {name[:90]}")
    if "--seq" in sys.argv:
        for name, us in seq:
            print(f"  {us:9.1f}  {name[:80]}")


if __name__ == "__main__":
    main()
