"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel: share, total, count."""
import csv
import sys
from collections import defaultdict


def main(path, title=""):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        ms = v / 1e6 if unit == "nsecond" else v / 1e3 if unit in ("usecond", "us") else v if unit == "msecond" else v / 1e6
        name = r["Kernel Name"]
        tot[name] += ms
        cnt[name] += 1
    total = sum(tot.values())
    if title:
        print(title)
    print(f"{len(rows)} launches, {total:.3f} ms total GPU time\n")
    print(f"{'share':>8} {'total_ms':>10} {'launches':>9}  kernel")
    for name, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{100 * ms / total:7.2f}% {ms:10.3f} {cnt[name]:9d}  {name[:110]}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
