"""Markdown summary of an `ncu --metrics gpu__time_duration.sum --csv --log-file X` launch list:
launches, total and share per kernel.  python tools/launch_list.py launches.csv > summary.md"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = next(r for r in rows if "Kernel Name" in r)
    ik, im, iv, iu = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows:
        if r is hdr or r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", "")) * {"ms": 1e3, "us": 1.0, "ns": 1e-3}.get(r[iu], 1.0)
        tot[r[ik]] += v
        cnt[r[ik]] += 1
    T = sum(tot.values())
    print("| kernel | launches | total µs | share |\n|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| `{k[:90]}` | {cnt[k]} | {v:.1f} | {100 * v / T:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
