"""Stall-reason mix of one kernel and its top stalled SASS instructions (with the dominant reason),
from `ncu -i REP --page source --csv --print-source sass -k regex:NAME > file.csv`:
python tools/stall_mix.py file.csv [N]"""
import csv
import sys


def main(path, n=12):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    col = {k: i for i, k in enumerate(hdr)}
    reasons = [k for k in hdr if k.startswith("stall_")]
    tot = {k: 0 for k in reasons}
    ins = []
    seen = set()
    for r in rows[hi + 1:]:
        if len(r) < len(hdr) or r[col["Address"]] in seen:
            continue
        seen.add(r[col["Address"]])
        v = {k: int(r[col[k]] or 0) for k in reasons if (r[col[k]] or "0").isdigit()}
        for k, x in v.items():
            tot[k] += x
        s = sum(v.values())
        if s:
            ins.append((s, r[col["Source"]].strip(), max(v, key=v.get)))
    allv = sum(tot.values()) or 1
    print(f"{path}: {allv} stall samples")
    for k, x in sorted(tot.items(), key=lambda kv: -kv[1]):
        if x:
            print(f"  {k:28s} {x / allv:6.1%}")
    print("top instructions:")
    for s, src, why in sorted(ins, reverse=True)[:n]:
        print(f"  {s / allv:6.1%}  {why:20s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], *(int(a) for a in sys.argv[2:]))
