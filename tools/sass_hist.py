"""Opcode histogram (executed instructions, stall samples) of one kernel from
`ncu -i X.ncu-rep --page source --csv --print-source sass -k regex:NAME > file.csv`."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Source" in r and "Instructions Executed" in r)
    iS, iN, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    tot, st = collections.Counter(), collections.Counter()
    for d in rows:
        if len(d) != len(hdr) or not d[iN].isdigit():
            continue
        toks = d[iS].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        tot[op] += int(d[iN])
        st[op] += int(d[iW] or 0)
    T, S = sum(tot.values()), max(1, sum(st.values()))
    print("executed warp instructions", T, "stall samples", S)
    for k, v in tot.most_common(top):
        print(f"{k:10s} {v:12d} {v / T:6.3f}  stall share {st[k] / S:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
