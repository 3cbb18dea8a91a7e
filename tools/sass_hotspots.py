"""Top SASS instructions by warp-stall samples from `ncu -i REP --page source --csv --print-source sass`
exports: python tools/sass_hotspots.py kernel_sass.csv [N] -> markdown table."""
import csv
import sys


def main(path, n=20):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    col = {k: i for i, k in enumerate(hdr)}
    data = []
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr):
            continue
        try:
            samples = int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        data.append((samples, r[col["Source"]].strip(), r[col["Instructions Executed"]]))
    total = sum(d[0] for d in data) or 1
    print(f"{rows[0][1][:100]}: {len(data)} SASS instructions, {total} stall samples\n")
    print("| share | samples | instruction | executed (warp-level) |\n|---|---|---|---|")
    for s, src, ex in sorted(data, key=lambda d: -d[0])[:n]:
        print(f"| {100 * s / total:.1f}% | {s} | `{src[:70]}` | {ex} |")
    kinds = {}
    for s, src, _ in data:
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        kinds[op] = kinds.get(op, 0) + s
    print("\nBy opcode: " + ", ".join(f"{k} {100 * v / total:.0f}%" for k, v in sorted(kinds.items(), key=lambda x: -x[1])[:10]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
