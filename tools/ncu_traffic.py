"""profiles/ncu_traffic.json from `ncu -i REPORT --page raw --csv` exports of full-size captures
(tools/profile_case.py c4 256 / c2 4096 / c5 32768): per kernel, DRAM bytes per launch next to
the algorithmic bytes (8 B per sample per transform).  bench.py reads the result as `traffic`.
python tools/ncu_traffic.py out.json c4=raw_c4.csv [c2=raw_c2.csv c5=raw_c5.csv]"""
import csv
import json
import sys

SAMPLES = {"c4": 256 * 2048 * 2048, "c2": 4096 * 65536, "c5": 32768 * 32768}


def kind(name):
    if "ana2d" in name or "ana1d" in name:
        return "analysis"
    if "syn2d" in name or "syn1d" in name:
        return "synthesis"
    return None


def main(out, *specs):
    res = {"_source": "ncu --set full --clock-control none on tools/profile_case.py <workload> at full size; "
                      "dram__bytes_read.sum + dram__bytes_write.sum per launch (largest launch of each kind)"}
    for spec in specs:
        wl, path = spec.split("=")
        rows = list(csv.reader(open(path)))
        hdr, units = rows[0], rows[1]
        col = {k: i for i, k in enumerate(hdr)}

        def val(r, k):
            u = units[col[k]]
            v = float(r[col[k]].replace(",", ""))
            return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1, "us": 1e-3}.get(u, 1)

        best = {}
        for r in rows[2:]:
            name = r[col["Kernel Name"]]
            k = kind(name)
            if not k:
                continue
            rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
            if k not in best or rd + wr > best[k]["dram_bytes_per_launch"]:
                alg = 8 * SAMPLES[wl]
                best[k] = {"kernel": name, "dram_bytes_per_launch": rd + wr, "dram_read_bytes_per_launch": rd,
                           "dram_write_bytes_per_launch": wr, "algorithmic_bytes_per_launch": alg,
                           "traffic_over_algorithmic": (rd + wr) / alg,
                           "ncu_duration_ms": val(r, "gpu__time_duration.sum"),
                           "dram_throughput_pct": r[col.get("dram__throughput.avg.pct_of_peak_sustained_elapsed",
                                                            col["gpu__time_duration.sum"])]}
        res[wl] = best
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
