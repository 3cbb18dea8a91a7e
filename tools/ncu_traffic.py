"""profiles/ncu_traffic.json from `ncu -i REPORT --page raw --csv` exports of full-size captures
(tools/profile_case.py c4 256 / c2 4096 / c5 32768): per kernel, the SURVEY §8(d) step-5 counters —
DRAM bytes per launch next to the algorithmic bytes (8 B per sample per transform), DRAM
throughput as % of peak, global store sectors per request, shared-memory bank conflicts.  bench.py
reads `dram_bytes_per_launch` as the roofline's `traffic`.
python tools/ncu_traffic.py out.json c4=raw_c4.csv [c2=raw_c2.csv c5=raw_c5.csv]"""
import csv
import json
import os
import sys

SAMPLES = {"c4": 256 * 2048 * 2048, "c2": 4096 * 65536, "c5": 32768 * 32768}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1, "us": 1e-3, "ns": 1e-6}


def kind(name):
    if "ana2d" in name or "ana1d" in name:
        return "analysis"
    if "syn2d" in name or "syn1d" in name:
        return "synthesis"
    return None


def main(out, *specs):
    res = {"_source": "ncu --set full --clock-control none on tools/profile_case.py <workload> at full size "
                      "(largest launch of each kind); dram bytes = dram__bytes_read.sum + dram__bytes_write.sum, "
                      "dram_throughput_pct = gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed, "
                      "store sectors/request = l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum / "
                      "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum (4 = full 128-B lines per request), "
                      "smem bank conflicts = l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_{ld,st}.sum"}
    if os.path.exists(out):   # merge: a capture per kernel file updates only that workload / kind
        old = json.load(open(out))
        old.update({k: v for k, v in res.items() if k == "_source"})
        res = old
    for spec in specs:
        wl, path = spec.split("=")
        rows = list(csv.reader(open(path)))
        hdr, units = rows[0], rows[1]
        col = {k: i for i, k in enumerate(hdr)}

        def val(r, k):
            if k not in col or not r[col[k]]:
                return None
            return float(r[col[k]].replace(",", "")) * SCALE.get(units[col[k]], 1)

        def ratio(r, a, b):
            x, y = val(r, a), val(r, b)
            return x / y if x is not None and y else None

        best = {}
        for r in rows[2:]:
            name = r[col["Kernel Name"]]
            k = kind(name)
            if not k:
                continue
            rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
            if k not in best or rd + wr > best[k]["dram_bytes_per_launch"]:
                alg = 8 * SAMPLES[wl]
                best[k] = {
                    "kernel": name, "dram_bytes_per_launch": rd + wr, "dram_read_bytes_per_launch": rd,
                    "dram_write_bytes_per_launch": wr, "algorithmic_bytes_per_launch": alg,
                    "traffic_over_algorithmic": (rd + wr) / alg,
                    "ncu_duration_ms": val(r, "gpu__time_duration.sum"),
                    "dram_throughput_pct": val(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                    "global_store_sectors_per_request": ratio(r, "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
                                                              "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum"),
                    "global_load_sectors_per_request": ratio(r, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
                                                             "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
                    "l2_write_sectors_per_request": ratio(r, "lts__t_sectors_srcunit_tex_op_write.sum",
                                                          "lts__t_requests_srcunit_tex_op_write.sum"),
                    "smem_bank_conflicts_ld": val(r, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
                    "smem_bank_conflicts_st": val(r, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"),
                    "smem_wavefronts_ld": val(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"),
                    "smem_wavefronts_st": val(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum"),
                    "registers_per_thread": val(r, "launch__registers_per_thread"),
                    "issue_active_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                }
        res.setdefault(wl, {}).update(best)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
