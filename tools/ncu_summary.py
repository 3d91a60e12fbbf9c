"""Summarise one ncu --set full report (first kernel) into the JSON kept under profiles/.

    python tools/ncu_summary.py gpurun_out/r/prof_c2_none.ncu-rep profiles/r01/ncu_ra_tc_c2_none_summary.json \
        [--traffic profiles/traffic_c2_none.json --label "C2 layer, mode none"]
"""
import argparse
import csv
import json
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--traffic")
    ap.add_argument("--label", default="")
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    summ = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            summ[k] = f"{vals[i]} {units[i]}".strip()
    json.dump(summ, open(a.out, "w"), indent=0)
    if a.traffic:
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(k)
            tot += float(vals[i].replace(",", "")) * SCALE.get(units[i], 1)
        json.dump({"dram_bytes_per_launch": int(tot), "source": f"ncu --set full, one ra_tc_kernel launch ({a.label}), {a.out}"},
                  open(a.traffic, "w"), indent=1)
    print(json.dumps(summ, indent=0))


if __name__ == "__main__":
    main()
