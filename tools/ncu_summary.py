"""Summarise one kernel of an `ncu --set full` report into a small JSON for profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep --kernel k6_gemm_i8 --config c3 --out profiles/gemm_ncu_summary.json

Reads `ncu -i REPORT --page raw --csv` and keeps the metrics the roofline and the VERDICT need:
duration, DRAM bytes read/written (the `traffic` field of bench.py's roofline object), achieved
DRAM bandwidth, SM / tensor-pipe / issue utilisation, registers, shared memory and occupancy.
"""
import argparse
import csv
import io
import json
import subprocess

KEEP = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_peak",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active": "pipe_uniform_pct",
    "sm__pipe_tensor_op_tmem_cycles_active.avg.pct_of_peak_sustained_active": "tensor_tmem_pct",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active": "tensor_tc_pct",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active": "issue_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1, "cycle/nsecond": 1e9,
         "cycle/usecond": 1e6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--config", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    name_col = hdr.index("Kernel Name")
    sel = [r for r in data if a.kernel in r[name_col]]
    if not sel:
        raise SystemExit(f"no kernel matching {a.kernel}")
    out = {"config": a.config, "kernel": sel[0][name_col], "launches_captured": len(sel), "note": a.note,
           "source": a.report.split("/")[-1]}
    per = []
    for r in sel:
        d = {}
        for m, key in KEEP.items():
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    d[key] = float(v) * SCALE.get(units[i], 1.0)
                    d[key + "_unit"] = "SI" if units[i] in SCALE else units[i]
                except ValueError:
                    d[key] = v
        per.append(d)
    first = per[0]
    out["metrics"] = {k: v for k, v in first.items() if not k.endswith("_unit")}
    if "dram_read" in first and "dram_write" in first:
        out["dram_bytes_per_launch"] = first["dram_read"] + first["dram_write"]
        if first.get("duration"):
            out["dram_gbps"] = out["dram_bytes_per_launch"] / first["duration"] / 1e9
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
