"""Summarise ncu `--page details --csv` + `--page raw --csv` exports (taken on
the GPU box, so the multi-GB .ncu-rep never travels) into one JSON object:
duration, DRAM bytes, L2 hit rate, IPC, instructions, occupancy, top stalls.
usage: python tools/ncu_csv_summary.py DETAILS.csv RAW.csv [label]"""
import csv
import json
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Executed Ipc Active", "Executed Instructions", "Achieved Active Warps Per SM",
        "Registers Per Thread", "Compute (SM) Throughput", "Warp Cycles Per Issued Instruction",
        "Grid Size", "Block Size", "Dynamic Shared Memory Per Block", "Theoretical Occupancy"]


def summarise(details, raw, label=""):
    out = {"label": label}
    rows = list(csv.reader(open(details)))
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in WANT and d["Metric Name"] not in out:
            out[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
        out.setdefault("kernel", d.get("Kernel Name", "")[:120])
    rows = list(csv.reader(open(raw)))
    hdr, units = rows[0], rows[1]
    d = dict(zip(hdr, rows[2]))
    u = dict(zip(hdr, units))
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
              "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct"):
        if k in d:
            out[k] = f"{d[k]} {u.get(k, '')}".strip()
    pre = "smsp__average_warps_issue_stalled_"
    st = {k[len(pre):].replace("_per_issue_active.ratio", ""): v for k, v in d.items()
          if k.startswith(pre) and k.endswith("_per_issue_active.ratio")}
    st = {k: float(v) for k, v in st.items() if v not in ("", "n/a")}
    out["stall_cycles_per_instruction"] = dict(sorted(st.items(), key=lambda x: -x[1])[:8])
    return out


if __name__ == "__main__":
    print(json.dumps(summarise(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""),
                     indent=1))
