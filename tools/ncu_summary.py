"""Summarise an ncu report (run in the build container: ncu -i works without
a GPU).  Prints and optionally writes the metrics the roofline needs."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "launch__occupancy_limit_registers": "occ_limit_regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_peak",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct_peak",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "")[:90]}
        for m, name in KEYS.items():
            if m in d:
                k[name] = d[m]
                k[name + "_unit"] = u.get(m, "")
        res.append(k)
    return res


def stalls(rep, top=8):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    d = dict(zip(hdr, rows[2]))
    pre = "smsp__average_warps_issue_stalled_"
    st = {k[len(pre):].replace("_per_issue_active.ratio", ""): v
          for k, v in d.items() if k.startswith(pre) and k.endswith("_per_issue_active.ratio")}
    st = {k: float(v.replace(",", "")) for k, v in st.items() if v not in ("", "n/a")}
    return dict(sorted(st.items(), key=lambda x: -x[1])[:top])


if __name__ == "__main__":
    rep = sys.argv[1]
    summary = {"kernels": raw(rep)}
    try:
        summary["stall_cycles_per_instruction"] = stalls(rep)
    except Exception as e:  # noqa: BLE001
        summary["stall_error"] = str(e)
    js = json.dumps(summary, indent=1)
    print(js)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(js)
