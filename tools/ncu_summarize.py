"""Summarise ncu --set full captures into profiles/ (dev helper):
  python tools/ncu_summarize.py TAG kernel=report.ncu-rep:units[:unit_name] ...
writes profiles/ncu_summary.json ("kernels": {kernel: {...}}, read by bench.py) and one
profiles/<TAG>_<kernel>_ncu_summary.txt per capture (key metrics + top source lines)."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "gpu__time_duration.sum": "time_ms_or_us",
    "sm__cycles_elapsed.max": "sm_cycles",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__inst_executed.avg.per_cycle_active": "ipc_per_sm",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__occupancy_limit_registers": "occupancy_limit_registers",
    "smsp__average_warp_latency_issue_stalled.ratio": "stall_ratio",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = {}
    for i, name in enumerate(h):
        if name in KEYS:
            try:
                val = float(v[i].replace(",", ""))
            except ValueError:
                continue
            unit = u[i]
            if name.startswith("dram__bytes"):
                val *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            if name == "gpu__time_duration.sum":
                val *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1)
                d["time_ms"] = val
                continue
            d[KEYS[name]] = val
    return d


def main():
    tag = sys.argv[1]
    outdir = os.environ.get("OUTDIR", os.path.join(ROOT, "profiles"))
    os.makedirs(outdir, exist_ok=True)
    path = os.path.join(outdir, "ncu_summary.json")
    try:
        summ = json.load(open(path))
        if "kernels" not in summ:
            summ = {"kernels": {}}
    except Exception:
        summ = {"kernels": {}}
    for spec in sys.argv[2:]:
        kern, rest = spec.split("=", 1)
        parts = rest.split(":")
        rep, units = parts[0], float(parts[1])
        uname = parts[2] if len(parts) > 2 else "accepted swap"
        d = raw(rep)
        d["dram_bytes_per_launch"] = d.pop("dram_read", 0.0) + d.pop("dram_write", 0.0)
        d["units"] = units
        d["unit"] = uname
        d["warp_instructions_per_unit"] = d.get("warp_instructions", 0) / units
        d["sm_cycles_per_unit"] = d.get("sm_cycles", 0) / units
        d["capture"] = f"{tag}: ncu --set full --clock-control none --import-source on, {os.path.basename(rep)}"
        summ["kernels"][kern] = d
        lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "25", str(units)],
                               capture_output=True, text=True).stdout
        with open(os.path.join(outdir, f"{tag}_{kern}_ncu_summary.txt"), "w") as f:
            f.write(f"{kern}: {d['capture']}\n")
            for k, v in d.items():
                if k != "capture":
                    f.write(f"  {k}: {v}\n")
            f.write(f"\nTop source lines by stall samples (inst/n = warp instructions per {uname}):\n")
            f.write(lines)
    summ["round"] = tag
    with open(path, "w") as f:
        json.dump(summ, f, indent=1)


if __name__ == "__main__":
    main()
