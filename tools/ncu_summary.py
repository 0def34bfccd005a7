"""Summarise an `ncu --set full` capture of the tile kernel into profiles/.

    python tools/ncu_summary.py gpurun_out/<tag>.ncu-rep <tag>

Writes profiles/<tag>_ncu.txt (pipe utilisation, issue, stalls, DRAM traffic, occupancy)
and profiles/ncu_summary.json (per-launch DRAM bytes, read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe (POPC) % of peak"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe (LOP3/VIMNMX) % of peak"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % of peak"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    d = {k: (v, u) for k, u, v in zip(head, units, vals)}
    out = [f"ncu --set full, {os.path.basename(rep)}: {d.get('Kernel Name', ('?', ''))[0]}"]
    for k, label in KEYS:
        if k in d:
            out.append(f"  {label:38s} {d[k][0]} {d[k][1]}")
    stalls = sorted(((k, float(v or 0)) for k, (v, u) in d.items()
                     if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")),
                    key=lambda t: -t[1])
    out.append("  stall reasons (warps per issue):")
    for k, v in stalls[:8]:
        out.append(f"    {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):24s} {v:.3f}")
    dram = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v, u = d[k]
        dram += float(v) * SCALE.get(u, 1)
    out.append(f"  DRAM bytes per launch (read+write)      {dram:.0f}")
    text = "\n".join(out) + "\n"
    print(text)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu.txt"), "w") as f:
        f.write(text)
    summ = {"dram_bytes_per_launch": dram, "source": f"profiles/{tag}_ncu.txt ({os.path.basename(rep)})",
            "xu_pct": float(d["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"][0]),
            "alu_pct": float(d["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"][0])}
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
        json.dump(summ, f, indent=1)


if __name__ == "__main__":
    main()
