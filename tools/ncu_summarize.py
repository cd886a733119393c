"""Summarise committed ncu --set full captures (profiles/ncu/*.ncu-rep) into
profiles/ncu_summary.json entries: duration, DRAM bytes per launch, pipe
utilisation, shared-memory wavefronts, stall reasons.

    python tools/ncu_summarize.py <kernel-key> <report> "<workload>" ["note"]
"""

from __future__ import annotations

import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "msecond": 1e3,
         "nsecond": 1e-3}


def raw(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(d: dict, k: str, unit_to=None):
    if k not in d:
        return None
    v, u = d[k]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    if unit_to == "bytes":
        x *= SCALE.get(u, 1)
    if unit_to == "us":
        x *= SCALE.get(u, 1)
    return x


def stalls(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, data = rows[1], rows[2:]
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0) for r in data) or 1.0
    agg = {r: sum(float(x[hdr.index(r)] or 0) for x in data) / tot for r in reasons}
    return {k[6:]: round(v, 3) for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v > 0.02}


def main() -> None:
    key, rep, workload = sys.argv[1], sys.argv[2], sys.argv[3]
    note = sys.argv[4] if len(sys.argv) > 4 else ""
    d = raw(rep)
    dram = (num(d, "dram__bytes_read.sum", "bytes") or 0) + (num(d, "dram__bytes_write.sum", "bytes") or 0)
    entry = {
        "report": str(Path(rep).relative_to(ROOT)) if Path(rep).is_absolute() else rep,
        "workload": workload,
        "duration_us": num(d, "gpu__time_duration.sum", "us"),
        "dram_bytes_per_launch": int(dram),
        "sm_active_pct_of_elapsed": round(100 * (num(d, "sm__cycles_active.avg") or 0) /
                                          max(num(d, "sm__cycles_elapsed.avg") or 1, 1), 1),
        "tensor_pipe_active_pct": num(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
        "alu_pipe_active_pct": num(d, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        "fma_pipe_active_pct": num(d, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "smem_lsu_wavefronts_pct_of_peak": num(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
        "smem_tc_wavefronts_pct_of_peak": num(d, "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
        "smem_bank_conflicts": num(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "issue_active_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "l2_red_sectors": num(d, "lts__t_sectors_srcunit_tex_op_red.sum"),
        "stall_share": stalls(rep),
        "note": note,
    }
    p = ROOT / "profiles" / "ncu_summary.json"
    summ = json.loads(p.read_text())
    if key in summ and summ[key].get("report") != entry["report"]:
        summ.setdefault("history", {})[key + "_" + Path(summ[key]["report"]).stem] = summ[key]
    summ[key] = entry
    summ["_note"] = ("Per-launch figures read from the committed ncu --set full captures (profiles/ncu/*.ncu-rep). "
                     "dram bytes = dram__bytes_read.sum + dram__bytes_write.sum.")
    p.write_text(json.dumps(summ, indent=1))
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    main()
