"""Summarise an ncu capture / launch list into profiles/ (JSON).

    python tools/ncu_summary.py report <file.ncu-rep | raw.csv> <out.json> <algorithmic_bytes | 0> [note]
    python tools/ncu_summary.py launches <launches.csv> <out.json>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def _scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
            "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}.get(unit, 1.0)


def _raw_rows(path):
    """Rows of `ncu -i <rep> --page raw --csv` (a .ncu-rep is exported first; a .csv is read as is)."""
    if path.endswith(".ncu-rep"):
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    else:
        raw = open(path).read()
    rows = list(csv.reader(io.StringIO(raw)))
    return rows[0], rows[1], rows[2:]


def _one(h, u, r, alg_bytes, peak_gbs):
    def g(k):
        return float(r[h.index(k)].replace(",", "")) * _scale(u[h.index(k)]) if k in h else None

    def f(k):
        return float(r[h.index(k)].replace(",", "")) if k in h else None

    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(r[h.index(k)])
              for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    stalls = {k: v for k, v in sorted(stalls.items(), key=lambda kv: -kv[1]) if v > 0.05}
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    dur = g("gpu__time_duration.sum")
    res = {"kernel": r[h.index("Kernel Name")], "duration_us": dur * 1e6,
           "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
           "dram_GBps_during_kernel": (rd + wr) / dur / 1e9,
           "dram_frac_of_measured_peak": (rd + wr) / dur / 1e9 / peak_gbs,
           "dram_throughput_pct_of_peak": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
           "registers_per_thread": f("launch__registers_per_thread"),
           "block_size": f("launch__block_size"), "grid_size": f("launch__grid_size"),
           "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
           "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
           "l2_hit_rate_pct": f("lts__t_sector_hit_rate.pct"),
           "fp64_pipe_pct": f("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
           "instructions": f("smsp__inst_executed.sum"), "stall_reasons_per_issue": stalls}
    if alg_bytes:
        res.update({"algorithmic_bytes_per_launch": alg_bytes, "traffic_over_algorithmic": (rd + wr) / alg_bytes,
                    "algorithmic_GBps": alg_bytes / dur / 1e9, "algorithmic_frac_of_measured_peak": alg_bytes / dur / 1e9 / peak_gbs})
    return res


def report(path, out, alg_bytes, note="", peak_gbs=6542.4):
    """Every captured launch of a `--set full` report (or its raw CSV export)."""
    h, u, rows = _raw_rows(path)
    launches_ = [_one(h, u, r, alg_bytes, peak_gbs) for r in rows if r and r[0] != ""]
    res = {"source": path, "note": note, "peak_GBps": peak_gbs, "launches": launches_}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:2500])


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = defaultdict(lambda: defaultdict(float))
    count = defaultdict(int)
    seen = set()
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0]
        key = (r[0], name)
        if key not in seen:
            seen.add(key)
            count[name] += 1
        per[name][r[mi]] += float(r[vi].replace(",", "")) * _scale(r[ui])
    tot = sum(v.get("gpu__time_duration.sum", 0.0) for v in per.values())
    res = {"source": path, "total_device_time_us": tot * 1e6, "kernels": {
        k: {"launches": count[k], "time_us": v.get("gpu__time_duration.sum", 0.0) * 1e6,
            "share": v.get("gpu__time_duration.sum", 0.0) / tot if tot else None,
            **({"dram_GB": (v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]) / 1e9}
               if "dram__bytes_read.sum" in v else {})}
        for k, v in sorted(per.items(), key=lambda kv: -kv[1].get("gpu__time_duration.sum", 0.0))}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    if sys.argv[1] == "report":
        report(sys.argv[2], sys.argv[3], float(sys.argv[4]), sys.argv[5] if len(sys.argv) > 5 else "")
    else:
        launches(sys.argv[2], sys.argv[3])
