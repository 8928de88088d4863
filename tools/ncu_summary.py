"""Summarise ncu captures into profiles/ (run here, after gpurun brought the
.ncu-rep / launch CSV back).

  python tools/ncu_summary.py --rep gpurun_out/prof_conv_r1.ncu-rep --out profiles/r1_conv_c2.json
  python tools/ncu_summary.py --launches gpurun_out/launches_c2.csv --out profiles/r1_launches_c2.json
"""
import argparse
import collections
import csv
import io
import json
import subprocess

METRICS = {
    "duration_ms": "gpu__time_duration.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_per_scheduler": "smsp__warps_active.avg.per_cycle_active",
    "warps_eligible_per_scheduler": "smsp__warps_eligible.avg.per_cycle_active",
    "instructions": "smsp__inst_executed.sum",
    "registers_per_thread": "launch__registers_per_thread",
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "sm_mhz": "smsp__cycles_elapsed.avg.per_second",
    "grid_size": "launch__grid_size",
    "block_size": "launch__block_size",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-3, "msecond": 1, "nsecond": 1e-6, "ns": 1e-6, "us": 1e-3, "ms": 1, "s": 1e3,
              "second": 1e3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def summarize_rep(rep):
    kernels, units = raw(rep)
    res = []
    for d in kernels:
        s = {"kernel": d.get("Kernel Name", "")[:120]}
        for k, m in METRICS.items():
            v = num(d.get(m))
            u = units.get(m, "")
            if v is not None and k.startswith("duration"):
                v *= UNIT_SCALE.get(u, 1)
            if v is not None and k.startswith("dram_bytes"):
                v *= UNIT_SCALE.get(u, 1)
            s[k] = v
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(v) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and num(v)}
        tot = sum(st.values()) or 1
        s["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
        if s.get("dram_bytes_read") is not None and s.get("dram_bytes_write") is not None:
            s["dram_bytes_per_launch"] = s["dram_bytes_read"] + s["dram_bytes_write"]
        res.append(s)
    return res


def summarize_launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    for i, r in enumerate(rows):
        if "Kernel Name" in r and "Metric Value" in r:
            hdr, start = r, i + 1
            break
    kn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = collections.defaultdict(lambda: [0, 0.0])
    order = []
    for r in rows[start:]:
        if len(r) <= mv:
            continue
        name = r[kn].split("(")[0]
        ms = num(r[mv]) * UNIT_SCALE.get(r[mu], 1)
        per[name][0] += 1
        per[name][1] += ms
        order.append((name, ms))
    total = sum(v[1] for v in per.values())
    return {"launches": len(order), "total_ms": total,
            "by_kernel": {k: {"launches": v[0], "ms": round(v[1], 4), "share": round(v[1] / total, 4)}
                          for k, v in sorted(per.items(), key=lambda x: -x[1][1])},
            "note": "ncu --metrics gpu__time_duration.sum --clock-control none: serialised, cold-cache; compare shares"}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    data = summarize_rep(a.rep) if a.rep else summarize_launches(a.launches)
    json.dump(data, open(a.out, "w"), indent=1)
    print(json.dumps(data, indent=1)[:3000])
