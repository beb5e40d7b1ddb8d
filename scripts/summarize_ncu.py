"""Summarise ncu artefacts (run here, no GPU needed) into profiles/.

    python scripts/summarize_ncu.py launches <launches.csv>      # per-kernel share of a step
    python scripts/summarize_ncu.py report <prof.ncu-rep>        # key counters of a --set full capture
"""
import csv
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_active.avg", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[r[ki]][0] += 1
        agg[r[ki]][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'launches':>8} {'total ms':>12} {'share':>8}  kernel")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:8d} {v / 1e6:12.3f} {100 * v / tot:7.2f}%  {k[:110]}")


def traffic(path, sass_hash=None, points=None, note="", config="5"):
    """k_label DRAM bytes per launch from a launch list taken with
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum"""
    import json
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = defaultdict(dict)
    for r in rows[1:]:
        if "k_label<" not in r[ki]:
            continue
        unit = r[h.index("Metric Unit")] if "Metric Unit" in h else ""
        v = float(r[vi].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
                 "second": 1e9}.get(unit, 1)
        per[r[ii]][r[mi]] = v * scale
    last = per[sorted(per, key=int)[-1]]
    rd, wr = last.get("dram__bytes_read.sum", 0.0), last.get("dram__bytes_write.sum", 0.0)
    pts = int(points) if points else None
    print(json.dumps({"kernel": "k_label<1,1,0>", "config": int(config), "sass_sha16": sass_hash, "points": pts,
                      "launches_seen": len(per), "dram_bytes_read": rd, "dram_bytes_write": wr,
                      "traffic_bytes": rd + wr,
                      "algorithmic_bytes": pts * (24 + 4 + 8) if pts else None,
                      "lts_bytes": last.get("lts__t_bytes.sum"), "gpu_time_ns_under_ncu": last.get("gpu__time_duration.sum"),
                      "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum of one full-mesh k_label launch",
                      "note": note}, indent=1))


FP32_PIPE = {"FFMA2": 2, "FADD2": 2, "FMUL2": 2, "FFMA": 1, "FADD": 1, "FMUL": 1}


def _opcode_counts(cell):
    """'235128 (FFMA2: 109; FADD2: 30; ...)' -> {'FFMA2': 109, ...}"""
    inner = cell[cell.index("(") + 1: cell.rindex(")")]
    out = {}
    for part in inner.split(";"):
        k, v = part.split(":")
        out[k.strip()] = int(v.strip())
    return out


def opcounts(path, sass_hash, evals, config, points, note=""):
    """FP32-pipe lane-ops per point-triangle evaluation of one k_label launch,
    from ncu --metrics sass__thread_inst_executed_true_per_opcode
    --print-metric-instances details (csv): 2 x packed (FFMA2/FADD2/FMUL2) +
    scalar FFMA/FADD/FMUL thread instructions with a true predicate."""
    import json
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    kcol = h.index("Kernel Name")
    if "Metric Name" in h:  # long format: one metric per row
        mi, vi = h.index("Metric Name"), h.index("Metric Value")
        last_id = [r for r in rows[1:] if "k_label<" in r[kcol]][-1][h.index("ID")]
        cells = {r[mi]: r[vi] for r in rows[1:] if r[h.index("ID")] == last_id}
        r = next(r for r in rows[1:] if r[h.index("ID")] == last_id)
    else:
        r = [r for r in rows[1:] if "k_label<" in r[kcol]][-1]
        cells = dict(zip(h, r))
    thr = _opcode_counts(cells["sass__thread_inst_executed_true_per_opcode"])
    warp = _opcode_counts(cells["sass__inst_executed_per_opcode"]) if "sass__inst_executed_per_opcode" in cells else {}
    lane_ops = sum(thr.get(k, 0) * w for k, w in FP32_PIPE.items())
    evals = int(evals)
    out = {"kernel": r[kcol], "grid": r[h.index("Grid Size")], "sass_sha16": sass_hash, "config": config, "points": int(points), "evals": evals,
           "fp32_lane_ops": lane_ops, "fp32_lane_ops_per_eval": lane_ops / evals,
           "mufu_per_eval": thr.get("MUFU", 0) / evals,
           "thread_inst_per_eval": {k: v / evals for k, v in sorted(thr.items(), key=lambda kv: -kv[1])[:16]},
           "warp_inst_total": sum(warp.values()) if warp else None,
           "source": "ncu --metrics sass__thread_inst_executed_true_per_opcode (thread instructions, predicate true)",
           "note": note}
    print(json.dumps(out, indent=1))


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        print("kernel:", d.get("Kernel Name", "?")[:100])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>20s} {u.get(k, '')}")
        stalls = {k: d[k] for k in d if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")}
        print("  stall reasons (warps per issued instruction):")
        for k, v in sorted(stalls.items(), key=lambda kv: -float(kv[1] or 0))[:10]:
            print(f"    {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {v}")


if __name__ == "__main__":
    {"launches": launches, "report": report, "traffic": traffic, "opcounts": opcounts}[sys.argv[1]](*sys.argv[2:])
