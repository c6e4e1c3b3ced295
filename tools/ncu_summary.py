"""Summarise ncu outputs into profiles/ (run here, no GPU needed).
    python tools/ncu_summary.py rep  <file.ncu-rep> <out_prefix> [--cells N]
    python tools/ncu_summary.py launches <launches.csv> <out_prefix>"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_active.avg",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    return hdr, units, vals


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, vals = rows[0], rows[2]
    d = dict(zip(hdr, vals))
    res = {}
    for k, v in d.items():
        if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio"):
            try:
                f = float(v.replace(",", ""))
            except ValueError:
                continue
            if f > 0.01:
                res[k.replace("smsp__average_warp_latency_issue_stalled_", "").replace(".ratio", "")] = f
    if not res:   # sm_100 reports: warp-state PC sampling shares instead
        samp = {}
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    samp[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v.replace(",", ""))
                except ValueError:
                    pass
        tot = sum(samp.values()) or 1.0
        res = {f"{k} (share of samples)": round(v / tot, 4) for k, v in samp.items() if v / tot > 0.002}
    return dict(sorted(res.items(), key=lambda x: -x[1]))


def summarize_rep(rep, prefix, cells=None):
    hdr, units, vals = raw(rep)
    kernels = []
    for v in vals:
        d = dict(zip(hdr, v))
        u = dict(zip(hdr, units))
        ent = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in KEYS:
            if k in d:
                ent[k] = f"{d[k]} {u.get(k, '')}".strip()
        kernels.append(ent)
    main = kernels[0] if kernels else {}
    summ = {"report": rep, "kernels": kernels, "stall_cycles_per_issue": stalls(rep)}

    def num(s):
        return float(s.split()[0].replace(",", ""))
    def nbytes(s):
        for unit, f in (("Tbyte", 1e12), ("Gbyte", 1e9), ("Mbyte", 1e6), ("Kbyte", 1e3)):
            if unit in s:
                return num(s) * f
        return num(s)
    try:
        summ["dram_bytes_per_launch"] = nbytes(main["dram__bytes_read.sum"]) + nbytes(main["dram__bytes_write.sum"])
    except Exception:
        pass
    if cells:
        try:
            summ["inst_per_cell"] = num(main["smsp__inst_executed.sum"]) * 32 / cells   # thread-instructions / cell
        except Exception:
            pass
    with open(prefix + ".json", "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps(summ, indent=1))


def summarize_launches(path, prefix):
    txt = open(path).read()
    lines = [ln for ln in txt.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][:80]
        val = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        agg[name][0] += 1
        agg[name][1] += val * scale
        total += val * scale
    out = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {k} | {n} | {us:.1f} | {us / total:.4f} |")
    md = "\n".join(out)
    with open(prefix + ".md", "w") as f:
        f.write(md + "\n")
    print(md)


if __name__ == "__main__":
    if sys.argv[1] == "rep":
        cells = None
        if "--cells" in sys.argv:
            cells = float(sys.argv[sys.argv.index("--cells") + 1])
        summarize_rep(sys.argv[2], sys.argv[3], cells)
    else:
        summarize_launches(sys.argv[2], sys.argv[3])
