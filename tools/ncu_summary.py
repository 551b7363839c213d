"""Compact text summary of ncu reports (for profiles/).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [...] > profiles/rNN_x.txt
    python tools/ncu_summary.py --launches gpurun_out/launches.csv [--step-flops F]

Per kernel launch in a report: duration, DMMA/tensor and FP64 pipe
utilisation, DRAM bytes (the roofline `traffic`), L2 hit rate, registers,
occupancy limits and the top warp-stall reasons.  For a launch list
(`--metrics gpu__time_duration.sum --csv`): time per kernel class and its
share of the total.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_pct"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma_issue_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_registers", "occ_limit_regs"),
    ("launch__occupancy_limit_shared_mem", "occ_limit_smem"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem_ld_conflicts"),
]


def summarize_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        print(f"# {path}: no data")
        return
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        print(f"## {path}\nkernel: {name[:160]}")
        for key, label in WANT:
            if key in d:
                print(f"  {label:18s} {d[key]} {u.get(key, '')}")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        top = sorted(stalls, reverse=True)[:8]
        print("  stalls             " + ", ".join(f"{n} {s / tot * 100:.0f}%" for s, n in top))


def summarize_launches(path, step_flops=None):
    text = open(path).read()
    lines = [l for l in text.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        ms = v * scale
        nm = d["Kernel Name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "")
        k = nm.split("(")[0].split("<")[0].split("::")[-1].strip()
        agg[k][0] += 1
        agg[k][1] += ms
        total += ms
    print(f"## {path}: {sum(a[0] for a in agg.values())} launches, {total:.3f} ms serialized (cold-cache)")
    for k, (cnt, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:60s} {cnt:5d} launches {ms:10.3f} ms  {ms / total * 100:5.1f}%")


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--launches":
        summarize_launches(args[1])
    else:
        for a in args:
            summarize_report(a)
