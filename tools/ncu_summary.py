"""Summarise ncu --set full reports of the stage kernel into profiles/.

    python tools/ncu_summary.py gpurun_out/r01_full_mixed.ncu-rep [...] --tag r01

Writes profiles/<tag>_ncu_<name>.md (one table row per profiled launch) and
updates profiles/stage_kernel_traffic.json (DRAM bytes per launch, read by
bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pipe_pct"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe_pct"),
    ("sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_active", "tma_pipe_pct"),
    ("smsp__inst_executed.sum", "warp_insts"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6,
         "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    tag = "r01"
    if "--tag" in sys.argv:
        tag = sys.argv[sys.argv.index("--tag") + 1]
        args = [a for a in args if a != tag]
    tfile = os.path.join(ROOT, "profiles", "stage_kernel_traffic.json")
    traffic = json.load(open(tfile)) if os.path.exists(tfile) else {}
    pfile = os.path.join(ROOT, "profiles", "stage_kernel_pipes.json")
    pipes = json.load(open(pfile)) if os.path.exists(pfile) else {}
    for rep in args:
        name = os.path.basename(rep).replace(".ncu-rep", "")
        hdr, units, rows = raw(rep)
        lines = [f"# ncu --set full: {name}", "",
                 "| launch | " + " | ".join(k for _, k in KEYS) + " | stalls (top 4) |",
                 "|---" * (len(KEYS) + 2) + "|"]
        tot_bytes = []
        pipe_rows = []
        for r in rows:
            kn = r[hdr.index("Kernel Name")]
            vals = []
            for m, _ in KEYS:
                i = hdr.index(m) if m in hdr else None
                vals.append(f"{r[i]} {units[i]}" if i is not None else "-")
            rd = float(r[hdr.index("dram__bytes_read.sum")]) * SCALE.get(
                units[hdr.index("dram__bytes_read.sum")], 1)
            wr = float(r[hdr.index("dram__bytes_write.sum")]) * SCALE.get(
                units[hdr.index("dram__bytes_write.sum")], 1)
            tot_bytes.append(rd + wr)
            st = [(float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                  for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith(
                      "not_issued") and r[i].replace(".", "").isdigit()]
            tot = sum(v for v, _ in st) or 1
            top = ", ".join(f"{h} {100 * v / tot:.0f}%" for v, h in sorted(st, reverse=True)[:4])
            lines.append(f"| {kn} | " + " | ".join(vals) + f" | {top} |")
            pr = {}
            for m, k in (("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pct"),
                         ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_fp32_pct"),
                         ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pct"),
                         ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct")):
                if m in hdr:
                    pr[k] = round(float(r[hdr.index(m)]), 1)
            pipe_rows.append(pr)
        mean = sum(tot_bytes) / len(tot_bytes)
        lines += ["", f"mean DRAM bytes per launch: {mean:.4e}"]
        open(os.path.join(ROOT, "profiles", f"{tag}_ncu_{name}.md"), "w").write(
            "\n".join(lines) + "\n")
        # C5 captures are named <tag>_full_<tier> (tier: mixed, f64, ddmixed,
        # ddfull); captures of other shapes do not feed bench.py's traffic
        if "_full_" in name:
            mode = name.rsplit("_", 1)[-1]
            traffic[f"{mode}_65536x512"] = mean
            pipes[f"{mode}_65536x512"] = {"source": f"profiles/{tag}_ncu_{name}.md",
                                          "per_launch": pipe_rows}
        print(name, mean)
    json.dump(traffic, open(tfile, "w"), indent=1)
    json.dump(pipes, open(pfile, "w"), indent=1)


if __name__ == "__main__":
    main()
