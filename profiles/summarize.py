"""Summarise one profiles/capture.sh run into committed evidence under profiles/.

usage: python profiles/summarize.py TAG [gpurun_out]

Writes
  profiles/TAG_launches.csv   the raw launch list (ncu --metrics gpu__time_duration.sum)
  profiles/TAG_summary.md     per-kernel shares of one steady-state frame + the whole run,
                              the --set full metrics of the traversal kernels, the bench line
  profiles/TAG_traffic.json   DRAM bytes per launch of the roofline kernel (read by bench.py)
Needs `ncu` on PATH for the --set full report (present in this image).
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def to_ms(value, unit):
    v = float(value.replace(",", ""))
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
    return scale.get(unit, 1.0) * v


def launches(path):
    rows = []
    with open(path, newline="") as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.reader(lines)
    header = next(rd)
    for rec in rd:
        d = dict(zip(header, rec))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].split("::")[-1]
        rows.append((int(d["ID"]), name, to_ms(d["Metric Value"], d["Metric Unit"])))
    return rows


def table(recs, title):
    agg = collections.defaultdict(lambda: [0, 0.0])
    for _, n, v in recs:
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(v for _, _, v in recs) or 1.0
    out = [f"### {title}", "", "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:24]:
        out.append(f"| `{n}` | {c} | {v:.3f} | {100 * v / tot:.1f}% |")
    out.append(f"| **all** | {len(recs)} | {tot:.3f} | 100% |")
    return out, agg, tot


def full_metrics(rep):
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__thread_inst_executed_per_inst_executed.ratio",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "lts__t_requests_srcunit_tex_op_atom_dot_alu.sum", "lts__t_requests_srcunit_tex_op_red.sum",
            "lts__t_sectors_srcunit_tex_op_atom_dot_alu.avg.per_cycle_elapsed",
            "lts__t_sectors_srcunit_tex_op_atom_dot_alu.avg.peak_sustained",
            "smsp__inst_executed_op_shared_atom.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rd = list(csv.reader(txt.splitlines()))
    header, units = rd[0], rd[1]
    out = []
    for rec in rd[2:]:
        d = dict(zip(header, rec))
        row = {"kernel": d["Kernel Name"].split("(")[0].split("::")[-1]}
        for k in keys:
            if k in d:
                u = units[header.index(k)]
                v = float(d[k].replace(",", "")) if d[k] else 0.0
                if u == "Gbyte":
                    v *= 1e9
                elif u == "Mbyte":
                    v *= 1e6
                elif u == "Kbyte":
                    v *= 1e3
                elif u == "ms":
                    v *= 1.0
                elif u == "us":
                    v *= 1e-3
                row[k] = v
        out.append(row)
    return out


def hbm_peak():
    """MEASURED_PEAKS.json hbm_gbs (driver-written), else B200_PROFILING.md's fallback."""
    try:
        with open(os.path.join(HERE, "..", "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6650.0


def main(tag, src="gpurun_out"):
    lc = os.path.join(src, f"{tag}_launches.csv")
    shutil.copy(lc, os.path.join(HERE, f"{tag}_launches.csv"))
    recs = launches(lc)
    starts = [i for i, (_, n, _) in enumerate(recs) if n == "k_frame_reset"]
    md = [f"# {tag} profile summary (C4, 1 B200)", "",
          "Recipe: `profiles/capture.sh` (plain bench, then the launch list, then one `ncu --set full`",
          "capture of the traversal kernels of a steady-state frame). Launch-list times are cold-cache and",
          "serialised: compare SHARES with the bench's stage times, not absolutes.", ""]
    last = recs[starts[-1]:] if starts else recs
    t, agg_last, tot_last = table(last, "Last steady-state frame (frame update -> verify -> retrace -> splat)")
    md += t + [""]
    t, _, _ = table(recs, "Whole command (cold frame 0 + warm-up + timed frames)")
    md += t + [""]
    import glob
    reps = sorted(glob.glob(os.path.join(src, f"{tag}_full*.ncu-rep")))
    traffic = {}
    if reps:
        fm = [row for rep in reps for row in full_metrics(rep)]
        md += ["### `ncu --set full` (one steady-state launch each)", "",
               "| kernel | ms | DRAM read GB | DRAM write GB | DRAM GB/s (% of HBM peak) | L2 hit % | L1 hit % | warps active % | issue active % | thr/inst | inst (M) | regs | global atom/red (L2 atomic unit busy %) | shared atom wavefronts |",
               "|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|"]
        for r in fm:
            ms = r.get("gpu__time_duration.sum", 0)
            gbs = (r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)) / (ms * 1e-3) / 1e9 if ms else 0.0
            md.append("| `{}` | {:.3f} | {:.3f} | {:.3f} | {:.0f} ({:.0f}%) | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.0f} | {:.0f} ({:.1f}%) | {:.0f} |".format(
                r["kernel"], ms, r.get("dram__bytes_read.sum", 0) / 1e9,
                r.get("dram__bytes_write.sum", 0) / 1e9, gbs, 100.0 * gbs / hbm_peak(),
                r.get("lts__t_sector_hit_rate.pct", 0),
                r.get("l1tex__t_sector_hit_rate.pct", 0),
                r.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0),
                r.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0),
                r.get("smsp__thread_inst_executed_per_inst_executed.ratio", 0),
                r.get("smsp__inst_executed.sum", 0) / 1e6,
                r.get("launch__registers_per_thread", 0),
                r.get("lts__t_requests_srcunit_tex_op_atom_dot_alu.sum", 0)
                + r.get("lts__t_requests_srcunit_tex_op_red.sum", 0),
                100.0 * r.get("lts__t_sectors_srcunit_tex_op_atom_dot_alu.avg.per_cycle_elapsed", 0)
                / max(r.get("lts__t_sectors_srcunit_tex_op_atom_dot_alu.avg.peak_sustained", 1.0), 1e-9),
                r.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", 0)))
            traffic[r["kernel"]] = {"dram_bytes": r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0),
                                    "ms": r.get("gpu__time_duration.sum", 0),
                                    "inst": r.get("smsp__inst_executed.sum", 0)}
        md.append("")
    bj = os.path.join(src, f"{tag}_bench.json")
    if os.path.exists(bj):
        with open(bj) as f:
            line = [ln for ln in f if ln.startswith("{")][-1]
        md += ["### Bench line of the same box", "", "```json", line.strip(), "```", ""]
    with open(os.path.join(HERE, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    with open(os.path.join(HERE, f"{tag}_traffic.json"), "w") as f:
        json.dump({"source": f"profiles/{tag}_summary.md (ncu --set full, one steady-state launch)",
                   "kernels": traffic}, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "gpurun_out")
