"""Summarise ncu artefacts from gpurun_out/ into profiles/ (tracked).

  python tools/profile_summary.py launches <launches.csv> <out.md> [title]
      per-kernel launch count, total and mean time and share of the run, from
      an `ncu --metrics gpu__time_duration.sum --csv` launch list
  python tools/profile_summary.py full <report.ncu-rep> <out.md> [traffic.json]
      the headline metrics of one `ncu --set full` capture; with traffic.json
      also writes dram bytes per launch for bench.py's roofline.traffic
  python tools/profile_summary.py source <report.ncu-rep> <out.md> [n]
      stall samples and executed instructions per source line (top n)
"""
import collections
import csv
import io
import json
import subprocess
import sys


def _ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def launches(path, out, title="launch list"):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, gi, bi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size"), h.index("Block Size")
    agg = collections.OrderedDict()
    total = 0.0
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("lrk::<unnamed>::", "").replace("<unnamed>::", "")
        t = float(r[vi].replace(",", "")) / 1e3  # ns -> us
        a = agg.setdefault(name, [0, 0.0, r[gi], r[bi]])
        a[0] += 1
        a[1] += t
        total += t
    lines = [f"# {title}", "", f"source: `{path}` ({len(rows) - 1} launches, {total:.1f} us of kernel time, "
             "cold-cache serialised ncu replay: shares matter, not absolutes)", "",
             "| kernel | launches | total us | mean us | share | grid | block |", "|---|---|---|---|---|---|---|"]
    for name, (n, t, g, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {name} | {n} | {t:.1f} | {t / n:.2f} | {100 * t / total:.1f}% | {g} | {b} |")
    open(out, "w").write("\n".join(lines) + "\n")


FULL = ["Kernel Name", "Grid Size", "Block Size", "launch__registers_per_thread", "gpu__time_duration.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]


def full(rep, out, traffic=None):
    rows = _ncu_csv(rep, "--page", "raw")
    h, units, vals = rows[0], rows[1], rows[2]
    lines = [f"# ncu --set full: `{rep.split('/')[-1]}`", "", "| metric | value | unit |", "|---|---|---|"]
    got = {}
    for w in FULL:
        if w in h:
            i = h.index(w)
            got[w] = vals[i]
            lines.append(f"| {w} | {vals[i]} | {units[i]} |")
    stalls = []
    for i, name in enumerate(h):
        if name.startswith("smsp__pcsamp_warps_issue_stalled") and not name.endswith("not_issued"):
            try:
                stalls.append((float(vals[i].replace(",", "")), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    lines += ["", "| warp state (pc samples) | share |", "|---|---|"]
    for s, n in sorted(stalls, reverse=True)[:10]:
        lines.append(f"| {n} | {100 * s / tot:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    if traffic:
        def mb(k):
            i = h.index(k)
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[i].strip()]
            return float(vals[i].replace(",", "")) * scale
        json.dump({"kernel": got.get("Kernel Name", "").split("(")[0].strip(), "report": rep.split("/")[-1],
                   "dram_bytes_per_launch": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
                   "duration_us": float(got.get("gpu__time_duration.sum", "0").replace(",", "")) *
                   {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}[units[h.index("gpu__time_duration.sum")].strip()]},
                  open(traffic, "w"), indent=1)


def source(rep, out, n=25):
    rows = _ncu_csv(rep, "--page", "source", "--print-source", "cuda,sass")
    cur, hdr = None, None
    agg, ins, src = collections.Counter(), collections.Counter(), {}
    stall = collections.defaultdict(collections.Counter)
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            ii = hdr.index("Instructions Executed")
            continue
        if hdr is None or len(r) < 6:
            continue
        try:
            ln, v = int(r[0]), int(r[4])
        except ValueError:
            continue
        agg[(cur, ln)] += v
        src[(cur, ln)] = r[1][:90].replace("|", "\\|")
        try:
            ins[(cur, ln)] += int(r[ii])
        except ValueError:
            pass
        for i, name in enumerate(hdr):
            if name.startswith("stall_") and "Not Issued" not in name and i < len(r):
                try:
                    stall[(cur, ln)][name[6:]] += int(r[i])
                except ValueError:
                    pass
    tot = sum(agg.values()) or 1
    lines = [f"# stall samples by source line: `{rep.split('/')[-1]}`", "",
             "| share | instructions | line | source | top stalls |", "|---|---|---|---|---|"]
    for k, v in agg.most_common(int(n)):
        top = ", ".join(f"{a}={b}" for a, b in stall[k].most_common(3))
        lines.append(f"| {100 * v / tot:.1f}% | {ins[k]} | {k[0]}:{k[1]} | `{src[k]}` | {top} |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    mode = sys.argv[1]
    {"launches": launches, "full": full, "source": source}[mode](*sys.argv[2:])
