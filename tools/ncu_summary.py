"""Key metrics of every kernel in an ncu --set full report (ncu -i ... --page raw --csv)."""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_%"),
    ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", "l1_lsu_wavefronts_%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "gld_requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "gld_sectors"),
    ("lts__t_sectors.sum.pct_of_peak_sustained_elapsed", "l2_sectors_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name', '?')[:90]}")
        for k, name in KEYS:
            if k in d:
                print(f"   {name:24s} {d[k]:>16s} {u.get(k, '')}")
        stalls = sorted(((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0)) for h, v in d.items()
                         if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")),
                        key=lambda x: -x[1])
        tot = sum(v for _, v in stalls) or 1
        print("   stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in stalls[:6]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
