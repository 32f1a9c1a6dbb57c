"""Summarise an ncu report (.ncu-rep) into a small text table for profiles/ (run here, no GPU)."""
import csv, io, subprocess, sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "lsu_wf_%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wf"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_act_%"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conf"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    print("| kernel | " + " | ".join(n for _, n in METRICS) + " |")
    print("|" + "---|" * (len(METRICS) + 1))
    for r in data:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")[:40]
        vals = []
        for m, _ in METRICS:
            if m in h:
                i = h.index(m)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("-")
        print(f"| {name} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
