"""Per-launch summary of an `ncu --set full` capture exported with
`ncu -i rep --page raw --csv`: duration, DRAM traffic, achieved occupancy,
issue activity, memory throughput, registers and shared memory."""
import csv
import sys

COLS = [
    ("Kernel Name", "kernel", None),
    ("Grid Size", "grid", None),
    ("gpu__time_duration.sum", "us", 1.0),
    ("dram__bytes_read.sum", "dram_rd", None),
    ("dram__bytes_write.sum", "dram_wr", None),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", None),
    ("sm__maximum_warps_per_active_cycle_pct", "occ_max%", None),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%", None),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%", None),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64pipe%", None),
    ("launch__registers_per_thread", "regs", None),
    ("launch__shared_mem_per_block_dynamic", "smem_dyn", None),
]


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = [(hdr.index(c) if c in hdr else -1, name, c) for c, name, _ in COLS]
    lines = ["  |  ".join(f"{name}[{units[i]}]" if i >= 0 and units[i] else name for i, name, _ in idx)]
    for r in rows[2:]:
        cells = []
        for i, name, _ in idx:
            v = r[i] if i >= 0 else "-"
            if name == "kernel":
                v = v.split("(")[0][:34]
            cells.append(v)
        lines.append("  |  ".join(cells))
    text = "\n".join(lines)
    if out:
        open(out, "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
