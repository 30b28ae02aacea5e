"""Key metrics of one-kernel `ncu --page raw --csv` exports as a markdown table.
Usage: python tools/ncu_summary.py name=file.csv [name=file.csv ...]"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles"),
    ("smsp__cycles_active.avg", "SMSP active cycles"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active % (of active cycles)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (of elapsed)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared-memory pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def load(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr, units, vals = rows[i], rows[i + 1], rows[i + 2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}, vals[hdr.index("Kernel Name")]


def main():
    cols = [a.rsplit("=", 1) for a in sys.argv[1:]]
    data = [(n,) + load(p) for n, p in cols]
    print("| metric | " + " | ".join(f"{n}" for n, _, _ in data) + " |")
    print("|---|" + "---|" * len(data))
    print("| kernel | " + " | ".join(f"`{k[:48]}`" for _, _, k in data) + " |")
    for key, label in KEYS:
        cells = []
        for _, d, _ in data:
            v, u = d.get(key, ("", ""))
            cells.append(f"{v} {u}".strip())
        if any(cells):
            print(f"| {label} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
