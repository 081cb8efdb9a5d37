"""Summarise an ncu --page raw --csv export: one line per launch.

    python scripts/ncu_table.py gpurun_out/prof_C4_raw.csv [--csv out.csv]
"""
import csv
import re
import sys

WANT = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rdMB"), ("dram__bytes_write.sum", "wrMB"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64i%"),
        ("launch__registers_per_thread", "regs"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("launch__block_size", "blk"), ("launch__grid_size", "grid"),
        ("launch__occupancy_limit_shared_mem", "oc_smem"), ("launch__occupancy_limit_registers", "oc_reg"),
        ("l1tex__t_sector_hit_rate.pct", "l1hit%"), ("lts__t_sector_hit_rate.pct", "l2hit%")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0,
         "us": 1.0, "msecond": 1e3, "ms": 1e3}


def rows(path):
    r = list(csv.reader(open(path)))
    hdr, units = r[0], r[1]
    out = []
    for row in r[2:]:
        if len(row) != len(hdr):
            continue
        d = {"kernel": re.search(r"(k_\w+)", row[hdr.index("Kernel Name")]).group(1)
             if re.search(r"(k_\w+)", row[hdr.index("Kernel Name")]) else row[hdr.index("Kernel Name")][:30]}
        for m, nm in WANT:
            if m not in hdr:
                d[nm] = None
                continue
            i = hdr.index(m)
            try:
                v = float(row[i].replace(",", ""))
            except ValueError:
                d[nm] = None
                continue
            u = units[i]
            if nm == "us":
                v *= SCALE.get(u, 1.0)
            elif nm in ("rdMB", "wrMB"):
                v = v * SCALE.get(u, 1.0) / 1e6
            d[nm] = v
        out.append(d)
    return out


if __name__ == "__main__":
    R = rows(sys.argv[1])
    cols = ["kernel"] + [nm for _, nm in WANT]
    print(" ".join(f"{c:>9}" if c != "kernel" else f"{c:<24}" for c in cols))
    for d in R:
        print(" ".join((f"{d[c]:>9.1f}" if isinstance(d[c], float) else f"{str(d[c]):>9}") if c != "kernel"
                       else f"{d[c]:<24}" for c in cols))
    if "--csv" in sys.argv:
        with open(sys.argv[sys.argv.index("--csv") + 1], "w") as f:
            w = csv.DictWriter(f, fieldnames=cols)
            w.writeheader()
            for d in R:
                w.writerow(d)
