"""Summarise an ncu --set full report: one line of key metrics per launch."""
import csv
import subprocess
import sys

WANT = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "MB"), ("dram__bytes_write.sum", "MB"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"), ("launch__registers_per_thread", "regs"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"), ("launch__grid_size", "grid"),
        ("launch__block_size", "blk"), ("smsp__inst_executed.sum", "winst"),
        ("launch__occupancy_limit_shared_mem", "occ_smem"), ("launch__occupancy_limit_registers", "occ_reg")]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("mfb::<unnamed>::", "")
    parts = [f"{name[:28]:28s}"]
    for key, short in WANT:
        if key not in hdr:
            continue
        i = hdr.index(key)
        v = float(r[i].replace(",", ""))
        if short in ("us", "MB"):
            v *= SCALE.get(units[i], 1.0)
        parts.append(f"{short}={v:.4g}")
    print(" ".join(parts))
