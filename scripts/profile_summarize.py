"""Turn scripts/profile_round.sh outputs (gpurun_out/prof_*) into profiles/:

  profiles/<round>_launches.csv   launch list (kernel, us) of the bench command
  profiles/<round>_ncu_full.csv   one line per kernel of one solve (ncu --set full)
  profiles/ncu_traffic.json       DRAM bytes per launch per bench kernel group (roofline.traffic)

    python scripts/profile_summarize.py [round tag, default r02]
"""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")

# bench.py kernel groups (Timeline names) -> kernels
GROUPS = {"basis_rows": ["k_basis_rows"], "gram_chol": ["k_gram_chol"], "fit_axis0": ["k_fit_axis0_tma"],
          "fit_last": ["k_last_contract_tma", "k_solve2d"], "epoch": ["k_epoch_regions", "k_epoch_finalize"],
          "pair_jumps": ["k_pair_jumps_regions"], "assemble": ["k_assemble"], "decode": ["k_decode_tma"],
          "reduce": ["k_reduce_partials"]}


def short(name):
    m = re.search(r"(k_\w+)", name)
    return m.group(1) if m else name


def launches():
    rows = [r for r in csv.reader(open(os.path.join(G, "prof_launches.csv"))) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[1:]:
        if "k_" not in r[ki] or "at::" in r[ki]:  # torch's synthetic-field kernels (outside the timed region)
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1000.0 if r[ui] == "nsecond" or r[ui] == "ns" else (v if r[ui] in ("usecond", "us") else v * 1000.0)
        out.append((short(r[ki]), v))
    with open(os.path.join(P, TAG + "_launches.csv"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 -- python bench.py --steps 2 "
                "--warmup 3 --no-cpu-baseline --no-e2e (C5); cold-cache, serialised per launch; graph-replayed "
                "solves show only their first direct launches\n")
        f.write("kernel,time_us\n")
        for k, v in out:
            f.write(f"{k},{v:.3f}\n")
    return out


WANT = [("gpu__time_duration.sum", "time_us"), ("dram__bytes_read.sum", "dram_read_B"),
        ("dram__bytes_write.sum", "dram_write_B"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"), ("launch__registers_per_thread", "regs"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"), ("launch__block_size", "block"),
        ("launch__grid_size", "grid"), ("smsp__inst_executed.sum", "warp_inst"),
        ("launch__occupancy_limit_shared_mem", "occ_limit_smem"), ("launch__occupancy_limit_registers", "occ_limit_regs")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
         "msecond": 1e3}


def full():
    rows = list(csv.reader(open(os.path.join(G, "prof_full_raw.csv"))))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        rec = {"kernel": short(r[hdr.index("Kernel Name")])}
        for key, nm in WANT:
            if key not in hdr:
                continue
            i = hdr.index(key)
            v = float(r[i].replace(",", ""))
            rec[nm] = v * SCALE.get(units[i], 1.0)
        recs.append(rec)
    cols = ["kernel"] + [nm for _, nm in WANT]
    with open(os.path.join(P, TAG + "_ncu_full.csv"), "w") as f:
        f.write(",".join(cols) + "\n")
        for rec in recs:
            f.write(",".join(str(round(rec[c], 3)) if isinstance(rec.get(c), float) else str(rec.get(c, ""))
                             for c in cols) + "\n")
    traffic = {}
    for g, ks in GROUPS.items():
        tot = 0.0
        seen = set()
        for rec in recs:
            if rec["kernel"] in ks and rec["kernel"] not in seen:  # first launch of each kernel of the group
                seen.add(rec["kernel"])
                tot += rec.get("dram_read_B", 0.0) + rec.get("dram_write_B", 0.0)
        if seen:
            traffic[g] = tot
    traffic["_source"] = ("profiles/" + TAG + "_ncu_full.csv: ncu --set full (C5, one solve, MFADD_HOST_LOOP=1 direct "
                          "launches), dram__bytes_read.sum + dram__bytes_write.sum per launch, summed over the "
                          "kernels of each bench.py group")
    with open(os.path.join(P, "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    return recs


if __name__ == "__main__":
    L = launches()
    R = full()
    for rec in R:
        print(f"{rec['kernel']:24s} {rec.get('time_us', 0):8.1f} us  dram {(rec.get('dram_read_B', 0) + rec.get('dram_write_B', 0)) / 1e6:8.1f} MB")
