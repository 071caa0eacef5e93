"""Summarise ncu reports (raw page): per launch duration, DRAM bytes, DRAM %,
tensor-pipe %, L2 %, registers, achieved occupancy.  Usage: ncu_summary.py rep..."""
import csv, io, subprocess, sys
WANT = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rd"), ("dram__bytes_write.sum", "wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("launch__registers_per_thread", "regs"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("launch__grid_size", "grid")]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"== {rep}")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0][:40]
        vals = []
        for key, short in WANT:
            if key in hdr:
                v, u = r[hdr.index(key)], units[hdr.index(key)]
                if u in ("byte", "Kbyte", "Mbyte", "Gbyte"):
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                    v = f"{float(v.replace(',', '')) * scale / 1e6:.1f}MB"
                elif u == "nsecond":
                    v = f"{float(v.replace(',', '')) / 1e3:.1f}"
                elif u == "usecond":
                    v = f"{float(v.replace(',', '')):.1f}"
                vals.append(f"{short}={v}")
        print(f"  {name:40s} " + " ".join(vals))
