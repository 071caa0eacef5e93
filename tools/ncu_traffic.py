"""Write profiles/k1_traffic.json (read by bench.py for roofline.traffic) from an
ncu --set full report of K1 on the profiling harness and the harness's own
algorithmic-byte count.  Usage: ncu_traffic.py <k1.ncu-rep> <harness.json> <out.json>"""
import csv, io, json, subprocess, sys
rep, harness, out = sys.argv[1:4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
def get(r, key):
    return float(r[hdr.index(key)].replace(",", "")) * scale[units[hdr.index(key)]]
r = rows[2]
traffic = get(r, "dram__bytes_read.sum") + get(r, "dram__bytes_write.sum")
h = json.loads(open(harness).read().strip().splitlines()[-1])
json.dump({"kernel": r[hdr.index("Kernel Name")].split("(")[0], "dram_bytes_per_launch": traffic,
           "algorithmic_bytes_per_launch": h["k1_algorithmic_bytes_first_decode_layer"],
           "ratio": traffic / h["k1_algorithmic_bytes_first_decode_layer"],
           "source": f"ncu --set full of {rep.split('/')[-1]} on tools/prof_harness.py "
                     f"({h['requests']} decode rows, context {h['ctx']}, {h.get('preset', 'gptj-6b')} shape, "
                     f"{h.get('layers', 28)} layers)"}, open(out, "w"), indent=1)
print(open(out).read())
