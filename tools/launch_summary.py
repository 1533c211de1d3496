"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_*])
by kernel: time per kernel name and, when captured, DRAM bytes per launch."""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, ui, vi = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"),
                  hdr.index("Metric Value"))
idi = hdr.index("ID")
t = collections.defaultdict(lambda: [0, 0.0, 0.0])  # launches, us, dram bytes
seen = set()
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    except ValueError:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("ngdb_dev::", "")[:60]
    if r[mi] == "gpu__time_duration.sum":
        t[name][0] += 1
        t[name][1] += v
    elif r[mi].startswith("dram__bytes"):
        t[name][2] += v
tot = sum(v[1] for v in t.values())
print(f"total {tot:.1f} us over {sum(v[0] for v in t.values())} launches")
for k, v in sorted(t.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    extra = f"  dram {v[2]/v[0]/1e6:8.2f} MB/launch {v[2]/1e3/max(v[1],1e-9):7.0f} GB/s" if v[2] else ""
    print(f"{v[1]:9.1f} us {100*v[1]/tot:5.1f}% {v[0]:4d} x {v[1]/v[0]:7.2f} us{extra}  {k}")
