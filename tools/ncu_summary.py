"""Summarise an ncu --set full report per launch: duration, grid, DRAM bytes
(read+write), achieved DRAM GB/s, tensor-pipe utilisation, occupancy."""
import csv
import io
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0,
         "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3, "ms": 1e3}

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]


def val(r, name):
    try:
        i = hdr.index(name)
    except ValueError:
        return None
    s = r[i].replace(",", "")
    try:
        return float(s) * SCALE.get(units[i], 1.0)
    except ValueError:
        return None


print("| kernel | grid | duration us | DRAM read+write MB | DRAM GB/s | tensor pipe % active | achieved occupancy % |")
print("|---|---|---|---|---|---|---|")
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:48]
    dur = val(r, "gpu__time_duration.sum") or 0.0
    rd = val(r, "dram__bytes_read.sum") or 0.0
    wr = val(r, "dram__bytes_write.sum") or 0.0
    tp = val(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
    occ = val(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
    grid = r[hdr.index("launch__grid_size")] if "launch__grid_size" in hdr else ""
    gbs = (rd + wr) / (dur * 1e-6) / 1e9 if dur else 0.0
    print(f"| {name} | {grid} | {dur:.2f} | {(rd + wr) / 1e6:.2f} | {gbs:.0f} | "
          f"{'' if tp is None else f'{tp:.1f}'} | {'' if occ is None else f'{occ:.1f}'} |")
