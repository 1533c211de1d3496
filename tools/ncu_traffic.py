"""Build profiles/ncu_traffic.json (the `roofline.traffic` source of bench.py)
from the per-config ncu launch lists of a profiling pass
(tools/profile_mn.sh / profile_r02.sh: gpu__time_duration + dram__bytes_read/
write per launch). For each config's reported families, the DRAM bytes per
launch of the family's dominant kernel, averaged over all its launches (every
tile width of the GEMM). Usage: python tools/ncu_traffic.py profiles/r02/ncu_r02n"""
import collections
import csv
import json
import pathlib
import sys

FAMILIES = {  # config -> family -> kernel name (namespace stripped, template args ignored)
    "c2": {"intersect": "tc_gemm_tma_kernel", "opt_entity": "entity_adam_kernel"},
    "c3": {"project": "tc_gemm_tma_kernel", "opt_entity": "beta_entity_adam_kernel"},
    "c4": {"opt_entity": "tc_gemm_tma_kernel", "entity_prep": "tc_gemm_tma_kernel"},
    "c5": {"intersect": "tc_gemm_tma_kernel", "opt_entity": "entity_adam_kernel"},
}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def per_launch_bytes(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, ui, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit",
                                                   "Metric Value", "ID"))
    launches = collections.defaultdict(float)
    names = {}
    for r in rows[1:]:
        if not r[mi].startswith("dram__bytes"):
            continue
        launches[r[ii]] += float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "").replace("ngdb_dev::", "")
    return launches, names


def main(d):
    d = pathlib.Path(d)
    root = pathlib.Path(__file__).resolve().parents[1]
    out = {"_about": "DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per launch of each "
           "family's dominant kernel, mean over its launches in the config's ncu launch list "
           f"(cold caches, serialised; {d.relative_to(root) if d.is_absolute() else d}/<config>_launches.csv, "
           "tools/ncu_traffic.py). bench.py copies it into roofline.traffic for the matching family; "
           "the algorithmic bytes per launch are the family's bytes_per_step / launches_per_step."}
    for cfg, fams in FAMILIES.items():
        f = d / f"{cfg}_launches.csv"
        if not f.exists():
            continue
        launches, names = per_launch_bytes(f)
        out[cfg] = {}
        for fam, kern in fams.items():
            ids = [i for i, n in names.items() if n.split("::")[-1].split("<")[0] == kern]
            if not ids:
                continue
            widths = sorted({names[i].split("::")[-1] for i in ids})
            out[cfg][fam] = {"kernel": f"{', '.join(widths)} (mean of {len(ids)} launches)",
                             "bytes_per_launch": round(sum(launches[i] for i in ids) / len(ids)),
                             "source": str(f.relative_to(root) if f.is_absolute() else f)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
