"""Print the key numbers of a bench.py JSON line: value, e2e, roofline, families."""
import json
import sys

for path in sys.argv[1:]:
    with open(path) as f:
        lines = [ln for ln in f if ln.strip().startswith("{")]
    if not lines:
        print(path, "no JSON line")
        continue
    d = json.loads(lines[-1])
    print(path, d.get("config", {}).get("workload"))
    print(f"  value {d['value']:.0f} q/s  ms/step {d.get('ms_per_step', 0):.3f}  launches "
          f"{d.get('gpu_launches')}  clocks {d.get('clocks')}")
    print("  e2e", json.dumps(d.get("e2e")))
    r = d.get("roofline") or {}
    print(f"  roofline {r.get('kernel')} {r.get('achieved', 0):.1f} / {r.get('peak')} "
          f"{r.get('unit')} frac {r.get('frac', 0):.3f} share {r.get('share_of_step', 0):.2f}")
    h = r.get("hbm_kernel") or {}
    if h:
        print(f"  hbm {h.get('kernel')} {h.get('achieved', 0):.0f} GB/s frac {h.get('frac', 0):.3f}")
    for k, v in (d.get("families") or {}).items():
        print(f"    {k:14s} {1000 * v['ms_per_step']:8.1f} us  {v['launches_per_step']:5.1f} launches"
              f"  {v['gbs']:7.0f} GB/s  {v['tflops']:6.2f} TF/s")
