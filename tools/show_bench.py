"""Summarise bench.py JSON lines (one row per workload)."""
import json
import sys

for line in open(sys.argv[1]):
    line = line.strip()
    if not line.startswith("{"):
        if line.startswith("[rank"):
            print(line)
        continue
    d = json.loads(line)

    def show(name, r):
        rf = r.get("roofline", {})
        print(f"{name:5s} value {r['value']:.4g} ms/step {r['ms_per_step']:.3f} "
              f"gcups {r.get('nw_gcups') or 0:.1f} e2e {r.get('e2e', {}).get('value', 0):.4g} "
              f"kern_ms {rf.get('kernel_ms', 0):.3f} hbm_frac {rf.get('frac', 0):.3f} "
              f"dp_frac {r.get('roofline_dp_alu', {}).get('frac', 0):.4f} "
              f"launches {r.get('gpu_launches')}/{r.get('gpu_launches_e2e')} "
              f"cpu {(r.get('cpu_baseline') or {}).get('value')}")

    show(d.get("impl", "main"), d)
    for k, v in d.get("workloads", {}).items():
        show(k, v)
    if "clocks" in d:
        print(d["clocks"])
