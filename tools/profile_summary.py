"""Summarise ncu --set full captures into profiles/ (text + raw metrics JSON).

Usage: python tools/profile_summary.py OUT_PREFIX TITLE rep1.ncu-rep [rep2 ...]
Writes OUT_PREFIX_ncu_full_summary.txt and OUT_PREFIX_ncu_raw_metrics.json with
one entry per profiled kernel (name without namespace/arguments).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

DETAILS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
           "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
           "Dynamic Shared Memory Per Block", "Block Limit Registers", "Block Limit Shared Mem",
           "Theoretical Active Warps per SM", "Achieved Active Warps Per SM",
           "Executed Instructions", "No Eligible", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size",
           "Block Size"]
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__warps_active.avg.pct_of_peak_sustained_active"]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def short(name):
    name = re.sub(r"\(.*$", "", name)
    name = re.sub(r"^void ", "", name)
    return name.replace("bm::", "")


def ncu(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    prefix, title, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    text = [f"# {title}"]
    raw_all = {}
    for rep in reps:
        rows = ncu(rep, "details")
        h = rows[0]
        ki, mi, ui, vi = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                          h.index("Metric Value"))
        # launches of the same kernel are kept apart (name#launch id) in the
        # text and summed per kernel name in the raw metrics
        ii = h.index("ID")
        names = {}
        for r in rows[1:]:
            names.setdefault(short(r[ki]), set()).add(r[ii])
        by = {}
        for r in rows[1:]:
            if int(os.environ.get("PROFILE_MAX_ID", "-1")) >= 0 and int(r[ii]) > int(
                    os.environ["PROFILE_MAX_ID"]):
                continue
            k = short(r[ki])
            if len(names[k]) > 1:
                k = f"{k}#{r[ii]}"
            by.setdefault(k, {})[r[mi]] = (r[vi], r[ui])
        raw = ncu(rep, "raw")
        rh, units = raw[0], raw[1]
        kcol = rh.index("Kernel Name")
        # normalised units: bytes and milliseconds
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                 "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
        sums = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "smsp__inst_executed.sum")
        max_id = int(os.environ.get("PROFILE_MAX_ID", "-1"))
        idc = rh.index("ID")
        for r in raw[2:]:
            if max_id >= 0 and int(r[idc]) > max_id:
                continue
            k = short(r[kcol])
            first = k not in raw_all
            ent = raw_all.setdefault(k, {})
            ent["launches"] = ent.get("launches", 0) + 1
            stalls = {}
            for i, name in enumerate(rh):
                if name in RAW:
                    v = float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
                    # additive metrics summed over launches; ratios from the longest
                    if name in sums:
                        ent[name] = ent.get(name, 0.0) + v
                    elif first or v > 0:
                        ent[name] = v
                elif name.startswith(STALLS) and not name.endswith("not_issued"):
                    try:
                        v = float(r[i].replace(",", ""))
                    except ValueError:
                        continue
                    if v > 0:
                        stalls[name[len(STALLS):]] = v
            tot = sum(stalls.values()) or 1.0
            ent["stall_share"] = {k2: round(v / tot, 3) for k2, v in
                                  sorted(stalls.items(), key=lambda x: -x[1])[:8]}
        for k, d in by.items():
            text.append(f"## {k}")
            for name in DETAILS:
                if name in d:
                    text.append(f"  {name:34s} {d[name][0]} {d[name][1]}")
            k = k.split("#")[0]
            if k in raw_all and "stall_share" in raw_all[k]:
                text.append("  stall share (pc sampling)         " +
                            ", ".join(f"{a} {b:.0%}" for a, b in raw_all[k]["stall_share"].items()))
    open(prefix + "_ncu_full_summary.txt", "w").write("\n".join(text) + "\n")
    raw_all["bytes_scale"] = 1.0
    raw_all["units"] = "dram bytes in bytes, gpu__time_duration.sum in ms"
    json.dump(raw_all, open(prefix + "_ncu_raw_metrics.json", "w"), indent=1)
    print("\n".join(text))


if __name__ == "__main__":
    main()
