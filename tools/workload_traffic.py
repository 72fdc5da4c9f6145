"""DRAM traffic and time per step of a workload from an ncu capture of ONE
step (tools/profile_workload.py), merged into profiles/<prefix>_kernels.json
under "workloads" (bench.py reads roofline.traffic from there):

  python tools/workload_traffic.py gpurun_out/c4.ncu-rep c4 profiles/r09_workloads
"""
import csv
import io
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
         "ms": 1e3, "msecond": 1e3}


def main(rep, wl, prefix):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    per = {}
    tot = {"kernels": 0, "duration_us": 0.0, "dram_bytes_per_step": 0.0}
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0]
        v = {}
        for key, metric in (("us", "gpu__time_duration.sum"), ("rd", "dram__bytes_read.sum"),
                            ("wr", "dram__bytes_write.sum")):
            i = col[metric]
            v[key] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
        e = per.setdefault(name, {"launches": 0, "duration_us": 0.0, "dram_bytes": 0.0})
        e["launches"] += 1
        e["duration_us"] += v["us"]
        e["dram_bytes"] += v["rd"] + v["wr"]
        tot["kernels"] += 1
        tot["duration_us"] += v["us"]
        tot["dram_bytes_per_step"] += v["rd"] + v["wr"]
    tot["per_kernel"] = per
    tot["capture"] = rep
    path = prefix + "_kernels.json"
    d = json.load(open(path)) if os.path.exists(path) else {}
    d.setdefault("note", "one step per workload under ncu (--clock-control none): cold-cache, serialised")
    d.setdefault("workloads", {})[wl] = tot
    with open(path, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps({wl: {k: v for k, v in tot.items() if k != "per_kernel"}}))
    for k, e in sorted(per.items(), key=lambda x: -x[1]["duration_us"]):
        print(f"  {e['duration_us']:10.1f} us {e['dram_bytes'] / 1e6:10.1f} MB x{e['launches']:3d}  {k[:100]}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
