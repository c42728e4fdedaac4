"""DRAM traffic of the branch kernels (k_dense_sublayer / k_branch_sublayer /
k_branch_x) per Rx-run launch, from an ncu metrics pass over one warm propagation of a bench
workload; merged into profiles/branch_traffic.json for bench.py's
roofline.traffic.

usage (on the GPU box): python tools/traffic.py <workload> [<workload> ...]
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "branch_traffic.json")
METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"


def measure(workload):
    log = os.path.join(ROOT, "gpurun_out", f"traffic_{workload}.csv")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    subprocess.run(["ncu", "--profile-from-start", "off", "--metrics", METRICS, "--clock-control", "none",
                    "-k", "regex:k_(dense_sublayer|branch_sublayer|branch_x)", "--csv", "--log-file", log, sys.executable,
                    os.path.join(ROOT, "tools", "profile_run.py"), workload, "--warm"],
                   check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(open(log)))
    for i, r in enumerate(rows):
        if "Metric Name" in r:
            hdr, body = r, rows[i + 1:]
            break
    ki, ni, vi, ui = (hdr.index(k) for k in ("ID", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}
    per, names = {}, {}
    kn = hdr.index("Kernel Name")
    for r in body:
        if len(r) <= vi:
            continue
        d = per.setdefault(r[ki], {})
        names[r[ki]] = r[kn]
        d[r[ni]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    # one "launch" = one Rx run: k_dense_sublayer plus the k_branch_sublayer pass behind it
    dense = sum(1 for v in names.values() if "k_dense_sublayer" in v)
    launches = dense if dense else len(per)
    rd = sum(d.get("dram__bytes_read.sum", 0) for d in per.values())
    wr = sum(d.get("dram__bytes_write.sum", 0) for d in per.values())
    t = sum(d.get("gpu__time_duration.sum", 0) for d in per.values())
    return {"launches": launches, "dram_bytes_per_launch": (rd + wr) / max(launches, 1),
            "dram_read_bytes": rd, "dram_write_bytes": wr, "kernel_s_serialized": t,
            "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (warm propagation, "
                      "all branch-kernel launches; per Rx run)"}


if __name__ == "__main__":
    data = {}
    if os.path.exists(OUT):
        data = json.load(open(OUT))
    for wl in sys.argv[1:]:
        data[wl] = measure(wl)
        print(wl, json.dumps(data[wl]))
    json.dump(data, open(OUT, "w"), indent=1)
