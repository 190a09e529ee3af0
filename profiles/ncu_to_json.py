"""ncu --set full report -> the per-kernel summary bench.py reads for roofline.traffic.
usage: python profiles/ncu_to_json.py REPORT.ncu-rep OUT.json LANES "source description"
"""
import csv
import json
import subprocess
import sys


def main(rep, out, lanes, source):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {k: hdr.index(k) for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
                                     "dram__bytes_write.sum")}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}
    kernels = {}
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        name = name.split("::")[-1]
        v = {}
        for key, field in (("duration_s", "gpu__time_duration.sum"), ("dram_read_bytes", "dram__bytes_read.sum"),
                           ("dram_write_bytes", "dram__bytes_write.sum")):
            i = col[field]
            v[key] = float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
        kernels.setdefault(name, v)  # first launch of each kernel
    traffic = sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in kernels.values())
    json.dump({"source": source, "lanes": int(lanes), "kernels": kernels, "traffic_bytes_per_sweep": traffic,
               "sum_duration_s": sum(k["duration_s"] for k in kernels.values()),
               "note": "per-launch cold-cache serialized ncu times (share, not absolute); traffic = dram read + "
                       "write summed over the kernels of one (batched) sweep"}, open(out, "w"), indent=1)
    print(json.dumps(kernels, indent=1), traffic)


if __name__ == "__main__":
    main(*sys.argv[1:5])
