"""Extract K3's DRAM traffic per launch from an `ncu --set full` capture of bench.py's timed
region and write profiles/k3_traffic.json (read by bench.py's roofline.traffic).

    ncu --set full --clock-control none --nvtx --nvtx-include "timed/" -k regex:attn_fwd_kernel \
        -c 1 -o gpurun_out/prof_k3_bench python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline
    python tools/k3_traffic.py gpurun_out/prof_k3_bench.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    rd = float(d["dram__bytes_read.sum"]) * SCALE[u["dram__bytes_read.sum"]]
    wr = float(d["dram__bytes_write.sum"]) * SCALE[u["dram__bytes_write.sum"]]
    res = {"bytes_per_launch": rd + wr, "read": rd, "write": wr, "kernel": d.get("Kernel Name"),
           "capture": os.path.basename(rep) + " (ncu --set full, bench.py timed region, n=131072)"}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "k3_traffic.json")
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    print(res)


if __name__ == "__main__":
    main(sys.argv[1])
