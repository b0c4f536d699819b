"""Extract K3's DRAM traffic per launch from an `ncu --set full` capture of bench.py's timed
region and write profiles/k3_traffic.json (read by bench.py's roofline.traffic).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "timed/" \
        -k regex:attn_fwd_kernel -c 2 -o gpurun_out/prof_k3_traffic python bench.py --steps 1 --warmup 1 --no-e2e \
        --no-cpu-baseline
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
    hdr, units = rows[0], rows[1]
    u = dict(zip(hdr, units))
    rd = wr = 0.0
    launches = 0
    name = None
    for vals in rows[2:]:  # the step's K3 launches (one per KV-head chunk) sum to one all-head launch
        d = dict(zip(hdr, vals))
        rd += float(d["dram__bytes_read.sum"]) * SCALE[u["dram__bytes_read.sum"]]
        wr += float(d["dram__bytes_write.sum"]) * SCALE[u["dram__bytes_write.sum"]]
        launches += 1
        name = d.get("Kernel Name")
    res = {"bytes_per_launch": rd + wr, "read": rd, "write": wr, "kernel": name, "launches_summed": launches,
           "capture": os.path.basename(rep) + " (ncu, bench.py timed region, n=131072: the step's K3 chunk launches "
                      "summed = the traffic of one all-head K3 launch)"}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "k3_traffic.json")
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    print(res)


if __name__ == "__main__":
    main(sys.argv[1])
