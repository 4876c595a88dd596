"""Turn `ncu --set full` reports into profiles/ncu_summary.json, the per-launch DRAM traffic that
bench.py reports as roofline.traffic (dram__bytes_read.sum + dram__bytes_write.sum of ONE launch).

usage: python profiles/ncu_to_json.py <config> <kernel_key>=<report.ncu-rep> [...]
e.g.   python profiles/ncu_to_json.py c2 mask_estimate=gpurun_out/mask_full.ncu-rep
       python profiles/ncu_to_json.py c4 mask_estimate=rep.ncu-rep#0 sparse_attention_prefill=rep.ncu-rep#1
"""
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "s": 1.0}


def launch_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, k):
        v = float(r[col[k]].replace(",", ""))
        return v * SCALE.get(units[col[k]], 1.0)
    res = []
    for r in data:
        res.append({"kernel": r[col["Kernel Name"]].split("(")[0],
                    "dram_bytes": val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
                    "dram_read_bytes": val(r, "dram__bytes_read.sum"),
                    "l2_bytes": val(r, "lts__t_bytes.sum") if "lts__t_bytes.sum" in col else None,
                    "duration_s": val(r, "gpu__time_duration.sum"),
                    "warp_instructions": val(r, "smsp__inst_executed.sum")})
    return res


def main():
    cfg = sys.argv[1]
    path = os.path.join(HERE, "ncu_summary.json")
    j = json.load(open(path)) if os.path.exists(path) else {}
    for arg in sys.argv[2:]:
        key, rep = arg.split("=", 1)
        i = 0
        if "#" in rep:  # report#i: the i-th launch of a multi-kernel report
            rep, i = rep.rsplit("#", 1)
            i = int(i)
        m = launch_metrics(rep)[i]
        m["report"] = os.path.basename(rep)
        j.setdefault(cfg, {})[key] = m
        print(cfg, key, m)
    json.dump(j, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
