#!/usr/bin/env python
"""Build profiles/ncu_traffic.json (dram__bytes_read.sum + dram__bytes_write.sum of ONE launch of
each benched kernel, the roofline `traffic` field) and a summary json from a directory of
ncu --set full reports named <key>.ncu-rep (tools/gpu_ncu_all.sh).
Usage: ncu_traffic.py gpurun_out/ncu_<tag> <summary.json> [<traffic.json>]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summarize  # noqa: E402


def to_bytes(s):
    val, unit = s.split()[0], (s.split()[1] if len(s.split()) > 1 else "byte")
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    return float(val.replace(",", "")) * mult


def main():
    d, out = sys.argv[1], sys.argv[2]
    summary, traffic = {}, {}
    for f in sorted(os.listdir(d)):
        if not f.endswith(".ncu-rep"):
            continue
        key = f[:-len(".ncu-rep")]
        recs = summarize(os.path.join(d, f))
        summary[key] = recs
        if recs:
            r = recs[0]
            traffic[key] = to_bytes(r["dram__bytes_read.sum"]) + to_bytes(r["dram__bytes_write.sum"])
    traffic["_source"] = (f"{out}: dram__bytes_read.sum + dram__bytes_write.sum of one launch per kernel "
                          f"(ncu --set full, tools/gpu_ncu_all.sh)")
    json.dump(summary, open(out, "w"), indent=1)
    json.dump(traffic, open(sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(out), "ncu_traffic.json"),
                            "w"), indent=1)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
