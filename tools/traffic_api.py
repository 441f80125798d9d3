"""ncu --set full raw CSV of the API kernels (tools/profile_rows.py, config 4) -> per-kernel DRAM traffic,
duration and throughput, written as profiles/r02_traffic_api.json.

    python tools/traffic_api.py gpurun_out/api_raw.csv profiles/r02_traffic_api.json
"""

import csv
import json
import sys


def main(src, dst):
    rows = list(csv.reader(open(src)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9,
             "us": 1e-6, "ms": 1e-3, "ns": 1e-9}
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[idx["Kernel Name"]].split("(")[0].replace("void ", "")}
        for w in want:
            if w not in idx:
                continue
            v = r[idx[w]].replace(",", "")
            u = units[idx[w]]
            try:
                x = float(v)
            except ValueError:
                continue
            if u in scale:
                x *= scale[u]
            rec[w] = x
        t = rec.get("gpu__time_duration.sum")
        rd, wr = rec.get("dram__bytes_read.sum", 0.0), rec.get("dram__bytes_write.sum", 0.0)
        if t:
            rec["dram_gbs"] = round((rd + wr) / t / 1e9, 1)
        rec["traffic_bytes"] = int(rd + wr)
        out.append(rec)
    json.dump({"source": src, "note": "ncu --set full --clock-control none, one launch per row (cold L2); "
                                     "config 4 (512^3) API calls of tools/profile_rows.py", "launches": out},
              open(dst, "w"), indent=1)
    print(f"{len(out)} launches -> {dst}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
